# A/B/C of older trees (build/<name>: own bench.py + library) against the current tree
for v in ${AB_ARMS:-prev n1 cur prev n1 cur}; do
  if [ $v = cur ]; then d=.; else d=build/$v; fi
  (cd $d && timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode > $GRAFT_REPO_ROOT/gpurun_out/ab_$v.log 2>&1 || \
            timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > $GRAFT_REPO_ROOT/gpurun_out/ab_$v.log 2>&1)
  python -c "import json; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print('$v', round(r['fused_ms_mean']*1e3,1), round(r.get('clean_step_ms', d['ms_per_step'])*1e3,1))" || tail -3 gpurun_out/ab_$v.log
done
