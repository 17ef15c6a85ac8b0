cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1])
print(round(d['value']), round(d['roofline']['fused_ms_median']*1e3,2), round(d['roofline']['frac'],4), d['roofline']['fused_le_step'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'], 'e2e', round(d['e2e']['value']))
for k,v in d['configs'].items(): print(k, round(v['value']), round(v['roofline']['frac'],3))
for k in ('sequence_mode','color_mode','batch_mode','anchor_mode','adjoint_mode'): print(k, round(d[k]['value']))
r=json.loads(open('gpurun_out/bench_ref.log').read().strip().splitlines()[-1]); print('ref', r['value'], r['ms_per_step'])
"
