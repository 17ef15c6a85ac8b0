cd $GRAFT_REPO_ROOT
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_full.log').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['roofline']['fused_ms_median'], d['e2e']['value'])
for k,v in d['configs'].items(): print(k, v['value'], v['roofline']['frac'], {kk: vv for kk, vv in v.items() if kk in ('batched',)})
for k in ('sequence_mode','color_mode','batch_mode','anchor_mode','adjoint_mode'): print(k, d[k]['value'])
"
