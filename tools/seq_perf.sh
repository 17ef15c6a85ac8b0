# sequence / colour / single-frame throughput (bench legs only)
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-adjoint-mode > gpurun_out/seq.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/seq.log').read().strip().splitlines()[-1]); print('render', round(d['value'],1), 'fused', round(d['roofline']['fused_ms_mean']*1e3,1), 'seq', round(d['sequence_mode']['value'],1), 'color', round(d['color_mode']['value'],1))"
