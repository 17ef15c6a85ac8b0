for n in ${NRINGS:-3 4 5 6 3}; do
  P2S_NRING=$n timeout 200 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode > gpurun_out/nr$n.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/nr$n.log').read().strip().splitlines()[-1]); print('nring $n', round(d['value'],1), 'fps', round(d['roofline']['fused_ms_mean']*1e3,1), 'us fused', d['plan']['stage_bytes'], d['plan']['nring'], d['clocks']['sm_mhz'])"
done
