# A/B of the steady item-list order (P2S_ORDER): bench lines for each, alternating
for o in ${ORDERS:-0 1 0 1}; do
  P2S_ORDER=$o timeout 200 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode > gpurun_out/ord$o.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ord$o.log').read().strip().splitlines()[-1]); print('order $o', round(d['value'],1), 'fps', round(d['roofline']['fused_ms_mean']*1e3,1), 'us fused', d['clocks']['sm_mhz'])"
done
