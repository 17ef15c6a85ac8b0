timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
P2S_EHALF=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
for e in 0 1; do
P2S_EHALF=$e python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-adjoint-mode 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['configs']
print('ehalf=$e', 'cfg3', round(d['value']), round(d['roofline']['fused_ms_median']*1e3,1), 'cfg5', round(c['cfg5_1024_rgb_K100_S65']['value']), round(c['cfg5_1024_rgb_K100_S65']['roofline']['frac'],3), 'cfg2', round(c['cfg2_256_gray_K100_S33']['value']), 'seq', round(d['sequence_mode']['value']), 'color', round(d['color_mode']['value']))" || true
done
