P2S_MLP_W0=160 timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_frames.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1
for w in 128 160 128 160; do
P2S_MLP_W0=$w python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-adjoint-mode --no-sequence-mode --no-color-mode 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['configs']
print('w0=$w stage', d['plan']['stage_bytes'], 'render', round(d['value']), round(d['ms_per_step']*1e3,1), round(d['roofline']['fused_ms_median']*1e3,1), 'cfg5', round(c['cfg5_1024_rgb_K100_S65']['value']), 'cfg2', round(c['cfg2_256_gray_K100_S33']['value']))" || true
done
