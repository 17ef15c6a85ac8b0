# scratch driver for one gpurun call (edited per call)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_frames.py -m gpu -q -p no:cacheprovider -k "dense or adjoint_cfg3 or anchor_grid_cfg3 or backward_cfg3" -rP > gpurun_out/t3.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|dense|dL/d|oracle|Error|assert" gpurun_out/t3.log | tail -40
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sampler_launches.csv python -c "
import torch, numpy as np
from paper_2107_11627_b200 import p2s, synth
s = p2s.Sampler(64, 33, spatial_cov=synth.anchor_cov_exp(64, 6.0))
a = torch.empty((50, 33, 64, 64), device='cuda')
for _ in range(3): s.sample(1, 0, 50, out=a)
torch.cuda.synchronize()
" > gpurun_out/ncu_s.log 2>&1
grep -E "k_draw_y|k_sample_dense" gpurun_out/sampler_launches.csv | tail -4
