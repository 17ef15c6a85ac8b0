"""Driver for one ncu capture of the fused kernel on the one-channel plan: a 32-frame cfg2 batch
(256x256 gray, K = 100, 33x33), a few p2s_debug_blur calls (the fused kernel alone). Tools only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
inp = synth.make_inputs(synth.CONFIGS[2], frames=range(32))
r = p2s.Renderer(inp.basis, inp.mlp)
img, z = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (inp.image, inp.zernike))
out = torch.empty_like(img)
for _ in range(n):
    r.debug_blur(img, z, out=out)
torch.cuda.synchronize()
print("c1_profile_run: ok", r.info()["c1_plan"])
r.close()
