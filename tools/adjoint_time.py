"""Time p2s_backward's pieces on cfg3 (GPU only; for ncu launch lists and quick A/B):
python tools/adjoint_time.py [iters] [image|beta|tilt|zernike|all|all4]  (all4: all + dL/dz)"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
what = sys.argv[2] if len(sys.argv) > 2 else "image"
spec = synth.CONFIGS[3]
inp = synth.make_inputs(spec)
g = synth.make_upstream_grad(spec)
r = p2s.Renderer(inp.basis, inp.mlp)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
img, z, t, gg = d(inp.image), d(inp.zernike), d(inp.tilt), d(g)
kw = dict(want_beta=what in ("beta", "all", "all4"), want_tilt=what in ("tilt", "all", "all4"),
          want_image=what in ("image", "all", "all4"), want_zernike=what in ("zernike", "all4"))
for _ in range(3):
    r.backward(img, z, t, gg, **kw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(iters):
    r.backward(img, z, t, gg, **kw)
e1.record()
torch.cuda.synchronize()
print(f"{what}: {e0.elapsed_time(e1) / iters * 1e3:.1f} us per backward (cfg3, L2 warm)")
info = r.info() if hasattr(r, "info") else None
