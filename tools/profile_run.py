"""Short driver for ncu captures: a few p2s_render calls of the bench workload (cfg3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2107_11627_b200 import p2s, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
spec = synth.CONFIGS[cfg]
inp = synth.make_inputs(spec, frames=range(1))
r = p2s.Renderer(inp.basis, inp.mlp)
img, z, t = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt))
out = torch.empty_like(img)
for _ in range(n):
    r.render(img, z, t, out=out)
torch.cuda.synchronize()
print("ok", out.abs().mean().item())
