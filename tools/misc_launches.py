"""One call each of the smaller entry points on cfg3 (for an ncu launch list): correlated anchor
sampling (50 frames, G = 16), dL/dbeta alone, the colour render."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

spec = synth.CONFIGS[3]
inp = synth.make_inputs(spec)
r = p2s.Renderer(inp.basis, inp.mlp)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
img, z, t = d(inp.image), d(inp.zernike), d(inp.tilt)
smp = p2s.Sampler(16, spec.n_in, 2.0)
g = d(synth.make_upstream_grad(spec))
zc = d(synth.make_zernike_color(spec))
for _ in range(2):
    smp.sample(1, 0, 50)
    r.backward(img, z, t, g, want_beta=True, want_tilt=False)
    r.render_color(img, zc, t)
torch.cuda.synchronize()
print("misc_launches: ok")
