"""Small invocations of every device entry point (for compute-sanitizer runs): render, anchors,
sequence, colour, sampler, backward (all three gradients, and dL/dz) on ragged shapes."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
for spec in (synth.custom("san1", 601, B=2, C=3, H=21, W=150, K=20, S=7, h1=48, h2=40, t_std=1.7),
             synth.custom("san2", 602, B=1, C=2, H=9, W=37, K=100, S=33, h1=200, h2=200, t_std=1.0)):
    inp = synth.make_inputs(spec)
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z, t = d(inp.image), d(inp.zernike), d(inp.tilt)
    r.render(img, z, t)
    anc = d(synth.make_anchors(spec, 5))
    r.render_anchors(img, anc, t)
    F = 3
    sinp = synth.make_inputs(spec, frames=range(F))
    r.render_sequence(d(sinp.image[:1]), d(sinp.zernike), d(sinp.tilt))
    r.render_color(img, d(synth.make_zernike_color(spec)), t)
    g = d(synth.make_upstream_grad(spec))
    r.backward(img, z, t, g, want_image=True)
    r.backward(img, z, None, g, want_tilt=False)
    r.backward(img, z, t, g, want_zernike=True)
    smp = p2s.Sampler(6, spec.n_in, 1.5)
    smp.sample(7, 0, 2)
    torch.cuda.synchronize()
    r.close()
print("sanitize_small: ok")
