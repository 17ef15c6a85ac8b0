"""Small invocations of every device entry point (for compute-sanitizer runs): render, anchors,
sequence, colour, both samplers, the host paths, the debug taps, backward (all gradients, dL/dz,
the colour adjoint, the anchor chain) on ragged shapes, on the three-channel plan (C = 3, 2) and
the one-channel plan (C = 1)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
for spec in (synth.custom("san1", 601, B=2, C=3, H=21, W=150, K=20, S=7, h1=48, h2=40, t_std=1.7),
             synth.custom("san2", 602, B=1, C=2, H=9, W=37, K=100, S=33, h1=200, h2=200, t_std=1.0),
             synth.custom("san3", 603, B=2, C=1, H=19, W=131, K=24, S=9, h1=64, h2=48, t_std=1.3)):
    inp = synth.make_inputs(spec)
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z, t = d(inp.image), d(inp.zernike), d(inp.tilt)
    r.render(img, z, t)
    r.debug_beta(z)
    r.debug_blur(img, z)
    a_np = synth.make_anchors(spec, 5)
    anc = d(a_np)
    r.render_anchors(img, anc, t)
    r.debug_blur_anchors(img, anc)
    F = 3
    sinp = synth.make_inputs(spec, frames=range(F))
    r.render_sequence(d(sinp.image[:1]), d(sinp.zernike), d(sinp.tilt))
    zc = d(synth.make_zernike_color(spec))
    r.render_color(img, zc, t)
    g = d(synth.make_upstream_grad(spec))
    r.backward(img, z, t, g, want_image=True)
    r.backward(img, z, None, g, want_tilt=False)
    r.backward(img, z, t, g, want_zernike=True)
    r.backward_anchors(img, anc, t, g, want_image=True)
    r.backward_color(img, zc, t, g, want_image=True, want_zernike=True)
    out_h = np.empty_like(inp.image)
    r.render_host(inp.image, inp.zernike, inp.tilt, out_h)
    r.render_anchors_host(inp.image, a_np, inp.tilt, out_h)
    smp = p2s.Sampler(6, spec.n_in, 1.5)
    smp.sample(7, 0, 2)
    smp.close()
    G = 6
    yy, xx = np.divmod(np.arange(G * G), G)
    cov = np.exp(-0.5 * ((yy[:, None] - yy[None, :]) ** 2 + (xx[:, None] - xx[None, :]) ** 2) / 1.5 ** 2)
    cov += 1e-6 * np.eye(G * G)
    dsm = p2s.Sampler(G, spec.n_in, spatial_cov=cov)
    dsm.sample(11, 1, 3)
    dsm.close()
    torch.cuda.synchronize()
    r.close()
print("sanitize_small: ok")
