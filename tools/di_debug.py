"""Debug aid for k_adjoint_image: dL/dI of one small case vs the oracle (argv: C K S H W)."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import oracle  # noqa: E402
from oracle import adjoint  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

C, K, S, H, W = (int(a) for a in sys.argv[1:6])
spec = synth.custom("dbg", 901, B=1, C=C, H=H, W=W, K=K, S=S, h1=16, h2=16, t_std=1.0)
inp = synth.make_inputs(spec)
g = synth.make_upstream_grad(spec)
r = p2s.Renderer(inp.basis, inp.mlp)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
_, _, gi = r.backward(d(inp.image), d(inp.zernike), d(inp.tilt), d(g), want_beta=False, want_tilt=False,
                      want_image=True)
torch.cuda.synchronize()
gi = gi.cpu().numpy()
beta = oracle.beta(inp.image, inp.zernike, inp.basis, inp.mlp)
ri = adjoint.backward(inp.image[0], beta[0], inp.tilt[0], inp.basis, g[0], coord_dtype=np.float32)[3][None]
err = np.abs(gi - ri)
print(sys.argv[1:6], "max err", err.max(), "ref max", np.abs(ri).max(), "rel l2",
      np.linalg.norm(gi - ri) / np.linalg.norm(ri))
