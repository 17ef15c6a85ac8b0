"""Timeline of one p2s_render_host call on the bench workload (P2S_HOST_TRACE=1; dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["P2S_HOST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

inp = synth.make_inputs(synth.CONFIGS[3], frames=range(1))
r = p2s.Renderer(inp.basis, inp.mlp)
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
img, z, t = pin(inp.image), pin(inp.zernike), pin(inp.tilt)
out = pin(np.empty_like(inp.image))
for i in range(4):
    print(f"--- call {i}", file=sys.stderr)
    r.render_host(img, z, t, out)
