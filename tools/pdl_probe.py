"""Back-to-back p2s_render calls on one stream (no flush, no per-call events): time per render with
the programmatic-dependent launch of the fused kernel on and off (P2S_NO_PDL) (dev tool)."""
import os
import subprocess
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) == 1:
    for m in ("pdl", "nopdl", "pdl", "nopdl"):
        env = dict(os.environ)
        env.pop("P2S_NO_PDL", None)
        if m == "nopdl":
            env["P2S_NO_PDL"] = "1"
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True).stdout
        print(m, out.strip())
    sys.exit(0)

import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402
inp = synth.make_inputs(synth.CONFIGS[3])
r = p2s.Renderer(inp.basis, inp.mlp)
img, z, t = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt))
out = torch.empty_like(img)
for _ in range(30):
    r.render(img, z, t, out=out)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    r.render(img, z, t, out=out)
e1.record()
torch.cuda.synchronize()
print(f"{e0.elapsed_time(e1) / 200 * 1e3:.1f} us per render (back to back, L2 warm)")
