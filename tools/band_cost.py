"""Fused-kernel time vs frame height (cost of small launches; dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

base = synth.CONFIGS[3]
for H in (16, 32, 64, 128, 136, 256, 512):
    spec = synth.custom("h", 3, B=1, C=3, H=H, W=512, K=100, S=33, h1=200, h2=200)
    inp = synth.make_inputs(spec)
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z, t = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt))
    out = torch.empty_like(img)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r.set_profile_events(e0, e1)
    ts = []
    for i in range(30):
        r.render(img, z, t, out=out)
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    print(f"H={H:4d} tiles={4*H:5d}: fused median {ts[len(ts)//2]:7.1f} us  min {ts[0]:7.1f}")
