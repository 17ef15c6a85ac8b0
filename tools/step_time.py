"""Step time (render = fused + warp) with and without the library's fused-kernel events (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

inp = synth.make_inputs(synth.CONFIGS[3], frames=range(1))
r = p2s.Renderer(inp.basis, inp.mlp)
img, z, t = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt))
out = torch.empty_like(img)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for mode in ("events", "none", "events", "none"):
    n = 50
    s0 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    s1 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    f0 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    f1 = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for i in range(n):
        flush.fill_(float(i))
        if mode == "events":
            r.set_profile_events(f0[i], f1[i])
        s0[i].record(st)
        r.render(img, z, t, out=out)
        s1[i].record(st)
    r.set_profile_events(None, None)
    torch.cuda.synchronize()
    step = np.array([a.elapsed_time(b) for a, b in zip(s0, s1)]) * 1e3
    msg = f"{mode:7s}: step mean {step[5:].mean():6.1f} us"
    if mode == "events":
        fu = np.array([a.elapsed_time(b) for a, b in zip(f0, f1)]) * 1e3
        msg += f"  fused mean {fu[5:].mean():6.1f} us"
    print(msg)
