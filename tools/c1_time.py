"""Times the fused kernel (p2s_debug_blur) and the render on one-channel frames: cfg2 (one 256x256
frame, and 8 per call) and a 512x512 gray frame of cfg3's model; run with and without P2S_NO_C1=1
to compare the one-channel plan with the three-channel one. Tools only (synthetic inputs)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_11627_b200 import p2s, synth  # noqa: E402


def timeit(fn, n=50):
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(10):
        fn()
    ts = []
    for i in range(n):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


res = {}
for name, cfg, B, H in (("cfg2", 2, 1, None), ("cfg2_x8", 2, 8, None), ("gray512", 3, 1, 512)):
    spec = synth.CONFIGS[cfg]
    if H:
        spec = synth.custom("g512", cfg, B=1, C=1, H=H, W=H, K=spec.K, S=spec.S, h1=spec.h1, h2=spec.h2)
    inp = synth.make_inputs(spec, frames=range(B))
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (inp.image, inp.zernike, inp.tilt))
    out = torch.empty_like(img)
    res[name] = {"render_us": timeit(lambda: r.render(img, z, t, out=out)),
                 "blur_us": timeit(lambda: r.debug_blur(img, z, out=out)), "c1_plan": r.info()["c1_plan"]}
    r.close()
print(json.dumps(res))
