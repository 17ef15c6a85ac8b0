"""Times step a1 alone (p2s_debug_beta: the P2S MLP -> beta [B,K,H,W]) on cfg3 frames, one per call
and 16 per call, L2 flushed: k_mlp_forward by default, the fused kernel's MLP-only mode with
P2S_BETA_FUSED=1. Tools only (synthetic inputs)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

spec = synth.CONFIGS[3]
inp = synth.make_inputs(spec, frames=[0])
r = p2s.Renderer(inp.basis, inp.mlp)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
res = {}
for B in (1, 16):
    z = torch.from_numpy(np.ascontiguousarray(np.repeat(inp.zernike, B, 0))).cuda()
    out = torch.empty((B, spec.K, spec.H, spec.W), device="cuda")
    for _ in range(5):
        r.debug_beta(z, out=out)
    ts = []
    for i in range(30):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r.debug_beta(z, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    res[f"B{B}_us_per_frame"] = round(float(np.median(ts)) / B, 1)
print(os.environ.get("P2S_BETA_FUSED", "k_mlp_forward"), json.dumps(res))
