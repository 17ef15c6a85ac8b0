"""Times p2s_mlp_backward (dL/dz through the P2S MLP) on one cfg3 frame and a 16-frame batch
(CUDA events, L2 warm and flushed). Tools only: no oracle, synthetic inputs."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_11627_b200 import p2s, synth  # noqa: E402


def main():
    spec = synth.CONFIGS[3]
    inp = synth.make_inputs(spec)
    r = p2s.Renderer(inp.basis, inp.mlp)
    res = {}
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for B in (1, 16):
        z = torch.from_numpy(np.ascontiguousarray(np.repeat(inp.zernike, B, 0))).cuda()
        gb = torch.randn((B, spec.K, 512, 512), device="cuda")
        out = torch.empty_like(z)
        for _ in range(3):
            r.mlp_backward(z, gb, out)
        for mode in ("warm", "flushed"):
            ts = []
            for _ in range(20):
                if mode == "flushed":
                    flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                r.mlp_backward(z, gb, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            us = float(np.median(ts))
            px = B * 512 * 512
            macs = px * (33 * 200 + 200 * 200 + 100 * 200 + 200 * 200 + 200 * 33)
            byts = px * (33 + 100 + 33) * 4
            res[f"B{B}_{mode}"] = {"us": us, "us_per_frame": us / B, "tflops": 2 * macs / us / 1e6,
                                   "gbs": byts / us / 1e3}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
