"""Times p2s_mlp_backward (dL/dz through the P2S MLP): one cfg3 frame and a 16-frame batch
(resident weights), cfg3 with the streamed variant forced (P2S_MB_MODE=stream), and one cfg5 frame
(33-256-256-100: the streamed variant). CUDA events, L2 warm and flushed. Tools only: synthetic
inputs, no oracle."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_11627_b200 import p2s, synth  # noqa: E402


def run(cfg, Bs, ring, res):
    spec = synth.CONFIGS[cfg]
    inp = synth.make_inputs(spec, frames=[0])
    if ring:
        os.environ["P2S_MB_MODE"] = "stream"
    r = p2s.Renderer(inp.basis, inp.mlp)
    os.environ.pop("P2S_MB_MODE", None)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    n_in, H, W = inp.zernike.shape[1:]
    h1, h2, K = inp.mlp["W1"].shape[0], inp.mlp["W2"].shape[0], spec.K
    for B in Bs:
        z = torch.from_numpy(np.ascontiguousarray(np.repeat(inp.zernike, B, 0))).cuda()
        gb = torch.randn((B, K, H, W), device="cuda")
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
            px = B * H * W
            macs = px * (n_in * h1 + h1 * h2 + K * h2 + h2 * h1 + h1 * n_in)
            byts = px * (2 * n_in + K) * 4
            res[f"cfg{cfg}{'_stream' if ring else ''}_B{B}_{mode}"] = {
                "us": us, "us_per_frame": us / B, "tflops": 2 * macs / us / 1e6, "gbs": byts / us / 1e3}
    r.close()


def main():
    res = {}
    run(3, (1, 16), False, res)
    run(3, (1,), True, res)
    run(5, (1,), False, res)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
