"""Fused-kernel time vs frame height and batch (the per-launch fixed cost; dev tool). Launches are
enqueued back to back behind a pre-warm (no host synchronisation between them: the B200 comes out
of idle slow); the library's events bracket each fused launch (p2s_debug_blur: the
fused kernel alone). L2 warm unless FLUSH=1."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda") if os.environ.get("FLUSH") else None
for H, B in ((16, 1), (32, 1), (64, 1), (128, 1), (256, 1), (512, 1), (512, 2), (512, 4), (512, 8)):
    spec = synth.custom("h", 3, B=B, C=3, H=H, W=512, K=100, S=33, h1=200, h2=200)
    inp = synth.make_inputs(spec, frames=range(B))
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike))
    J = torch.empty_like(img)
    n = 30
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(n)]
    for e in ev:
        e[0].record(), e[1].record()
    torch.cuda.synchronize()
    for _ in range(20):
        r.debug_blur(img, z, out=J)
    for i in range(n):
        if flush is not None:
            flush.fill_(float(i))
        r.set_profile_events(ev[i][0], ev[i][1])
        r.debug_blur(img, z, out=J)
    r.set_profile_events(None, None)
    torch.cuda.synchronize()
    ts = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    tiles = 4 * H * B
    print(f"H={H:4d} B={B}: tiles={tiles:5d} ({tiles / 148:5.1f} per CTA)  fused median {np.median(ts):8.1f} us"
          f"  per frame {np.median(ts) / B:7.1f} us  per tile-round {np.median(ts) / np.ceil(tiles / 148):6.2f} us")
    r.close()
