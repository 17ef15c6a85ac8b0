"""Launch-phase timeline of CTA 0 of the fused kernel (needs a -DP2S_STARTUP_PROF build passed as
P2S_LIB; dev tool): globaltimer stamps relative to kernel entry, for a one-tile-per-CTA launch
(H = 16) and a full cfg3 frame, back to back behind a pre-warm (L2 warm)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2107_11627_b200 import p2s, synth  # noqa: E402

names = ["entry", "tables copied", "barriers+TMEM+cluster sync", "first A1 built (builder)",
         "first E built (epilogue warps)", "first UMMA (L1 chunk 0)", "first conv UMMA", "tile 1 ACC_FULL",
         "tile 1 TMEM_FREE", "epilogue done", "issuer done"]
for H in (16, 512):
    spec = synth.custom("h", 3, B=1, C=3, H=H, W=512, K=100, S=33, h1=200, h2=200)
    inp = synth.make_inputs(spec)
    r = p2s.Renderer(inp.basis, inp.mlp)
    img, z = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike))
    J = torch.empty_like(img)
    buf = torch.zeros(16 + 2 * 160, dtype=torch.int64, device="cuda")
    for _ in range(20):
        r.debug_blur(img, z, out=J)
    r.debug_profile_buffer(buf)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r.set_profile_events(e0, e1)
    r.debug_blur(img, z, out=J)
    r.set_profile_events(None, None)
    r.debug_profile_buffer(None)
    torch.cuda.synchronize()
    t = buf.cpu().numpy().astype(np.int64)
    print(f"H = {H}: event time {e0.elapsed_time(e1) * 1e3:.1f} us; stamps (us after entry):")
    for i, n in enumerate(names):
        if t[i]:
            print(f"  {n:32s} {(t[i] - t[0]) / 1e3:8.2f}")
    ent, ext = t[16:16 + 148], t[176:176 + 148]
    ok = (ent > 0) & (ext > 0)
    e, x = ent[ok], ext[ok]
    print(f"  all CTAs ({ok.sum()}): entry spread {(e.max() - e.min()) / 1e3:.2f} us, first entry -> last exit "
          f"{(x.max() - e.min()) / 1e3:.2f} us, CTA 0 exit at {(ext[0] - t[0]) / 1e3:.2f} us, exit spread "
          f"{(x.max() - x.min()) / 1e3:.2f} us")
    if H == 512:
        rel = (ext[ok] - e.min()) / 1e3
        print("  exit percentiles (us):", {q: round(float(np.percentile(rel, q)), 1) for q in (0, 10, 25, 50, 75, 90, 100)})
        print("  exit by CTA (us):", [round(float(v), 1) for v in (ext[:148] - e.min()) / 1e3])
    r.close()
