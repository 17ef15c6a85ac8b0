"""Per-role cycle breakdown of k_fused_p2s (needs libp2s_prof.so, built with -DP2S_PROFILE).

Usage: P2S_LIB=paper_2107_11627_b200/libp2s_prof.so python tools/role_profile.py [cfg]
       (ADJ=image: the adjoint's fused pass instead of the render; ANCHOR_G=G: anchor mode;
        TRACE_B=n: n frames per call)
Counters (clock64 cycles, averaged over CTAs), per role:
  MMA issuer : 0 wait A1_FULL, 1 wait BETA_FREE, 2 wait SCR_FREE, 3 wait E_FULL,
               4 wait ring (MLP), 5 wait ring (conv), 6 wait ACC_FREE (first conv stage), 19 total
  producer   : 7 wait ring_empty, 19 total
  builder t0 : 9 wait A1_EMPTY, 11 wait E_EMPTY, 12 build E, 19 total
  epilogue t0: 13 wait MLP_DONE, 15 wait ACC_FULL, 19 total
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2107_11627_b200 import p2s, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
spec = synth.CONFIGS[cfg]
if os.environ.get("TRACE_H"):
    spec = synth.custom("h", cfg, B=1, C=spec.C, H=int(os.environ["TRACE_H"]), W=spec.W, K=spec.K, S=spec.S, h1=spec.h1, h2=spec.h2)
NB = int(os.environ.get("TRACE_B", "1"))  # frames per call
inp = synth.make_inputs(spec, frames=range(NB))
r = p2s.Renderer(inp.basis, inp.mlp)
img, z, t = (torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt))
out = torch.empty_like(img)
ANCH = int(os.environ.get("ANCHOR_G", "0"))  # >0: anchor-grid mode (p2s_render_anchors) with this G
ADJ = os.environ.get("ADJ")  # "image": the adjoint's fused pass (mode 3: J + U = beta dL/dJ)
if ADJ:
    gg = torch.from_numpy(synth.make_upstream_grad(spec, frames=range(1))).cuda()
    render = lambda: r.backward(img, z, t, gg, want_beta=False, want_tilt=False, want_image=True)  # noqa: E731
elif ANCH:
    anc = torch.from_numpy(synth.make_anchors(spec, ANCH, frames=range(1))).cuda()
    render = lambda: r.render_anchors(img, anc, t, out=out)  # noqa: E731
else:
    render = lambda: r.render(img, z, t, out=out)  # noqa: E731
for _ in range(3):
    render()
buf = torch.zeros(148 * 4 * 20 + 4 * 256, dtype=torch.int64, device="cuda")
r.debug_profile_buffer(buf)
render()
torch.cuda.synchronize()
r.debug_profile_buffer(None)
c = buf[:148 * 4 * 20].view(148, 4, 20).cpu().numpy().astype(np.float64)
names = {0: {0: "wait A1_FULL", 1: "wait TMEM_FREE", 2: "wait SCR_FREE", 3: "wait E_FULL", 5: "wait ring",
             4: "conv UMMA loops", 6: "MLP UMMA loops", 19: "total"},
         1: {7: "wait ring_empty", 19: "total"},
         2: {9: "wait A1_EMPTY", 11: "wait E_EMPTY", 12: "build E", 19: "total"},
         3: {13: "wait MLP_DONE", 15: "wait ACC_FULL", 16: "conv epi to release", 17: "MLP drain work", 18: "drain fence+arrive", 19: "total"}}
roles = ["MMA", "producer", "builder", "epilogue"]
ntiles = NB * spec.H * ((spec.W + 127) // 128)
print(f"cfg{cfg}: {ntiles} tiles over 148 CTAs (~{ntiles / 148:.1f} tiles/CTA); cycles per CTA (mean / max)")
for ri, role in enumerate(roles):
    for k, n in names[ri].items():
        v = c[0::2, ri, k] if ri == 0 else c[:, ri, k]  # MMA issuer runs in the leader CTAs only
        print(f"  {role:9s} {n:18s} {v.mean():12.0f} {v.max():12.0f}")

# wall-clock phases (globaltimer ns): kernel entry (slot 10), MMA loop start (11), role end (12)
t0 = c[:, :, 10][c[:, :, 10] > 0].min()
ent = c[0::2, 0, 10] - t0
lst = c[0::2, 0, 11] - t0
lend = c[0::2, 0, 12] - t0
eend = c[:, 3, 12] - t0
print(f"wall (us, rel. first CTA entry): entry max {ent.max()/1e3:.1f}; MMA loop start mean {lst.mean()/1e3:.1f} "
      f"max {lst.max()/1e3:.1f}; MMA loop end min {lend.min()/1e3:.1f} mean {lend.mean()/1e3:.1f} max {lend.max()/1e3:.1f}; "
      f"epilogue end max {eend.max()/1e3:.1f}")
