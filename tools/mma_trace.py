"""Per-item UMMA issue timeline of leader CTA 0 (needs a -DP2S_PROFILE build).

Usage: P2S_LIB=paper_2107_11627_b200/libp2s_prof.so python tools/mma_trace.py [cfg] [first] [count]
(TRACE_SEQ=F traces a p2s_render_sequence of F frames; TRACE_H=h a frame of h rows)
Columns: item, kind (conv/mlp + flags), slabs, N, start (cycles since kernel entry), wait cycles,
issue cycles (waits end -> commits done), cycles since the previous item start, and the ideal
tensor time of that item (56 cyc per M=256 N=112 UMMA, scaled by N).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2107_11627_b200 import p2s, synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
count = int(sys.argv[3]) if len(sys.argv) > 3 else 80
spec = synth.CONFIGS[cfg]
if os.environ.get("TRACE_H"):  # e.g. TRACE_H=16: one tile per CTA (launch-latency view)
    spec = synth.custom("h", cfg, B=1, C=spec.C, H=int(os.environ["TRACE_H"]), W=spec.W, K=spec.K, S=spec.S,
                        h1=spec.h1, h2=spec.h2)
SEQ = int(os.environ.get("TRACE_SEQ", "0"))  # > 0: a p2s_render_sequence of SEQ frames instead
inp = synth.make_inputs(spec, frames=range(max(1, SEQ)))
r = p2s.Renderer(inp.basis, inp.mlp)
img, z, t = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (inp.image[:1], inp.zernike, inp.tilt))
out = torch.empty((max(1, SEQ),) + tuple(img.shape[1:]), device="cuda")


def call():
    if SEQ:
        r.render_sequence(img, z, t, out=out)
    else:
        r.render(img, z, t, out=out)


for _ in range(3):
    call()
buf = torch.zeros(148 * 4 * 20 + 4 * 256, dtype=torch.int64, device="cuda")
r.debug_profile_buffer(buf)
call()
torch.cuda.synchronize()
r.debug_profile_buffer(None)
tr = buf[148 * 4 * 20:].view(256, 4).cpu().numpy().astype(np.int64)
FL = {1: "CONV", 2: "WA1", 4: "WSCR", 8: "WE", 16: "CA1", 32: "CMLP", 64: "CACC"}
prev = None
tot_gap = tot_ideal = 0
print(f"{'#':>4} {'kind':22s} {'sl':>3} {'N':>4} {'start':>8} {'wait':>6} {'issue':>6} {'dt':>6} {'ideal':>6}")
for i in range(256):
    a, b, c, f = tr[i]
    if a == 0 and i > 0:
        break
    flags = int(f) & 0xffff
    ns, n16 = (int(f) >> 16) & 0xff, (int(f) >> 24) & 0xff
    conv = flags & 1
    ideal = ns * (3 if conv else 1) * 56 * (n16 * 16) / 112
    dt = a - prev if prev is not None else 0
    if first <= i < first + count:
        kind = "+".join(v for k, v in FL.items() if flags & k) or "mlp"
        print(f"{i:4d} {kind:22s} {ns:3d} {n16*16:4d} {a:8d} {b - a:6d} {c - b:6d} {dt:6d} {ideal:6.0f}")
    prev = a
