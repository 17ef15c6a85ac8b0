"""Where CUDA events put the fused kernel's time (dev tool): orderings of the L2 flush, torch
events and the library's fused-kernel events around p2s_render."""
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


def E():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)  # create it now
    return e


def run(mode, n=40):
    ev = [[E() for _ in range(6)] for _ in range(n)]
    torch.cuda.synchronize()
    for i in range(n):
        a = ev[i]
        if mode != "noflush":
            flush.fill_(float(i))
        if mode in ("A", "noflush"):
            r.set_profile_events(a[2], a[3])
            r.render(img, z, t, out=out)
        elif mode == "B":
            r.set_profile_events(a[2], a[3])
            a[0].record(st)
            r.render(img, z, t, out=out)
            a[1].record(st)
        elif mode == "C":
            r.set_profile_events(None, None)
            a[0].record(st)
            r.render(img, z, t, out=out)
            a[1].record(st)
        elif mode == "D":
            r.set_profile_events(None, None)
            a[0].record(st)
            a[4].record(st)
            r.render(img, z, t, out=out)
            a[1].record(st)
        elif mode == "F":  # flush, torch event, lib events; no outer end event
            r.set_profile_events(a[2], a[3])
            a[0].record(st)
            r.render(img, z, t, out=out)
    r.set_profile_events(None, None)
    torch.cuda.synchronize()
    res = {}
    sl = slice(5, None)
    if mode in ("A", "B", "noflush", "F"):
        res["fused"] = np.mean([x[2].elapsed_time(x[3]) for x in ev[sl]]) * 1e3
    if mode in ("B", "C", "D"):
        res["step"] = np.mean([x[0].elapsed_time(x[1]) for x in ev[sl]]) * 1e3
    if mode == "D":
        res["step_from_2nd_event"] = np.mean([x[4].elapsed_time(x[1]) for x in ev[sl]]) * 1e3
    if mode in ("B", "F"):
        res["outer_to_fused_begin"] = np.mean([x[0].elapsed_time(x[2]) for x in ev[sl]]) * 1e3
    return res


for rep in range(2):
    for mode in ("A", "B", "C", "D", "F", "noflush"):
        print(rep, mode, {k: round(v, 1) for k, v in run(mode).items()}, flush=True)
