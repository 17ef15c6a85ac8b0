"""Pinned host<->device copy rates for the e2e path's transfer sizes (dev tool)."""
import torch

def t_copy(dst, src, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        dst.copy_(src, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

for mb in (3.1, 8.6, 34.6, 39.8):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    ms = t_copy(d, h)
    ms2 = t_copy(h, d)
    print(f"{mb:5.1f} MB: H2D {ms*1e3:7.1f} us ({mb/ms:5.1f} GB/s)  D2H {ms2*1e3:7.1f} us ({mb/ms2:5.1f} GB/s)")
