import sys; sys.path.insert(0, '.')
import torch
from paper_2107_11627_b200 import p2s, synth
GD, FD = 64, 50
dsmp = p2s.Sampler(GD, 33, spatial_cov=synth.anchor_cov_exp(GD, 6.0))
danc = torch.empty((FD, 33, GD, GD), device="cuda", dtype=torch.float32)
for i in range(4):
    dsmp.sample(7, 0, FD, out=danc)
torch.cuda.synchronize()
print("ok")
