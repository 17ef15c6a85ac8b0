import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2107_11627_b200 import p2s, synth
name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
specs = {"tiny": synth.custom("t", 1, B=1, C=1, H=4, W=100, K=8, S=5, h1=16, h2=16),
         "one": synth.custom("t", 1, B=1, C=1, H=1, W=100, K=8, S=5, h1=16, h2=16),
         "cfg1": synth.CONFIGS[1], "cfg3": synth.CONFIGS[3]}
inp = synth.make_inputs(specs[name])
r = p2s.Renderer(inp.basis, inp.mlp)
t0 = time.time()
out = r.render(*(torch.from_numpy(a).cuda() for a in (inp.image, inp.zernike, inp.tilt)))
torch.cuda.synchronize()
print(name, "ok", time.time() - t0, float(out.abs().mean()))
