import os, time, json, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2107_11627_b200 import p2s, synth
spec=synth.CONFIGS[3]; inp=synth.make_inputs(spec, frames=[0]); r=p2s.Renderer(inp.basis, inp.mlp)
pin=lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
i,z,t=pin(inp.image),pin(inp.zernike),pin(inp.tilt); o=pin(np.zeros_like(inp.image))
for _ in range(5): r.render_host(i,z,t,o)
res=[]
for rep in range(5):
    t0=time.perf_counter()
    for _ in range(40): r.render_host(i,z,t,o)
    res.append(40/(time.perf_counter()-t0))
print(os.environ.get('P2S_HOST_ONEWARP','banded'), [round(x) for x in res])
