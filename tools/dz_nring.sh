# Sweep of the streamed dL/dz variant's ring depth (P2S_MB_NRING, clamped to what two CTAs per SM
# leave room for) on cfg3 and cfg5; run via gpurun.
for n in 4 6 8 12 16; do echo "nring=$n"; P2S_MB_NRING=$n P2S_MB_MODE=stream python - <<'PY'
import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_2107_11627_b200 import p2s, synth
for cfg in (3,5):
    spec=synth.CONFIGS[cfg]; inp=synth.make_inputs(spec, frames=[0]); r=p2s.Renderer(inp.basis, inp.mlp)
    z=torch.from_numpy(inp.zernike).cuda(); gb=torch.randn((1,spec.K)+inp.zernike.shape[2:],device='cuda'); out=torch.empty_like(z)
    for _ in range(3): r.mlp_backward(z,gb,out)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): r.mlp_backward(z,gb,out)
    e1.record(); torch.cuda.synchronize(); print(f"  cfg{cfg}: {e0.elapsed_time(e1)/20*1e3:.1f} us")
    r.close()
PY
done
