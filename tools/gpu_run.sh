cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "host or reserve" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t.log
for v in 0 1 0 1; do
if [ $v = 1 ]; then export P2S_HOST_ONEWARP=1; else unset P2S_HOST_ONEWARP; fi
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-anchor-mode --no-adjoint-mode --no-configs --no-batch-mode --no-sequence-mode --no-color-mode --e2e-steps 60 > gpurun_out/e2e_$v.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/e2e_$v.log').read().strip().splitlines()[-1])
print('ONEWARP=$v', round(d['value']), 'e2e', round(d['e2e']['value'],1))"
done
P2S_HOST_TRACE=1 python -c "
import numpy as np, torch
from paper_2107_11627_b200 import p2s, synth
spec=synth.CONFIGS[3]; inp=synth.make_inputs(spec, frames=[0]); r=p2s.Renderer(inp.basis, inp.mlp)
pin=lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
i,z,t=pin(inp.image),pin(inp.zernike),pin(inp.tilt); o=pin(np.zeros_like(inp.image))
for _ in range(4): r.render_host(i,z,t,o)
" 2>&1 | tail -24
