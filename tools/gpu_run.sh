# scratch driver of one gpurun call
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "mlp_backward or backward_anchors or adjoint_chain or envelope or color" > gpurun_out/dz_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/dz_tests.log
timeout 300 python tools/dz_time.py > gpurun_out/dz_time.log 2>&1; echo "dz rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/dz_time.log').read().strip().splitlines()[-1])
print({k: round(v['us_per_frame'],1) for k,v in d.items()})"
P2S_MB_NOZSEP=1 timeout 300 python tools/dz_time.py > gpurun_out/dz_time_nozsep.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/dz_time_nozsep.log').read().strip().splitlines()[-1])
print('nozsep', {k: round(v['us_per_frame'],1) for k,v in d.items()})"
