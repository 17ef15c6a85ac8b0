cd $GRAFT_REPO_ROOT
P2S_LIB=paper_2107_11627_b200/abl_dzv2.so timeout 600 python -m pytest tests -m gpu -x -q -k "mlp_backward or anchors_chain or adjoint_chain" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t.log
for L in abl_dzv abl_dzv2 abl_dzv abl_dzv2; do
P2S_LIB=paper_2107_11627_b200/$L.so timeout 300 python tools/dz_time.py > gpurun_out/dz_$L.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/dz_$L.log').read().strip().splitlines()[-1])
print('$L', {k: round(v['us_per_frame'],1) for k,v in d.items() if 'stream' not in k and 'cfg5' not in k})"
done
