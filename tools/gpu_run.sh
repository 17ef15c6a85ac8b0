cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "backward or adjoint" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t.log
for L in libp2s abl_nou libp2s; do
P2S_LIB=paper_2107_11627_b200/$L.so python tools/adjoint_time.py 20 image 2>&1 | tail -1 | sed "s/^/$L /"
done
