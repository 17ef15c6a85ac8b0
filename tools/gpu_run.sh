# scratch driver of one gpurun call
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -x -q -k "mlp_backward or backward_anchors or adjoint_chain or envelope or color" > gpurun_out/dz_tests.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/dz_tests.log
timeout 300 python tools/dz_time.py > gpurun_out/dz_time.log 2>&1; echo "dz rc=$?"
tail -2 gpurun_out/dz_time.log
