# scratch driver of one gpurun call
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "reserve or backward or host or graph or anchors" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/t.log
