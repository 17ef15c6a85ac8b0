cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -k "in_bounds or h224" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/t.log
