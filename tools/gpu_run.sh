cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/gputest.log
python tools/beta_time.py
