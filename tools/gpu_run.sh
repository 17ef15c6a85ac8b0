cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -k "info_reports" > gpurun_out/t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t.log
