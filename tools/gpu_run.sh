# evidence: full GPU tests, bench (default), reference arm, smoke, launch list, ncu of the fused kernel
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; tail -2 gpurun_out/gputest.log
bash tools/evidence_run.sh
bash tools/ncu_full_run.sh
