# scratch driver for one gpurun call (edited per call)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "dense or backward or sampler or host_checks or two_handles" -rP > gpurun_out/t2.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|dense|dL/dt|dL/dI" gpurun_out/t2.log | tail -60
timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --no-cpu-baseline --no-e2e > gpurun_out/bench2.log 2>&1; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench2.log
