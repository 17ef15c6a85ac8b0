# scratch driver for one gpurun call (edited per call)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/gputest.log 2>&1; tail -3 gpurun_out/gputest.log
timeout 300 python bench.py > gpurun_out/bench.log 2>gpurun_out/bench.err; tail -c 3000 gpurun_out/bench.log
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -c 1500 gpurun_out/bench_ref.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
