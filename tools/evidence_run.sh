# One gpurun call: default bench line (with cpu_baseline), the reference arm, smoke(), and the
# ncu launch list of a short device-path bench run (the only profiler in this call).
set -e
python bench.py > gpurun_out/bench_full.log 2>&1
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --no-configs > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --no-configs > gpurun_out/ncu_launch.log 2>&1
tail -1 gpurun_out/bench_full.log; tail -1 gpurun_out/bench_ref.log; tail -2 gpurun_out/smoke.log
