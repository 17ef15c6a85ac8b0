# ncu evidence for the current build (run under gpurun; one ncu tool per call)
set -e
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python tools/profile_run.py 3 3 > gpurun_out/prof_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
    -o gpurun_out/prof_fused python tools/profile_run.py 3 3 > gpurun_out/ncu_full.log 2>&1
echo CAPTURED
