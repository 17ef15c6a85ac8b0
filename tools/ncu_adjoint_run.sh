# One gpurun call: the adjoint's launch list (all four gradients, cfg3) and one ncu --set full
# capture of k_adjoint_image, each after the same driver ran clean without ncu.
set -e
python tools/adjoint_time.py 5 all4 > gpurun_out/adj_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/adj_launches.csv \
    python tools/adjoint_time.py 1 all4 > gpurun_out/adj_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_adjoint_image -c 1 \
    -o gpurun_out/prof_adjoint -f python tools/adjoint_time.py 1 image > gpurun_out/adj_ncu_full.log 2>&1
tail -1 gpurun_out/adj_plain.log; tail -2 gpurun_out/adj_ncu_full.log
