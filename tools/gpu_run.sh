cd $GRAFT_REPO_ROOT
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --no-configs > gpurun_out/plain_bench.log 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-anchor-mode --no-batch-mode --no-sequence-mode --no-adjoint-mode --no-color-mode --no-configs > gpurun_out/ncu_launch.log 2>&1; echo "ncu launch rc=$?"
timeout 120 python tools/profile_run.py 3 3 > gpurun_out/prof_plain.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
    -o gpurun_out/prof_fused -f python tools/profile_run.py 3 3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 300 python tools/dz_time.py > gpurun_out/dz_time.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_mlp_backward -s 3 -c 1 \
    -o gpurun_out/prof_dz_res -f python tools/dz_time.py > gpurun_out/ncu_dz_res.log 2>&1; echo "ncu dz rc=$?"
