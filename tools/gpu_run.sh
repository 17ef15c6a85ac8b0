# scratch driver of one gpurun call: full GPU suite, default bench, smoke, dL/dz timing + ncu capture
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -rf > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 300 python tools/dz_time.py > gpurun_out/dz_time.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_mlp_backward -s 3 -c 1 \
    -o gpurun_out/prof_dz_res -f python tools/dz_time.py > gpurun_out/ncu_dz_res.log 2>&1
echo done
