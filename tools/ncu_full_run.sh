# One gpurun call: one ncu --set full capture of k_fused_p2s (after the same driver ran clean).
set -e
python tools/profile_run.py 3 3 > gpurun_out/prof_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused -s 1 -c 1 \
    -o gpurun_out/prof_fused -f python tools/profile_run.py 3 3 > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
