# One gpurun call: dL/dz evidence — the timing tool clean, then one ncu --set full capture of the
# resident kernel (cfg3) and one of the streamed kernel (cfg5 frame), each after a clean run.
set -e
python tools/dz_time.py > gpurun_out/dz_time.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mlp_backward -s 3 -c 1 \
    -o gpurun_out/prof_dz_res -f python tools/dz_time.py > gpurun_out/ncu_dz_res.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_mlp_backward_s -s 3 -c 1 \
    -o gpurun_out/prof_dz_str -f python tools/dz_time.py > gpurun_out/ncu_dz_str.log 2>&1
tail -1 gpurun_out/dz_time.log
