# scratch driver for one gpurun call (edited per call)
timeout 300 python tools/adjoint_time.py 50 image; python tools/adjoint_time.py 50 all
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_frames.py -m gpu -q -p no:cacheprovider -x -k "backward_parity or image_gradient or backward_cfg3 or adjoint_cfg3 or backward_color or two_handles or adjoint_chain or mlp_backward_parity or mlp_backward_cfg3" > gpurun_out/t7.log 2>&1; tail -3 gpurun_out/t7.log; grep -E "dL/dI|fp64 masks" gpurun_out/t7.log | head -30
ncu --metrics gpu__time_duration.sum,lts__t_bytes.sum --clock-control none --csv --log-file gpurun_out/adj_launches.csv python tools/adjoint_time.py 3 image > /dev/null 2>&1
grep k_adjoint_image gpurun_out/adj_launches.csv | tail -2
