timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_frames.py -m gpu -q -p no:cacheprovider -x -k "image or backward or adjoint or color" 2>&1 | tail -3
for w in image all; do python tools/adjoint_time.py 20 $w 2>&1 | head -1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fused|k_adjoint_image" --csv python tools/adjoint_time.py 2 image 2>/dev/null | grep -E "k_fused|k_adjoint" | tail -2 | awk -F'","' '{print $5, $NF}'
