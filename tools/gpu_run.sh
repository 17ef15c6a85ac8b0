timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "sampl or dense" 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_draw_y|k_sample_dense" --csv python tools/draw_run.py 2>/dev/null | grep -E "k_draw_y|k_sample_dense" | tail -2 | awk -F'","' '{print $5, $NF}'
