for lib in paper_2107_11627_b200/libp2s.so paper_2107_11627_b200/abl_nou.so; do
for w in image all beta tilt; do P2S_LIB=$lib python tools/adjoint_time.py 20 $w 2>&1 | head -1; done
P2S_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fused --csv python tools/adjoint_time.py 2 image 2>/dev/null | grep k_fused | tail -1 | awk -F'","' '{print $5, $NF}'
done
