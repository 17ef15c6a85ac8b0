python tools/profile_run.py 3 3 > gpurun_out/pp.log 2>&1 && ncu --set full --clock-control none -k regex:k_fused -s 1 -c 1 -o gpurun_out/prof_good python tools/profile_run.py 3 3 > /dev/null 2>&1
P2S_LIB=paper_2107_11627_b200/libp2s_alt.so python tools/profile_run.py 3 3 > gpurun_out/pp2.log 2>&1 && P2S_LIB=paper_2107_11627_b200/libp2s_alt.so ncu --set full --clock-control none -k regex:k_fused -s 1 -c 1 -o gpurun_out/prof_prog python tools/profile_run.py 3 3 > /dev/null 2>&1
echo done
