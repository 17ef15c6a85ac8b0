cd $GRAFT_REPO_ROOT
L=paper_2107_11627_b200/libp2s_prof.so
P2S_LIB=$L timeout 120 python tools/mma_trace.py 2 0 60 > gpurun_out/trace_c1.txt 2>&1
P2S_LIB=$L timeout 120 python tools/role_profile.py 2 > gpurun_out/roles_c1.txt 2>&1
