P2S_LIB=paper_2107_11627_b200/abl_mbprof.so python tools/dz_trace.py
