cd $GRAFT_REPO_ROOT
python tools/c1_time.py; P2S_NO_C1=1 python tools/c1_time.py; python tools/c1_time.py
