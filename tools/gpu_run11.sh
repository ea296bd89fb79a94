cd $GRAFT_REPO_ROOT
python tools/ntt_micro.py c2 128 2>&1 | tail -7
python tools/ntt_micro.py c2 32 2>&1 | tail -7 | head -2
