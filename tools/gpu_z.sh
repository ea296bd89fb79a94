cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "ntt or c2s or binary64 or composite" 2>&1 | tail -2
IMPLS=7,0 timeout 300 python tools/ntt_micro.py c2 128 2>&1 | tail -2
