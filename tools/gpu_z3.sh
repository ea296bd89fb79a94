cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "ntt or c3 or hypercube or composite" 2>&1 | tail -2
timeout 300 python tools/ntt_phi.py c3 32
