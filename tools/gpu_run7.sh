cd $GRAFT_REPO_ROOT
python tools/ntt_micro.py c2 128 2>&1 | tail -12
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --timeout 500 -p no:cacheprovider 2>&1 | tail -3
