cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_edges.py -q -m gpu -p no:cacheprovider 2>&1 | tail -4
IMPLS=0,12,13 timeout 300 python tools/ntt_micro.py c5 32 2>&1 | tail -3
IMPLS=0,12,13 BC_LIB_PATH=variants/lib_e89_4.so timeout 300 python tools/ntt_micro.py c5 32 2>&1 | tail -3
