cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --timeout 500 -p no:cacheprovider 2>&1 | tail -15
timeout 900 python bench.py --pairs 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -3
