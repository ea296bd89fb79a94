cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "non_blocking or full" --timeout 500 -p no:cacheprovider --durations=5 2>&1 | tail -30
timeout 900 python bench.py --pairs 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "slow" --timeout 800 -p no:cacheprovider --durations=5 2>&1 | tail -20
