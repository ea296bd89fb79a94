# GPU pass: bivariate parity (c1b), compaction, C3 full-size decrypt, C3 bench (small)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 1100 -p no:cacheprovider -x -k "bivariate or compaction or c3" 2>&1 | tail -4
timeout 1200 python bench.py --config c3 --pairs 16 --steps 1 --warmup 1 2>&1 | tail -2 | cut -c1-1200
