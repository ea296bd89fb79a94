# FP64 NTT: micro (all impls, equality vs radix-2), GPU parity tests, short bench
cd $GRAFT_REPO_ROOT
timeout 600 python tools/ntt_micro.py c2 64 2>&1 | tail -12
timeout 1500 python -m pytest tests -q -m gpu --timeout 1400 -p no:cacheprovider -x 2>&1 | tail -4
timeout 900 python bench.py --pairs 256 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-400
