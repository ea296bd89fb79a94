cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "ntt or binary64 or c2s or ops or tournament or sort or edges or select" 2>&1 | tail -3
timeout 300 python tools/ntt_micro.py c2 64 2>&1 | grep '"impl": [07],'
timeout 900 python bench.py --pairs 256 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
