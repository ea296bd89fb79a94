cd $GRAFT_REPO_ROOT
python tools/ntt_micro.py c2 128 2>&1 | grep -E '"group_mb": (48|4096)' | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 800 -p no:cacheprovider 2>&1 | tail -3
timeout 900 python bench.py --pairs 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/ct', d['ms_per_ct_compare'], 'value', d['value'], 'ntt frac', d['roofline']['frac'], 'verified', d['verified'])"
