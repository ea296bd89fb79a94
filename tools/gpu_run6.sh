cd $GRAFT_REPO_ROOT
python tools/ntt_micro.py c2 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow" --timeout 500 -p no:cacheprovider 2>&1 | tail -4
for impl in 0 2; do BC_NTT_IMPL=$impl timeout 900 python bench.py --pairs 64 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('impl', $impl, 'ms/ct', d['ms_per_ct_compare'], 'value', d['value'], 'ntt frac', d['roofline']['frac'])"; done
