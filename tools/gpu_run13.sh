cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 800 -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r4.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench4.log 2>&1
timeout 900 python bench.py --pairs 128 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms/ct', d['ms_per_ct_compare'], 'value', d['value'], 'ntt frac', d['roofline']['frac'], 'verified', d['verified'], 'launches', d['gpu_launches'])"
