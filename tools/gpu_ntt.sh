# GPU pass: NTT parity + live-roofline bench after an NTT kernel change
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 800 -p no:cacheprovider -x -k "ntt or compare_matches or ops_match" 2>&1 | tail -3
timeout 600 python bench.py --pairs 128 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_c2_ntt.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_ntt.json')); print('c2 ms/ct', d['ms_per_ct_compare'], 'verified', d['verified'], 'roof', {k: d['roofline'].get(k) for k in ('frac','per_launch_ms','limb_transforms_per_launch','share_of_step')})"
timeout 300 python tools/ntt_probe.py 2>&1 | tail -1
