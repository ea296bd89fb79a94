# GPU pass: new parity tests (tournament / sort), short C2 bench with the live NTT roofline,
# small C4 / C5 vector workloads (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 800 -p no:cacheprovider -x -k "tournament or sort or tables" 2>&1 | tail -4
timeout 600 python bench.py --pairs 64 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_c2_live.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_live.json')); print('c2 ms/ct', d['ms_per_ct_compare'], 'roof', {k: d['roofline'].get(k) for k in ('frac','per_launch_ms','limb_transforms_per_launch','share_of_step')})"
timeout 900 python bench.py --config c4 --T 2 --steps 1 --warmup 1 2>&1 | tail -2 | cut -c1-900
timeout 900 python bench.py --config c5 --T 4 --steps 1 --warmup 1 2>&1 | tail -2 | cut -c1-900
