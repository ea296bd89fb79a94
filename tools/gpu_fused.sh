# GPU pass: full parity suite (fused ModDown+modswitch, alpha = 4), C2 bench, ncu full capture of the NTT passes
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu --timeout 1400 -p no:cacheprovider -x 2>&1 | tail -6
timeout 600 python bench.py --pairs 128 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_c2_fused.json
python -c "import json; d=json.load(open('gpurun_out/bench_c2_fused.json')); print('c2 ms/ct', d['ms_per_ct_compare'], 'verified', d['verified'], 'roof', {k: d['roofline'].get(k) for k in ('frac','per_launch_ms','limb_transforms_per_launch','share_of_step')})"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 6 -c 3 -o gpurun_out/ntt_full python tools/ntt_probe.py > gpurun_out/ntt_full.log 2>&1
tail -2 gpurun_out/ntt_full.log
