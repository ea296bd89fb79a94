# C3 on the paper's p10 ring: hypercube + composite-m parity tests, then a short compact_compare bench
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 1400 -p no:cacheprovider -k "c3 or hypercube or tables or ntt" 2>&1 | tail -15
timeout 900 python bench.py --config c3 --pairs 4 --steps 1 --warmup 1 --no-cpu 2>gpurun_out/bench_c3r.err | tail -1 > gpurun_out/bench_c3r.json
cut -c1-400 gpurun_out/bench_c3r.json; tail -3 gpurun_out/bench_c3r.err
timeout 300 python tools/ntt_micro.py c2 64 2>&1 | tail -6
