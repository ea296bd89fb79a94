cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "c3 or hypercube or composite or ntt_forward" 2>&1 | tail -3
timeout 300 python tools/ntt_phi.py c3 32
timeout 900 python bench.py --config c3 --steps 2 --warmup 2 2>gpurun_out/bench_c3.err | tail -1 > gpurun_out/bench_c3.json
cut -c1-300 gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
