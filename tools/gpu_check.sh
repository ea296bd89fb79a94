# GPU sanity pass: parity tests, smoke, short bench (run under gpurun from the repo root)
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -q -m gpu --timeout 1100 -p no:cacheprovider -x 2>&1 | tail -5
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 900 python bench.py --pairs 128 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 > gpurun_out/bench_short.json
cat gpurun_out/bench_short.json | cut -c1-600
