cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "not slow and not full" --timeout 400 -p no:cacheprovider 2>&1 | tail -60 > gpurun_out/r1_tests.txt
cat gpurun_out/r1_tests.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -5
timeout 600 python bench.py --pairs 16 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -5
