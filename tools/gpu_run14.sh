cd $GRAFT_REPO_ROOT
free -g | head -2; nproc
timeout 1200 python bench.py 2>&1 | tail -2 > gpurun_out/bench_r1_default.json
cat gpurun_out/bench_r1_default.json
