cd $GRAFT_REPO_ROOT
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench3.log 2>&1
tail -1 gpurun_out/ncu_bench3.log | cut -c1-300
timeout 900 python bench.py --pairs 128 --steps 2 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-600
