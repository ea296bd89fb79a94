# GPU pass: full-size C4 tournament (T=16) and C5 sort (T=16) one step each; launch list of a C2 step
cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --config c4 --T 16 --steps 1 --warmup 1 --vec-chunk 40 2>&1 | tail -1 > gpurun_out/bench_c4_T16.json
cut -c1-400 gpurun_out/bench_c4_T16.json
timeout 1500 python bench.py --config c5 --T 16 --steps 1 --warmup 1 --vec-chunk 40 2>&1 | tail -1 > gpurun_out/bench_c5_T16.json
cut -c1-400 gpurun_out/bench_c5_T16.json
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_v3.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1
python tools/launches.py gpurun_out/launches_c2_v3.csv | head -30
