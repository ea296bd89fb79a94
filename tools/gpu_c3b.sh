cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --config c3 --steps 2 --warmup 3 2>gpurun_out/bench_c3.err | tail -1 > gpurun_out/bench_c3.json
cut -c1-300 gpurun_out/bench_c3.json; tail -2 gpurun_out/bench_c3.err
timeout 900 ncu --nvtx --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --pairs 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1
python tools/launches.py gpurun_out/launches_c3.csv | head -25
