# Round pass: GPU parity suite, default bench line, launch shares, C3/C4/C5 workload lines
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu --timeout 1400 -p no:cacheprovider -x 2>&1 | tail -3
timeout 1200 python bench.py 2>gpurun_out/bench_default.err | tail -1 > gpurun_out/bench_default.json
cut -c1-250 gpurun_out/bench_default.json
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | head -12
for c in c3 c4 c5; do
  timeout 1500 python bench.py --config $c --steps 2 --warmup 3 2>gpurun_out/bench_$c.err | tail -1 > gpurun_out/bench_$c.json
  cut -c1-300 gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err
done
