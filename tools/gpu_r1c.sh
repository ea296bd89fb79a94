# Re-entry GPU pass: parity tests, smoke, default bench line, launch list of a short C2 step, ncu full of the NTT probe
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
nproc
timeout 1500 python -m pytest tests -q -m gpu --timeout 1400 -p no:cacheprovider 2>&1 | tail -8 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python bench.py 2>gpurun_out/bench_default.err | tail -1 > gpurun_out/bench_default.json
cut -c1-300 gpurun_out/bench_default.json
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | head -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 6 -c 3 -o gpurun_out/ntt_full python tools/ntt_probe.py > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
