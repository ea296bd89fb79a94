# Round-1 measurement pass: full GPU parity suite + smoke, default bench line, launch list, ncu full of the NTT passes
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -q -m gpu --timeout 2300 -p no:cacheprovider 2>&1 | tail -4
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py 2>gpurun_out/bench_default.err | tail -1 > gpurun_out/bench_default.json
cut -c1-250 gpurun_out/bench_default.json
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | head -14
timeout 900 ncu --set full --clock-control none --import-source on -k regex:kf_pass -s 6 -c 3 -o gpurun_out/nttf_full3 python tools/ntt_probe.py > gpurun_out/nttf_full3.log 2>&1
tail -1 gpurun_out/nttf_full3.log
timeout 900 ncu --set full --clock-control none -k regex:"k_kip_f|k_lift_f|k_tensor_f|k_scale_sub" -s 10 -c 4 -o gpurun_out/elem_full python bench.py --pairs 16 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/elem_full.log 2>&1
tail -1 gpurun_out/elem_full.log
