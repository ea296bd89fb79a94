cd $GRAFT_REPO_ROOT
timeout 1500 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_default.csv python bench.py --no-e2e --no-cpu > gpurun_out/r1_ncu_launch.log 2>&1
tail -1 gpurun_out/r1_ncu_launch.log | cut -c1-200
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 6 -c 3 -o gpurun_out/r1_probe_full python tools/ntt_probe.py > gpurun_out/r1_ncu_full.log 2>&1
tail -2 gpurun_out/r1_ncu_full.log
