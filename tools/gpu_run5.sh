cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_r2.csv python bench.py --pairs 16 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench2.log 2>&1
tail -2 gpurun_out/ncu_bench2.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_pass|k_lift|k_kip" -s 40 -c 6 -o gpurun_out/prof_v2 python bench.py --pairs 16 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_full2.log 2>&1
tail -2 gpurun_out/ncu_full2.log
