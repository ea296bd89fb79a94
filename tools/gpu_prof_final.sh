cd $GRAFT_REPO_ROOT
timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"kf_pass" -c 3 -o gpurun_out/nttf_full4 python tools/ntt_probe.py > gpurun_out/nttf_full4.log 2>&1
tail -1 gpurun_out/nttf_full4.log
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | head -30
