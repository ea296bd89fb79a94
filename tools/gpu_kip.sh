cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -p no:cacheprovider -k "binary64 or ops or c2s or tournament" 2>&1 | tail -3
timeout 900 python bench.py --pairs 256 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | cut -c1-200
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_launch_c2.log 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | grep -E "total|kip"
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --pairs 2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1
python tools/launches.py gpurun_out/launches_c3.csv | head -24
