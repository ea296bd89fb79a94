cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -k "ops or binary64 or c2s or edges" 2>&1 | tail -2
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | grep -E "total|tensor"
