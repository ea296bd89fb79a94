# Round-end measurement pass (one GPU): parity suite + smoke, bench lines for C2 (default), C3 (313 dense pairs),
# C4, C5, private_q, the C2 launch list, and one ncu --set full capture of the NTT passes at a representative size
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -q -m gpu --timeout 2300 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 1200 python bench.py 2>gpurun_out/bench_default.err | tail -1 > gpurun_out/bench_default.json
cut -c1-200 gpurun_out/bench_default.json
for c in ${CFGS:-c3 c4 c5 p3q}; do
  P=""; [ $c = c3 ] && P="--pairs 313"
  timeout 2400 python bench.py --config $c $P --steps 2 --warmup 3 2>gpurun_out/bench_$c.err | tail -1 > gpurun_out/bench_$c.json
  cut -c1-200 gpurun_out/bench_$c.json
done
timeout 900 ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --pairs 32 --steps 1 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
python tools/launches.py gpurun_out/launches_c2.csv | head -16
NPOLY=384 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"kf_pass" -c 3 -o gpurun_out/ntt_final python tools/ntt_probe.py > gpurun_out/ntt_final.log 2>&1
tail -1 gpurun_out/ntt_final.log
