# parity suite + A/B of tuning knobs inside a C2 compare (tools/kip_ab.py) + optional bench configs
cd $GRAFT_REPO_ROOT
timeout 2400 python -m pytest tests -q -m gpu -x --timeout 2300 -p no:cacheprovider 2>&1 | tail -3
for kv in ${AB:-ntt_epi:0,1,0,1 ntt_lean:0,4,0,4}; do
  KNOB=${kv%%:*} VALS=${kv#*:} timeout 600 python tools/kip_ab.py 200 2>&1 | tail -1
done
for c in ${CFGS:-}; do
  timeout 1800 python bench.py --config $c --steps 2 --warmup 3 2>gpurun_out/bench_$c.err | tail -1 > gpurun_out/bench_$c.json
  cut -c1-300 gpurun_out/bench_$c.json; tail -2 gpurun_out/bench_$c.err
done
