cd $GRAFT_REPO_ROOT
timeout 600 python tools/ntt_micro.py c2 64 2>&1 | tail -9
timeout 600 python tools/ntt_micro.py c5 32 2>&1 | grep '"impl": 0, "group_mb": 4096\|"impl": 7'
timeout 1500 python -m pytest tests -q -m gpu --timeout 1400 -p no:cacheprovider -x 2>&1 | tail -4
timeout 800 ncu --set full --clock-control none --import-source on -k regex:kf_pass -s 6 -c 3 -o gpurun_out/nttf_full2 python tools/ntt_probe.py > gpurun_out/nttf_full2.log 2>&1; tail -1 gpurun_out/nttf_full2.log
