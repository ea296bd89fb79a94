cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k2_pass -s 3 -c 3 -o gpurun_out/prof_ntt_e8 python tools/ntt_prof.py > gpurun_out/ncu_ntt.log 2>&1
tail -2 gpurun_out/ncu_ntt.log
