cd $GRAFT_REPO_ROOT
for r in 255 64 56; do echo "REG $r"; BC_LIB_PATH=variants/lib_r$r.so python tools/ntt_micro.py c2 128 2>&1 | grep '"impl": 0'; done
for g in 48 192 768; do echo "GROUP $g"; BC_NTT_GROUP_MB=$g python tools/ntt_micro.py c2 128 2>&1 | grep '"impl": 0'; done
