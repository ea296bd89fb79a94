# GPU pass: NTT register-cap variants (micro) + parity of the default build
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 500 -p no:cacheprovider -x -k "ntt" 2>&1 | tail -2
for r in 64 72 80 96; do echo "REG $r"; BC_LIB_PATH=variants/lib_r$r.so timeout 300 python tools/ntt_micro.py c2 64 2>&1 | grep '"impl": 0'; done
for r in 64 80; do echo "REG $r c4"; BC_LIB_PATH=variants/lib_r$r.so timeout 300 python tools/ntt_micro.py c4 32 2>&1 | grep '"impl": 0'; done
