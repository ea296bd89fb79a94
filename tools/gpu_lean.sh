# persistent column-pass variants (bc_tune ntt_lean 0/1/2): per-limb-transform time and bit-identity
cd $GRAFT_REPO_ROOT
for cfg in c2 c3 c4 c5; do
  IMPLS=${IMPLS:-0} LEAN=${LEANV:-0,2,3,0,2,3} timeout 600 python tools/ntt_micro.py $cfg ${NPOLY:-128} 2>&1 | grep -v Warn
done
