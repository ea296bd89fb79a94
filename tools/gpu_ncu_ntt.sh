# ncu --set full of the NTT probe passes (forward C2, 704 limb-transforms) for the persistent column-pass variants
cd $GRAFT_REPO_ROOT
for L in ${LEANS:-0 2}; do
  NTT_LEAN=$L timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "probe/" -k regex:"kf_pass" -c 3 \
    -o gpurun_out/ntt_lean$L python tools/ntt_probe.py > gpurun_out/ntt_lean$L.log 2>&1
  tail -1 gpurun_out/ntt_lean$L.log
done
