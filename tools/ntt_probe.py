"""The bench roofline probe launch (64 polys x 11 limbs forward Bluestein at C2), for ncu.
NTT_IMPL selects the kernel family (0 = three binary64 passes, 20 = fused cluster kernel), NTT_LEAN the
persistent column-pass variant (bc_tune ntt_lean)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

bc.set_ntt_impl(int(os.environ.get("NTT_IMPL", "0")))
if "NTT_LEAN" in os.environ:
    bc._lib.bc_tune(b"ntt_lean", int(os.environ["NTT_LEAN"]))
ctx = bc.Context(bc.load_params(os.environ.get("NTT_CFG", "c2")))
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("probe")      # ncu --nvtx --nvtx-include probe/ (context creation runs small NTTs)
r = bc.profile_ntt(ctx, npoly=int(os.environ.get("NPOLY", "64")))
torch.cuda.nvtx.range_pop()
print(r)
