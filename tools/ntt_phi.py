"""Composite m (C3): inverse NTT time with the sparse Barrett quotient (default) vs the convolution."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

ctx = bc.Context(bc.load_params(sys.argv[1] if len(sys.argv) > 1 else "c3"))
L, npoly = ctx.n_cipher, int(sys.argv[2]) if len(sys.argv) > 2 else 32
x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device="cuda")
ws = ctx.workspace(npoly * L * ctx.M * 8 * 3 + (256 << 20))
y = ctx.ntt_fwd(x, ws=ws)
for conv in (0, 1, 0):
    bc._lib.bc_tune(b"phi_conv", conv)
    for _ in range(2):
        z = ctx.ntt_inv(y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        z = ctx.ntt_inv(y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    print("phi_conv=%d inv %.3f us/limb roundtrip=%s" % (conv, 1000 * e0.elapsed_time(e1) / 5 / (npoly * L),
                                                       bool(torch.equal(z, x))), flush=True)
bc._lib.bc_tune(b"phi_conv", 0)
