"""Timing sensitivity of the binary64 NTT passes to their table reads (bc_tune ntt_dbg bits; results invalid
while set): forward C2 transform of 64 polys x 11 limbs, CUDA events, per dbg mask."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

ctx = bc.Context(bc.load_params(sys.argv[1] if len(sys.argv) > 1 else "c2"))
L, npoly = ctx.n_cipher, 64
x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device="cuda")
ws = ctx.workspace(npoly * L * ctx.M * 8 + (64 << 20))
names = {0: "baseline", 1: "A: no input chirp", 2: "A: no cross twiddle", 4: "B: no D^", 8: "B: no cross twiddle",
         16: "C: no output chirp", 32: "C: no pos gather", 64: "A: no input load", 127: "all tables/loads off"}
for dbg in [0, 1, 2, 4, 8, 16, 32, 64, 127, 0]:
    bc._lib.bc_tune(b"ntt_dbg", dbg)
    for _ in range(2):
        ctx.ntt_fwd(x, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ctx.ntt_fwd(x, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print("%-24s %7.3f ms  %6.3f us/limb" % (names[dbg], ms, 1000 * ms / (npoly * L)), flush=True)
bc._lib.bc_tune(b"ntt_dbg", 0)
