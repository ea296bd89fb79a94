"""Fused cluster NTT: per-limb-transform time vs the number of persistent clusters (C2, forward + inverse)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

ctx = bc.Context(bc.load_params(sys.argv[1] if len(sys.argv) > 1 else "c2"))
L = ctx.n_cipher
npoly = int(sys.argv[2]) if len(sys.argv) > 2 else 256
x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device="cuda")
ws = ctx.workspace(npoly * L * ctx.M * 8 + (64 << 20))
bc.set_ntt_impl(10)
ref = ctx.ntt_fwd(x, ws=ws)
refi = ctx.ntt_inv(ref, ws=ws)
bc.set_ntt_impl(20)
runs = [(int(a), int(v)) for a in os.environ.get("VAR", "0").split(",") for v in os.environ.get("NCL", "0").split(",")]
for var, ncl in runs:
    bc._lib.bc_tune(b"nttc_variant", var)
    act = bc._lib.bc_tune(b"nttc_clusters", ncl)
    for _ in range(2):
        y = ctx.ntt_fwd(x, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        y = ctx.ntt_fwd(x, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    f = e0.elapsed_time(e1) / 5
    e0.record()
    for _ in range(5):
        z = ctx.ntt_inv(y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    i = e0.elapsed_time(e1) / 5
    print(json.dumps({"variant": var, "clusters": ncl, "active_max": bc._lib.bc_tune(b"nttc_clusters", ncl), "occupancy_max": act, "limbs": npoly * L,
                      "us_fwd": round(1000 * f / (npoly * L), 4), "us_inv": round(1000 * i / (npoly * L), 4),
                      "exact": bool(torch.equal(y, ref)) and bool(torch.equal(z, refi))}), flush=True)
bc._lib.bc_tune(b"nttc_clusters", 0)
bc.set_ntt_impl(0)
