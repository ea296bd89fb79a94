"""Microbenchmark of the batched Bluestein NTT (forward + inverse) per kernel family / group size."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

cfg = bc.load_params(sys.argv[1] if len(sys.argv) > 1 else "c2")
ctx = bc.Context(cfg)
L = ctx.n_cipher
npoly = int(sys.argv[2]) if len(sys.argv) > 2 else 128
x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device="cuda")
ws = ctx.workspace(2 * npoly * L * ctx.M * 8 + (64 << 20))   # composite m: two slots per job
work = bc.ntt_work(ctx) * npoly * L
ref = None
ref_inv = None
bc._lib.bc_tune(b"ntt_split", int(os.environ.get("SPLIT", "0")))
for impl, gmb, lean in [(int(a), int(g), int(ln)) for a in os.environ.get("IMPLS", "7,0").split(",")
                        for g in os.environ.get("GMB", "4096").split(",") for ln in os.environ.get("LEAN", "0").split(",")]:
    bc.set_ntt_impl(impl)
    bc._lib.bc_tune(os.environ.get("KNOB", "ntt_lean").encode(), lean)
    bc._lib.bc_tune(b"ntt_group_bytes", gmb << 20)
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
    if ref is None:
        ref = y.clone()
    if ref_inv is None:
        ref_inv = z.clone()
    ok = bool(torch.equal(y, ref)) and bool(torch.equal(z, ref_inv))
    print(json.dumps({"limbs": npoly * L, "impl": impl, "group_mb": gmb, "knob": os.environ.get("KNOB", "ntt_lean"), "value": lean, "fwd_ms": round(f, 3), "inv_ms": round(i, 3),
                      "us_per_limb_fwd": round(1000 * f / (npoly * L), 3),
                      "Tmulmod_s": round(work / (f / 1e3) / 1e12, 3), "matches_radix2": ok, "roundtrip": bool(torch.equal(ctx.ntt_inv(y, ws=ws), x))}), flush=True)
bc.set_ntt_impl(0)
bc._lib.bc_tune(b"ntt_group_bytes", 48 << 20)
