"""Fig. 12 analog (m from 941 to 41,761, transform sizes 2,048 to 131,072): forward + inverse
Bluestein time per limb-transform vs m, at the power-of-two length and at the R25 mixed-radix length
where the library implements it (prime m, 9 x 32 / 3 x 128 rows).  Small chains (2 + 1 primes): the
transform does not depend on the chain length.  Prints one JSON object per (m, length)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

RINGS = [(13, 859), (17, 1423), (3, 1871), (11, 15797), (5, 19531), (7, 20197), (19, 29989), (13, 30941),
         (3, 34511), (17, 41761), (31, 52053)]
npoly = int(sys.argv[1]) if len(sys.argv) > 1 else 64
rows = []
for p, m in RINGS:
    for blu in ("pow2", "mixed"):
        cfg = {"name": "sweep", "p": p, "m": m, "circuit": "U", "d": 1, "l": 1, "n_cipher": 2, "cipher_bits": 50,
               "n_special": 1, "special_bits": 50, "alpha": 1, "bluestein": blu}
        try:
            ctx = bc.Context(cfg)
        except bc.BoostComError as e:
            if blu == "mixed":
                rows.append({"m": m, "bluestein": blu, "unsupported": str(e)[:120]})
                print(json.dumps(rows[-1]), flush=True)
                continue
            raise
        if blu == "mixed" and ctx.M == rows[-1].get("M"):
            continue                        # the mixed rule kept the power of two
        L = ctx.n_cipher + ctx.n_special
        x = torch.randint(0, 1 << 40, (npoly, L, ctx.n), dtype=torch.int64, device="cuda")
        ws = ctx.workspace(npoly * L * ctx.M * 8 * 2 + (64 << 20))
        for _ in range(2):
            y = ctx.ntt_fwd(x, ws=ws)
            z = ctx.ntt_inv(y, ws=ws)
        torch.cuda.synchronize()
        ok = bool(torch.equal(z, x))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            y = ctx.ntt_fwd(x, ws=ws)
            z = ctx.ntt_inv(y, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        us = 1000 * e0.elapsed_time(e1) / 5 / (npoly * L) / 2
        rows.append({"m": m, "p": p, "n": ctx.n, "M": ctx.M, "bluestein": blu, "us_per_limb_transform": round(us, 4),
                     "ns_per_point_of_M": round(1000 * us / ctx.M, 4), "roundtrip": ok})
        print(json.dumps(rows[-1]), flush=True)
        del ctx, x, y, z, ws
        torch.cuda.empty_cache()
