"""A/B of the KIP kernels inside a C2 compare (bits identical; step time and a launch list)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402
from inputs import word_pairs  # noqa: E402

ctx = bc.Context(bc.load_params("c2"))
keys = ctx.keygen(0xB00C0001)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(5)
A, Bw = word_pairs(rng, B * ctx.ints_per_ct, ctx.base, ctx.d * ctx.l)
ca = ctx.encrypt(keys, np.array(A, dtype=np.uint64).reshape(B, -1), 3, 0)
cb = ctx.encrypt(keys, np.array(Bw, dtype=np.uint64).reshape(B, -1), 3, B)
ws = ctx.workspace(max(ctx.workspace_bytes(B), 1 << 30))
res = {}
knob = os.environ.get("KNOB", "kip_blocked").encode()
vals = [int(v) for v in os.environ.get("VALS", "0,2,1,0,2,1").split(",")]
for kb in vals:
    bc._lib.bc_tune(knob, kb)
    r = ctx.compare_lt(keys, ca, cb, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        r = ctx.compare_lt(keys, ca, cb, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    res.setdefault(kb, []).append(e0.elapsed_time(e1) / 3 / B)
    if kb == vals[0]:
        ref = r.clone()
    else:
        assert torch.equal(r, ref), "blocked KIP changed the bits"
print(json.dumps({"ms_per_compare": res, "identical": True}))
bc._lib.bc_tune(knob, 1)
