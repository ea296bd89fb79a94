"""f1: choose the key-switching digit size alpha (dnum = ceil(L / alpha)) and special-prime
count K >= alpha by measurement.  C2 ring and circuit, B ciphertext pairs, every result bit verified;
prints ms per ct compare_lt and the transform count per key switch for each (alpha, K)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402
from inputs import word_pairs  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 200
base = bc.load_params(sys.argv[2] if len(sys.argv) > 2 else "c2")
for alpha, K in [(2, 2), (3, 3), (4, 4), (6, 6), (11, 11)]:
    cfg = dict(base, alpha=alpha, n_special=K)
    ctx = bc.Context(cfg)
    keys = ctx.keygen(0xB00C0001)
    rng = np.random.default_rng(9)
    A, Bw = word_pairs(rng, B * ctx.ints_per_ct, ctx.base, ctx.d * ctx.l)
    A = np.array(A, dtype=np.uint64).reshape(B, -1)
    Bw = np.array(Bw, dtype=np.uint64).reshape(B, -1)
    ca = ctx.encrypt(keys, A, 3, 0)
    cb = ctx.encrypt(keys, Bw, 3, B)
    free, _ = torch.cuda.mem_get_info()
    ws = ctx.workspace(int(min(max(ctx.workspace_bytes(1), int(free * 0.8)), free - (2 << 30))))
    r = ctx.compare_lt(keys, ca, cb, ws=ws)
    ok = bool(np.array_equal(ctx.decrypt(keys, r, as_bits=True), (A < Bw).astype(np.uint64)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        r = ctx.compare_lt(keys, ca, cb, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    L = ctx.n_cipher
    dnum = -(-L // alpha)
    print(json.dumps({"alpha": alpha, "K": K, "dnum_top": dnum, "transforms_per_ks_top": dnum * (L + K) + 2 * K + 2 * L,
                      "ms_per_ct_compare": round(e0.elapsed_time(e1) / 3 / B, 4), "verified": ok}), flush=True)
    del ctx, keys, ca, cb, ws, r
    torch.cuda.empty_cache()
