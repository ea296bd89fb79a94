"""private_q probe: host enqueue time vs device time, blocking vs non-blocking, side-stream priority."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_07308_b200 as bc  # noqa: E402

cfg = bc.load_params("p3q")
ctx = bc.Context(cfg)
keys = ctx.keygen(0xB00C0001)
N = int(sys.argv[1]) if len(sys.argv) > 1 else 100
e = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ints = ctx.ints_per_ct
rng = np.random.default_rng(1)
X = np.zeros((N, ctx.S, ctx.D), dtype=np.int16)
X[:, :, 0] = rng.integers(0, ctx.p, (N, ctx.S))
data = ctx.encrypt_slots(keys, X, 3, ct_index0=0)
op1 = ctx.encrypt_slots(keys, X[:1], 3, ct_index0=N)
q = ctx.encrypt(keys, np.array([[3] * ints], dtype=np.uint64), 3, ct_index0=N + 1)
codes = ctx.encrypt(keys, np.array([[c] * ints for c in (1, 2, 3)], dtype=np.uint64), 3, ct_index0=N + 2)
wsm = ctx.workspace(int(bc._lib.bc_private_query_workspace_bytes(ctx._h, N, 13, 13, 13, e, 0)))
wss = torch.empty(int(bc._lib.bc_private_query_workspace_bytes(ctx._h, N, 13, 13, 13, e, 1)), dtype=torch.uint8,
                  device="cuda")
for prio, impl in ((-1, 0), (-1, 17)):
    bc.set_ntt_impl(impl)
    side = torch.cuda.Stream(priority=prio)
    graphs = {}
    for name, fn in (("blocking", lambda: ctx.private_query(keys, data, q, codes, op1, e, ws=wsm)),
                     ("nonblocking", lambda: ctx.private_query(keys, data, q, codes, op1, e, side_stream=side, ws=wsm,
                                                               ws_side=wss)),
                     ("branch", lambda: ctx.compare_eq(keys, torch.cat([q, q, q]), codes, ws=wsm))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(3):
            fn()
        t1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"prio": prio, "ntt_impl": impl, "what": name, "host_enqueue_ms": round((t1 - t0) * 1e3 / 3, 2),
                          "device_ms": round(e0.elapsed_time(e1) / 3, 2)}), flush=True)
bc.set_ntt_impl(0)
