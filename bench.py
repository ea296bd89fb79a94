#!/usr/bin/env python
"""bench.py -- batched encrypted comparison throughput on B200 (BASELINE.json metric).

Step = one compare_lt (all §8(a) rows: extraction, digit circuits, lexicographic
combination, key switching, modulus switching, Bluestein NTTs) over a batch of ciphertext
pairs already resident in HBM.  Default workload: C2 = Table 3 p5 univariate, 64-bit words,
1000 ciphertext pairs per GPU (weak scaling; pairs are sharded, no collective on the path).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl product|reference]

Under torchrun (N > 1) every rank runs its own batch; timing = max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted slot-comparisons/s and ms per ciphertext compare_lt at 1/2/4/8 B200"
SEED_KEYS, SEED_INPUT, SEED_ENC = 0xB00C0001, 0xB00C0002, 0xB00C0003


def load_json(p):
    with open(p) as f:
        return json.load(f)


def shard(rank, world, pairs):
    """Weak scaling: rank r owns global pairs [r*pairs, (r+1)*pairs); its a-ciphertexts use global
    ciphertext indices [2*pairs*r, 2*pairs*r + pairs) and its b-ciphertexts the next `pairs`
    (the counter-based sampler makes every ciphertext independent of the rank layout, R7)."""
    base = 2 * pairs * rank
    return {"pair0": rank * pairs, "ct_a0": base, "ct_b0": base + pairs, "input_seed": SEED_INPUT + rank}


def max_over_ranks(x, world, device=None):
    """max of a per-rank float over the process group (the timing rule: max over ranks)."""
    if world <= 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------
# CPU oracle baseline (bounded sample, extrapolated by the oracle's own operation count)
# ------------------------------------------------------------------------------------------
def oracle_sample(cfg, budget_s=20.0):
    """Time the oracle's dominant primitive (schoolbook product mod (q, Phi_m) at the full ring)
    and extrapolate a compare_lt by counting the oracle's ring products for the schedule."""
    from oracle import bgv, circuits
    from oracle.cyclo import Ring
    import oracle._c as oc
    P = bgv.Params(cfg)
    rng = np.random.default_rng(1)
    q = P.moduli[0]
    a = rng.integers(0, q, size=P.n, dtype=np.uint64)
    b = rng.integers(0, q, size=P.n, dtype=np.uint64)
    t0 = time.perf_counter()
    reps = 0
    while True:
        P.ring.mul(a, b, q)
        reps += 1
        if time.perf_counter() - t0 > budget_s / 2 or reps >= 8:
            break
    t_mul = (time.perf_counter() - t0) / reps
    count = circuits_product_count(P)
    cores = os.cpu_count()
    try:
        import ctypes
        cores = int(os.environ.get("OMP_NUM_THREADS", cores))
    except Exception:
        pass
    return t_mul, count, reps, cores


def circuits_product_count(P):
    """ring products (per limb) an oracle compare_lt makes, counted by running the schedule on
    a cost evaluator that mirrors oracle/bgv.py operation by operation."""
    from oracle import circuits

    class CV:
        def __init__(self, lvl, parts=2):
            self.level, self.parts = lvl, parts

    class CostEval:
        def __init__(self):
            self.p = P.p
            self.alg = None
            self.n = 0

        def _ms(self, x, lvl):
            return CV(lvl)

        def ks(self, lvl):
            nd = sum(1 for j in range(P.dnum) if P.digit_group(j, lvl))
            self.n += nd * (lvl + P.K) * 2

        def mul(self, a, b):
            lv = min(a.level, b.level)
            self.n += 4 * lv
            self.ks(lv)
            return CV(lv - 1)

        def add(self, a, b):
            return CV(min(a.level, b.level))

        def scalar(self, a, c):
            return CV(a.level)

        def add_const(self, a, c):
            return CV(a.level)

        def ptmul(self, a, s):
            self.n += 2 * a.level
            return CV(a.level)

        def add_pt(self, a, s):
            return CV(a.level)

        def rotate(self, a, k):
            self.ks(a.level)
            return CV(a.level)

        def frobenius(self, a, k):
            self.ks(a.level)
            return CV(a.level)

    class AlgStub:
        def __init__(self):
            self.S = 1
            self.D = P.alg.D if P.n < 5000 else _ord(P.p, P.m)

    def _ord(p, m):
        k, x = 1, p % m
        while x != 1:
            x = x * p % m
            k += 1
        return k

    ev = CostEval()
    alg = AlgStub()
    ev.alg = alg
    # replace mask / kappa constructors by stubs (cost only)
    orig_mask, orig_kappa = circuits.block_mask, circuits.kappa_slots
    circuits.block_mask = lambda *a, **k: np.zeros((1, 2), dtype=np.int64)
    circuits.kappa_slots = lambda *a, **k: np.zeros((1, 2), dtype=np.int64)
    try:
        circuits.compare(ev, CV(P.L1), CV(P.L1), P.circuit, P.d, P.l, 1)
    finally:
        circuits.block_mask, circuits.kappa_slots = orig_mask, orig_kappa
    return ev.n


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return
    steps = []
    info = None
    for i in range(args.warmup + args.steps):
        t_mul, count, reps, cores = oracle_sample(cfg, budget_s=6.0)
        if i >= args.warmup:
            steps.append(t_mul * count)
        info = (t_mul, count, reps, cores)
    t_cmp = float(np.mean(steps))
    from oracle import bgv
    P = bgv.Params(cfg)
    ints = P.ints_per_ct if P.n < 5000 else None
    if ints is None:
        from oracle.nt import mult_order
        ints = (P.n // mult_order(P.p, P.m)) // P.l
    val = ints / t_cmp
    line = {"metric": METRIC, "value": val, "unit": "int-compares/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t_cmp,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": {"workload": cfg["name"], "pairs_per_step": 1,
                                           "note": "oracle compare_lt extrapolated from timed primitives"},
            "cpu_baseline": {"value": val, "unit": "int-compares/s", "cores": info[3], "kind": "oracle",
                             "sample": "%d schoolbook ring products mod (q, Phi_m) at n=%d timed (%.3f s each) "
                                       "x %d products per compare_lt (oracle op count)" %
                                       (info[2], P.n, info[0], info[1])},
            "e2e": {"value": val, "unit": "int-compares/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--pairs", type=int, default=1000)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verify", type=int, default=1)
    args = ap.parse_args()
    cfg = load_json(os.path.join(ROOT, "params", args.config + ".json"))
    rank, world, local = dist_env()

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2407_07308_b200 as bc
    from inputs import word_pairs

    ctx = bc.Context(cfg, device=local)
    keys = ctx.keygen(SEED_KEYS)
    ints = ctx.ints_per_ct
    B = args.pairs
    # shard: rank r owns global pairs [r*B, (r+1)*B) (weak scaling, no collective on the path)
    sh = shard(rank, world, B)
    rng = np.random.default_rng(sh["input_seed"])
    A, Bw = word_pairs(rng, B * ints, ctx.base, ctx.d * ctx.l)
    A = np.array(A, dtype=np.uint64).reshape(B, ints)
    Bw = np.array(Bw, dtype=np.uint64).reshape(B, ints)
    ws = ctx.workspace(max(ctx.workspace_bytes(1), 4 << 30))
    ca = ctx.encrypt(keys, A, SEED_ENC, ct_index0=sh["ct_a0"], ws=ws)
    cb = ctx.encrypt(keys, Bw, SEED_ENC, ct_index0=sh["ct_b0"], ws=ws)
    lvl_out = ctx.out_level(ctx.n_cipher, 0)
    out = ctx.ct_empty(B, lvl_out)
    free, total = torch.cuda.mem_get_info(dev)
    need1 = ctx.workspace_bytes(1)
    ws_bytes = int(min(max(need1, int(free * 0.80)), free - (2 << 30)))
    ws = ctx.workspace(ws_bytes)
    wsp = bc._ptr(ws)
    st = bc._stream

    def step(a, b, o):
        bc._check(bc._lib.bc_compare_lt(ctx._h, keys.keys, ctx.view(a), ctx.view(b), ctx.view(o), wsp,
                                        ws.numel(), st()), "bc_compare_lt")

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    verified = None
    for w in range(args.warmup):
        step(ca, cb, out)
        if w == 0 and args.verify:
            torch.cuda.synchronize()
            bits = ctx.decrypt(keys, out, as_bits=True, ws=None)
            want = (A < Bw).astype(np.uint64)
            verified = bool(np.array_equal(bits, want))
            if not verified:
                bad = int((bits != want).sum())
                print("VERIFY FAILED: %d of %d result bits wrong" % (bad, bits.size), file=sys.stderr)
                sys.exit(3)
    barrier()
    bc.launch_count(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.nvtx.range_push("step")
        e0.record()
        for _ in range(args.steps):
            step(ca, cb, out)
        e1.record()
        torch.cuda.nvtx.range_pop()
        barrier()
    launches = bc.launch_count(reset=True)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    total_pairs = B * world
    value = total_pairs * ints / (ms / 1000.0)
    clocks = clk.summary()

    # ---- e2e: host buffers through the C ABI, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        ha = ca.cpu().pin_memory()
        hb = cb.cpu().pin_memory()
        ho = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        da, db = torch.empty_like(ca), torch.empty_like(cb)
        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(args.steps):
            da.copy_(ha, non_blocking=True)
            db.copy_(hb, non_blocking=True)
            step(da, db, out)
            ho.copy_(out, non_blocking=True)
        e3.record()
        barrier()
        ms2 = max_over_ranks(e2.elapsed_time(e3) / args.steps, world, dev)
        e2e = {"value": total_pairs * ints / (ms2 / 1000.0), "unit": "int-compares/s",
               "h2d_bytes_per_step": int(ha.numel() * 8 + hb.numel() * 8),
               "d2h_bytes_per_step": int(ho.numel() * 8), "ms_per_step": ms2}

    roof = roofline(ctx, keys, bc, torch, cfg)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        t_mul, count, reps, cores = oracle_sample(cfg)
        t_cmp = t_mul * count
        cpu = {"value": ints / t_cmp, "unit": "int-compares/s", "cores": cores, "kind": "oracle",
               "sample": "%d schoolbook ring products mod (q, Phi_m) at n=%d timed (%.3f s each) x %d products "
                         "per compare_lt (oracle op count); extrapolated" % (reps, ctx.n, t_mul, count)}
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "int-compares/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": "C2: Table 3 p5 univariate (p=13, m=30941, (d,l)=(4,6), 64-bit words), "
                                       "%d ciphertext pairs per GPU" % B if args.config == "c2" else args.config,
                           "params": args.config, "pairs_per_gpu": B, "ints_per_ct": ints,
                           "n_cipher": ctx.n_cipher, "n_special": ctx.n_special, "alpha": cfg["alpha"],
                           "l2": "inputs (%.1f GB) larger than L2 (126 MB)" % (2 * ca.numel() * 8 / 1e9)},
                "ms_per_ct_compare": ms / B, "slot_compares_per_s": total_pairs * ctx.S / (ms / 1000.0),
                "verified": verified, "gpu_launches": launches, "clocks": clocks,
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def roofline(ctx, keys, bc, torch, cfg):
    """Dominant kernel (Bluestein NTT passes, integer-pipe bound): algorithmic 64-bit modular
    multiplications per launch / measured duration vs the IMAD-derived peak."""
    try:
        prof = bc.profile_ntt(ctx)
    except Exception as e:  # pragma: no cover
        return {"bound": "alu", "error": str(e)}
    return prof


if __name__ == "__main__":
    main()
