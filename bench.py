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
# CPU oracle baseline: a bounded sample of the SAME workload, timed as it stands
# ------------------------------------------------------------------------------------------
def host_info():
    """CPU model, logical cores, clock and the threads the oracle's OpenMP helper uses."""
    model, mhz = None, []
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name") and model is None:
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("cpu MHz"):
                    mhz.append(float(line.split(":", 1)[1]))
    except OSError:
        pass
    n = os.cpu_count() or 1
    threads = int(os.environ.get("OMP_NUM_THREADS", n))
    return {"cpu_model": model, "nproc": n, "cpu_mhz": float(np.median(mhz)) if mhz else None,
            "omp_threads": threads}


class OracleSample:
    """One real operation of the compare_lt schedule, at the benchmarked configuration's full size:
    the oracle's R15 product (tensor, ModUp with exact big-integer CRT lifts, key inner product,
    fused ModDown + modulus switch) of two full-size ciphertexts at level 2 -- the last product of
    the schedule.  Ring products dominate the oracle (schoolbook, O(n^2)); the sample's count is
    checked against the oracle's own call counter, and the compare_lt's count comes from running
    the R16 schedule on a cost evaluator (circuits_product_count, checked against the counter on
    C2's shadow ring in tests/test_bench_host.py).  The compare time is extrapolated as
    (sample time / sample products) x compare products and labelled as such."""

    def __init__(self, cfg, level=2):
        from oracle import bgv
        self.bgv = bgv
        P = bgv.Params(cfg)
        self.P = P
        t0 = time.perf_counter()
        self.K = bgv.keygen(P, SEED_KEYS, (), relin=True)
        z = np.zeros(P.n, dtype=np.int64)                  # the product's cost does not depend on the message
        self.a = bgv.modswitch_to(P, bgv.encrypt(P, self.K, z, SEED_ENC, 0), level)
        self.b = bgv.modswitch_to(P, bgv.encrypt(P, self.K, z, SEED_ENC, 1), level)
        self.setup_s = time.perf_counter() - t0
        self.level = level
        ndig = sum(1 for j in range(P.dnum) if P.digit_group(j, level))
        self.products = 4 * level + 2 * ndig * (level + P.K)
        self.compare_products = circuits_product_count(P)

    def run(self):
        import oracle._c as oc
        c0 = oc.CALLS["ring_mul"]
        t0 = time.perf_counter()
        self.bgv.mul(self.P, self.K, self.a, self.b)
        dt = time.perf_counter() - t0
        assert oc.CALLS["ring_mul"] - c0 == self.products, "oracle product count changed"
        return dt

    def describe(self, t):
        P = self.P
        return ("oracle R15 product (tensor + ModUp/KIP + fused ModDown/modswitch, big-integer CRT lifts) of two "
                "full-size ciphertexts at level %d (n=%d, %d+%d primes): %d schoolbook ring products, %.2f s; "
                "= %.5f of one compare_lt (%d ring products by the oracle's schedule)"
                % (self.level, P.n, P.L1, P.K, self.products, t, self.products / self.compare_products,
                   self.compare_products))

    def extrapolated_compare_s(self, t):
        return t / self.products * self.compare_products


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

        def frobenius_hoisted(self, a, ks):
            for _ in ks:
                self.ks(a.level)
            return [CV(a.level) for _ in ks]

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
    """--impl reference: the oracle as it stands on the host cores (rank 0 only; other ranks exit).
    Each step runs one real operation of the compare_lt workload at full size (OracleSample); the
    line reports the measured step time and the fraction of a compare_lt it covers, so
    value = units_per_step / step time with units = int-compares (fraction x ints per ciphertext)."""
    if rank != 0:
        return
    S = OracleSample(cfg)
    times = []
    for i in range(args.warmup + args.steps):
        t = S.run()
        if i >= args.warmup:
            times.append(t)
    t_step = float(np.mean(times))
    ints = compare_ints(cfg, S.P)
    units = ints * S.products / S.compare_products
    val = units / t_step
    hi = host_info()
    line = {"metric": METRIC, "value": val, "unit": "int-compares/s", "impl": "reference",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * t_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic", "config": product_config(args, cfg, ints),
            "units_per_step": units,
            "extrapolated_ms_per_ct_compare": 1000 * S.extrapolated_compare_s(t_step),
            "setup_s": S.setup_s,
            "cpu_baseline": dict({"value": val, "unit": "int-compares/s", "cores": hi["omp_threads"],
                                  "kind": "oracle", "sample": S.describe(t_step)}, **hi),
            "e2e": {"value": val, "unit": "int-compares/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def compare_ints(cfg, P):
    if P.n < 5000:
        return P.ints_per_ct
    from oracle.nt import mult_order
    return (P.n // mult_order(P.p, P.m)) // P.l


def product_config(args, cfg, ints, B=None):
    """the config object of the product arm's line (the reference arm prints the same one)"""
    B = B if B is not None else (args.pairs or 1000)
    return {"workload": "C2: Table 3 p5 univariate (p=13, m=30941, (d,l)=(4,6), 64-bit words), "
                        "%d ciphertext pairs per GPU" % B if args.config == "c2" else args.config,
            "params": args.config, "pairs_per_gpu": B, "ints_per_ct": ints,
            "n_cipher": cfg["n_cipher"], "n_special": cfg["n_special"], "alpha": cfg["alpha"],
            "schedule": cfg.get("schedule", "r16"),
            "l2": "inputs (%.1f GB) larger than L2 (126 MB)" % (2 * B * 2 * cfg["n_cipher"] * _n_of(cfg) * 8 / 1e9)}


def _n_of(cfg):
    from oracle.nt import euler_phi
    return euler_phi(int(cfg["m"]))


# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="product", choices=["product", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--pairs", type=int, default=None,
                    help="ciphertext pairs per GPU (default: 1000 for compare (C2), 16 dense pairs for c3 compact_compare)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=8, help="chunks of the pipelined host-buffer compare (e2e)")
    ap.add_argument("--schedule", default=None, help="override the config's digit-circuit schedule (r16/r23/r26/r27)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--verify", type=int, default=1)
    ap.add_argument("--workload", default=None,
                    choices=[None, "compare", "tournament", "sort", "compact_compare", "private_q"],
                    help="compare (default; C2), tournament (C4 min over T vectors), sort (C5 rank sort)")
    ap.add_argument("--T", type=int, default=16, help="tournament / sort: number of elements")
    ap.add_argument("--cts", type=int, default=0, help="ciphertexts per element (tournament: 5 -> 4096 words)")
    ap.add_argument("--vec-chunk", type=int, default=0, help="max ct pairs per batched compare (0 = all)")
    ap.add_argument("--exps", default="64,128,256,512,1024", help="private_q: exponents op2 swept (Fig. 14)")
    args = ap.parse_args()
    cfg = load_json(os.path.join(ROOT, "params", args.config + ".json"))
    if args.schedule:
        cfg["schedule"] = args.schedule          # digit-circuit reading override (r16 / r23 / r26 / r27)
    rank, world, local = dist_env()

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    workload = args.workload or {"c4": "tournament", "c5": "sort", "c3": "compact_compare",
                                 "p3q": "private_q"}.get(args.config, "compare")
    if args.pairs is None:
        args.pairs = 16 if workload == "compact_compare" else 1000
    if workload in ("tournament", "sort"):
        run_vector_workload(args, cfg, rank, world, local, workload)
        return
    if workload == "compact_compare":
        run_compact_compare(args, cfg, rank, world, local)
        return
    if workload == "private_q":
        run_private_q(args, cfg, rank, world, local)
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
    bc.ntt_timing(True)
    bc.ntt_timing()                      # drop anything recorded before the timed region
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
    live = bc.ntt_timing(split=True)
    bc.ntt_timing(False)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, world, dev)
    total_pairs = B * world
    # per-phase breakdown (Fig. 3 analog): one extra step with phase events (not timed above)
    phases = None
    if rank == 0:
        bc.phase_timing(True)
        bc.phase_timing()
        step(ca, cb, out)
        torch.cuda.synchronize()
        ph = bc.phase_timing()
        bc.phase_timing(False)
        tot = sum(v[0] for v in ph.values())
        phases = {k: {"ms": round(v[0], 3), "share_of_step": round(v[0] / ms_local, 4)} for k, v in ph.items() if v[1]}
        phases["unattributed_share"] = round(max(0.0, 1 - tot / ms_local), 4)
    value = total_pairs * ints / (ms / 1000.0)
    clocks = clk.summary()

    # ---- e2e: host buffers through the C ABI, copies inside the timed region ----
    e2e = None
    if not args.no_e2e:
        # bc_compare_lt_host: the public host-buffer call; its H2D / compare / D2H run pipelined in chunks
        # (copy stream + events inside the library), every copy inside the timed region
        ha = ca.cpu().pin_memory()
        hb = cb.cpu().pin_memory()
        ho = torch.empty(out.shape, dtype=out.dtype).pin_memory()
        chunk = max(1, (B + args.e2e_chunks - 1) // args.e2e_chunks)
        stage = torch.empty(int(bc._lib.bc_host_stage_bytes(ctx._h, chunk, ctx.n_cipher)), dtype=torch.uint8, device=dev)
        ctx.compare_lt_host(keys, ha, hb, ho, chunk=chunk, ws=ws, stage=stage)      # warm-up (untimed)
        torch.cuda.synchronize()
        if not torch.equal(ho, out.cpu()):
            raise SystemExit("bc_compare_lt_host words differ from bc_compare_lt")
        barrier()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record()
        for _ in range(args.steps):
            ctx.compare_lt_host(keys, ha, hb, ho, chunk=chunk, ws=ws, stage=stage)
        e3.record()
        barrier()
        ms2 = max_over_ranks(e2.elapsed_time(e3) / args.steps, world, dev)
        e2e = {"value": total_pairs * ints / (ms2 / 1000.0), "unit": "int-compares/s",
               "h2d_bytes_per_step": int(ha.numel() * 8 + hb.numel() * 8),
               "d2h_bytes_per_step": int(ho.numel() * 8), "ms_per_step": ms2,
               "how": "bc_compare_lt_host on pinned host buffers: %d chunks of %d pairs, host->device copy of the "
                      "next chunk and device->host copy of the previous one on a copy stream while a chunk is "
                      "compared; words checked equal to bc_compare_lt" % ((B + chunk - 1) // chunk, chunk)}
        del stage

    # ---- single-pair latency, eager and replayed as a CUDA graph (bc_graph_*) ----
    latency = None
    if rank == 0 and not args.no_e2e:
        a1, b1, o1 = ca[:1].clone(), cb[:1].clone(), out[:1].clone()
        cap = torch.cuda.Stream(device=dev)
        res = {}
        with torch.cuda.stream(cap):
            for _ in range(2):
                step(a1, b1, o1)
            cap.synchronize()
            g = bc.Graph()
            with g:
                step(a1, b1, o1)
            for nm, fn in (("eager_ms", lambda: step(a1, b1, o1)), ("graph_ms", g.launch)):
                fn()
                cap.synchronize()
                l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                l0.record()
                for _ in range(5):
                    fn()
                l1.record()
                cap.synchronize()
                res[nm] = l0.elapsed_time(l1) / 5
            ok1 = bool(torch.equal(o1[0], out[0]))
        latency = dict(res, pairs=1, identical_to_batch=ok1, launches_per_compare=int(launches / args.steps))

    # ---- keygen / encrypt / decrypt, timed separately (reported, not counted) ----
    client = None
    if not args.no_e2e:
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        _ = ctx.encrypt(keys, A, SEED_ENC, ct_index0=sh["ct_a0"], ws=ws)
        ev[1].record()
        _ = ctx.decrypt(keys, out, as_bits=True, ws=ws)
        ev[2].record()
        barrier()
        import time as _time
        t0 = _time.perf_counter()
        k2 = ctx.keygen(SEED_KEYS)
        torch.cuda.synchronize()
        kg_ms = 1000 * (_time.perf_counter() - t0)
        del k2
        client = {"encrypt_ms_per_ct": ev[0].elapsed_time(ev[1]) / B,
                  "decrypt_bits_ms_per_ct": ev[1].elapsed_time(ev[2]) / B,
                  "keygen_ms": kg_ms, "n_galois_keys": ctx.n_galois,
                  "note": "encode (int8 slot-basis GEMM) + public-key encryption of one ct of %d words; decrypt = "
                          "s-dot-product + exact CRT + decode of the result bits (host wall time for keygen)" % ints}

    roof = roofline(ctx, bc, live, ms_local * args.steps)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        S = OracleSample(cfg)
        t = S.run()
        units = ints * S.products / S.compare_products
        cpu = dict({"value": units / t, "unit": "int-compares/s", "cores": host_info()["omp_threads"],
                    "kind": "oracle", "sample": S.describe(t),
                    "extrapolated_ms_per_ct_compare": 1000 * S.extrapolated_compare_s(t)}, **host_info())
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "int-compares/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": product_config(args, cfg, ints, B),
                "ms_per_ct_compare": ms / B, "slot_compares_per_s": total_pairs * ctx.S / (ms / 1000.0),
                "verified": verified, "gpu_launches": launches, "clocks": clocks,
                "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "client_ops": client, "phases": phases,
                "single_pair_latency": latency}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_vector_workload(args, cfg, rank, world, local, workload):
    """C4: slot-wise min over T encrypted vectors of 4096 32-bit words (T x 4096 = 2^16 words at T = 16),
    R20 fixed tree; elements sharded contiguously over ranks, cross-rank rounds via NCCL send/recv
    (paper_2407_07308_b200/dist.py) -> strong scaling (total work fixed).
    C5: R21 rank sort of T = 16 encrypted elements per GPU (one ciphertext each: ints_per_ct
    independent groups of 16 words) -> weak scaling, no collective."""
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2407_07308_b200 as bc
    from paper_2407_07308_b200 import dist as bdist
    ctx = bc.Context(cfg, device=local)
    keys = ctx.keygen(SEED_KEYS)
    ints = ctx.ints_per_ct
    T = args.T
    if args.vec_chunk:
        bc._lib.bc_tune(b"vec_chunk", args.vec_chunk)
    cap = min(ctx.base ** (ctx.d * ctx.l), 2 ** 64)
    if workload == "tournament":
        V = args.cts or 5
        words_per_vec = min(4096, V * ints)
        lo, hi = bdist.shard(T, world, rank)
        rng = np.random.default_rng(SEED_INPUT)            # every rank regenerates all vectors (verify on rank 0)
        W = rng.integers(0, cap, size=(T, V * ints), dtype=np.uint64)
        W[:, words_per_vec:] = 0
        mine = list(range(lo, hi))
    else:
        V = args.cts or 1
        rng = np.random.default_rng(SEED_INPUT + rank)
        W = rng.integers(0, cap, size=(T, V * ints), dtype=np.uint64)
        W[:, ::7] = W[0, ::7]                              # ties (stable by index)
        mine = list(range(T))
    elems = [ctx.encrypt(keys, W[t].reshape(V, ints), SEED_ENC,
                         ct_index0=(t if workload == "tournament" else rank * T + t) * V) for t in mine]
    levels = [ctx.n_cipher] * len(elems)
    op = "min" if workload == "tournament" else "sort"
    need = ctx.vec_workspace_bytes(op, levels, V) if len(elems) > 1 else 0
    if workload == "tournament":
        need = max(need, ctx.workspace_bytes(V))
    free, _ = torch.cuda.mem_get_info(dev)
    vc = args.vec_chunk
    while need > free - (1 << 30) and not args.vec_chunk and len(elems) > 1:
        # the batched pairwise compares do not fit: cap the ciphertext pairs per batched compare (halving)
        vc = (T * (T - 1) // 2 if vc == 0 else vc) // 2
        if vc < 1:
            break
        bc._lib.bc_tune(b"vec_chunk", vc)
        need = ctx.vec_workspace_bytes(op, levels, V)
        if workload == "tournament":
            need = max(need, ctx.workspace_bytes(V))
    args.vec_chunk = vc
    if need > free - (1 << 30):
        raise SystemExit("workspace %.1f GB > free %.1f GB: use --vec-chunk" % (need / 1e9, free / 1e9))
    ctx.workspace(need)
    ops = bdist.ProductOps(ctx, keys)

    def step():
        if workload == "tournament":
            return bdist.tournament(ops, elems, "min")
        return ctx.sort(keys, elems)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    verified = None
    for w in range(args.warmup):
        r = step()
        if w == 0 and args.verify:
            torch.cuda.synchronize()
            if workload == "tournament":
                if rank == 0:
                    got = ctx.decrypt(keys, r).reshape(-1)
                    verified = bool(np.array_equal(got, W.min(axis=0)))
            else:
                got = np.stack([ctx.decrypt(keys, o).reshape(-1) for o in r])
                verified = bool(np.array_equal(got, np.sort(W, axis=0)))
            if verified is False:
                print("VERIFY FAILED", file=sys.stderr)
                sys.exit(3)
    barrier()
    bc.launch_count(reset=True)
    bc.ntt_timing(True)
    bc.ntt_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record()
        torch.cuda.nvtx.range_push("step")
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.nvtx.range_pop()
        barrier()
    launches = bc.launch_count(reset=True)
    live = bc.ntt_timing(split=True)
    bc.ntt_timing(False)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, world, dev)
    if workload == "tournament":
        words = T * words_per_vec
        line = {"metric": "encrypted min over %d 32-bit words (R20 tournament, %d vectors)" % (words, T),
                "value": words / (ms / 1e3), "unit": "words/s", "scaling": "strong",
                "ms_per_tournament": ms}
    else:
        words = world * T * V * ints
        line = {"metric": "encrypted rank sort of groups of %d 32-bit words (R21)" % T,
                "value": words / (ms / 1e3), "unit": "words sorted/s", "scaling": "weak",
                "ms_per_sort": ms, "groups_per_gpu": V * ints}
    if rank == 0:
        line.update({"n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                     "higher_is_better": True, "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                     "config": {"workload": args.config + " " + workload, "params": args.config, "T": T,
                                "cts_per_element": V, "ints_per_ct": ints, "n_cipher": ctx.n_cipher,
                                "n_special": ctx.n_special, "alpha": cfg["alpha"], "vec_chunk": args.vec_chunk,
                                "l2": "inputs larger than L2"},
                     "verified": verified, "gpu_launches": launches, "clocks": clk.summary(),
                     "roofline": roofline(ctx, bc, live, ms_local * args.steps), "e2e": None,
                     "cpu_baseline": None})
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_compact_compare(args, cfg, rank, world, local):
    """C3: sparse ciphertext pairs at 25% block utilisation (blocks = 3 mod 4 useful, Fig. 7) are
    compacted 4 -> 1 (R17: one mask product + rotation per (block set, offset) bucket, one batched
    modulus switch), then the dense pairs are compared (bivariate circuit).  --pairs = dense pairs
    per GPU (4x as many sparse pairs); weak scaling, no collective."""
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
    Bd = args.pairs
    Bs = 4 * Bd
    rng = np.random.default_rng(SEED_INPUT + rank)
    A, Bw = word_pairs(rng, Bs * ints, ctx.base, ctx.d * ctx.l)
    A = np.array(A, dtype=np.uint64).reshape(Bs, ints)
    Bw = np.array(Bw, dtype=np.uint64).reshape(Bs, ints)
    useful = np.zeros((Bs, ints), dtype=np.uint8)
    useful[:, 3::4] = 1
    A[useful == 0] = 0
    Bw[useful == 0] = 0
    base = 2 * Bs * rank
    ws = ctx.workspace(max(ctx.workspace_bytes(1), 4 << 30))
    ca = ctx.encrypt(keys, A, SEED_ENC, ct_index0=base, ws=ws)
    cb = ctx.encrypt(keys, Bw, SEED_ENC, ct_index0=base + Bs, ws=ws)
    free, _ = torch.cuda.mem_get_info(dev)
    ws = ctx.workspace(int(min(max(ctx.workspace_bytes(1), int(free * 0.80)), free - (2 << 30))))
    lvl_c = ctx.n_cipher - 1
    lvl_out = ctx.out_level(lvl_c, 0)
    out = ctx.ct_empty(Bd, lvl_out)
    da, db = ctx.ct_empty(Bd + 2, lvl_c), ctx.ct_empty(Bd + 2, lvl_c)   # Fig. 7 pattern: 4 -> 1
    dest = np.zeros((Bs, ints), dtype=np.int32)
    nout = bc._u32(0)
    uptr = useful.ctypes.data
    wsp = bc._ptr(ws)

    def step():
        for src, dst in ((ca, da), (cb, db)):
            bc._check(bc._lib.bc_compact(ctx._h, keys.keys, ctx.view(src), uptr, ctx.view(dst), bc.ctypes.byref(nout),
                                         dest.ctypes.data, wsp, ws.numel(), bc._stream()), "bc_compact")
        n = nout.value
        bc._check(bc._lib.bc_compare_lt(ctx._h, keys.keys, ctx.view(da[:n]), ctx.view(db[:n]), ctx.view(out[:n]), wsp,
                                        ws.numel(), bc._stream()), "bc_compare_lt")
        return n

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    verified = None
    for w in range(args.warmup):
        n = step()
        if w == 0 and args.verify:
            torch.cuda.synchronize()
            bits = ctx.decrypt(keys, out[:n], as_bits=True)
            ok = True
            for c in range(Bs):
                for j in range(3, ints, 4):
                    ct_i, blk = divmod(int(dest[c, j]), ints)
                    ok &= int(bits[ct_i][blk]) == int(A[c, j] < Bw[c, j])
            verified = bool(ok and n == Bd)
            if not verified:
                print("VERIFY FAILED (n_out %d)" % n, file=sys.stderr)
                sys.exit(3)
    barrier()
    bc.launch_count(reset=True)
    bc.ntt_timing(True)
    bc.ntt_timing()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record()
        torch.cuda.nvtx.range_push("step")
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.nvtx.range_pop()
        barrier()
    launches = bc.launch_count(reset=True)
    live = bc.ntt_timing(split=True)
    bc.ntt_timing(False)
    ms_local = e0.elapsed_time(e1) / args.steps
    ms = max_over_ranks(ms_local, world, dev)
    useful_ints = int(useful.sum()) * world
    phases = None
    if rank == 0:
        bc.phase_timing(True)
        bc.phase_timing()
        step()
        torch.cuda.synchronize()
        ph = bc.phase_timing()
        bc.phase_timing(False)
        tot = sum(v[0] for v in ph.values())
        phases = {k: {"ms": round(v[0], 3), "share_of_step": round(v[0] / ms_local, 4)} for k, v in ph.items() if v[1]}
        phases["unattributed_share"] = round(max(0.0, 1 - tot / ms_local), 4)
    if rank == 0:
        line = {"metric": "encrypted slot-comparisons/s after slot compaction (C3, bivariate p=31)",
                "value": useful_ints / (ms / 1e3), "unit": "int-compares/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {"workload": "c3 compact_compare", "params": args.config, "sparse_pairs_per_gpu": Bs,
                           "dense_pairs_per_gpu": Bd, "ints_per_ct": ints, "utilisation": 0.25,
                           "n_cipher": ctx.n_cipher, "n_special": ctx.n_special, "alpha": cfg["alpha"],
                           "l2": "inputs larger than L2"},
                "ms_per_dense_compare": ms / Bd, "verified": verified, "gpu_launches": launches,
                "clocks": clk.summary(), "roofline": roofline(ctx, bc, live, ms_local * args.steps), "e2e": None,
                "cpu_baseline": None, "phases": phases}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_private_q(args, cfg, rank, world, local):
    """f4 private_q (Listings 3-5, R24): a database of --pairs ciphertexts (default 100) on the p3
    ring; one step = one private query (3 EQs + broadcasts, Data + op1, Data * op1, Data^e, combination),
    blocking (Listing 4, one stream) and non-blocking (Listing 5: the EQs on a second stream), for every
    exponent of --exps (Fig. 14).  Both are checked bit-identical and by decryption in warm-up.  Weak
    scaling over ranks (each rank its own database shard, no collective)."""
    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    import paper_2407_07308_b200 as bc
    ctx = bc.Context(cfg, device=local)
    keys = ctx.keygen(SEED_KEYS)
    N = args.pairs if args.pairs and args.pairs != 1000 else 100
    ints = ctx.ints_per_ct
    rng = np.random.default_rng(SEED_INPUT + rank)
    X = np.zeros((N, ctx.S, ctx.D), dtype=np.int16)
    X[:, :, 0] = rng.integers(0, ctx.p, (N, ctx.S))
    Y = np.zeros((1, ctx.S, ctx.D), dtype=np.int16)
    Y[:, :, 0] = rng.integers(0, ctx.p, (1, ctx.S))
    base = (N + 8) * rank
    data = ctx.encrypt_slots(keys, X, SEED_ENC, ct_index0=base)
    op1 = ctx.encrypt_slots(keys, Y, SEED_ENC, ct_index0=base + N)
    qv = 3                                   # the power branch (the expensive one, Fig. 14)
    q = ctx.encrypt(keys, np.array([[qv] * ints], dtype=np.uint64), SEED_ENC, ct_index0=base + N + 1)
    codes = ctx.encrypt(keys, np.array([[c] * ints for c in (1, 2, 3)], dtype=np.uint64), SEED_ENC,
                        ct_index0=base + N + 2)
    side = torch.cuda.Stream(device=dev, priority=-1)   # the branch evaluation first when SMs free up
    exps = [int(x) for x in args.exps.split(",")]
    emax = max(exps)
    wsm = ctx.workspace(int(bc._lib.bc_private_query_workspace_bytes(ctx._h, N, data.shape[2], q.shape[2],
                                                                     op1.shape[2], emax, 0)))
    wss = torch.empty(int(bc._lib.bc_private_query_workspace_bytes(ctx._h, N, data.shape[2], q.shape[2],
                                                                   op1.shape[2], emax, 1)), dtype=torch.uint8,
                      device=dev)
    S1 = ctx.S // 2 if cfg["m"] == 20197 else ctx.S
    rows = []

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()

    def timed(fn):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            fn()
        e1.record()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)

    verified = True
    launches = {}
    q3 = torch.cat([q, q, q])
    lvl_eq = ctx.out_level(q.shape[2], 1)
    eq_out = ctx.ct_empty(3, lvl_eq)
    with ClockSampler(local) as clk:
        for e in exps:
            lvl = int(bc._lib.bc_private_query_level(ctx._h, N, data.shape[2], q.shape[2], op1.shape[2], e))
            out_b, out_n = ctx.ct_empty(N, lvl), ctx.ct_empty(N, lvl)
            blk = lambda: ctx.private_query(keys, data, q, codes, op1, e, ws=wsm, out=out_b)             # noqa: E731
            nbl = lambda: ctx.private_query(keys, data, q, codes, op1, e, side_stream=side, ws=wsm,      # noqa: E731
                                            ws_side=wss, out=out_n)
            eqo = lambda: bc._check(bc._lib.bc_compare_eq(ctx._h, keys.keys, ctx.view(q3), ctx.view(codes),  # noqa
                                                          ctx.view(eq_out), bc._ptr(wsm), wsm.numel(), bc._stream()),
                                    "bc_compare_eq")
            for w in range(args.warmup):
                blk()
                nbl()
                eqo()
                if w == 0 and args.verify:
                    torch.cuda.synchronize()
                    same = bool(torch.equal(out_b, out_n))
                    dec = ctx.decrypt_slots(keys, out_n[: min(N, 4)])
                    want = np.vectorize(lambda t: pow(int(t), e, ctx.p))(X[: min(N, 4), :, 0].astype(np.int64))
                    cov = np.array([(s % S1) < (S1 // ctx.l) * ctx.l for s in range(ctx.S)])
                    ok = same and np.array_equal(dec[:, cov, 0], want[:, cov])
                    verified &= bool(ok)
                    if not ok:
                        print("VERIFY FAILED (exponent %d, identical %s)" % (e, same), file=sys.stderr)
                        sys.exit(3)
            bc.launch_count(reset=True)
            tb = timed(blk)
            launches[e] = bc.launch_count(reset=True) // args.steps
            tn = timed(nbl)
            tc = timed(eqo)
            # the same three calls captured once as CUDA graphs (host planning and launches not repeated)
            graphs = {}
            cap = torch.cuda.Stream(device=dev)
            torch.cuda.synchronize()
            with torch.cuda.stream(cap):
                for nm, fn in (("b", blk), ("n", nbl), ("c", eqo)):
                    g = bc.Graph()
                    with g:
                        fn()
                    graphs[nm] = g
            torch.cuda.synchronize()
            with torch.cuda.stream(cap):
                ref_b = out_b.clone()
                graphs["n"].launch()
                cap.synchronize()
                gsame = bool(torch.equal(out_n, ref_b))
                graphs["b"].launch()
                cap.synchronize()
                gsame &= bool(torch.equal(out_b, ref_b))
            if not gsame:
                print("VERIFY FAILED (graph replay, exponent %d)" % e, file=sys.stderr)
                sys.exit(3)
            with torch.cuda.stream(cap):
                tgb = timed(graphs["b"].launch)
                tgn = timed(graphs["n"].launch)
                tgc = timed(graphs["c"].launch)
            rows.append({"exponent": e, "blocking_ms": tb, "nonblocking_ms": tn, "branch_eval_ms": tc,
                         "hidden_ms": tb - tn, "speedup": tb / tn,
                         "graph": {"blocking_ms": tgb, "nonblocking_ms": tgn, "branch_eval_ms": tgc,
                                   "hidden_ms": tgb - tgn, "hidden_frac_of_branch": (tgb - tgn) / tgc if tgc else None,
                                   "speedup": tgb / tgn}})
    if rank == 0:
        last = rows[-1]
        line = {"metric": "private_q queries/s (database of %d ciphertexts x %d slots, non-blocking comparison, "
                          "CUDA graph)" % (N, ctx.S),
                "value": world * 1e3 / last["graph"]["nonblocking_ms"], "unit": "queries/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": last["graph"]["nonblocking_ms"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic",
                "config": {"workload": "f4 private_q (P:670, Listings 3-5, R24)", "params": args.config,
                           "m": cfg["m"], "database_cts": N, "slots_per_ct": ctx.S, "query": "power (q = 3)",
                           "exponent": last["exponent"], "n_cipher": ctx.n_cipher, "l2": "inputs larger than L2"},
                "sweep": rows, "verified": verified, "gpu_launches_blocking": launches,
                "clocks": clk.summary(), "roofline": None, "e2e": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def roofline(ctx, bc, live, step_ms_total):
    """Dominant kernel family (Bluestein NTT passes, integer-pipe bound), measured LIVE in the timed
    region: CUDA event pairs around every NTT call on the launching stream (bc_ntt_timing).
    achieved = limb-transforms x algorithmic 64-bit modular multiplications per limb-transform
     / summed NTT time; peak = FP64-pipe modular-butterfly rate at the max SM clock."""
    if len(live) == 4:
        ms, jobs, inv_jobs, calls = live
    else:
        (ms, jobs, calls), inv_jobs = live, 0
    if not calls or ms <= 0:
        return {"bound": "alu", "error": "no NTT calls timed"}
    work = bc.ntt_work(ctx)
    bw = bc.barrett_work(ctx)       # composite m: the Barrett division inside every inverse (C3)
    achieved = (jobs * work + inv_jobs * bw) / (ms / 1e3) / 1e12
    peak = bc.ntt_peak(1965.0)
    traffic = None
    try:
        prof = load_json(os.path.join(ROOT, "profiles", "ntt_traffic.json"))
        if prof.get("n") == ctx.n:
            traffic = prof["dram_bytes_per_limb_transform"] * jobs / calls
    except Exception:
        traffic = None
    return {"bound": "alu", "kernel": "bluestein_ntt (passA+passB+passC [+reduce]) per ntt_forward/ntt_inverse call",
            "achieved": achieved, "peak": peak, "unit": "T modmul/s", "frac": achieved / peak,
            "traffic": traffic, "per_launch_ms": ms / calls, "limb_transforms_per_launch": jobs / calls,
            "work_per_limb_transform": work, "barrett_work_per_inverse": bw, "inverse_limb_transforms": inv_jobs,
            "launches_timed": calls, "share_of_step": ms / step_ms_total,
            "how": "CUDA events on the launching stream around every NTT call inside the timed region",
            "traffic_note": "ncu --set full dram__bytes_read+write per limb-transform (profiles/ntt_traffic.json) x "
                            "limb-transforms per call",
            "peak_note": "148 SM x 64 DFMA/clk (measured 18.2e12/s, tools/micro/bfly_micro.cu) x 1965 MHz / %d "
                         "binary64 ops per modular butterfly (ntt3.cu)" % bc.FP64_PER_MODBFLY}


if __name__ == "__main__":
    main()
