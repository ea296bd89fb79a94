"""World-size-2 host-side path of the multi-GPU bench on CPU (gloo): sharding of ciphertext pairs,
bit-identical key regeneration per rank, independent per-rank compare (oracle on C1 stands in for
the device), max-over-ranks timing and the aggregated result check on rank 0."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import json
    import hashlib
    import bench
    from inputs import word_pairs
    from oracle import bgv, circuits, slots
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    cfg = json.load(open(os.path.join(ROOT, "params", "c1.json")))
    P = bgv.Params(cfg)
    A = P.alg
    gal = [pow(P.p, k, P.m) for k in range(1, A.D)]
    K = bgv.keygen(P, bench.SEED_KEYS, gal)
    pairs = 2
    sh = bench.shard(rank, world, pairs)
    rng = np.random.default_rng(sh["input_seed"])
    ints = P.ints_per_ct
    a, b = word_pairs(rng, pairs * ints, P.base, P.d * P.l)
    ev = circuits.OracleEval(P, K)
    bits = []
    for i in range(pairs):
        wa, wb = a[i * ints:(i + 1) * ints], b[i * ints:(i + 1) * ints]
        ca = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wa, A, P.d, P.l, P.base)), bench.SEED_ENC, sh["ct_a0"] + i)
        cb = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wb, A, P.d, P.l, P.base)), bench.SEED_ENC, sh["ct_b0"] + i)
        lt, _ = circuits.compare(ev, ca, cb, P.circuit, P.d, P.l, ints)
        dec = A.decode(bgv.decrypt(P, K, lt))
        bits += [int(dec[j * P.l, 0]) for j in range(ints)]
    key_hash = hashlib.sha256(K.pk[0].tobytes() + K.ksk[0][0][0].tobytes()).hexdigest()
    mx = bench.max_over_ranks(float(rank + 1) * 1.5, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, {"rank": rank, "bits": bits, "want": [int(x < y) for x, y in zip(a, b)],
                                      "cts": list(range(sh["ct_a0"], sh["ct_a0"] + pairs)) +
                                             list(range(sh["ct_b0"], sh["ct_b0"] + pairs)),
                                      "key": key_hash, "max": mx})
    if rank == 0:
        out.put(gathered)
    dist.destroy_process_group()


def test_two_rank_sharded_compare_gloo():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len({r["key"] for r in res}) == 1                    # bit-identical keys on every rank
    cts = [c for r in res for c in r["cts"]]
    assert len(cts) == len(set(cts))                             # disjoint ciphertext indices
    for r in res:
        assert r["bits"] == r["want"]                            # each shard's compare is correct
        assert r["max"] == 3.0                                   # max over ranks


class _OracleOps:
    """stand-in for ProductOps on CPU: the oracle evaluates tree/pair steps; ciphertexts travel
    as int64 tensors [1, 2, level, n] (coefficient form) so dist.tournament's transport is real."""

    def __init__(self, P, K):
        from oracle import circuits
        self.P, self.K, self.c = P, K, circuits
        self.ev = circuits.OracleEval(P, K)

    def to_t(self, ct):
        import torch
        return torch.from_numpy(np.stack(ct.parts).view(np.int64)[None].copy())

    def from_t(self, t):
        from oracle import bgv
        a = t[0].numpy().view(np.uint64)
        return bgv.Ciphertext([a[0].copy(), a[1].copy()], a.shape[1])

    def tree(self, op, elems):
        P = self.P
        return self.to_t(self.c.tournament(self.ev, [self.from_t(e) for e in elems], op, P.circuit, P.d, P.l,
                                           P.ints_per_ct))

    def pair(self, op, a, b):
        P = self.P
        f = self.c.vmin if op == "min" else self.c.vmax
        return self.to_t(f(self.ev, self.from_t(a), self.from_t(b), P.circuit, P.d, P.l, P.ints_per_ct))

    def empty(self, shape):
        import torch
        return torch.empty(shape, dtype=torch.int64)


def _tour_worker(rank, world, port, T, out):
    import sys
    sys.path.insert(0, ROOT)
    import json
    from oracle import bgv, slots
    from paper_2407_07308_b200 import dist as bdist
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    P = bgv.Params(json.load(open(os.path.join(ROOT, "params", "c1t.json"))))
    A = P.alg
    gal = {pow(P.p, k, P.m) for k in range(1, A.D)} | {A.g, pow(A.g, -1, P.m)}
    K = bgv.keygen(P, 0xB00C0001, sorted(gal))
    ops = _OracleOps(P, K)
    rng = np.random.default_rng(99)
    W = [[int(x) for x in rng.integers(0, 4, size=P.ints_per_ct)] for _ in range(T)]
    cts = [bgv.encrypt(P, K, A.encode(slots.words_to_slots(w, A, P.d, P.l, P.base)), 0xB00C0003, 700 + t)
           for t, w in enumerate(W)]
    lo, hi = bdist.shard(T, world, rank)
    res = bdist.tournament(ops, [ops.to_t(c) for c in cts[lo:hi]], "min")
    if rank == 0:
        ref = ops.to_t(ops.c.tournament(ops.ev, cts, "min", P.circuit, P.d, P.l, P.ints_per_ct))
        dec = slots.slots_to_words(A.decode(bgv.decrypt(P, K, ops.from_t(res))), P.d, P.l, P.base, P.ints_per_ct)
        out.put({"bit_exact": bool((res == ref).all()), "dec": dec,
                 "want": [min(W[t][j] for t in range(T)) for j in range(P.ints_per_ct)]})
    else:
        assert res is None
    dist.destroy_process_group()


def test_cross_schedule_matches_element_tree():
    """rank-level rounds == the element tree's rounds restricted to shard leaders (R20)."""
    from paper_2407_07308_b200 import dist as bdist
    for world in (1, 2, 3, 4, 5, 8):
        sched = bdist.cross_schedule(world)
        # element tree over `world` leaders with per-rank block size 1
        alive = set(range(world))
        sh = 1
        while sh < world:
            for i in range(0, world, 2 * sh):
                if i + sh < world:
                    assert (sh, "recv", i + sh) in sched[i]
                    assert (sh, "send", i) in sched[i + sh]
                    alive.discard(i + sh)
            sh *= 2
        assert alive == {0}


def test_two_rank_tournament_gloo_bit_exact():
    """world 2, T = 4 elements (2 per rank): the distributed tournament (local tree + one
    send/recv cross round) equals the single-process oracle tournament bit for bit."""
    world, T = 2, 4
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tour_worker, args=(r, world, port, T, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res["bit_exact"]
    assert res["dec"] == res["want"]
