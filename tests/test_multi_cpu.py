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
