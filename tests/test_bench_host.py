"""bench.py's host-side pieces (CPU): the oracle cost model used for the labelled compare_lt
extrapolation of the CPU baseline equals the oracle's own ring-product count on a real run
(C2's circuit and chain on its shadow ring), and the reference arm's sample is one real R15
product whose count the oracle confirms."""
import json
import os
import sys

import numpy as np

from conftest import ROOT, load_cfg

sys.path.insert(0, ROOT)


def test_cost_model_matches_oracle_counter():
    import bench
    import oracle._c as oc
    from inputs import word_pairs
    from oracle import bgv, circuits, slots
    cfg = load_cfg("c2s")
    P = bgv.Params(cfg)
    A = P.alg
    gal = sorted({pow(P.p, k, P.m) for k in range(1, A.D)} | {pow(A.g, s, P.m) for s in (1, 2, 4) if s < P.l})
    K = bgv.keygen(P, 0xB00C0001, gal)
    a, b = word_pairs(np.random.default_rng(5), P.ints_per_ct, P.base, P.d * P.l)
    oa = bgv.encrypt(P, K, A.encode(slots.words_to_slots(a, A, P.d, P.l, P.base)), 0xB00C0003, 0)
    ob = bgv.encrypt(P, K, A.encode(slots.words_to_slots(b, A, P.d, P.l, P.base)), 0xB00C0003, 1)
    c0 = oc.CALLS["ring_mul"]
    circuits.compare(circuits.OracleEval(P, K), oa, ob, P.circuit, P.d, P.l, P.ints_per_ct)
    assert oc.CALLS["ring_mul"] - c0 == bench.circuits_product_count(P)


def test_oracle_sample_is_one_real_product():
    import bench
    S = bench.OracleSample(load_cfg("c2s"))
    t = S.run()                         # asserts the oracle's counter matches S.products
    assert t > 0 and 0 < S.products < S.compare_products
    assert "R15 product" in S.describe(t)


def test_host_info_fields():
    import bench
    h = bench.host_info()
    assert h["nproc"] >= 1 and h["omp_threads"] >= 1
