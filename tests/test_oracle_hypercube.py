"""Oracle pins for non-cyclic (hypercube) slot structures -- C3's p10 ring (m = 52053 = 3 x 17351,
Z_m^*/<31> = Z_3470 x Z_2), its shadow m = 1851 = 3 x 617 (Z_56 x Z_2) and the tiny m = 33 = 3 x 11
(Z_2 x Z_2).  R5 (slot generators), R6 (row-aligned integers), R17 (compaction within rows)."""
import math

import numpy as np
import pytest

from oracle import bgv, circuits, slots

SEED_KEYS, SEED_ENC = 0xB00C0001, 0xB00C0003


@pytest.mark.parametrize("cfg", ["c3h", "c3s2"])
def test_hypercube_generators(oracle_params, cfg):
    """every unit of Z_m is p^k g^i g2^j for exactly one (k, i, j) (brute force over the units),
    g2^S2 = 1 (mod m), and no smaller power of g or g2 falls in the subgroup generated before it"""
    P = oracle_params(cfg)
    A, m, p = P.alg, P.m, P.p
    assert A.S1 * A.S2 == A.S and A.S2 > 1
    units = {t for t in range(1, m) if math.gcd(t, m) == 1}
    img = [pow(p, k, m) * pow(A.g, i, m) * pow(A.g2, j, m) % m
           for k in range(A.D) for i in range(A.S1) for j in range(A.S2)]
    assert len(img) == len(units) and set(img) == units
    assert pow(A.g2, A.S2, m) == 1
    H = {pow(p, k, m) for k in range(A.D)}
    assert all(pow(A.g, i, m) not in H for i in range(1, A.S1))
    # no cyclic generator exists: every unit has quotient order < S
    assert max(A.quotient_order(t) for t in units) == A.S1 < A.S


@pytest.mark.parametrize("cfg", ["c3h", "c3s2"])
def test_hypercube_encode_decode(oracle_params, cfg):
    P = oracle_params(cfg)
    A = P.alg
    rng = np.random.default_rng(5)
    beta = rng.integers(0, P.p, size=(A.S, A.D))
    assert np.array_equal(A.decode(A.encode(beta)), beta)


def test_hypercube_rotation_is_a_row_shift(oracle_params):
    """sigma_g moves slot (i+1, j) to (i, j) inside each row (no Frobenius twist away from the row
    end, by t_(i+1, j) = g t_(i, j)); the row index j never changes"""
    P = oracle_params("c3s2")
    A = P.alg
    ev = circuits.PlainEval(A)
    rng = np.random.default_rng(6)
    beta = rng.integers(0, P.p, size=(A.S, A.D))
    out = ev.rotate(circuits.PlainValue(beta), 1).v
    for j in range(A.S2):
        for i in range(A.S1 - 1):
            assert np.array_equal(out[j * A.S1 + i], beta[j * A.S1 + i + 1])


def test_hypercube_words_row_aligned(oracle_params):
    """R6: floor(S1/l) integers per row; C3's shadow: 18 per row, 36 per ciphertext"""
    P = oracle_params("c3s2")
    A = P.alg
    assert P.ints_per_ct == 36 and A.words_per_row(P.l) == 18
    w = list(range(1, 37))
    sl = slots.words_to_slots(w, A, P.d, P.l, P.base)
    assert slots.slots_to_words(sl, P.d, P.l, P.base, 36, A) == w
    # slots 54, 55 of each row (56 = 18*3 + 2) stay empty
    for j in range(A.S2):
        assert not sl[j * A.S1 + 54:j * A.S1 + 56].any()


def test_hypercube_compare_plain_all_pairs(oracle_params):
    """the R16 schedules with row-aligned masks on C3's shadow slots: LT and EQ of 36 word pairs per
    evaluation equal brute force (plaintext evaluator: the circuits' slot semantics)"""
    P = oracle_params("c3s2")
    A = P.alg
    ints = P.ints_per_ct
    import random
    rng = random.Random(7)
    cap = P.base ** (P.d * P.l)
    for _ in range(3):
        wa = [rng.randrange(cap) for _ in range(ints)]
        wb = [x if k % 3 == 0 else rng.randrange(cap) for k, x in enumerate(wa)]
        wb[1] = wa[1] + 1 if wa[1] + 1 < cap else wa[1] - 1
        ev = circuits.PlainEval(A)
        lt, eq = circuits.compare(ev, circuits.PlainValue(slots.words_to_slots(wa, A, P.d, P.l, P.base)),
                                  circuits.PlainValue(slots.words_to_slots(wb, A, P.d, P.l, P.base)),
                                  P.circuit, P.d, P.l, ints)
        for j in range(ints):
            s0 = A.word_slot(j, P.l)
            assert int(lt.v[s0, 0]) == int(wa[j] < wb[j])
            assert int(eq.v[s0, 0]) == int(wa[j] == wb[j])


def test_hypercube_compaction_stays_in_rows(oracle_params):
    """R17 plan with rows: a block moves by delta within its row only (Fig. 7 pattern, 4 inputs)"""
    P = oracle_params("c3s2")
    ints, wpr = P.ints_per_ct, P.alg.words_per_row(P.l)
    useful = [[b for b in range(ints) if b % 4 == 3]] * 4
    groups, n_out, dest = circuits.plan_compaction(useful, ints, 3, wpr)
    for (c, b), (cp, b2) in dest.items():
        assert b // wpr == b2 // wpr
    # row 1 holds 5 useful blocks per input (positions 1, 5, 9, 13, 17): 20 > 18 needs a second output
    per_row = [sum(1 for b in useful[0] if b // wpr == r) * 4 for r in range(2)]
    assert n_out == max(-(-k // wpr) for k in per_row) == 2 and len(dest) == 4 * len(useful[0])


@pytest.mark.parametrize("sched", ["r16", "r23", "r26", "r27"])
def test_hypercube_compare_bgv(oracle_params, sched):
    """full BGV compare_lt / compare_eq on the tiny hypercube ring (p = 31 bivariate, m = 33):
    decrypted block slot 0 equals brute force for 2 integers (one per row) per ciphertext, with the
    R16 and the R23 (f2) digit circuits"""
    from oracle import bgv as _bgv
    from conftest import load_cfg
    P = oracle_params("c3h") if sched == "r16" else _bgv.Params(dict(load_cfg("c3h"), schedule=sched))
    A = P.alg
    gal = [pow(P.p, k, P.m) for k in range(1, A.D)]
    sh = 1
    while sh < P.l:
        gal += [pow(A.g, sh, P.m), pow(A.g, -sh, P.m)]
        sh *= 2
    K = bgv.keygen(P, SEED_KEYS, gal)
    ints = P.ints_per_ct
    ev = circuits.OracleEval(P, K)
    cases = [([5, 923520], [7, 923520]), ([31 * 31 + 4, 0], [31 * 31 + 3, 1])]
    for c0, (wa, wb) in enumerate(cases):
        ca = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wa, A, P.d, P.l, P.base)), SEED_ENC, 10 + c0)
        cb = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wb, A, P.d, P.l, P.base)), SEED_ENC, 20 + c0)
        lt, eq = circuits.compare(ev, ca, cb, P.circuit, P.d, P.l, ints)
        dl, de = A.decode(bgv.decrypt(P, K, lt)), A.decode(bgv.decrypt(P, K, eq))
        for j in range(ints):
            s0 = A.word_slot(j, P.l)
            assert int(dl[s0, 0]) == int(wa[j] < wb[j])
            assert int(de[s0, 0]) == int(wa[j] == wb[j])
