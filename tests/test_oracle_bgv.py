"""Pins for the oracle BGV scheme and the ciphertext-level comparison (C1, SPEC's toy set).

Pins: decryption correctness, homomorphism against plaintext slot arithmetic
(S:770), relinearised == unrelinearised, modulus-switch invariance, the lift's
defining congruences, and compare_lt/eq against brute-force integer comparison in every block.
"""
import math

import numpy as np
import pytest

from oracle import bgv, circuits, nt, slots

SEED_KEYS, SEED_ENC = 0xB00C0001, 0xB00C0003


@pytest.fixture(scope="module")
def c1(oracle_params):
    P = oracle_params("c1")
    A = P.alg
    gal = [pow(P.p, k, P.m) for k in range(1, A.D)] + [A.g, pow(A.g, -1, P.m)]
    K = bgv.keygen(P, SEED_KEYS, gal)
    return P, K


def _enc_slots(P, K, beta, idx):
    return bgv.encrypt(P, K, P.alg.encode(beta), SEED_ENC, idx)


def test_public_key_relation(c1):
    """pk: b + a s = p e (mod Q) with e small (R8)."""
    P, K = c1
    b, a = K.pk
    idx = list(range(P.L1))
    s_r = bgv.int_poly_to_rns(P, K.s, idx)
    x = bgv._add(b, bgv._mul(a, s_r, P, idx), P, idx)
    vals, _ = bgv.lift_centered(P, x, idx)
    assert all(v % P.p == 0 for v in vals)
    assert max(abs(v) for v in vals) <= P.p * 21


def test_decrypt_encrypt(c1):
    P, K = c1
    rng = np.random.default_rng(1)
    for i in range(3):
        beta = rng.integers(0, P.p, size=(P.alg.S, P.alg.D))
        ct = _enc_slots(P, K, beta, i)
        assert np.array_equal(P.alg.decode(bgv.decrypt(P, K, ct)), beta)
    z = _enc_slots(P, K, np.zeros((P.alg.S, P.alg.D), dtype=np.int64), 9)
    assert not bgv.decrypt(P, K, z).any()


def test_lift_congruences(c1):
    P, K = c1
    rng = np.random.default_rng(2)
    idx = [0, 1, 2]
    arr = np.stack([rng.integers(0, P.moduli[i], size=P.n, dtype=np.uint64) for i in idx])
    vals, Q = bgv.lift_centered(P, arr, idx)
    for r, i in enumerate(idx):
        assert all(v % P.moduli[i] == int(x) for v, x in zip(vals, arr[r]))
    assert all(-(Q // 2) <= v <= Q // 2 for v in vals)


def test_homomorphism(c1):
    P, K = c1
    A = P.alg
    rng = np.random.default_rng(3)
    b1 = rng.integers(0, P.p, size=(A.S, A.D))
    b2 = rng.integers(0, P.p, size=(A.S, A.D))
    c1_, c2_ = _enc_slots(P, K, b1, 10), _enc_slots(P, K, b2, 11)
    dec = lambda c: A.decode(bgv.decrypt(P, K, c))
    assert np.array_equal(dec(bgv.add(P, c1_, c2_)), (b1 + b2) % P.p)
    assert np.array_equal(dec(bgv.mul(P, K, c1_, c2_)), A.gf.mul(b1, b2))
    t = bgv.tensor(P, c1_, c2_)
    assert np.array_equal(dec(t), A.gf.mul(b1, b2))                   # 3-part decrypt
    assert np.array_equal(dec(bgv.relinearize(P, K, t)), dec(t))
    assert np.array_equal(dec(bgv.modswitch(P, c1_)), b1)
    assert np.array_equal(dec(bgv.rotate(P, K, c1_, 1)), np.roll(b1, -1, axis=0))
    assert np.array_equal(dec(bgv.rotate(P, K, c1_, -1)), np.roll(b1, 1, axis=0))
    assert np.array_equal(dec(bgv.frobenius(P, K, c1_, 2)), A.gf.pow(b1, P.p ** 2))
    assert np.array_equal(dec(bgv.mul_scalar(P, c1_, 2)), 2 * b1 % P.p)


@pytest.mark.parametrize("cfg", ["c1", "c1l2"])
def test_compare_exhaustive_2bit(oracle_params, cfg):
    """compare_lt / compare_eq on every pair of 2-bit words (brute force), every block."""
    P = oracle_params(cfg)
    A = P.alg
    gal = [pow(P.p, k, P.m) for k in range(1, A.D)]
    sh = 1
    while sh < P.l:
        gal += [pow(A.g, sh, P.m), pow(A.g, -sh, P.m)]
        sh *= 2
    K = bgv.keygen(P, SEED_KEYS, gal)
    ints = P.ints_per_ct
    pairs = [(x, y) for x in range(4) for y in range(4)]
    ev = circuits.OracleEval(P, K)
    for c0 in range(0, len(pairs), ints):
        chunk = pairs[c0:c0 + ints]
        wa = [x for x, _ in chunk] + [0] * (ints - len(chunk))
        wb = [y for _, y in chunk] + [0] * (ints - len(chunk))
        ca = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wa, A, P.d, P.l, P.base)), SEED_ENC, 100 + c0)
        cb = bgv.encrypt(P, K, A.encode(slots.words_to_slots(wb, A, P.d, P.l, P.base)), SEED_ENC, 200 + c0)
        lt, eq = circuits.compare(ev, ca, cb, P.circuit, P.d, P.l, ints)
        dl, de = A.decode(bgv.decrypt(P, K, lt)), A.decode(bgv.decrypt(P, K, eq))
        for j in range(ints):
            assert int(dl[j * P.l, 0]) == int(wa[j] < wb[j])
            assert int(de[j * P.l, 0]) == int(wa[j] == wb[j])
        nb, Qb = bgv.noise_bits(P, K, lt)
        assert nb < Qb - math.log2(P.p) - 2


def test_min_select_ciphertext(oracle_params):
    P = oracle_params("c1l2")
    A = P.alg
    gal = [pow(P.p, k, P.m) for k in range(1, A.D)] + [A.g, pow(A.g, -1, P.m)]
    K = bgv.keygen(P, SEED_KEYS, gal)
    ints = P.ints_per_ct
    rng = np.random.default_rng(4)
    wa = [int(x) for x in rng.integers(0, 4, size=ints)]
    wb = [int(x) for x in rng.integers(0, 4, size=ints)]
    # the chain has 3 primes: compare uses 2 levels; select needs one more -> use fresh 3-prime
    # ciphertexts only for the compare/select structure check at plaintext level
    ev = circuits.PlainEval(A)
    va = circuits.PlainValue(slots.words_to_slots(wa, A, P.d, P.l, P.base))
    vb = circuits.PlainValue(slots.words_to_slots(wb, A, P.d, P.l, P.base))
    mn = circuits.vmin(ev, va, vb, P.circuit, P.d, P.l, ints)
    assert slots.slots_to_words(mn.v, P.d, P.l, P.base, ints) == [min(x, y) for x, y in zip(wa, wb)]


def _gal_all(P):
    A = P.alg
    gal = {pow(P.p, k, P.m) for k in range(1, A.D)}
    sh = 1
    while sh < P.l:
        gal |= {pow(A.g, sh, P.m), pow(A.g, -sh, P.m)}
        sh *= 2
    return sorted(gal)


@pytest.fixture(scope="module")
def c1t(oracle_params):
    P = oracle_params("c1t")
    return P, bgv.keygen(P, SEED_KEYS, _gal_all(P))


@pytest.mark.parametrize("op", ["min", "max"])
def test_tournament_ciphertext(c1t, op):
    """R20 fixed-tree min/max of 4 encrypted vectors decrypts to the brute-force min/max."""
    P, K = c1t
    A, ints = P.alg, P.ints_per_ct
    rng = np.random.default_rng(11)
    W = [[int(x) for x in rng.integers(0, 4, size=ints)] for _ in range(4)]
    cts = [bgv.encrypt(P, K, A.encode(slots.words_to_slots(w, A, P.d, P.l, P.base)), SEED_ENC, 300 + t)
           for t, w in enumerate(W)]
    ev = circuits.OracleEval(P, K)
    r = circuits.tournament(ev, cts, op, P.circuit, P.d, P.l, ints)
    f = min if op == "min" else max
    got = slots.slots_to_words(A.decode(bgv.decrypt(P, K, r)), P.d, P.l, P.base, ints)
    assert got == [f(W[t][j] for t in range(4)) for j in range(ints)]
    assert r.level == P.L1 - 6


def test_sort_ciphertext(c1t):
    """R21 rank sort of 3 encrypted vectors (S:555 sort [3,1,2] -> [1,2,3] in block 0)."""
    P, K = c1t
    A, ints = P.alg, P.ints_per_ct
    rng = np.random.default_rng(12)
    W = [[int(x) for x in rng.integers(0, 4, size=ints)] for _ in range(3)]
    W[0][0], W[1][0], W[2][0] = 3, 1, 2
    cts = [bgv.encrypt(P, K, A.encode(slots.words_to_slots(w, A, P.d, P.l, P.base)), SEED_ENC, 400 + t)
           for t, w in enumerate(W)]
    ev = circuits.OracleEval(P, K)
    out = circuits.sort_rank(ev, cts, P.circuit, P.d, P.l, ints)
    got = [slots.slots_to_words(A.decode(bgv.decrypt(P, K, o)), P.d, P.l, P.base, ints) for o in out]
    for j in range(ints):
        assert [got[k][j] for k in range(3)] == sorted(W[t][j] for t in range(3))
    assert [got[k][0] for k in range(3)] == [1, 2, 3]


def test_fused_mul_decrypts_like_two_step(c1):
    """R15 fused ModDown + modulus switch: same plaintext and level as relinearise -> modswitch
    (the two-step definition), noise within 2 bits of it; a dropped P factor, a wrong delta sign or
    a missing D^{-1} breaks one of these."""
    P, K = c1
    A = P.alg
    rng = np.random.default_rng(5)
    for idx in range(3):
        b1 = rng.integers(0, P.p, size=(A.S, A.D))
        b2 = rng.integers(0, P.p, size=(A.S, A.D))
        c1_, c2_ = _enc_slots(P, K, b1, 20 + 2 * idx), _enc_slots(P, K, b2, 21 + 2 * idx)
        f = bgv.mul(P, K, c1_, c2_)
        u = bgv.mul_unfused(P, K, c1_, c2_)
        assert f.level == u.level == c1_.level - 1
        want = A.gf.mul(b1, b2)
        assert np.array_equal(A.decode(bgv.decrypt(P, K, f)), want)
        assert np.array_equal(A.decode(bgv.decrypt(P, K, u)), want)
        assert bgv.noise_bits(P, K, f)[0] <= bgv.noise_bits(P, K, u)[0] + 2


def test_mul_sum_lazy_scale_down(c1):
    """R27 (lazy ModDown): mul_sum of one pair IS mul (every word); of three pairs at two
    levels it decrypts to sum b1_i * b2_i at the level mul would give the lowest pair, with noise within 2 bits
    of the sum of separate products, and its words differ from that sum (one rounding instead of three)."""
    P, K = c1
    A = P.alg
    rng = np.random.default_rng(9)
    bs = [(rng.integers(0, P.p, size=(A.S, A.D)), rng.integers(0, P.p, size=(A.S, A.D))) for _ in range(3)]
    cs = [(_enc_slots(P, K, x, 60 + 2 * i), _enc_slots(P, K, y, 61 + 2 * i)) for i, (x, y) in enumerate(bs)]
    one = bgv.mul_sum(P, K, [cs[0]])
    ref = bgv.mul(P, K, *cs[0])
    assert one.level == ref.level and all(np.array_equal(u, v) for u, v in zip(one.parts, ref.parts))
    pairs = [cs[0], (bgv.modswitch(P, cs[1][0]), cs[1][1]), cs[2]]      # one operand a level lower
    lz = bgv.mul_sum(P, K, pairs)
    sep = bgv.add(P, bgv.add(P, bgv.mul(P, K, *pairs[0]), bgv.mul(P, K, *pairs[1])), bgv.mul(P, K, *pairs[2]))
    assert lz.level == sep.level == P.L1 - 2
    want = sum(A.gf.mul(x, y) for x, y in bs) % P.p
    assert np.array_equal(A.decode(bgv.decrypt(P, K, lz)), want)
    assert np.array_equal(A.decode(bgv.decrypt(P, K, sep)), want)
    assert bgv.noise_bits(P, K, lz)[0] <= bgv.noise_bits(P, K, sep)[0] + 2
    assert not np.array_equal(lz.parts[0], sep.parts[0])


def test_hoisted_automorphisms_decrypt_like_plain(c1):
    """R22 hoisted key switching: every sigma_t of one ciphertext decrypts exactly like the
    non-hoisted automorphism (Frobenius: slot-wise p^k power; rotations: slot
    shift) with noise within 2 bits; the bits differ (sigma_t(lift(c1)) vs lift(sigma_t(c1)))."""
    P, K = c1
    A = P.alg
    rng = np.random.default_rng(6)
    b1 = rng.integers(0, P.p, size=(A.S, A.D))
    c = _enc_slots(P, K, b1, 30)
    ts = [pow(P.p, k, P.m) for k in range(1, A.D)] + [A.g, pow(A.g, -1, P.m)]
    hs = bgv.automorphisms_hoisted(P, K, c, ts)
    dec = lambda x: A.decode(bgv.decrypt(P, K, x))
    for t, h in zip(ts, hs):
        plain = bgv.automorphism(P, K, c, t)
        assert np.array_equal(dec(h), dec(plain))
        assert bgv.noise_bits(P, K, h)[0] <= bgv.noise_bits(P, K, plain)[0] + 2
    for k in range(1, A.D):
        assert np.array_equal(dec(hs[k - 1]), A.gf.pow(b1, P.p ** k))
    assert np.array_equal(dec(hs[A.D - 1]), np.roll(b1, -1, axis=0))
    assert not np.array_equal(hs[0].parts[1], bgv.automorphism(P, K, c, ts[0]).parts[1])
