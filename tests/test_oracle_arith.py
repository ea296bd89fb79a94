"""Pins for the oracle's number theory and ring arithmetic (not self-referential).

Each test checks the oracle against something other than itself: sympy (library routines),
closed forms, the paper's printed numbers (tests/golden), or brute force.
"""
import random

import numpy as np
import pytest
import sympy

from conftest import golden
from oracle import _c, cyclo, nt


def test_is_prime_matches_sympy():
    rng = random.Random(1)
    for _ in range(300):
        x = rng.randrange(2, 1 << 62)
        assert nt.is_prime(x) == sympy.isprime(x)
    for x in range(2, 2000):
        assert nt.is_prime(x) == sympy.isprime(x)


def test_prime_chain_spec_pin():
    g = golden("spec_examples.json")["gen_ntt_primes"]
    M = nt.bluestein_pad(g["m"])
    assert M == g["M"]
    qs = nt.prime_chain(nt.lcm(3, g["m"], M), g["bits"], g["count"])
    assert len(qs) == 3 and len(set(qs)) == 3
    for q in qs:
        assert sympy.isprime(q)
        assert q % g["modulus"] == 1            # = 1 mod lcm(2m, M) = 23296
        assert q.bit_length() == g["bits"]
    # "smallest": no prime = 1 (mod lcm) between 2^58 and the first returned one
    L = nt.lcm(3, g["m"], M)
    x = (1 << 58) + ((1 - (1 << 58)) % L)
    while x < qs[0]:
        assert not sympy.isprime(x)
        x += L


def test_bluestein_pad_pins():
    for m, M in golden("spec_examples.json")["bluestein_pad"]["pairs"]:
        assert nt.bluestein_pad(m) == M


def test_root_of_unity_exact_order():
    for m in (91, 859, 30941):
        M = nt.bluestein_pad(m)
        q = nt.prime_chain(nt.lcm(13, m, M), 50, 1)[0]
        w = nt.root_of_unity(m, q)
        assert pow(w, m, q) == 1
        assert sympy.n_order(w, q) == m


def test_crt_roundtrip_and_center():
    rng = random.Random(3)
    mods = nt.prime_chain(nt.lcm(3, 91, 256), 59, 3)
    Q = mods[0] * mods[1] * mods[2]
    for _ in range(200):
        x = rng.randrange(-(Q // 2), Q // 2 + 1)
        r = [x % q for q in mods]
        y, QQ = nt.crt(r, mods)
        assert QQ == Q and nt.centered(y, Q) == x


@pytest.mark.parametrize("m", [3, 6, 7, 15, 45, 91, 105, 859])
def test_cyclotomic_matches_sympy(m):
    x = sympy.Symbol("x")
    ref = sympy.Poly(sympy.cyclotomic_poly(m, x), x).all_coeffs()[::-1]
    assert cyclo.cyclotomic(m) == [int(c) for c in ref]


def test_cyclotomic_spec_examples():
    for m, c in golden("spec_examples.json")["cyclotomic"]["cases"]:
        assert cyclo.cyclotomic(m) == c


def test_filter_spec_examples():
    # Listing 1/2: keep i with gcd(i, m) = 1, ascending
    for m, vals, out in golden("spec_examples.json")["filter"]["cases"]:
        z = cyclo.zm_star(m)
        assert [vals[i] for i in z] == out


def _rand_poly(rng, n, q):
    return np.array([rng.randrange(q) for _ in range(n)], dtype=np.uint64)


@pytest.mark.parametrize("m", [7, 45, 91, 859])
def test_ring_mul_vs_sympy(m):
    """schoolbook mod (q, Phi_m) vs sympy polynomial remainder over GF(q)."""
    rng = random.Random(m)
    R = cyclo.Ring(m)
    q = nt.prime_chain(nt.lcm(3, m, nt.bluestein_pad(m)), 40, 1)[0]
    x = sympy.Symbol("x")
    phi = sympy.Poly(sympy.cyclotomic_poly(m, x), x, modulus=q)
    for _ in range(2 if m > 100 else 4):
        a, b = _rand_poly(rng, R.n, q), _rand_poly(rng, R.n, q)
        got = R.mul(a, b, q)
        pa = sympy.Poly([int(v) for v in a[::-1]], x, modulus=q)
        pb = sympy.Poly([int(v) for v in b[::-1]], x, modulus=q)
        rem = (pa * pb).rem(phi)
        coeffs = [int(c) % q for c in rem.all_coeffs()[::-1]]
        coeffs += [0] * (R.n - len(coeffs))
        assert [int(v) for v in got] == coeffs


@pytest.mark.parametrize("m", [7, 31, 45, 91])
def test_eval_is_homomorphic_and_pins(m):
    """R3 evaluation form: naive evaluation at omega^{z_k}; products map to pointwise products;
    constants -> constant vectors; x -> omega^{z_k}."""
    rng = random.Random(10 + m)
    R = cyclo.Ring(m)
    M = nt.bluestein_pad(m)
    q = nt.prime_chain(nt.lcm(3, m, M), 45, 1)[0]
    w = nt.root_of_unity(m, q)
    a, b = _rand_poly(rng, R.n, q), _rand_poly(rng, R.n, q)
    ea, eb = R.to_eval(a, w, q), R.to_eval(b, w, q)
    eab = R.to_eval(R.mul(a, b, q), w, q)
    assert [int(x) * int(y) % q for x, y in zip(ea, eb)] == [int(v) for v in eab]
    c = np.zeros(R.n, dtype=np.uint64)
    c[0] = 12345
    assert set(int(v) for v in R.to_eval(c, w, q)) == {12345}
    xpoly = np.zeros(R.n, dtype=np.uint64)
    xpoly[1] = 1
    assert [int(v) for v in R.to_eval(xpoly, w, q)] == [pow(w, int(zk), q) for zk in R.z]


@pytest.mark.parametrize("m", [7, 31, 45, 91])
def test_bluestein_literal_equals_naive_dft(m):
    """The paper's BluesteinNTT steps reproduce the naive DFT at Z_m^*."""
    rng = random.Random(m)
    R = cyclo.Ring(m)
    M = nt.bluestein_pad(m)
    q = nt.prime_chain(nt.lcm(3, m, M), 41, 1)[0]
    w = nt.root_of_unity(m, q)
    f = _rand_poly(rng, R.n, q)
    assert cyclo.bluestein_literal(f, m, w, q, M) == [int(v) for v in R.to_eval(f, w, q)]


def test_automorphism_composition():
    """sigma_s o sigma_t = sigma_{st}; sigma_1 = id; sigma_{p^D} = id (C4 pins)."""
    rng = random.Random(5)
    m = 91
    R = cyclo.Ring(m)
    q = nt.prime_chain(nt.lcm(3, m, 256), 59, 1)[0]
    a = _rand_poly(rng, R.n, q)
    s, t = 2, 5
    st = R.automorph_mod(R.automorph_mod(a, t, q), s, q)
    assert np.array_equal(st, R.automorph_mod(a, s * t % m, q))
    assert np.array_equal(R.automorph_mod(a, 1, q), a)
    assert np.array_equal(R.automorph_mod(a, pow(3, 6, m), q), a)
    # the automorphism is a ring homomorphism
    b = _rand_poly(rng, R.n, q)
    lhs = R.automorph_mod(R.mul(a, b, q), 4, q)
    rhs = R.mul(R.automorph_mod(a, 4, q), R.automorph_mod(b, 4, q), q)
    assert np.array_equal(lhs, rhs)


def test_vec_helpers():
    q = (1 << 61) - 1
    rng = np.random.default_rng(0)
    a = rng.integers(0, q, size=1000, dtype=np.uint64)
    b = rng.integers(0, q, size=1000, dtype=np.uint64)
    got = _c.vec_mulmod(a, b, q)
    assert [int(x) for x in got] == [int(x) * int(y) % q for x, y in zip(a, b)]


@pytest.mark.parametrize("m", [33, 45, 91, 211])
def test_reduce_int_matches_sympy(m):
    """Ring.reduce_int (integer polynomial mod Phi_m over Z, any length) = sympy's remainder."""
    x = sympy.symbols("x")
    R = cyclo.Ring(m)
    rng = np.random.default_rng(m)
    c = [int(v) for v in rng.integers(-50, 50, size=3 * m)]
    r = sympy.Poly(c[::-1], x).rem(sympy.cyclotomic_poly(m, x, polys=True))
    want = [int(v) for v in r.all_coeffs()[::-1]]
    assert R.reduce_int(c) == want + [0] * (R.n - len(want))


def test_bluestein_pad_mixed_lengths():
    """R25 (f3): the mixed-radix Bluestein length of each large ring, by hand from the candidate set
    {2^k} U {256 r N' : r in {3,5,7,9}, N' in {32,64,128}}: C4 (m = 34511, 2m-1 = 69021) -> 9*8192 =
    73728; C5 (41761 -> 83521) -> 3*32768 = 98304; C3 (52053 -> 104105) -> 7*16384 = 114688;
    p3 (20197 -> 40393) -> 5*8192 = 40960; C2 (30941 -> 61881) stays 65536 (P:316's power of two);
    the minimum over the candidate set by brute force; primes = 1 mod lcm(p, m, M)"""
    assert nt.bluestein_pad(34511, True) == 73728
    assert nt.bluestein_pad(41761, True) == 98304
    assert nt.bluestein_pad(52053, True) == 114688
    assert nt.bluestein_pad(20197, True) == 40960
    assert nt.bluestein_pad(30941, True) == 65536
    cands = sorted({2 ** k for k in range(1, 20)} | {256 * r * nn for r in (3, 5, 7, 9) for nn in (32, 64, 128)})
    for m in (91, 859, 1423, 1871, 20197, 30941, 34511, 41761, 52053):
        assert nt.bluestein_pad(m, True) == min(L for L in cands if L >= 2 * m - 1)
        assert nt.bluestein_pad(m, True) <= nt.bluestein_pad(m)
    from oracle import bgv
    from conftest import load_cfg
    cfg = dict(load_cfg("c4"), bluestein="mixed")
    P = bgv.Params(cfg)
    assert P.M == 73728 and all(q % nt.lcm(P.p, P.m, 73728) == 1 for q in P.moduli)
