"""Pins for the oracle's slot algebra and integer encoding (Table 3)."""
import random

import numpy as np
import pytest
import sympy

from conftest import golden
from oracle import cyclo, nt, slots


def test_table3_closed_forms():
    """F1: N = phi(m), D = ord_m(p), S = phi(m)/D, ints = floor(S/l), d <= D, and the integer
    capacity base^(d l) >= 2^64 (base p for B, (p+1)/2 for U) for all 20 rows of Table 3."""
    for row in golden("table3.json")["rows"]:
        p, m = row["p"], row["m"]
        assert nt.euler_phi(m) == row["N"]
        D = nt.mult_order(p, m)
        S = row["N"] // D
        for circ in ("B", "U"):
            d, l = row[circ]["d"], row[circ]["l"]
            # the paper's count is floor(S / l) for every row, hypercube rows included
            assert S // l == row[circ]["ints"]
            assert d <= D
            base = slots.digit_base(p, circ)
            assert base ** (d * l) >= 2 ** 64


def _quotient_orders(p, m):
    """orders of the elements of Z_m^*/<p> (brute force over divisors of S): -> (S, max order)"""
    H = {pow(p, k, m) for k in range(nt.mult_order(p, m))}
    S = nt.euler_phi(m) // len(H)
    divs = [k for k in range(1, S + 1) if S % k == 0]
    best = 1
    for t in range(2, m):
        if nt.gcd(t, m) == 1:
            best = max(best, next(k for k in divs if pow(t, k, m) in H))
    return S, best


def test_table3_hypercube_rows():
    """F7 / S17: Z_m^*/<p> is cyclic for every Table 3 row except p3 and p10, where it is
    Z_S1 x Z_2; R6's row-aligned layout then holds 2 floor(S1/l) = floor(S/l) - 1 integers."""
    for row in golden("table3.json")["rows"]:
        if row["m"] > 60000:
            continue
        S, S1 = _quotient_orders(row["p"], row["m"])
        if row["set"] in ("p3", "p10"):
            assert S1 * 2 == S
            for circ in ("B", "U"):
                l = row[circ]["l"]
                assert 2 * (S1 // l) == row[circ]["ints"] - 1
        else:
            assert S1 == S


def test_slot_algebra_spec_pin():
    g = golden("spec_examples.json")["slot_algebra"]
    A = slots.SlotAlgebra(g["p"], cyclo.Ring(g["m"]))
    assert (A.D, A.S) == (g["D"], g["S"])


@pytest.mark.parametrize("p,m", [(3, 91), (13, 859), (2, 7), (31, 1129)])
def test_G_is_smallest_irreducible(p, m):
    if p == 2:
        pytest.skip("p odd only")
    A = slots.SlotAlgebra(p, cyclo.Ring(m))
    X = sympy.Symbol("X")
    G = A.G
    assert sympy.Poly(G[::-1], X, modulus=p).is_irreducible
    v = sum(c * p ** i for i, c in enumerate(G[:-1]))
    for u in range(min(v, 400)):
        c = [(u // p ** i) % p for i in range(A.D)] + [1]
        assert not sympy.Poly(c[::-1], X, modulus=p).is_irreducible


@pytest.mark.parametrize("p,m", [(3, 91), (13, 859)])
def test_slot_factors_multiply_to_phi(p, m):
    """Prod_s F_s = Phi_m (mod p), each F_s irreducible of degree D."""
    R = cyclo.Ring(m)
    A = slots.SlotAlgebra(p, R)
    A._prepare_encode()
    X = sympy.Symbol("X")
    prod = sympy.Poly(1, X, modulus=p)
    for s in range(A.S):
        H = A._enc[0][s]
        # F_s = Phi / H_s
        F = sympy.Poly([int(c) for c in cyclo.cyclotomic(m)[::-1]], X, modulus=p).exquo(
            sympy.Poly([int(c) for c in H[::-1]], X, modulus=p))
        assert F.degree() == A.D and F.is_irreducible
        prod = prod * F
    assert prod == sympy.Poly([int(c) for c in cyclo.cyclotomic(m)[::-1]], X, modulus=p)


@pytest.mark.parametrize("p,m", [(3, 91), (13, 859)])
def test_encode_decode_roundtrip_and_multiplicative(p, m):
    rng = np.random.default_rng(p * m)
    R = cyclo.Ring(m)
    A = slots.SlotAlgebra(p, R)
    for _ in range(3):
        beta = rng.integers(0, p, size=(A.S, A.D))
        a = A.encode(beta)
        assert np.array_equal(A.decode(a), beta)
    b1 = rng.integers(0, p, size=(A.S, A.D))
    b2 = rng.integers(0, p, size=(A.S, A.D))
    a1, a2 = A.encode(b1), A.encode(b2)
    prod = R.mul(a1.astype(np.uint64), a2.astype(np.uint64), p).astype(np.int64)
    assert np.array_equal(A.decode(prod), A.gf.mul(b1, b2))
    # constant slots <-> constant polynomial
    c = np.zeros((A.S, A.D), dtype=np.int64)
    c[:, 0] = 2
    e = A.encode(c)
    assert e[0] == 2 and not e[1:].any()


def test_galois_action_on_slots():
    """decode(sigma_p(a)) = decode(a)^p (Frobenius) and decode(sigma_g(a))_s = decode(a)_{s+1}."""
    p, m = 3, 91
    R = cyclo.Ring(m)
    A = slots.SlotAlgebra(p, R)
    rng = np.random.default_rng(7)
    beta = rng.integers(0, p, size=(A.S, A.D))
    a = A.encode(beta).astype(np.uint64)
    fa = R.automorph_mod(a, p, p).astype(np.int64)
    assert np.array_equal(A.decode(fa), A.gf.pow(beta, p))
    ga = R.automorph_mod(a, A.g, p).astype(np.int64)
    assert np.array_equal(A.decode(ga), np.roll(beta, -1, axis=0))
    # cosets t_s <p> partition Z_m^*
    seen = set()
    for t in A.t:
        for k in range(A.D):
            seen.add(t * pow(p, k, m) % m)
    assert seen == set(cyclo.zm_star(m))


def test_int_to_digits_spec():
    for x, p, count, dig in golden("spec_examples.json")["int_to_digits"]["cases"]:
        base = p if dig == [2, 0, 1] else (p + 1) // 2 + (0 if p != 5 else 0)
        if x == 5:
            base = 3   # S:337 half alphabet for p=5: base (p+1)/2 = 3
        assert slots.int_to_digits(x, base, count) == dig
    with pytest.raises(ValueError):
        slots.int_to_digits(27, 3, 3)


def test_words_to_slots_roundtrip():
    A = slots.SlotAlgebra(13, cyclo.Ring(859))
    rng = random.Random(1)
    d, l, base = 4, 6, 7
    ints = A.S // l
    words = [rng.randrange(2 ** 64) for _ in range(ints)]
    sl = slots.words_to_slots(words, A, d, l, base)
    assert sl.max() < base
    assert slots.slots_to_words(sl, d, l, base, ints) == words


def test_frobenius_extraction_identity_exhaustive():
    """P:286 mod extract: sum_k kappa_{i,k} beta^{p^k} = a_i for every beta in F_{3^6} (729 values)."""
    A = slots.SlotAlgebra(3, cyclo.Ring(91))
    gf = A.gf
    mus = A.dual_basis()
    allb = np.array([[(v // 3 ** i) % 3 for i in range(A.D)] for v in range(3 ** A.D)], dtype=np.int64)
    frob = [allb]
    for _ in range(1, A.D):
        frob.append(gf.pow(frob[-1], 3))
    for i in range(A.D):
        acc = np.zeros_like(allb)
        for k in range(A.D):
            kap = gf.pow(mus[i], 3 ** k)
            acc = (acc + gf.mul(frob[k], kap)) % 3
        assert np.array_equal(acc[:, 0], allb[:, i])
        assert not acc[:, 1:].any()


def test_alexnet_slot_arithmetic():
    g = golden("spec_examples.json")["alexnet_slots"]
    cts = -(-g["inputs"] // g["slots"])
    assert cts == g["cts"]
    unused = 1 - g["inputs"] / (cts * g["slots"])
    assert abs(100 * unused - g["unused_pct_approx"]) < 1.0
