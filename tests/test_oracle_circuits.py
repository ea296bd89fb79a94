"""Pins for the oracle's comparison circuits.

The schedules run on plaintext slot values (PlainEval) so they can be checked exhaustively
against brute-force comparison; the ciphertext versions are pinned in test_oracle_bgv.py.
"""
import math
import random

import numpy as np
import pytest

from conftest import golden
from oracle import circuits, cyclo, slots

PRIMES = [3, 5, 7, 11, 13, 17, 19, 23, 29, 31]


@pytest.mark.parametrize("p", PRIMES)
def test_digit_polys_truth_tables(p):
    h = (p - 1) // 2
    lt = circuits.lt_univariate_coeffs(p)
    eq = circuits.eq_coeffs(p)
    for x in range(h + 1):
        for y in range(h + 1):
            z = (x - y) % p
            assert circuits.eval_poly_fp(lt, z, p) == (1 if x < y else 0)
            assert circuits.eval_poly_fp(eq, z, p) == (1 if x == y else 0)
    # structure (A.5): odd powers plus ((p+1)/2) z^{p-1}
    assert lt[p - 1] == (p + 1) // 2 and lt[0] == 0
    assert all(lt[k] == 0 for k in range(2, p - 1, 2))


@pytest.mark.parametrize("p", [3, 5, 7, 11, 13])
def test_bivariate_truth_table_and_structure(p):
    c = circuits.lt_bivariate_coeffs(p)
    for x in range(p):
        for y in range(p):
            v = 0
            for j in range(len(c)):
                for k in range(len(c[j])):
                    if c[j][k]:
                        v += c[j][k] * pow(y, j, p) * pow((x - y) % p, k, p)
            assert v % p == (1 if x < y else 0)
    assert all(c[0][k] == 0 for k in range(len(c[0])))          # no Y^0 terms (A.5)
    assert max(j + k for j in range(len(c)) for k in range(len(c[j])) if c[j][k]) == p  # total degree p


def test_spec_lt_digit_examples():
    g = golden("spec_examples.json")["lt_digit"]
    c = circuits.lt_bivariate_coeffs(3)
    for x, y, want in g["bivariate_p3"]:
        v = sum(c[j][k] * pow(y, j, 3) * pow((x - y) % 3, k, 3) for j in range(len(c)) for k in range(len(c[j])))
        assert v % 3 == want
    lt5 = circuits.lt_univariate_coeffs(5)
    for z, want in g["univariate_p5_sign"]:
        assert circuits.eval_poly_fp(lt5, z, 5) == want


class _FpAlg:
    """minimal stand-in for a slot algebra whose slots are F_p (D = 1)."""

    def __init__(self, p, S):
        self.p, self.D, self.S = p, 1, S
        self.gf = slots.GF(p, [0, 1])


def _digit_run(p, kind, r23=False, k=None):
    """run the schedule on one F_p value per slot covering every digit pair."""
    h = (p - 1) // 2 if kind == "U" else p - 1
    A = _FpAlg(p, (h + 1) ** 2)       # F_p itself (D = 1): one digit pair per slot
    ev = circuits.PlainEval(A)
    h = (p - 1) // 2 if kind == "U" else p - 1
    pairs = [(x, y) for x in range(h + 1) for y in range(h + 1)]
    res = []
    for i0 in range(0, len(pairs), A.S):
        chunk = pairs[i0:i0 + A.S]
        X = np.zeros((A.S, A.D), dtype=np.int64)
        Y = np.zeros((A.S, A.D), dtype=np.int64)
        for s, (x, y) in enumerate(chunk):
            X[s, 0], Y[s, 0] = x, y
        ev.counts["mul"] = 0
        if kind == "U":
            z = circuits.PlainValue((X - Y) % p)
            lt, eq = circuits.univariate_lt_eq_r23(ev, z, p, k) if r23 else circuits.univariate_lt_eq(ev, z, p)
        elif r23 in ("r26", "r27"):
            lt, eq = circuits.bivariate_lt_eq_r26(ev, circuits.PlainValue(X), circuits.PlainValue(Y), p, *k,
                                                  lazy=r23 == "r27")
        elif r23:
            lt, eq = circuits.bivariate_lt_eq_r23(ev, circuits.PlainValue(X), circuits.PlainValue(Y), p, k)
        else:
            lt, eq = circuits.bivariate_lt_eq(ev, circuits.PlainValue(X), circuits.PlainValue(Y), p)
        for s, (x, y) in enumerate(chunk):
            res.append((x, y, int(lt.v[s, 0]), int(eq.v[s, 0])))
            assert not lt.v[s, 1:].any() and not eq.v[s, 1:].any()
    return res, ev.counts["mul"], max(lt.depth, eq.depth if hasattr(eq, "depth") else 0)


@pytest.mark.parametrize("p", PRIMES)
def test_univariate_schedule_truth_and_budget(p):
    res, mults, depth = _digit_run(p, "U")
    for x, y, lt, eq in res:
        assert (lt, eq) == (int(x < y), int(x == y))
    # sqrt(p-3) + O(log p); SPEC budget: <= 2 ceil(sqrt p) + 2 ceil(log2 p)
    assert mults <= 2 * math.ceil(math.sqrt(p)) + 2 * math.ceil(math.log2(p))
    assert depth <= math.ceil(math.log2(p)) + 2


@pytest.mark.parametrize("p", [3, 5, 7, 11, 13, 17])
def test_bivariate_schedule_truth_and_3p_minus_5(p):
    res, mults, _ = _digit_run(p, "B")
    for x, y, lt, eq in res:
        assert (lt, eq) == (int(x < y), int(x == y))
    assert mults == 3 * p - 5      # P:71 [Tan]: 3p-5 non-scalar multiplications (with EQ)


@pytest.mark.parametrize("p", PRIMES)
@pytest.mark.parametrize("kind", ["U", "B"])
def test_r23_schedule_truth_tables(p, kind):
    """R23 (f2): the baby-step / giant-step digit circuits give [x < y], [x = y] on every digit
    pair at every baby-step size k, with no more products and no more depth than R16 at the k the
    rule selects."""
    kmax = (p - 1) // 2 if kind == "U" else p - 1
    ks = sorted({1, 2, max(kmax, 1), (circuits.r23_univariate_k(p) if kind == "U" else circuits.r23_bivariate_k(p))})
    r16 = _digit_run(p, kind)
    for k in ks:
        if k > max(kmax, 1):
            continue
        res, mults, depth = _digit_run(p, kind, r23=True, k=k)
        for x, y, lt, eq in res:
            assert (lt, eq) == (int(x < y), int(x == y)), (p, kind, k, x, y)
        if k == (circuits.r23_univariate_k(p) if kind == "U" else circuits.r23_bivariate_k(p)):
            assert mults <= r16[1] and depth <= r16[2]


def test_r23_product_counts_closed_form():
    """R23 product counts against the hand count of the schedule (R23):
    U, p = 13, k = 3: W; W^2, W^3; (A = 2: no giant beyond W^3); W^3 B_1; W^6 = W^3 W^3; z g -> 6
      (R16: 7);
    B, p = 31, k = 4: Z^2..Z^30 (29); Y^2..Y^4 (3); G_2..G_7 = Y^8..Y^28 (6); I_0..I_6: 3 each (21),
      I_7 (j = 29, 30): 2; G_a I_a, a = 1..7 (7) -> 68 at depth 7;
    B, p = 31, k = 14: 29 + Y^2..Y^14 (13) + G_2 (1) + I_0 13 + I_1 13 + I_2 2 + 2 outer -> 73 at
      depth 6 = R16's depth (88 products, P:71's 3p - 5), the rule's choice."""
    assert circuits._r23_cost(circuits.univariate_lt_eq_r23, 13, 3) == (6, 5)
    assert circuits._r23_cost(circuits.bivariate_lt_eq_r23, 31, 4) == (68, 7)
    assert circuits._r23_cost(circuits.bivariate_lt_eq_r23, 31, 14) == (73, 6)
    assert circuits.r23_univariate_k(13) == 3 and circuits.r23_bivariate_k(31) == 14
    # k = 1 is the R16 bivariate tree: 3p - 5 products
    for p in (5, 7, 11, 13):
        assert circuits._r23_cost(circuits.bivariate_lt_eq_r23, p, 1)[0] == 3 * p - 5
    # fewer products than 3p - 5 for every bivariate p >= 5 (toward P:77's 2p - 6)
    for p in PRIMES:
        if p >= 5:
            assert circuits._r23_cost(circuits.bivariate_lt_eq_r23, p, circuits.r23_bivariate_k(p))[0] < 3 * p - 5


def test_spec_lex_example():
    g = golden("spec_examples.json")["lex"]
    p = g["p"]
    A = slots.SlotAlgebra(p, cyclo.Ring(91))
    ev = circuits.PlainEval(A)
    a = g["a_msb_first"][::-1]
    b = g["b_msb_first"][::-1]
    lts, eqs = [], []
    for x, y in zip(a, b):
        v = np.zeros((A.S, A.D), dtype=np.int64)
        v[:, 0] = int(x < y)
        w = np.zeros((A.S, A.D), dtype=np.int64)
        w[:, 0] = int(x == y)
        lts.append(circuits.PlainValue(v))
        eqs.append(circuits.PlainValue(w))
    lt, _ = circuits.lex_tree(ev, lts, eqs)
    assert int(lt.v[0, 0]) == g["lt"]


def _plain_words(A, words, d, l, base):
    return circuits.PlainValue(slots.words_to_slots(words, A, d, l, base))


@pytest.mark.parametrize("circ,p,m,d,l", [("U", 3, 91, 2, 2), ("U", 13, 859, 4, 6), ("B", 3, 91, 2, 2),
                                          ("B", 5, 31, 3, 1)])
def test_compare_plain_vs_bruteforce(circ, p, m, d, l):
    A = slots.SlotAlgebra(p, cyclo.Ring(m))
    base = slots.digit_base(p, circ)
    ints = A.S // l
    cap = min(base ** (d * l), 2 ** 64)
    rng = random.Random(p * 31 + d)
    ev = circuits.PlainEval(A)
    for trial in range(3):
        wa = [rng.randrange(cap) for _ in range(ints)]
        wb = [rng.randrange(cap) for _ in range(ints)]
        for j in range(0, ints, 3):
            wb[j] = wa[j]
        if ints > 1:
            wb[1] = min(wa[1] + 1, cap - 1)
        lt, eq = circuits.compare(ev, _plain_words(A, wa, d, l, base), _plain_words(A, wb, d, l, base),
                                  circ, d, l, ints)
        for j in range(ints):
            assert int(lt.v[j * l, 0]) == int(wa[j] < wb[j])
            assert int(eq.v[j * l, 0]) == int(wa[j] == wb[j])


def test_spec_compare_min_examples():
    """(5,7) -> lt=1, eq=0; x vs x -> (0,1); min [3,1,2,9] -> 1."""
    A = slots.SlotAlgebra(3, cyclo.Ring(91))
    d, l, base = 2, 2, 2   # 4-bit words, 6 per ciphertext
    ev = circuits.PlainEval(A)
    ints = A.S // l
    g = golden("spec_examples.json")
    wa = [c[0] for c in g["compare_ints"]["cases"]] + [0] * (ints - 2)
    wb = [c[1] for c in g["compare_ints"]["cases"]] + [0] * (ints - 2)
    lt, eq = circuits.compare(ev, _plain_words(A, wa, d, l, base), _plain_words(A, wb, d, l, base), "U", d, l, ints)
    for j, c in enumerate(g["compare_ints"]["cases"]):
        assert (int(lt.v[j * l, 0]), int(eq.v[j * l, 0])) == (c[2], c[3])
    vals = g["min"]["values"]
    cur = [_plain_words(A, [v] * ints, d, l, base) for v in vals]
    while len(cur) > 1:
        cur = [circuits.vmin(ev, cur[i], cur[i + 1], "U", d, l, ints) for i in range(0, len(cur), 2)]
    got = slots.slots_to_words(cur[0].v, d, l, base, ints)
    assert got == [g["min"]["min"]] * ints


def test_select_and_broadcast_plain():
    A = slots.SlotAlgebra(13, cyclo.Ring(859))
    d, l, base = 4, 6, 7
    ints = A.S // l
    rng = random.Random(9)
    ev = circuits.PlainEval(A)
    wa = [rng.randrange(2 ** 64) for _ in range(ints)]
    wb = [rng.randrange(2 ** 64) for _ in range(ints)]
    a, b = _plain_words(A, wa, d, l, base), _plain_words(A, wb, d, l, base)
    mn = circuits.vmin(ev, a, b, "U", d, l, ints)
    mx = circuits.vmax(ev, a, b, "U", d, l, ints)
    assert slots.slots_to_words(mn.v, d, l, base, ints) == [min(x, y) for x, y in zip(wa, wb)]
    assert slots.slots_to_words(mx.v, d, l, base, ints) == [max(x, y) for x, y in zip(wa, wb)]


def _words_matrix(rng, T, ints, cap, tie_rate=4):
    """T word vectors; every tie_rate-th block copies a value from another element (ties)."""
    W = [[rng.randrange(cap) for _ in range(ints)] for _ in range(T)]
    for j in range(0, ints, tie_rate):
        if T > 1:
            W[rng.randrange(T)][j] = W[rng.randrange(T)][j]
    return W


def test_spec_sort_example():
    """sort [3,1,2] -> [1,2,3], slot-wise in every block, at p = 3 (T = 3 <= p)."""
    g = golden("spec_examples.json")["sort"]
    A = slots.SlotAlgebra(3, cyclo.Ring(91))
    d, l, base = 2, 2, 2
    ints = A.S // l
    ev = circuits.PlainEval(A)
    import itertools
    perms = list(itertools.permutations(g["values"]))
    cols = [perms[j % len(perms)] for j in range(ints)]       # block j holds a permutation
    xs = [_plain_words(A, [cols[j][t] for j in range(ints)], d, l, base) for t in range(len(g["values"]))]
    out = circuits.sort_rank(ev, xs, "U", d, l, ints)
    for k, o in enumerate(out):
        assert slots.slots_to_words(o.v, d, l, base, ints) == [g["sorted"][k]] * ints


@pytest.mark.parametrize("circ,p,m,d,l,T", [("U", 5, 31, 2, 2, 5), ("B", 5, 31, 2, 1, 4), ("U", 3, 91, 1, 2, 3)])
def test_sort_plain_vs_bruteforce(circ, p, m, d, l, T):
    A = slots.SlotAlgebra(p, cyclo.Ring(m))
    base = slots.digit_base(p, circ)
    ints = A.S // l
    cap = base ** (d * l)
    rng = random.Random(1000 + p * T)
    ev = circuits.PlainEval(A)
    W = _words_matrix(rng, T, ints, cap, tie_rate=2)
    xs = [_plain_words(A, W[t], d, l, base) for t in range(T)]
    out = circuits.sort_rank(ev, xs, circ, d, l, ints)
    got = [slots.slots_to_words(o.v, d, l, base, ints) for o in out]
    for j in range(ints):
        assert [got[k][j] for k in range(T)] == sorted(W[t][j] for t in range(T))


@pytest.mark.parametrize("op", ["min", "max"])
@pytest.mark.parametrize("T", [1, 2, 4, 5, 7])
def test_tournament_plain_vs_bruteforce(op, T):
    A = slots.SlotAlgebra(5, cyclo.Ring(31))
    d, l, base = 2, 2, 3
    ints = A.S // l
    rng = random.Random(77 + T)
    ev = circuits.PlainEval(A)
    W = _words_matrix(rng, T, ints, base ** (d * l))
    xs = [_plain_words(A, W[t], d, l, base) for t in range(T)]
    r = circuits.tournament(ev, xs, op, "U", d, l, ints)
    f = min if op == "min" else max
    assert slots.slots_to_words(r.v, d, l, base, ints) == [f(W[t][j] for t in range(T)) for j in range(ints)]


def test_spec_min_tournament_example():
    """min_tournament [3,1,2,9] -> 1 through the R20 fixed tree."""
    g = golden("spec_examples.json")["min"]
    A = slots.SlotAlgebra(3, cyclo.Ring(91))
    d, l, base = 2, 2, 2
    ints = A.S // l
    ev = circuits.PlainEval(A)
    xs = [_plain_words(A, [v] * ints, d, l, base) for v in g["values"]]
    r = circuits.tournament(ev, xs, "min", "U", d, l, ints)
    assert slots.slots_to_words(r.v, d, l, base, ints) == [g["min"]] * ints


def _p3s_plain():
    from oracle import bgv
    from conftest import load_cfg
    P = bgv.Params(load_cfg("p3s"))
    return P, P.alg


@pytest.mark.parametrize("e,products", [(1, 0), (2, 1), (5, 3), (8, 3), (1024, 10), (1023, 18)])
def test_power_product_count(e, products):
    """R24 left-to-right binary power: one squaring per bit below the top, one product per further 1 bit;
    every product extends the one chain, so the depth equals the product count"""
    ev = circuits.CountEval(7)
    r = circuits.power(ev, circuits.CountValue(), e)
    assert ev.counts["mul"] == products == (e.bit_length() - 1) + (bin(e).count("1") - 1)
    assert getattr(r, "depth", 0) == products


@pytest.mark.parametrize("qv", [1, 2, 3, 0, 5])
def test_private_query_semantics(qv):
    """R24 private_q (Listings 3-4) on plaintext slots of the p3 shadow ring (m = 111, 4 x 2
    hypercube, (d,l) = (8,4)): query type add (1), mult (2), power (3) or none gives
    Data + op1, Data * op1, Data^e, 0 in every slot of an integer block (slots outside the row-aligned
    blocks are 0)"""
    P, A = _p3s_plain()
    ev = circuits.PlainEval(A)
    rng = np.random.default_rng(qv)
    ints = P.ints_per_ct

    def words(w):
        return circuits.PlainValue(slots.words_to_slots(w, A, P.d, P.l, P.base))

    def fp_slots():
        v = np.zeros((A.S, A.D), dtype=np.int64)
        v[:, 0] = rng.integers(0, P.p, A.S)
        return v
    for e in (1, 5):
        data = [circuits.PlainValue(fp_slots()) for _ in range(2)]
        op1 = circuits.PlainValue(fp_slots())
        out = circuits.private_query(ev, data, words([qv] * ints), [words([c] * ints) for c in (1, 2, 3)],
                                     op1, e, P.circuit, P.d, P.l, ints)
        covered = np.array([(s % A.S1) < (A.S1 // P.l) * P.l for s in range(A.S)])
        for D, o in zip(data, out):
            x, y = D.v[:, 0], op1.v[:, 0]
            want = {1: (x + y) % P.p, 2: (x * y) % P.p, 3: np.array([pow(int(t), e, P.p) for t in x])}.get(qv, 0 * x)
            assert np.array_equal(o.v[covered, 0], want[covered])
            assert not o.v[~covered].any() and not o.v[:, 1:].any()


def test_private_query_bgv_decrypts():
    """R24 on the oracle BGV (p3 shadow ring, 13 + 4 primes): the decrypted result equals the plaintext
    semantics of a power query (e = 3)"""
    from oracle import bgv
    P, A = _p3s_plain()
    gal = sorted({pow(P.p, k, P.m) for k in range(1, A.D)} | {pow(A.g, s, P.m) for s in (1, 2)}
                 | {pow(A.g, -s, P.m) for s in (1, 2)})
    K = bgv.keygen(P, 0xB00C0001, gal)
    ev = circuits.OracleEval(P, K)
    ints = P.ints_per_ct
    rng = np.random.default_rng(7)

    def enc_words(w, idx):
        return bgv.encrypt(P, K, A.encode(slots.words_to_slots(w, A, P.d, P.l, P.base)), 0xB00C0003, idx)

    def enc_slots(v, idx):
        return bgv.encrypt(P, K, A.encode(v), 0xB00C0003, idx)
    x = np.zeros((A.S, A.D), dtype=np.int64)
    x[:, 0] = rng.integers(0, P.p, A.S)
    y = np.zeros((A.S, A.D), dtype=np.int64)
    y[:, 0] = rng.integers(0, P.p, A.S)
    codes = [enc_words([c] * ints, 10 + c) for c in (1, 2, 3)]
    covered = np.array([(s % A.S1) < (A.S1 // P.l) * P.l for s in range(A.S)])
    for qv, want in ((3, np.array([pow(int(t), 3, P.p) for t in x[:, 0]])),):
        out = circuits.private_query(ev, [enc_slots(x, 1)], enc_words([qv] * ints, 2), codes, enc_slots(y, 3), 3,
                                     P.circuit, P.d, P.l, ints)
        dec = A.decode(bgv.decrypt(P, K, out[0]))
        assert np.array_equal(dec[covered, 0], want[covered])
        assert not dec[~covered].any()


@pytest.mark.parametrize("p", PRIMES)
def test_r26_schedule_truth_tables(p):
    """R26 (f2): the two-dimensional Paterson-Stockmeyer bivariate circuit gives [x < y], [x = y]
    on every digit pair at the selected block sizes and at a few others; at the selected ones it uses no
    more products than R23 for p >= 11 and is no deeper than R16"""
    sel = circuits.r26_bivariate_k(p)
    r16 = _digit_run(p, "B")
    for k in sorted({sel, (1, 1), (2, 3), (min(4, p - 1), min(4, p - 1))}):
        res, mults, depth = _digit_run(p, "B", r23="r26", k=k)
        for x, y, lt, eq in res:
            assert (lt, eq) == (int(x < y), int(x == y)), (p, k, x, y)
        if k == sel:
            assert depth <= r16[2] and mults <= r16[1]
            if p >= 11:
                assert mults <= circuits._r23_cost(circuits.bivariate_lt_eq_r23, p, circuits.r23_bivariate_k(p))[0]


@pytest.mark.parametrize("p", PRIMES)
def test_r27_lazy_schedule_truth_tables(p):
    """R27 (R26 with one scale-down per sum of products, f1): [x < y], [x = y] on every digit pair at the
    selected and at other block sizes, with exactly R26's product count and depth (the lazy sums regroup
    the same products)"""
    sel = circuits.r26_bivariate_k(p)
    for k in sorted({sel, (1, 1), (2, 3), (min(4, p - 1), min(4, p - 1))}):
        res, mults, depth = _digit_run(p, "B", r23="r27", k=k)
        for x, y, lt, eq in res:
            assert (lt, eq) == (int(x < y), int(x == y)), (p, k, x, y)
        _, m26, d26 = _digit_run(p, "B", r23="r26", k=k)
        assert (mults, depth) == (m26, d26)


def test_r26_counts():
    """R26 counts: (k1, k2) = (1, 1) is the R16 tree (3p - 5 products); at p = 31 the rule picks
    (8, 8) with 59 products at depth 6 (R16: 88, R23: 73 at the same depth); at depth 7, (4, 8) needs 54,
    below the paper's asymptotic 2p - 6 = 56; at p = 13, 26 (R23: 28)"""
    for p in (5, 7, 11, 13):
        assert circuits._r26_cost(p, 1, 1)[0] == 3 * p - 5
    assert circuits.r26_bivariate_k(31) == (8, 8)
    assert circuits._r26_cost(31, 8, 8) == (59, 6)
    assert circuits._r26_cost(31, 4, 8) == (54, 7)
    assert circuits._r26_cost(13, *circuits.r26_bivariate_k(13)) == (26, 5)
