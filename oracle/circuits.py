"""Comparison circuits for the oracle (TEST INFRASTRUCTURE ONLY).

P:71, P:77 (§1): digit LT/EQ, 3p-5 multiplications [Tan]; bivariate vs univariate (PS).
P:282-290 (§2.1): decomposition -> mod extract -> digit EQ/LT -> lexicographic combination
  (first within each block of d digits, then across the l slots: ShiftMul / ShiftAdd).
P:490-506 (§5.3, Fig. 7): slot compaction.  P:557-573 (Listings 3-5): select by straightlining.
Readings: R16 schedules (the exact expression trees below are the contract both
sides follow; only ct x ct products, key switches and modulus switches can change bits),
R17 select/min/max/compaction.

Schedules are written once against an evaluator interface and run either on the oracle BGV
(OracleEval) or on plaintext slot values (PlainEval, used to pin the schedules).
Values are either ciphertext objects or python ints (plaintext constants in F_p).
"""
import functools
import math

import numpy as np

from . import bgv


# ----------------------------------------------------------------------------------------
# digit polynomials over F_p (definitions by interpolation)
# ----------------------------------------------------------------------------------------
def _binom_row(n, p):
    row = [1]
    for k in range(1, n + 1):
        row.append(row[-1] * (n - k + 1) // k)
    return [r % p for r in row]


def indicator_poly(p, target):
    """Lagrange interpolation over F_p: f(z) = sum_v target(v) (1 - (z - v)^{p-1}).
    Returns coefficients c_0..c_{p-1}."""
    c = [0] * p
    row = _binom_row(p - 1, p)
    for v in range(p):
        if target(v):
            c[0] = (c[0] + 1) % p
            # (z - v)^{p-1} = sum_k C(p-1,k) z^k (-v)^{p-1-k}
            for k in range(p):
                c[k] = (c[k] - row[k] * pow(-v, p - 1 - k, p)) % p
    return c


def lt_univariate_coeffs(p):
    """LT_U(z) = 1 iff z in {-1, ..., -(p-1)/2} (i.e. a_i < b_i with digits <= (p-1)/2)."""
    h = (p - 1) // 2
    return indicator_poly(p, lambda v: (p - h) <= v <= p - 1)


def eq_coeffs(p):
    return indicator_poly(p, lambda v: v == 0)


@functools.lru_cache(maxsize=None)
def _lt_bivariate_coeffs_cached(p):
    return tuple(tuple(r) for r in _lt_bivariate_coeffs(p))


def lt_bivariate_coeffs(p):
    """cached copy of _lt_bivariate_coeffs (pure function of p)"""
    return [list(r) for r in _lt_bivariate_coeffs_cached(p)]


def _lt_bivariate_coeffs(p):
    """LT_B(x, y) = [x < y] on [0,p)^2 by 2-D Lagrange interpolation, rewritten in
    (Y = y, Z = x - y): returns c[j][k] with LT = sum_{j,k} c[j][k] Y^j Z^k."""
    # f(x, y) = sum_{u<v} (1 - (x-u)^{p-1}) (1 - (y-v)^{p-1})
    fx = {}
    for u in range(p):
        fx[u] = indicator_poly(p, lambda t, u=u: t == u)
    C = [[0] * p for _ in range(p)]          # C[a][b] coefficient of x^a y^b
    for u in range(p):
        for v in range(u + 1, p):
            for a_ in range(p):
                if fx[u][a_]:
                    for b_ in range(p):
                        if fx[v][b_]:
                            C[a_][b_] = (C[a_][b_] + fx[u][a_] * fx[v][b_]) % p
    # substitute x = Z + Y: x^a = sum_r C(a, r) Z^r Y^(a-r)
    out = [[0] * (2 * p) for _ in range(2 * p)]   # out[j][k]: Y^j Z^k
    for a_ in range(p):
        row = _binom_row(a_, p) if a_ else [1]
        for b_ in range(p):
            c = C[a_][b_]
            if c:
                for r in range(a_ + 1):
                    out[(a_ - r) + b_][r] = (out[(a_ - r) + b_][r] + c * row[r]) % p
    return out


def eval_poly_fp(c, z, p):
    return sum(ci * pow(z, i, p) for i, ci in enumerate(c)) % p


# ----------------------------------------------------------------------------------------
# value helpers: python ints are plaintext constants
# ----------------------------------------------------------------------------------------
def is_const(x):
    return isinstance(x, (int, np.integer))


def vmul(ev, a, b):
    if is_const(a) and is_const(b):
        return int(a) * int(b) % ev.p
    if is_const(a):
        return ev.scalar(b, a)
    if is_const(b):
        return ev.scalar(a, b)
    return ev.mul(a, b)


def vadd(ev, a, b):
    if is_const(a) and is_const(b):
        return (int(a) + int(b)) % ev.p
    if is_const(a):
        return ev.add_const(b, a)
    if is_const(b):
        return ev.add_const(a, b)
    return ev.add(a, b)


def lincomb(ev, terms, const):
    """sum of c * x over terms with c != 0 (in the listed order) plus const (skipped if 0).
    R16: zero coefficients are dropped; a combination with no ciphertext term is a constant."""
    acc = None
    for c, x in terms:
        c %= ev.p
        if c == 0:
            continue
        t = vmul(ev, x, c)
        acc = t if acc is None else vadd(ev, acc, t)
    const %= ev.p
    if acc is None:
        return const
    if const:
        acc = vadd(ev, acc, const)
    return acc


def vmul_sum(ev, pairs):
    """R27: sum of the ct x ct products of pairs with one scale-down (ev.mul_sum); one pair is ev.mul"""
    if len(pairs) == 1:
        return ev.mul(*pairs[0])
    return ev.mul_sum(pairs)


class Powers:
    """R16 power rule: x^1 given; x^j (j >= 2) = x^a * x^(j-a), a = largest power of two < j."""

    def __init__(self, ev, x):
        self.ev = ev
        self.pw = {1: x}

    def __call__(self, j):
        if j not in self.pw:
            a = 1 << ((j - 1).bit_length() - 1)
            self.pw[j] = vmul(self.ev, self(a), self(j - a))
        return self.pw[j]


# ----------------------------------------------------------------------------------------
# digit circuits (a7)
# ----------------------------------------------------------------------------------------
def univariate_lt_eq(ev, z, p):
    """R16 univariate: W = z^2; e = (p-3)/2; LT = z*g(W) + ((p+1)/2) W^{e+1}, EQ = 1 - W^{e+1}
    (both read off the interpolated LT_U / EQ coefficients).  g(W) = sum_k c_{2k+1} W^k is
    evaluated Paterson-Stockmeyer style: baby step k0 = 2^ceil(log2 sqrt(e+1)), powers W^1..W^k0
    built in increasing order, chunks B_i = sum_{j<k0} c_{2(i k0 + j)+1} W^j, recursive split
    g[lo,hi) = g[lo,lo+h) + W^{k0 h} * g[lo+h,hi), h = largest power of two < hi-lo."""
    c = lt_univariate_coeffs(p)
    e = (p - 3) // 2
    assert all(c[2 * k] == 0 for k in range(1, (p - 1) // 2)) and c[0] == 0
    g = [c[2 * k + 1] for k in range(e + 1)]
    top = c[p - 1]
    W = vmul(ev, z, z)
    pw = Powers(ev, W)
    k0 = 1
    while k0 * k0 < e + 1:      # k0 = 2^ceil(log2 sqrt(e+1)): smallest power of two with k0^2 >= e+1
        k0 *= 2
    for j in range(2, k0 + 1):
        pw(j)
    nchunks = -(-(e + 1) // k0)

    def chunk(i):
        terms = [(g[i * k0 + j], pw(j)) for j in range(1, k0) if i * k0 + j <= e]
        return lincomb(ev, terms, g[i * k0])

    def ps(lo, hi):
        if hi - lo == 1:
            return chunk(lo)
        h = 1 << ((hi - lo - 1).bit_length() - 1)
        low = ps(lo, lo + h)
        high = ps(lo + h, hi)
        return vadd(ev, low, vmul(ev, pw(k0 * h), high))

    gval = ps(0, nchunks)
    We = pw(e + 1)
    lt = vadd(ev, vmul(ev, z, gval), vmul(ev, We, top))
    eq = vadd(ev, vmul(ev, We, -1), 1)
    return lt, eq


def bivariate_lt_eq(ev, x, y, p):
    """R16 bivariate: Z = x - y; powers Z^2..Z^{p-1} then Y^2..Y^{p-1} by the power rule;
    LT = sum_{j=1}^{p-1} Y^j * R_j(Z), R_j = sum_k c_{jk} Z^k; EQ = 1 - Z^{p-1}."""
    c = lt_bivariate_coeffs(p)
    assert all(c[0][k] == 0 for k in range(len(c[0]))), "LT_B has a Y^0 term"
    Z = vadd(ev, x, vmul(ev, y, -1))
    zp = Powers(ev, Z)
    for j in range(2, p):
        zp(j)
    yp = Powers(ev, y)
    for j in range(2, p):
        yp(j)
    lt = None
    for j in range(1, p):
        terms = [(c[j][k], zp(k)) for k in range(1, p)]
        R = lincomb(ev, terms, c[j][0])
        if is_const(R) and R == 0:
            continue
        t = vmul(ev, yp(j), R)
        lt = t if lt is None else vadd(ev, lt, t)
    eq = vadd(ev, vmul(ev, zp(p - 1), -1), 1)
    return lt, eq


# ----------------------------------------------------------------------------------------
# R23: baby-step / giant-step digit circuits (§8(f) f2; "2p-6 (Bivariate case) and
# sqrt(p-3) + O(log p) (Univariate case)", the paper's counts are asymptotic: DESIGN.md R23)
# ----------------------------------------------------------------------------------------
class CountValue:
    """stand-in ciphertext for counting products and depth (no arithmetic)"""

    def __init__(self, depth=0):
        self.depth = depth


class CountEval:
    """evaluator that only counts ct x ct products and tracks the multiplicative depth"""

    def __init__(self, p):
        self.p = p
        self.counts = {"mul": 0}

    def mul(self, a, b):
        self.counts["mul"] += 1
        return CountValue(max(a.depth, b.depth) + 1)

    def add(self, a, b):
        return CountValue(max(a.depth, b.depth))

    def mul_sum(self, pairs):
        self.counts["mul"] += len(pairs)
        return CountValue(max(max(a.depth, b.depth) for a, b in pairs) + 1)

    def scalar(self, a, c):
        return CountValue(a.depth)

    def add_const(self, a, c):
        return CountValue(a.depth)


def _largest_pow2_below(j):
    return 1 << ((j - 1).bit_length() - 1)


class Giant:
    """giant powers G_a = B^(a k) of a base power B = x^k (a >= 1): G_1 = B, G_a = G_a' * G_(a - a'),
    a' = the largest power of two < a (the R16 power rule on multiples of k)"""

    def __init__(self, ev, base):
        self.ev = ev
        self.g = {1: base}

    def __call__(self, a):
        if a not in self.g:
            a1 = _largest_pow2_below(a)
            self.g[a] = vmul(self.ev, self(a1), self(a - a1))
        return self.g[a]


def univariate_lt_eq_r23(ev, z, p, k=None):
    """R23 univariate: W = z^2, e = (p-3)/2, E = e + 1, g(W) = sum_i c_(2i+1) W^i (as R16).
    Baby powers W^2..W^k (power rule), giant powers G_a = W^(a k), a = 2..A-1, A = ceil((e+1)/k);
    chunks B_a = sum_(b<k) c_(2(ak+b)+1) W^b; g = B_0 + sum_(a=1)^(A-1) G_a B_a (a ascending);
    W^E = W^E (E <= k), G_a (E = a k) or G_a W^b (E = a k + b); LT = z g + ((p+1)/2) W^E,
    EQ = 1 - W^E.  k = r23_univariate_k(p) unless given."""
    c = lt_univariate_coeffs(p)
    e = (p - 3) // 2
    E = e + 1
    assert all(c[2 * i] == 0 for i in range(1, (p - 1) // 2)) and c[0] == 0
    g = [c[2 * i + 1] for i in range(e + 1)]
    top = c[p - 1]
    if k is None:
        k = r23_univariate_k(p)
    W = vmul(ev, z, z)
    pw = Powers(ev, W)
    for j in range(2, k + 1):
        pw(j)
    A = -(-(e + 1) // k)
    G = Giant(ev, pw(k))
    for a in range(2, A):
        G(a)

    def chunk(a):
        terms = [(g[a * k + b], pw(b)) for b in range(1, k) if a * k + b <= e]
        return lincomb(ev, terms, g[a * k])

    gval = chunk(0)
    for a in range(1, A):
        B = chunk(a)
        if is_const(B) and B == 0:
            continue
        gval = vadd(ev, gval, vmul(ev, G(a), B))
    if E <= k:
        WE = pw(E)
    else:
        a, b = divmod(E, k)
        WE = G(a) if b == 0 else vmul(ev, G(a), pw(b))
    lt = vadd(ev, vmul(ev, z, gval), vmul(ev, WE, top))
    eq = vadd(ev, vmul(ev, WE, -1), 1)
    return lt, eq


def bivariate_lt_eq_r23(ev, x, y, p, k=None):
    """R23 bivariate: Z = x - y, Z^2..Z^(p-1) by the power rule (EQ = 1 - Z^(p-1) is free);
    LT = sum_(j=1)^(p-1) Y^j R_j(Z) (as R16) evaluated baby-step / giant-step in Y: j = a k + b,
    baby powers Y^2..Y^k (power rule), giant powers G_a = Y^(a k), a = 2..A-1, A = floor((p-1)/k) + 1;
    I_a = sum_(b<k, 1<=ak+b<=p-1) Y^b R_(ak+b)(Z) (b ascending; the b = 0 term is R_(ak) itself);
    LT = I_0 + sum_(a=1)^(A-1) G_a I_a (a ascending).  k = 1 is the R16 tree.  k = r23_bivariate_k(p)
    unless given."""
    c = lt_bivariate_coeffs(p)
    assert all(c[0][i] == 0 for i in range(len(c[0]))), "LT_B has a Y^0 term"
    if k is None:
        k = r23_bivariate_k(p)
    Z = vadd(ev, x, vmul(ev, y, -1))
    zp = Powers(ev, Z)
    for j in range(2, p):
        zp(j)
    yp = Powers(ev, y)
    for j in range(2, k + 1):
        yp(j)
    A = (p - 1) // k + 1
    G = Giant(ev, yp(k))
    for a in range(2, A):
        G(a)

    def R(j):
        return lincomb(ev, [(c[j][i], zp(i)) for i in range(1, p)], c[j][0])

    def inner(a):
        acc = None
        for b in range(k):
            j = a * k + b
            if j < 1 or j > p - 1:
                continue
            r = R(j)
            if is_const(r) and r == 0:
                continue
            t = r if b == 0 else vmul(ev, yp(b), r)
            acc = t if acc is None else vadd(ev, acc, t)
        return 0 if acc is None else acc

    lt = inner(0)
    for a in range(1, A):
        I = inner(a)
        if is_const(I) and I == 0:
            continue
        t = vmul(ev, G(a), I)
        lt = t if (is_const(lt) and lt == 0) else vadd(ev, lt, t)
    eq = vadd(ev, vmul(ev, zp(p - 1), -1), 1)
    return lt, eq


def bivariate_lt_eq_r26(ev, x, y, p, k1=None, k2=None, lazy=False):
    """R26 bivariate, two-dimensional Paterson-Stockmeyer: LT = sum_(j,i) c_ji Y^j Z^i (Z = x - y, the R16
    coefficients) split into blocks j = k1 C + a, i = k2 D + b (a < k1, b < k2):
    L_CD = sum c Y^a Z^b (baby monomials Y^a Z^b = Y^a * Z^b, created when first needed, a and b ascending),
    inner_C = L_C0 + sum_(D>=1) Z^(k2 D) L_CD (D ascending), LT = inner_0 + sum_(C>=1) Y^(k1 C) inner_C
    (C ascending); every power of Y and of Z by the R16 power rule (one memo each, shared with EQ);
    zero blocks are skipped.  EQ = 1 - Z^(p-1).  (k1, k2) = r26_bivariate_k(p) unless given.
    lazy (R27): the products of each sum take one scale-down -- inner_C = L_C0, then the
    scalar terms c Z^(k2 D) of constant blocks (D ascending), then vmul_sum([(Z^(k2 D), L_CD) : D >= 1, L_CD
    a ciphertext]); LT likewise from inner_0 and the (Y^(k1 C), inner_C), C >= 1.  Same products and depth."""
    c = lt_bivariate_coeffs(p)
    if k1 is None:
        k1, k2 = r26_bivariate_k(p)
    Z = vadd(ev, x, vmul(ev, y, -1))
    zp = Powers(ev, Z)
    yp = Powers(ev, y)
    mono = {}

    def M(a, b):
        if (a, b) not in mono:
            mono[(a, b)] = zp(b) if a == 0 else (yp(a) if b == 0 else vmul(ev, yp(a), zp(b)))
        return mono[(a, b)]

    terms = {(j, i): c[j][i] % p for j in range(p) for i in range(p) if c[j][i] % p}
    Cm = max(j for j, _ in terms) // k1
    Dm = max(i for _, i in terms) // k2
    def acc(s, t):
        return t if (is_const(s) and s == 0) else vadd(ev, s, t)

    def lazy_sum(s, prs):
        """s, then the scalar terms, then one vmul_sum of the ciphertext pairs (R27)"""
        cts = []
        for g, v in prs:
            if is_const(v):
                s = acc(s, vmul(ev, g, v))
            else:
                cts.append((g, v))
        return acc(s, vmul_sum(ev, cts)) if cts else s

    lt = 0
    outer = []
    for C in range(Cm + 1):
        inner = 0
        prs = []
        for D in range(Dm + 1):
            L = lincomb(ev, [(terms[(k1 * C + a, k2 * D + b)], M(a, b)) for a in range(k1) for b in range(k2)
                             if (a, b) != (0, 0) and (k1 * C + a, k2 * D + b) in terms],
                        terms.get((k1 * C, k2 * D), 0))
            if is_const(L) and L == 0:
                continue
            if D == 0:
                inner = L
            elif lazy:
                prs.append((zp(k2 * D), L))
            else:
                inner = acc(inner, vmul(ev, zp(k2 * D), L))
        if lazy:
            inner = lazy_sum(inner, prs)
        if is_const(inner) and inner == 0:
            continue
        if C == 0:
            lt = inner
        elif lazy:
            outer.append((yp(k1 * C), inner))
        else:
            lt = acc(lt, vmul(ev, yp(k1 * C), inner))
    if lazy:
        lt = lazy_sum(lt, outer)
    eq = vadd(ev, vmul(ev, zp(p - 1), -1), 1)
    return lt, eq


@functools.lru_cache(maxsize=None)
def r26_bivariate_k(p):
    """R26: among (k1, k2) in [1, p-1]^2 whose circuit is no deeper than R16's, the fewest products, then
    the smallest k1, then the smallest k2"""
    cap = _r16_depth("B", p)
    best = None
    for k1 in range(1, p):
        for k2 in range(1, p):
            mu, d = _r26_cost(p, k1, k2)
            if d <= cap and (best is None or mu < best[0]):
                best = (mu, k1, k2)
    return best[1], best[2]


def _r26_cost(p, k1, k2):
    ev = CountEval(p)
    lt, eq = bivariate_lt_eq_r26(ev, CountValue(), CountValue(), p, k1, k2)
    return ev.counts["mul"], max(getattr(lt, "depth", 0), getattr(eq, "depth", 0))


def _r23_cost(fn, p, k):
    ev = CountEval(p)
    args = (CountValue(),) if fn is univariate_lt_eq_r23 else (CountValue(), CountValue())
    lt, eq = fn(ev, *args, p, k=k)
    d = max(getattr(lt, "depth", 0), getattr(eq, "depth", 0))
    return ev.counts["mul"], d


def _r16_depth(kind, p):
    ev = CountEval(p)
    if kind == "U":
        lt, eq = univariate_lt_eq(ev, CountValue(), p)
    else:
        lt, eq = bivariate_lt_eq(ev, CountValue(), CountValue(), p)
    return max(getattr(lt, "depth", 0), getattr(eq, "depth", 0))


def r23_univariate_k(p):
    """R23: among the baby-step sizes k in [1, (p-1)/2] whose circuit is no deeper than R16's (the
    modulus chains are sized for that depth), the one with the fewest products, then the smallest k"""
    cap = _r16_depth("U", p)
    ks = [k for k in range(1, max((p - 1) // 2, 1) + 1) if _r23_cost(univariate_lt_eq_r23, p, k)[1] <= cap]
    return min(ks, key=lambda k: (_r23_cost(univariate_lt_eq_r23, p, k)[0], k))


def r23_bivariate_k(p):
    """R23: among k in [1, p-1] with depth <= R16's, the fewest products, then the smallest k"""
    cap = _r16_depth("B", p)
    ks = [k for k in range(1, p) if _r23_cost(bivariate_lt_eq_r23, p, k)[1] <= cap]
    return min(ks, key=lambda k: (_r23_cost(bivariate_lt_eq_r23, p, k)[0], k))


# ----------------------------------------------------------------------------------------
# extraction (a8), lexicographic combination (a9), compare
# ----------------------------------------------------------------------------------------
def kappa_slots(alg, i, k):
    """kappa_{i,k} = mu_i^{p^k} in every slot (mu = trace-dual basis of {X^i})."""
    mu = alg.dual_basis()[i]
    v = alg.gf.pow(mu, alg.p ** k)
    return np.tile(v, (alg.S, 1))


def extract_digits(ev, ct, d):
    """digit_i = sum_{k<D} kappa_{i,k} (.) sigma_{p^k}(ct), i < d  ("mod extract")."""
    D = ev.alg.D
    F = [ct] + ev.frobenius_hoisted(ct, list(range(1, D)))    # R22: one ModUp for the D-1 maps
    out = []
    for i in range(d):
        acc = None
        for k in range(D):
            t = ev.ptmul(F[k], kappa_slots(ev.alg, i, k))
            acc = t if acc is None else ev.add(acc, t)
        out.append(acc)
    return out


def lex_tree(ev, lts, eqs):
    """Within a slot: merge adjacent pairs (hi = 2i+1, lo = 2i): LT = LT_hi + EQ_hi LT_lo,
    EQ = EQ_hi EQ_lo; an unpaired most-significant element passes through."""
    lts, eqs = list(lts), list(eqs)
    while len(lts) > 1:
        nl, ne = [], []
        for i in range(0, len(lts) - 1, 2):
            nl.append(vadd(ev, lts[i + 1], vmul(ev, eqs[i + 1], lts[i])))
            ne.append(vmul(ev, eqs[i + 1], eqs[i]))
        if len(lts) % 2:
            nl.append(lts[-1])
            ne.append(eqs[-1])
        lts, eqs = nl, ne
    return lts[0], eqs[0]


def block_mask(alg, l, ints, pred):
    """1 at the slots of the first `ints` integer blocks whose position in the block satisfies pred
    (R6 rows: slot s is position i = s mod S1 of its row; blocks cover i < floor(S1/l) l)"""
    m = np.zeros((alg.S, alg.D), dtype=np.int64)
    wpr = alg.S1 // l
    for s in range(alg.S):
        row, i = divmod(s, alg.S1)
        if i < wpr * l and row * wpr + i // l < ints and pred(i % l):
            m[s, 0] = 1
    return m


def lex_slots(ev, lt, eq, l, ints):
    """Across slots (ShiftMul/ShiftAdd), Kogge-Stone: round r, shift 2^r:
    mask[s] = [(s mod l) + 2^r < l]; hiLT = mask (.) rot(LT); hiEQ = mask (.) rot(EQ) + (1-mask);
    LT = hiLT + hiEQ * LT; EQ = hiEQ * EQ.  Result in slot 0 of each block."""
    r = 0
    while (1 << r) < l:
        sh = 1 << r
        mask = block_mask(ev.alg, l, ints, lambda t: t + sh < l)
        inv = (1 - mask) % ev.p
        inv[:, 1:] = 0
        hi_lt = ev.ptmul(ev.rotate(lt, sh), mask)
        hi_eq = ev.add_pt(ev.ptmul(ev.rotate(eq, sh), mask), inv)
        lt = vadd(ev, hi_lt, vmul(ev, hi_eq, lt))
        eq = vmul(ev, hi_eq, eq)
        r += 1
    return lt, eq


def compare(ev, a, b, circuit, d, l, ints):
    """(LT, EQ) of the words packed in a and b (block slot 0 holds the result).  circuit: "U" / "B"
    (R16 digit circuits), "U:r23" / "B:r23" (R23), "U:r26" / "B:r26" (R26 bivariate; univariate = R23) or
    "U:r27" / "B:r27" (R26 with R27's lazy scale-down of its sums)."""
    p = ev.p
    sched = circuit.partition(":")[2] or "r16"   # R16, R23 or R26 digit circuits (params "schedule")
    if circuit[0] == "U":
        z = ev.add(a, ev.scalar(b, -1))
        digs = extract_digits(ev, z, d)
        f = univariate_lt_eq_r23 if sched in ("r23", "r26", "r27") else univariate_lt_eq   # R26 / R27 univariate = R23
        res = [f(ev, x, p) for x in digs]
    else:
        da = extract_digits(ev, a, d)
        db = extract_digits(ev, b, d)
        f = {"r23": bivariate_lt_eq_r23, "r26": bivariate_lt_eq_r26,
             "r27": functools.partial(bivariate_lt_eq_r26, lazy=True)}.get(sched, bivariate_lt_eq)
        res = [f(ev, x, y, p) for x, y in zip(da, db)]
    lt, eq = lex_tree(ev, [r[0] for r in res], [r[1] for r in res])
    if l > 1:
        lt, eq = lex_slots(ev, lt, eq, l, ints)
    return lt, eq


def broadcast(ev, c, l, ints):
    """Copy block slot 0 to every slot of its block: c = mask0 (.) c, then for r:
    c = c + [(s mod l) >= 2^r] (.) rot_{-2^r}(c)."""
    c = ev.ptmul(c, block_mask(ev.alg, l, ints, lambda t: t == 0))
    r = 0
    while (1 << r) < l:
        sh = 1 << r
        c = ev.add(c, ev.ptmul(ev.rotate(c, -sh), block_mask(ev.alg, l, ints, lambda t: t >= sh)))
        r += 1
    return c


def select(ev, cond, x1, x2, l, ints):
    """x2 + bcast(cond) * (x1 - x2)  (Listing 4 straightlining)."""
    bc = broadcast(ev, cond, l, ints)
    diff = ev.add(x1, ev.scalar(x2, -1))
    return ev.add(x2, ev.mul(bc, diff))


def power(ev, x, e):
    """R24 x^e, e >= 1, left-to-right binary: acc = x; for each bit of e below the top one:
    acc = acc * acc, then acc = acc * x if the bit is 1 (e = 2^k: k squarings)."""
    assert e >= 1
    acc = x
    for bit in bin(e)[3:]:
        acc = ev.mul(acc, acc)
        if bit == "1":
            acc = ev.mul(acc, x)
    return acc


def private_query(ev, data, q, codes, op1, e, circuit, d, l, ints):
    """R24 private_q (Listing 4 straightlined, Listing 5 non-blocking -- the same values):
    c_j = bcast(EQ(q, code_j)), j = 0, 1, 2 (add, mult, power; the query type q and the codes are
    words in every integer block); for every database ciphertext D_i:
    out_i = ((D_i + op1) c_0 + (D_i op1) c_1) + D_i^e c_2."""
    masks = []
    for code in codes:
        _, eq = compare(ev, q, code, circuit, d, l, ints)
        masks.append(broadcast(ev, eq, l, ints))
    out = []
    for D in data:
        d1 = ev.add(D, op1)
        d2 = ev.mul(D, op1)
        d3 = power(ev, D, e)
        acc = ev.add(ev.mul(d1, masks[0]), ev.mul(d2, masks[1]))
        out.append(ev.add(acc, ev.mul(d3, masks[2])))
    return out


def vmin(ev, a, b, circuit, d, l, ints):
    lt, _ = compare(ev, a, b, circuit, d, l, ints)
    return select(ev, lt, a, b, l, ints)


def vmax(ev, a, b, circuit, d, l, ints):
    lt, _ = compare(ev, a, b, circuit, d, l, ints)
    return select(ev, lt, b, a, l, ints)


def tournament(ev, elems, op, circuit, d, l, ints):
    """R20 min/max over T elements (slot-wise), fixed tree over element indices (SURVEY §8(e),
    S:540-548 min_tournament): round r pairs (i, i + 2^r) for i = 0 mod 2^(r+1), the lower index
    is `a`, result stored at i; an element without a partner passes through unchanged."""
    f = vmin if op == "min" else vmax
    cur = list(elems)
    T = len(cur)
    sh = 1
    while sh < T:
        for i in range(0, T, 2 * sh):
            if i + sh < T:
                cur[i] = f(ev, cur[i], cur[i + sh], circuit, d, l, ints)
        sh *= 2
    return cur[0]


def sort_rank(ev, xs, circuit, d, l, ints):
    """R21 rank sort of T elements slot-wise (S:549-557 sort_rank, ties broken by index).
    For i < j: (lt, eq) = compare(x_i, x_j), le_ij = lt + eq = [x_i <= x_j].
    S_j = sum_{i<j} le_ij + sum_{i>j} (-1) * le_ji (i ascending); rank_j = S_j + (T-1-j), so
    rank_j = #{i : x_i < x_j or (x_i = x_j and i < j)}.
    v_jk = S_j + (T-1-j-k) (one constant, mod p) = rank_j - k;  e_jk = 1 - v_jk^(p-1) (power rule,
    = [rank_j = k] since |rank_j - k| < T <= p);  out_k = sum_j bcast(e_jk) * x_j (j ascending).
    Needs T <= p (ranks distinct in F_p)."""
    p = ev.p
    T = len(xs)
    assert 1 <= T <= p, "sort_rank needs T <= p"
    le = {}
    for i in range(T):
        for j in range(i + 1, T):
            lt, eq = compare(ev, xs[i], xs[j], circuit, d, l, ints)
            le[(i, j)] = ev.add(lt, eq)
    outs = [None] * T
    e = {}
    for j in range(T):
        S = None
        for i in range(T):
            if i == j:
                continue
            t = le[(i, j)] if i < j else ev.scalar(le[(j, i)], -1)
            S = t if S is None else ev.add(S, t)
        for k in range(T):
            c = (T - 1 - j - k) % p
            v = S if S is not None else None
            if v is None:                      # T == 1: rank 0 = k
                e[(j, k)] = 1
                continue
            v = ev.add_const(v, c) if c else v
            w = Powers(ev, v)(p - 1)
            e[(j, k)] = ev.add_const(ev.scalar(w, -1), 1)
    for k in range(T):
        acc = None
        for j in range(T):
            if is_const(e[(j, k)]):
                t = xs[j]
            else:
                t = ev.mul(broadcast(ev, e[(j, k)], l, ints), xs[j])
            acc = t if acc is None else ev.add(acc, t)
        outs[k] = acc
    return outs


# ----------------------------------------------------------------------------------------
# evaluators
# ----------------------------------------------------------------------------------------
class OracleEval:
    """Evaluator over the oracle BGV (bgv.py)."""

    def __init__(self, P, K):
        self.P, self.K = P, K
        self.p = P.p
        self.alg = P.alg
        self._pt = {}
        self.counts = {"mul": 0, "ks": 0}

    def _encode(self, slots):
        key = np.asarray(slots, dtype=np.int64).tobytes()
        if key not in self._pt:
            self._pt[key] = self.alg.encode(slots)
        return self._pt[key]

    def mul(self, a, b):
        self.counts["mul"] += 1
        self.counts["ks"] += 1
        return bgv.mul(self.P, self.K, a, b)

    def add(self, a, b):
        return bgv.add(self.P, a, b)

    def mul_sum(self, pairs):
        self.counts["mul"] += len(pairs)
        self.counts["ks"] += len(pairs)
        return bgv.mul_sum(self.P, self.K, pairs)

    def scalar(self, a, c):
        return bgv.mul_scalar(self.P, a, c)

    def add_const(self, a, c):
        return bgv.add_const(self.P, a, c)

    def ptmul(self, a, slots):
        return bgv.mul_plain(self.P, a, self._encode(slots))

    def add_pt(self, a, slots):
        return bgv.add_plain(self.P, a, self._encode(slots))

    def rotate(self, a, k):
        self.counts["ks"] += 1
        return bgv.rotate(self.P, self.K, a, k)

    def frobenius(self, a, k):
        self.counts["ks"] += 1
        return bgv.frobenius(self.P, self.K, a, k)

    def frobenius_hoisted(self, a, ks):
        self.counts["ks"] += len(ks)
        return bgv.automorphisms_hoisted(self.P, self.K, a, [pow(self.P.p, k, self.P.m) for k in ks])

    def modswitch(self, a):
        return bgv.modswitch(self.P, a)


class PlainValue:
    def __init__(self, v, depth=0):
        self.v = np.asarray(v, dtype=np.int64)
        self.depth = depth


class PlainEval:
    """Evaluator over plaintext slot values in F_{p^D} (pins the schedules; depth = number of
    ct x ct multiplications on the longest path)."""

    def __init__(self, alg):
        self.alg = alg
        self.p = alg.p
        self.gf = alg.gf
        self.counts = {"mul": 0, "ks": 0}

    def mul(self, a, b):
        self.counts["mul"] += 1
        return PlainValue(self.gf.mul(a.v, b.v), max(a.depth, b.depth) + 1)

    def add(self, a, b):
        return PlainValue((a.v + b.v) % self.p, max(a.depth, b.depth))

    def mul_sum(self, pairs):
        self.counts["mul"] += len(pairs)
        v = sum(self.gf.mul(a.v, b.v) for a, b in pairs) % self.p
        return PlainValue(v, max(max(a.depth, b.depth) for a, b in pairs) + 1)

    def scalar(self, a, c):
        return PlainValue(a.v * int(c) % self.p, a.depth)

    def add_const(self, a, c):
        v = a.v.copy()
        v[..., 0] = (v[..., 0] + int(c)) % self.p
        return PlainValue(v, a.depth)

    def ptmul(self, a, slots):
        return PlainValue(self.gf.mul(a.v, slots), a.depth)

    def add_pt(self, a, slots):
        return PlainValue((a.v + slots) % self.p, a.depth)

    def _rot_map(self, k):
        """slot s of sigma_{g^k}(a) is a(zeta^{g^k t_s}) = beta_{s'}^{p^j} with g^k t_s = t_{s'} p^j."""
        key = k % (self.alg.m * self.alg.S)
        if not hasattr(self, "_rm"):
            self._rm = {}
        if key not in self._rm:
            alg = self.alg
            t = pow(alg.g, k, alg.m)
            ppow = {pow(alg.p, j, alg.m): j for j in range(alg.D)}
            tindex = {ts: s for s, ts in enumerate(alg.t)}
            src, fj = [], []
            for s in range(alg.S):
                target = t * alg.t[s] % alg.m
                for jm, j in ppow.items():
                    cand = target * pow(jm, -1, alg.m) % alg.m
                    if cand in tindex:
                        src.append(tindex[cand])
                        fj.append(j)
                        break
            self._rm[key] = (np.array(src), np.array(fj))
        return self._rm[key]

    def rotate(self, a, k):
        src, fj = self._rot_map(k)
        out = a.v[src].copy()
        for j in set(fj.tolist()):
            if j:
                sel = fj == j
                out[sel] = self.gf.pow(out[sel], self.alg.p ** j)
        return PlainValue(out, a.depth)

    def frobenius(self, a, k):
        return PlainValue(self.gf.pow(a.v, self.p ** k), a.depth)

    def frobenius_hoisted(self, a, ks):
        return [self.frobenius(a, k) for k in ks]

    def modswitch(self, a):
        return PlainValue(a.v, a.depth + 1)


# ----------------------------------------------------------------------------------------
# slot compaction (a10, Fig. 7; R17)
# ----------------------------------------------------------------------------------------
def compaction_offsets(span):
    """candidate block offsets in preference order: 0, 1, -1, 2, -2, ..., span, -span."""
    out = [0]
    for k in range(1, span + 1):
        out += [k, -k]
    return out


def plan_compaction(useful, ints, span, wpr=None):
    """R17 greedy plan.  useful[c] = sorted useful block indices of input ct c.  For each input
    in order, repeatedly pick (existing output c', offset delta) placing the most remaining blocks
    b at free blocks b - delta of c' (first maximum in the order outputs ascending x offsets
    0, 1, -1, ...); if nothing fits anywhere, open a new output with delta = 0.
    Returns (groups [(c, c', delta, blocks)], n_out, dest {(c, b): (c', b')})."""
    wpr = wpr or ints          # blocks per row (R6 rows): a rotation by delta l moves blocks within a row

    def fits(b, dl):
        return 0 <= b - dl < ints and 0 <= b % wpr - dl < wpr

    occ = []
    groups = []
    dest = {}
    for c, blocks in enumerate(useful):
        rem = list(blocks)
        while rem:
            best, best_cnt = None, 0
            for cp in range(len(occ)):
                for dl in compaction_offsets(span):
                    cnt = sum(1 for b in rem if fits(b, dl) and (b - dl) not in occ[cp])
                    if cnt > best_cnt:
                        best, best_cnt = (cp, dl), cnt
            if best is None:
                occ.append(set())
                best = (len(occ) - 1, 0)
            cp, dl = best
            moved = [b for b in rem if fits(b, dl) and (b - dl) not in occ[cp]]
            for b in moved:
                occ[cp].add(b - dl)
                dest[(c, b)] = (cp, b - dl)
            groups.append((c, cp, dl, moved))
            rem = [b for b in rem if b not in set(moved)]
    return groups, len(occ), dest


def compaction_galois(alg, l, span):
    """rotation elements g^{+-delta l}, delta in [1, span]."""
    return sorted({pow(alg.g, s * k * l, alg.m) for k in range(1, span + 1) for s in (1, -1)})


def compact(ev, cts, useful, l, ints, span, modswitch=True):
    """out_{c'} = sum over groups (c, c', delta) of rot_{delta l}(cts[c] (.) mask(blocks)), then one
    modulus switch per output (R17).  Blocks of an output not written by any group are zero."""
    groups, n_out, dest = plan_compaction(useful, ints, span, ev.alg.S1 // l)
    outs = [None] * n_out
    for c, cp, dl, blocks in groups:
        if not blocks:
            continue
        bs = set(blocks)
        mask = block_mask_sets(ev.alg, l, bs)
        t = ev.ptmul(cts[c], mask)
        if dl:
            t = ev.rotate(t, dl * l)
        outs[cp] = t if outs[cp] is None else ev.add(outs[cp], t)
    if modswitch:
        outs = [ev.modswitch(o) for o in outs]
    return outs, dest


def block_mask_sets(alg, l, blocks):
    m = np.zeros((alg.S, alg.D), dtype=np.int64)
    for b in blocks:
        w0 = alg.word_slot(b, l)
        m[w0:w0 + l, 0] = 1
    return m
