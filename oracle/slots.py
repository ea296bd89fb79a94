"""Plaintext slot algebra for the oracle (TEST INFRASTRUCTURE ONLY).

P:271 (§2.1): SIMD slots via the ring isomorphism F_p[x]/Phi_m = prod_s F_p[x]/F_s.
P:284-286 (§2.1): an integer is decomposed into l slots of F_{p^d}, each split into digits.
Table 3: (d l) = d base-digits per F_{p^D} slot, l slots per integer (F1).

Readings: R5 (G, zeta, slot generator, slot order), R6 (integer encoding).
Elements of F_{p^D} = F_p[X]/G are int64 arrays of D coefficients (1, X, ..., X^{D-1}).
"""
import numpy as np

from .nt import factorize, mult_order, gcd


# ----------------------------------------------------------------------------------------
# polynomials over F_p as python lists (low -> high), used for small-degree work
# ----------------------------------------------------------------------------------------
def _trim(a):
    a = list(a)
    while len(a) > 1 and a[-1] == 0:
        a.pop()
    return a


def pmod(a, b, p):
    """a mod b over F_p (b nonzero)."""
    a = [x % p for x in a]
    b = _trim([x % p for x in b])
    db = len(b) - 1
    inv = pow(b[-1], -1, p)
    for k in range(len(a) - 1, db - 1, -1):
        c = a[k] * inv % p
        if c:
            for j in range(db + 1):
                a[k - db + j] = (a[k - db + j] - c * b[j]) % p
    return _trim(a[:db] if db > 0 else [0])


def pmul(a, b, p):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] = (out[i + j] + x * y) % p
    return _trim(out)


def psub(a, b, p):
    n = max(len(a), len(b))
    a = list(a) + [0] * (n - len(a))
    b = list(b) + [0] * (n - len(b))
    return _trim([(x - y) % p for x, y in zip(a, b)])


def pgcd(a, b, p):
    a, b = _trim(a), _trim(b)
    while b != [0]:
        a, b = b, pmod(a, b, p)
    return a


def ppowmod(base, e, mod, p):
    result = [1]
    base = pmod(base, mod, p)
    while e:
        if e & 1:
            result = pmod(pmul(result, base, p), mod, p)
        base = pmod(pmul(base, base, p), mod, p)
        e >>= 1
    return result


def is_irreducible(G, p):
    """Rabin's test: X^{p^D} = X mod G and gcd(X^{p^{D/r}} - X, G) = 1 for primes r | D."""
    D = len(G) - 1
    X = [0, 1]

    def frob_pow(k):  # X^{p^k} mod G
        y = X
        for _ in range(k):
            y = ppowmod(y, p, G, p)
        return y

    if psub(frob_pow(D), X, p) != [0]:
        return False
    for r in factorize(D):
        g = pgcd(G, psub(frob_pow(D // r), X, p), p)
        if len(g) > 1:
            return False
    return True


def smallest_irreducible(p, D):
    """R5: G = X^D + sum_{i<D} c_i X^i with the smallest v = sum c_i p^i that is irreducible."""
    for v in range(p ** D):
        c = [(v // p ** i) % p for i in range(D)]
        G = c + [1]
        if D == 1 or is_irreducible(G, p):
            return G
    raise ValueError("no irreducible polynomial")


class GF:
    """F_{p^D} = F_p[X]/G with vectorised (leading-axis batch) arithmetic."""

    def __init__(self, p, G):
        self.p = p
        self.G = np.array(G, dtype=np.int64)
        self.D = len(G) - 1

    def mul(self, a, b):
        a = np.asarray(a, dtype=np.int64)
        b = np.asarray(b, dtype=np.int64)
        D, p = self.D, self.p
        shape = np.broadcast_shapes(a.shape[:-1], b.shape[:-1])
        prod = np.zeros(shape + (2 * D - 1,), dtype=np.int64)
        for i in range(D):
            prod[..., i:i + D] += a[..., i:i + 1] * b
            prod %= p
        for k in range(2 * D - 2, D - 1, -1):
            c = prod[..., k:k + 1]
            prod[..., k - D:k] = (prod[..., k - D:k] - c * self.G[:D]) % p
        return prod[..., :D] % p

    def one(self, shape=()):
        e = np.zeros(tuple(shape) + (self.D,), dtype=np.int64)
        e[..., 0] = 1
        return e

    def pow(self, a, e):
        a = np.asarray(a, dtype=np.int64)
        r = self.one(a.shape[:-1])
        while e:
            if e & 1:
                r = self.mul(r, a)
            a = self.mul(a, a)
            e >>= 1
        return r

    def inv(self, a):
        return self.pow(a, self.p ** self.D - 2)

    def from_int(self, v):
        return np.array([(v // self.p ** i) % self.p for i in range(self.D)], dtype=np.int64)

    def trace(self, a):
        """Tr(a) = sum_k a^{p^k} (an element of F_p, returned as int)."""
        s = np.zeros(self.D, dtype=np.int64)
        x = np.asarray(a, dtype=np.int64)
        for _ in range(self.D):
            s = (s + x) % self.p
            x = self.pow(x, self.p)
        assert all(int(v) == 0 for v in s[1:])
        return int(s[0])


def _solve_mod_p(A, b, p):
    """Solve A x = b over F_p (A square invertible) by Gauss-Jordan elimination."""
    A = [[int(v) % p for v in row] + [int(bb) % p] for row, bb in zip(A, b)]
    n = len(A)
    for c in range(n):
        piv = next(r for r in range(c, n) if A[r][c])
        A[c], A[piv] = A[piv], A[c]
        inv = pow(A[c][c], -1, p)
        A[c] = [v * inv % p for v in A[c]]
        for r in range(n):
            if r != c and A[r][c]:
                f = A[r][c]
                A[r] = [(x - f * y) % p for x, y in zip(A[r], A[c])]
    return [A[r][n] for r in range(n)]


class SlotAlgebra:
    """R5: D = ord_m(p), S = n/D; G smallest irreducible; zeta = beta^((p^D-1)/m) for the first
    beta (integer order, v = 1, 2, ...) giving exact order m; slot s <-> zeta^{t_s}, t_s = g^s."""

    def __init__(self, p, ring):
        self.p = p
        self.ring = ring
        m, n = ring.m, ring.n
        self.m, self.n = m, n
        self.D = mult_order(p, m)
        self.S = n // self.D
        self.G = smallest_irreducible(p, self.D)
        self.gf = GF(p, self.G)
        self.zeta = self._find_zeta()
        # R5: slot s = j*S1 + i <-> t_s = g^i g2^j (cyclic quotient: S1 = S, g2 = 1)
        self.g, self.S1, self.g2, self.S2 = self._slot_generators()
        self.t = [pow(self.g, s % self.S1, m) * pow(self.g2, s // self.S1, m) % m for s in range(self.S)]
        # zeta^e for e < m (evaluation table)
        zp = np.zeros((m, self.D), dtype=np.int64)
        x = self.gf.one()
        for e in range(m):
            zp[e] = x
            x = self.gf.mul(x, self.zeta)
        self.zpow = zp
        self._enc = None

    # --- structure -------------------------------------------------------------------
    def _find_zeta(self):
        p, D, m = self.p, self.D, self.m
        e = (p ** D - 1) // m
        primes_m = list(factorize(m))
        for v in range(1, p ** D):
            z = self.gf.pow(self.gf.from_int(v), e)
            if all(not np.array_equal(self.gf.pow(z, m // r), self.gf.one()) for r in primes_m):
                return z
        raise ValueError("no element of order m")

    def _powers_of_p(self):
        return {pow(self.p, k, self.m) for k in range(self.D)}

    def _order(self, t):
        """multiplicative order of t mod m: divide n = phi(m) by its prime factors while t^(o/r) = 1"""
        if getattr(self, "_nf", None) is None:
            self._nf = factorize(self.n)
        o = self.n
        for r in self._nf:
            while o % r == 0 and pow(t, o // r, self.m) == 1:
                o //= r
        return o

    def quotient_order(self, t):
        """order of t in Z_m^* / <p>: the exponents k with t^k in <p> are the multiples of it, so
        start from ord(t) and divide by primes r while t^(k/r) stays in <p>"""
        if getattr(self, "_H", None) is None:
            self._H = self._powers_of_p()
        k = self._order(t)
        for r in self._nf:
            while k % r == 0 and pow(t, k // r, self.m) in self._H:
                k //= r
        return k

    def _slot_generators(self):
        """R5.  Cyclic Z_m^*/<p>: g = the smallest t of quotient order S with t^S = 1 (mod m) if one
        exists ("good" generator), else the smallest of quotient order S; (S1, g2, S2) = (S, 1, 1).
        Otherwise (hypercube Z_S1 x Z_S2, S1 = the largest quotient order): g = the smallest t of
        quotient order S1 with t^S1 = 1 (mod m) if one exists, else the smallest of that order;
        g2 = the smallest t outside <p, g> with t^S2 in <p, g>, preferring t^S2 = 1 (mod m); every
        unit must be p^k g^i g2^j for exactly one (k, i, j)."""
        m, S = self.m, self.S
        if S == 1:
            return 1, 1, 1, 1
        units = [t for t in range(2, m) if gcd(t, m) == 1]
        qo = {}
        first = None
        for t in units:
            o = self.quotient_order(t)
            if o == S:
                if pow(t, S, m) == 1:
                    return t, S, 1, 1
                if first is None:
                    first = t
            qo[t] = o
        if first is not None:
            return first, S, 1, 1
        S1 = max(qo.values())
        S2 = S // S1
        cands = [t for t in units if qo[t] == S1]
        g = next((t for t in cands if pow(t, S1, m) == 1), cands[0])
        Hg = {pow(self.p, k, m) * pow(g, i, m) % m for k in range(self.D) for i in range(S1)}
        c2 = [t for t in units if t not in Hg and pow(t, S2, m) in Hg
              and all(pow(t, j, m) not in Hg for j in range(1, S2))]
        if not c2:
            raise NotImplementedError("Z_m^*/<p> is not Z_S1 x Z_S2")
        g2 = next((t for t in c2 if pow(t, S2, m) == 1), c2[0])
        cover = {h * pow(g2, j, m) % m for h in Hg for j in range(S2)}
        if len(cover) != self.n:
            raise NotImplementedError("Z_m^*/<p> is not generated by (p, g, g2)")
        return g, S1, g2, S2

    def words_per_row(self, l):
        """R6 (hypercube rows): floor(S1 / l) integers per row of S1 slots"""
        return self.S1 // l

    def ints(self, l):
        return self.S2 * (self.S1 // l)

    def word_slot(self, w, l):
        """first slot of integer w: row w // wpr, position (w mod wpr) * l in the row"""
        wpr = self.S1 // l
        return (w // wpr) * self.S1 + (w % wpr) * l

    # --- decode / encode ---------------------------------------------------------------
    def decode(self, a, chunk=512):
        """beta_s = a(zeta^{t_s}) for every slot s (definition).  a: ints mod p, len n."""
        a = np.asarray(a, dtype=np.int64) % self.p
        m, p = self.m, self.p
        j = np.arange(self.n, dtype=np.int64)
        out = np.zeros((self.S, self.D), dtype=np.int64)
        for s0 in range(0, self.S, chunk):
            ts = np.array(self.t[s0:s0 + chunk], dtype=np.int64)
            idx = (ts[:, None] * j[None, :]) % m                 # (c, n)
            vals = self.zpow[idx]                                # (c, n, D)
            out[s0:s0 + chunk] = np.einsum("cnd,n->cd", vals % p, a) % p
        return out

    def _prepare_encode(self):
        """Per slot: F_s = prod_k (x - zeta^{t_s p^k}), H_s = Phi_m / F_s (mod p),
        h_s^{-1} = H_s(zeta^{t_s})^{-1}, and the map V_s^{-1}: F_{p^D} -> F_p[x]/F_s."""
        p, D, m = self.p, self.D, self.m
        phi = [int(c) % p for c in self.ring.phi]
        Hs, hinv, Vinv = [], [], []
        gf = self.gf
        for s in range(self.S):
            ts = self.t[s]
            # F_s coefficients in F_{p^D}[x]: start with 1
            F = [gf.one()]
            for k in range(D):
                r = self.zpow[(ts * pow(p, k, m)) % m]
                newF = [np.zeros(D, dtype=np.int64) for _ in range(len(F) + 1)]
                for i, c in enumerate(F):
                    newF[i + 1] = (newF[i + 1] + c) % p
                    newF[i] = (newF[i] - gf.mul(c, r)) % p
                F = newF
            assert all(int(v) == 0 for c in F for v in c[1:]), "F_s not over F_p"
            Fp = [int(c[0]) for c in F]
            # H_s = Phi / F_s exactly over F_p
            H = self._pdiv_exact(phi, Fp)
            Hs.append(H)
            y = self.zpow[ts % m]
            hval = np.zeros(D, dtype=np.int64)
            for e, c in enumerate(H):
                if c:
                    hval = (hval + c * self.zpow[(ts * e) % m]) % p
            hinv.append(gf.inv(hval))
            # V_s columns: coefficients of y^j, j < D
            cols = [self.zpow[(ts * j) % m] for j in range(D)]
            Vinv.append(np.array(cols, dtype=np.int64).T)   # V_s (D x D); solved per encode
        self._enc = (Hs, hinv, Vinv)

    def _pdiv_exact(self, a, b):
        p = self.p
        a = list(a)
        db = len(b) - 1
        q = [0] * (len(a) - db)
        for k in range(len(a) - 1, db - 1, -1):
            c = a[k] % p
            q[k - db] = c
            if c:
                for j in range(db + 1):
                    a[k - db + j] = (a[k - db + j] - c * b[j]) % p
        assert all(v % p == 0 for v in a[:db]), "F_s does not divide Phi_m mod p"
        return q

    def encode(self, beta):
        """The unique a in F_p[x]/Phi_m with a(zeta^{t_s}) = beta_s (CRT):
        a = sum_s H_s * w_s, w_s(zeta^{t_s}) = beta_s * H_s(zeta^{t_s})^{-1}, deg w_s < D."""
        if self._enc is None:
            self._prepare_encode()
        Hs, hinv, Vs = self._enc
        p = self.p
        beta = np.asarray(beta, dtype=np.int64) % p
        a = np.zeros(self.n, dtype=np.int64)
        for s in range(self.S):
            if not beta[s].any():
                continue
            gam = self.gf.mul(beta[s], hinv[s])
            w = _solve_mod_p(Vs[s], gam, p)
            H = np.array(Hs[s], dtype=np.int64)
            for i, wi in enumerate(w):
                if wi:
                    a[i:i + len(H)] = (a[i:i + len(H)] + wi * H) % p
        return a

    # --- Frobenius digit extraction constants ------------------------------------
    def dual_basis(self):
        """mu_i with Tr(mu_i X^j) = delta_ij (trace-dual of the power basis {X^i})."""
        if getattr(self, "_dual", None) is None:
            self._dual = self._dual_basis()
        return self._dual

    def _dual_basis(self):
        D, p, gf = self.D, self.p, self.gf
        basis = [gf.from_int(p ** i) for i in range(D)]       # X^i
        # Tr matrix T[i][j] = Tr(X^i X^j); mu = T^{-1} applied to the power basis
        T = [[gf.trace(gf.mul(basis[i], basis[j])) for j in range(D)] for i in range(D)]
        mus = []
        for i in range(D):
            e = [1 if k == i else 0 for k in range(D)]
            c = _solve_mod_p(T, e, p)       # mu_i = sum_k c_k X^k with sum_k c_k T[k][j] = delta
            mus.append(np.array(c, dtype=np.int64) % p)
        # T symmetric, so solving T c = e_i gives sum_k c_k Tr(X^k X^j) = delta_ij
        return mus


# ----------------------------------------------------------------------------------------
# integer <-> slot encoding (R6, Table 3 pins)
# ----------------------------------------------------------------------------------------
def digit_base(p, circuit):
    """Bivariate digits in [0, p); univariate digits in [0, (p-1)/2] i.e. base (p+1)/2."""
    return p if circuit[0] == "B" else (p + 1) // 2


def int_to_digits(x, base, count):
    if x < 0 or x >= base ** count:
        raise ValueError("OutOfRange")
    return [(x // base ** i) % base for i in range(count)]


def words_to_slots(words, alg, d, l, base):
    """Word j occupies slots w0 .. w0+l-1, w0 = alg.word_slot(j, l) (= j*l for a cyclic slot
    structure); slot w0+s holds sum_{i<d} a_{s,i} X^i where x = sum_s sum_i a_{s,i} base^{s d + i}
    (little-endian).  Unused slots are 0."""
    S, D = alg.S, alg.D
    assert d <= D
    cap = alg.ints(l)
    assert len(words) <= cap
    out = np.zeros((S, D), dtype=np.int64)
    for j, x in enumerate(words):
        dig = int_to_digits(int(x), base, d * l)
        w0 = alg.word_slot(j, l)
        for s in range(l):
            for i in range(d):
                out[w0 + s, i] = dig[s * d + i]
    return out


def slots_to_words(slots, d, l, base, count, alg=None):
    out = []
    for j in range(count):
        w0 = alg.word_slot(j, l) if alg is not None else j * l
        x = 0
        for s in range(l):
            for i in range(d):
                x += int(slots[w0 + s][i]) * base ** (s * d + i)
        out.append(x)
    return out
