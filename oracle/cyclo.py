"""Cyclotomic ring R_q = Z_q[x]/Phi_m(x) for the oracle (TEST INFRASTRUCTURE ONLY).

P:267 (§2.1): R_Q = Z_Q[x]/(Phi_m(x)), N = phi(m).  Non-power-of-two m.
P:313-316 (§2.2): evaluation ("integer DFT") representation and BluesteinNTT.
Listing 1/2: filtering keeps the Z_m^* positions in ascending order.
"""
import numpy as np

from . import _c
from .nt import factorize, gcd


def mobius(n):
    f = factorize(n)
    if any(e > 1 for e in f.values()):
        return 0
    return -1 if len(f) % 2 else 1


def _polymul_int(a, b):
    out = [0] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x:
            for j, y in enumerate(b):
                out[i + j] += x * y
    return out


def _polydiv_exact_int(a, b):
    """Exact division of integer polys (b monic); asserts zero remainder."""
    a = list(a)
    db = len(b) - 1
    q = [0] * (len(a) - db)
    for k in range(len(a) - 1, db - 1, -1):
        c = a[k]
        q[k - db] = c
        if c:
            for j in range(db + 1):
                a[k - db + j] -= c * b[j]
    assert all(v == 0 for v in a[:db]), "inexact division"
    return q


def cyclotomic(m):
    """Phi_m over Z via Phi_m = prod_{d|m} (x^d - 1)^{mu(m/d)}; coefficients low->high (len n+1)."""
    divs = [d for d in range(1, m + 1) if m % d == 0]
    num, den = [1], [1]
    for d in divs:
        mu = mobius(m // d)
        b = [-1] + [0] * (d - 1) + [1]
        if mu == 1:
            num = _polymul_int(num, b)
        elif mu == -1:
            den = _polymul_int(den, b)
    return _polydiv_exact_int(num, den)


def zm_star(m):
    """Z_m^* in ascending order (Listing 1 loop order)."""
    return [i for i in range(m) if gcd(i, m) == 1]


class Ring:
    """Z[x]/Phi_m with per-prime helpers.  Polynomials are uint64 residue vectors of length n."""

    def __init__(self, m):
        self.m = m
        self.phi = np.array(cyclotomic(m), dtype=np.int64)
        self.n = len(self.phi) - 1
        self.z = np.array(zm_star(m), dtype=np.int32)
        assert len(self.z) == self.n

    # --- coefficient-form primitives -------------------------------------------------
    def mul(self, a, b, q):
        """Schoolbook product, folded mod x^m - 1, reduced mod (q, Phi_m) (C helper)."""
        return _c.ring_mul(a, b, self.phi, q, self.m)

    def reduce_int(self, coeffs):
        """Exact reduction of an integer polynomial (any length) modulo Phi_m over Z: fold the
        exponents mod m (x^m = 1 modulo Phi_m, which divides x^m - 1), then long division."""
        t = [0] * self.m
        for k, c in enumerate(coeffs):
            t[k % self.m] += int(c)
        n = self.n
        ph = [int(c) for c in self.phi]
        for k in range(len(t) - 1, n - 1, -1):
            c = t[k]
            if c:
                for j in range(n + 1):
                    t[k - n + j] -= c * ph[j]
        t = t[:n] + [0] * max(0, n - len(t))
        return t

    def automorph_int(self, coeffs, t):
        """sigma_t(f)(x) = f(x^t) mod Phi_m over Z (exponents reduced mod m first)."""
        out = [0] * self.m
        for j, c in enumerate(coeffs):
            if c:
                out[(j * t) % self.m] += int(c)
        return self.reduce_int(out)

    def automorph_mod(self, a, t, q):
        """sigma_t on residues mod q."""
        out = np.zeros(self.m, dtype=np.uint64)
        idx = (np.arange(self.n, dtype=np.int64) * t) % self.m
        # distinct j give distinct j*t mod m (t invertible mod m), so plain assignment is exact
        out[idx] = np.asarray(a, dtype=np.uint64) % np.uint64(q)
        return _c.poly_mod_phi(out, self.phi, q)

    # --- evaluation form (kernel parity only) ----------------------------------------
    def omega_pows(self, w, q):
        pw = np.empty(self.m, dtype=np.uint64)
        x = 1
        for e in range(self.m):
            pw[e] = x
            x = x * w % q
        return pw

    def to_eval(self, a, w, q):
        """E[k] = a(w^{z_k}), z_k ascending in Z_m^* -- naive evaluation (DESIGN R3)."""
        return _c.eval_naive(np.asarray(a, dtype=np.uint64), self.z, self.m, self.omega_pows(w, q), q)


def bluestein_literal(f, m, w, q, M):
    """The paper's BluesteinNTT, step by step, with the zero-padded product computed
    by schoolbook convolution (no NTT).  Returns the filtered length-n vector.

    h = 2^{-1} mod m (m odd) so that j*k = h(j^2 + k^2 - (k-j)^2) (mod m):
      1. C_j = f_j * TF1_j, TF1_j = w^(h j^2)                  ("multiplied element-wise by TF1")
      2. C_pad (length M >= 2m-1) times D_pad, D_t = w^(-h t^2) ("padded ... multiplied by D_pad")
      3. truncate to m, adding the exceeding coefficients      ("the exceeding coefficient being added")
      4. multiply element-wise by TF1                          ("multiplied element-wise by TF1")
      5. keep the Z_m^* positions in ascending order           ("filtered ... from m to N", Listing 1)
    D_pad holds D_t for t in [0, m) and zeros up to M; the linear product has length 2m-1 <= M,
    and y_k = lin_k + lin_{k+m} is the length-m cyclic product sum_j C_j D_{(k-j) mod m}.
    """
    assert M >= 2 * m - 1
    h = pow(2, -1, m)
    fm = [int(f[j]) if j < len(f) else 0 for j in range(m)]
    tf1 = [pow(w, h * j * j % m, q) for j in range(m)]
    C = [fm[j] * tf1[j] % q for j in range(m)]
    winv = pow(w, -1, q)
    Dpad = [pow(winv, h * t * t % m, q) for t in range(m)] + [0] * (M - m)
    lin = [0] * (2 * m - 1)
    for j, c in enumerate(C):
        if c:
            for t in range(m):
                lin[j + t] = (lin[j + t] + c * Dpad[t]) % q
    y = [(lin[k] + (lin[k + m] if k + m < len(lin) else 0)) % q for k in range(m)]
    E = [y[k] * tf1[k] % q for k in range(m)]
    return [E[k] for k in range(m) if gcd(k, m) == 1]
