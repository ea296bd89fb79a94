"""Leveled BGV over R_Q = Z_Q[x]/Phi_m in RNS, coefficient form (TEST INFRASTRUCTURE ONLY).

P:254-271 (§2.1): BGV, C = R_Q x R_Q, Q = prod q_i (Table 1), modulus chain, SIMD slots.
P:313 (§2.2): RNS residue matrix (L+1) x phi(m).  P:403 (§4): CRT with big integers.
Readings: R1 chain, R7 sampling, R8 keys (hybrid key switching), R9 encrypt,
R10 decrypt, R11 linear ops, R12 level alignment, R13 modulus switching, R14 key switching.

Representation: an RNS polynomial is a uint64 array [len(idx), n] of canonical residues,
idx = indices into Params.moduli (0..L cipher primes, L+1..L+K special primes).
Every lift is the exact centered CRT representative computed with Python big integers.
"""
import math

import numpy as np

from . import _c, prng
from .cyclo import Ring
from .nt import bluestein_pad, centered, lcm, prime_chain, root_of_unity
from .slots import SlotAlgebra, digit_base


class Params:
    """R1: q_0..q_L = the n_cipher smallest primes >= 2^(bits-1), q = 1 mod lcm(p, m, M);
    special primes P_0..P_{K-1} continue the same ascending search (so P_k > every q_i)."""

    def __init__(self, cfg):
        self.cfg = dict(cfg)
        self.name = cfg.get("name", "")
        self.p = int(cfg["p"])
        self.m = int(cfg["m"])
        self.schedule = cfg.get("schedule", "r16")     # digit-circuit reading: R16, R23, R26 or R27
        assert self.schedule in ("r16", "r23", "r26", "r27")
        self.circuit = cfg.get("circuit", "U") + ("" if self.schedule == "r16" else ":" + self.schedule)
        self.d = int(cfg["d"])
        self.l = int(cfg["l"])
        self.ring = Ring(self.m)
        self.n = self.ring.n
        self.bluestein = cfg.get("bluestein", "pow2")      # R25: "mixed" -> mixed-radix length
        assert self.bluestein in ("pow2", "mixed")
        self.M = bluestein_pad(self.m, self.bluestein == "mixed")
        mod = lcm(self.p, self.m, self.M)
        self.q = prime_chain(mod, int(cfg["cipher_bits"]), int(cfg["n_cipher"]), exclude={self.p})
        self.P = prime_chain(mod, int(cfg["special_bits"]), int(cfg["n_special"]),
                             after=max(self.q), exclude={self.p})
        self.moduli = self.q + self.P
        self.L1 = len(self.q)              # number of cipher primes (top level)
        self.K = len(self.P)
        self.special = list(range(self.L1, self.L1 + self.K))
        self.alpha = int(cfg["alpha"])
        self.dnum = math.ceil(self.L1 / self.alpha)
        self.omega = [root_of_unity(self.m, q) for q in self.moduli]
        self._alg = None
        self.base = digit_base(self.p, self.circuit)

    @property
    def alg(self):
        if self._alg is None:
            self._alg = SlotAlgebra(self.p, self.ring)
        return self._alg

    @property
    def ints_per_ct(self):
        return self.alg.ints(self.l)

    def digit_group(self, j, level):
        """R8: G_j = {j*alpha, ..., (j+1)*alpha-1} restricted to the primes present at `level`."""
        return [i for i in range(j * self.alpha, min((j + 1) * self.alpha, self.L1)) if i < level]


# ----------------------------------------------------------------------------------------
# RNS helpers
# ----------------------------------------------------------------------------------------
def int_poly_to_rns(P, coeffs, idx):
    """Embed an integer polynomial (python/numpy ints, length n) into the limbs idx."""
    c = [int(x) for x in coeffs]
    out = np.empty((len(idx), P.n), dtype=np.uint64)
    for r, i in enumerate(idx):
        q = P.moduli[i]
        out[r] = np.array([x % q for x in c], dtype=np.uint64)
    return out


def lift_centered(P, arr, idx):
    """Exact centered CRT lift of the limbs `idx` of arr (rows aligned with idx) -> list of ints
    in (-Q^/2, Q^/2], Q^ = prod of those primes (textbook CRT, "big integer")."""
    mods = [P.moduli[i] for i in idx]
    Q = 1
    for q in mods:
        Q *= q
    acc = np.zeros(arr.shape[1], dtype=object)
    for r, q in enumerate(mods):
        Qi = Q // q
        c = Qi * pow(Qi, -1, q)
        acc = acc + arr[r].astype(object) * c
    acc = acc % Q
    half = Q // 2
    return [int(x) - Q if x > half else int(x) for x in acc], Q


def _ints_mod(vals, q):
    return np.array([v % q for v in vals], dtype=np.uint64)


def _add(a, b, P, idx):
    out = np.empty_like(a)
    for r, i in enumerate(idx):
        q = np.uint64(P.moduli[i])
        s = a[r] + b[r]
        out[r] = np.where(s >= q, s - q, s)
    return out


def _sub(a, b, P, idx):
    out = np.empty_like(a)
    for r, i in enumerate(idx):
        q = np.uint64(P.moduli[i])
        out[r] = np.where(a[r] >= b[r], a[r] - b[r], a[r] + (q - b[r]))
    return out


def _mul(a, b, P, idx):
    out = np.empty_like(a)
    for r, i in enumerate(idx):
        out[r] = P.ring.mul(a[r], b[r], P.moduli[i])
    return out


def _scal(a, c, P, idx):
    """multiply limb r by the integer c (any sign) mod q."""
    out = np.empty_like(a)
    for r, i in enumerate(idx):
        q = P.moduli[i]
        out[r] = _c.vec_mulscalar(a[r], int(c) % q, q)
    return out


# ----------------------------------------------------------------------------------------
# keys
# ----------------------------------------------------------------------------------------
class Ciphertext:
    def __init__(self, parts, level):
        self.parts = parts      # list of uint64 [level, n] arrays
        self.level = level

    def copy(self):
        return Ciphertext([x.copy() for x in self.parts], self.level)


class Keys:
    def __init__(self):
        self.s = None           # int64[n] ternary secret
        self.pk = None          # (b, a) over cipher limbs 0..L
        self.ksk = {}           # key id -> list over digits of (b_j, a_j) over all QP limbs


def keygen(P, seed, galois=(), relin=True):
    """R8.  s ternary; pk = (-a s + p e, a) over Q; for key id t (0 = relinearisation with
    s' = s^2, else s' = sigma_t(s)) and digit j: swk_j = (-a_j s + p e_j + P W_j s', a_j) over QP,
    with P W_j = [i in G_j] * (P mod q_i) on cipher limb i and 0 on special limbs."""
    K = Keys()
    n = P.n
    s = prng.ternary(seed, prng.TAG_S, 0, n)
    K.s = s
    qidx = list(range(P.L1))
    a = np.stack([prng.uniform(seed, prng.TAG_PK_A, 0, n, i, P.moduli[i]) for i in qidx])
    e = prng.cbd21(seed, prng.TAG_PK_E, 0, n)
    s_r = int_poly_to_rns(P, s, qidx)
    pe = int_poly_to_rns(P, P.p * e, qidx)
    b = _sub(pe, _mul(a, s_r, P, qidx), P, qidx)
    K.pk = (b, a)
    for t in ([0] if relin else []) + [int(t) for t in galois]:
        gen_switch_key(P, K, seed, t)
    return K


def gen_switch_key(P, K, seed, t):
    n = P.n
    allidx = list(range(P.L1 + P.K))
    s = K.s
    if t == 0:
        s2 = P.ring.reduce_int(np.convolve(s, s).tolist())     # s^2 mod Phi_m over Z
    else:
        s2 = P.ring.automorph_int(s, t)
    s_r = int_poly_to_rns(P, s, allidx)
    sp_r = int_poly_to_rns(P, s2, allidx)
    Pprod = 1
    for q in P.P:
        Pprod *= q
    keys = []
    for j in range(P.dnum):
        stream = t * 64 + j
        a = np.stack([prng.uniform(seed, prng.TAG_KS_A, stream, n, i, P.moduli[i]) for i in allidx])
        e = prng.cbd21(seed, prng.TAG_KS_E, stream, n)
        pe = int_poly_to_rns(P, P.p * e, allidx)
        b = _sub(pe, _mul(a, s_r, P, allidx), P, allidx)
        G = P.digit_group(j, P.L1)
        for i in G:
            q = P.moduli[i]
            term = _c.vec_mulscalar(sp_r[i], Pprod % q, q)
            bi = b[i] + term
            b[i] = np.where(bi >= np.uint64(q), bi - np.uint64(q), bi)
        keys.append((b, a))
    K.ksk[t] = keys


# ----------------------------------------------------------------------------------------
# encrypt / decrypt
# ----------------------------------------------------------------------------------------
def encrypt(P, K, pt, seed, ct_index):
    """R9: (c0, c1) = ([b u + p e0 + m~]_Q, [a u + p e1]_Q), m~ centered lift of pt (mod p)."""
    n = P.n
    qidx = list(range(P.L1))
    u = prng.ternary(seed, prng.TAG_ENC_U, ct_index, n)
    e0 = prng.cbd21(seed, prng.TAG_ENC_E0, ct_index, n)
    e1 = prng.cbd21(seed, prng.TAG_ENC_E1, ct_index, n)
    mt = np.array([centered(int(x), P.p) for x in pt], dtype=np.int64)
    u_r = int_poly_to_rns(P, u, qidx)
    b, a = K.pk
    c0 = _add(_mul(b, u_r, P, qidx), int_poly_to_rns(P, P.p * e0 + mt, qidx), P, qidx)
    c1 = _add(_mul(a, u_r, P, qidx), int_poly_to_rns(P, P.p * e1, qidx), P, qidx)
    return Ciphertext([c0, c1], P.L1)


def decrypt_raw(P, K, ct):
    """R10: x = [c0 + c1 s (+ c2 s^2)]_{Q_l} (centered ints)."""
    idx = list(range(ct.level))
    s_r = int_poly_to_rns(P, K.s, idx)
    acc = ct.parts[0].copy()
    spow = s_r
    for part in ct.parts[1:]:
        acc = _add(acc, _mul(part, spow, P, idx), P, idx)
        spow = _mul(spow, s_r, P, idx)
    x, Q = lift_centered(P, acc, idx)
    return x, Q


def decrypt(P, K, ct):
    x, _ = decrypt_raw(P, K, ct)
    return np.array([v % P.p for v in x], dtype=np.int64)


def noise_bits(P, K, ct):
    """log2 of the largest |[c0 + c1 s]_Q| coefficient (noise-budget probe, R19)."""
    x, Q = decrypt_raw(P, K, ct)
    mx = max(abs(v) for v in x)
    return math.log2(mx) if mx else 0.0, math.log2(Q)


# ----------------------------------------------------------------------------------------
# modulus switching, key switching
# ----------------------------------------------------------------------------------------
def _scale_down(P, c, idx, drop_idx, r_vals, Qdrop):
    """Return (c_i - delta) * Qdrop^{-1} mod q_i for i in idx, delta = r + Qdrop * [-r]_p."""
    p = P.p
    delta = [r + Qdrop * centered(-r, p) for r in r_vals]
    out = np.empty((len(idx), P.n), dtype=np.uint64)
    for row, i in enumerate(idx):
        q = P.moduli[i]
        dq = _ints_mod(delta, q)
        diff = np.where(c[row] >= dq, c[row] - dq, c[row] + (np.uint64(q) - dq))
        out[row] = _c.vec_mulscalar(diff, pow(Qdrop, -1, q), q)
    return out


def modswitch(P, ct):
    """R13: drop q_{l-1}: r = [c]_{q}, delta = r + q [-r]_p, c'_i = (c_i - delta) q^{-1} mod q_i."""
    lv = ct.level
    assert lv >= 2, "OutOfLevels"
    idx = list(range(lv - 1))
    q = P.moduli[lv - 1]
    parts = []
    for c in ct.parts:
        r = [centered(int(v), q) for v in c[lv - 1]]
        parts.append(_scale_down(P, c[:lv - 1], idx, lv - 1, r, q))
    return Ciphertext(parts, lv - 1)


def modswitch_to(P, ct, level):
    while ct.level > level:
        ct = modswitch(P, ct)
    return ct


def modup(P, d, level):
    """R14 ModUp: for each digit j the exact centered lift x_j of d restricted to G_j, embedded
    in every target limb (rows: cipher 0..level-1, then special).  -> [(j, x_j rows)]."""
    tgt = list(range(level)) + P.special
    out = []
    for j in range(P.dnum):
        G = P.digit_group(j, level)
        if not G:
            continue
        x, _ = lift_centered(P, d[G], G)
        out.append((j, int_poly_to_rns(P, x, tgt)))
    return out


def kip(P, K, digits, level, key_id):
    """R14 key inner product: (u0, u1) = sum_j x_j (b_j, a_j) over the target limbs."""
    key = K.ksk[key_id]
    tgt = list(range(level)) + P.special
    u0 = np.zeros((len(tgt), P.n), dtype=np.uint64)
    u1 = np.zeros((len(tgt), P.n), dtype=np.uint64)
    for j, xr in digits:
        b, a = key[j]
        u0 = _add(u0, _mul(xr, b[tgt], P, tgt), P, tgt)
        u1 = _add(u1, _mul(xr, a[tgt], P, tgt), P, tgt)
    return u0, u1


def keyswitch_up(P, K, d, level, key_id):
    """R14 ModUp + key inner product (rows: cipher 0..level-1, then special)."""
    return kip(P, K, modup(P, d, level), level, key_id)


def moddown(P, u0, u1, level):
    """R14 ModDown: r = [u]_P, delta = r + P [-r]_p, u' = (u - delta) P^{-1}."""
    Pprod = 1
    for q in P.P:
        Pprod *= q
    out = []
    sp_rows = list(range(level, level + P.K))
    for u in (u0, u1):
        r, _ = lift_centered(P, u[sp_rows], P.special)
        out.append(_scale_down(P, u[:level], list(range(level)), None, r, Pprod))
    return out[0], out[1]


def keyswitch(P, K, d, level, key_id):
    """R14 (hybrid): ModUp and KIP (keyswitch_up), then ModDown."""
    u0, u1 = keyswitch_up(P, K, d, level, key_id)
    return moddown(P, u0, u1, level)


# ----------------------------------------------------------------------------------------
# homomorphic operations (R11, R12, R15)
# ----------------------------------------------------------------------------------------
def align(P, a, b):
    lv = min(a.level, b.level)
    return modswitch_to(P, a, lv), modswitch_to(P, b, lv)


def add(P, a, b):
    a, b = align(P, a, b)
    idx = list(range(a.level))
    n = max(len(a.parts), len(b.parts))
    parts = []
    for k in range(n):
        if k < len(a.parts) and k < len(b.parts):
            parts.append(_add(a.parts[k], b.parts[k], P, idx))
        else:
            parts.append((a.parts[k] if k < len(a.parts) else b.parts[k]).copy())
    return Ciphertext(parts, a.level)


def neg(P, a):
    idx = list(range(a.level))
    z = np.zeros_like(a.parts[0])
    return Ciphertext([_sub(z, c, P, idx) for c in a.parts], a.level)


def sub(P, a, b):
    return add(P, a, neg(P, b))


def mul_scalar(P, a, c):
    """multiply by the integer centered lift of c in F_p."""
    cc = centered(int(c), P.p)
    idx = list(range(a.level))
    return Ciphertext([_scal(x, cc, P, idx) for x in a.parts], a.level)


def pt_poly_rns(P, pt, level):
    """centered lift of a plaintext polynomial (coeffs mod p) into limbs 0..level-1."""
    mt = [centered(int(x), P.p) for x in pt]
    return int_poly_to_rns(P, mt, list(range(level)))


def add_plain(P, a, pt):
    idx = list(range(a.level))
    parts = [x.copy() for x in a.parts]
    parts[0] = _add(parts[0], pt_poly_rns(P, pt, a.level), P, idx)
    return Ciphertext(parts, a.level)


def add_const(P, a, c):
    pt = np.zeros(P.n, dtype=np.int64)
    pt[0] = int(c) % P.p
    return add_plain(P, a, pt)


def mul_plain(P, a, pt):
    idx = list(range(a.level))
    ptr = pt_poly_rns(P, pt, a.level)
    return Ciphertext([_mul(x, ptr, P, idx) for x in a.parts], a.level)


def tensor(P, a, b):
    idx = list(range(a.level))
    a0, a1 = a.parts
    b0, b1 = b.parts
    d0 = _mul(a0, b0, P, idx)
    d1 = _add(_mul(a0, b1, P, idx), _mul(a1, b0, P, idx), P, idx)
    d2 = _mul(a1, b1, P, idx)
    return Ciphertext([d0, d1, d2], a.level)


def relinearize(P, K, ct):
    d0, d1, d2 = ct.parts
    u0, u1 = keyswitch(P, K, d2, ct.level, 0)
    idx = list(range(ct.level))
    return Ciphertext([_add(d0, u0, P, idx), _add(d1, u1, P, idx)], ct.level)


def mul_unfused(P, K, a, b):
    """align -> tensor -> relinearise (ModDown by P) -> modswitch (by q_{l-1}): the two-step
    definition; decrypts like mul() (a test pin), different rounding bits."""
    a, b = align(P, a, b)
    return modswitch(P, relinearize(P, K, tensor(P, a, b)))


def mul(P, K, a, b):
    """R15 (fused ModDown + modulus switch): align -> tensor (d0, d1, d2) -> ModUp + KIP of d2 ->
    w_k = P d_k + u_k (k = 0, 1) over the cipher limbs of the level and the special limbs ->
    one scale-down by D = P q_{l-1}: r = [w]_D (exact centered CRT over the special primes and
    q_{l-1}), delta = r + D [-r]_p, w'_i = (w_i - delta) D^{-1} mod q_i for i < l-1 (R13/R14 with
    Qdrop = D; D = 1 mod p keeps the plaintext)."""
    a, b = align(P, a, b)
    lv = a.level
    assert lv >= 2, "OutOfLevels"
    d0, d1, d2 = tensor(P, a, b).parts
    u0, u1 = keyswitch_up(P, K, d2, lv, 0)
    Pprod = 1
    for q in P.P:
        Pprod *= q
    D = Pprod * P.moduli[lv - 1]
    cidx = list(range(lv))
    drop_rows = list(range(lv, lv + P.K)) + [lv - 1]
    drop_idx = P.special + [lv - 1]
    parts = []
    for dk, u in ((d0, u0), (d1, u1)):
        w = u.copy()
        w[:lv] = _add(_scal(dk, Pprod, P, cidx), u[:lv], P, cidx)
        r, _ = lift_centered(P, w[drop_rows], drop_idx)
        parts.append(_scale_down(P, w[:lv - 1], list(range(lv - 1)), None, r, D))
    return Ciphertext(parts, lv - 1)


def mul_sum(P, K, pairs):
    """R27 (lazy ModDown of a sum of products): sum_i a_i b_i with ONE scale-down.  Every
    operand is switched to lv = the lowest level of all of them (R12); per pair the w_k = P d_k + u_k of mul()
    (R15: tensor, ModUp + KIP of d2, over the cipher limbs of lv and the special limbs) are summed limb-wise;
    the sum takes mul()'s single scale-down by D = P q_{lv-1}.  One pair: exactly mul() (a test pin); more
    pairs: decrypts to the sum of the products, different bits from summing mul() results (one rounding)."""
    lv = min(min(a.level, b.level) for a, b in pairs)
    assert lv >= 2, "OutOfLevels"
    Pprod = 1
    for q in P.P:
        Pprod *= q
    D = Pprod * P.moduli[lv - 1]
    cidx = list(range(lv))
    rows = cidx + P.special
    W = [None, None]
    for a, b in pairs:
        a, b = modswitch_to(P, a, lv), modswitch_to(P, b, lv)
        d0, d1, d2 = tensor(P, a, b).parts
        u0, u1 = keyswitch_up(P, K, d2, lv, 0)
        for k, (dk, u) in enumerate(((d0, u0), (d1, u1))):
            w = u.copy()
            w[:lv] = _add(_scal(dk, Pprod, P, cidx), u[:lv], P, cidx)
            W[k] = w if W[k] is None else _add(W[k], w, P, rows)
    drop_rows = list(range(lv, lv + P.K)) + [lv - 1]
    drop_idx = P.special + [lv - 1]
    parts = []
    for w in W:
        r, _ = lift_centered(P, w[drop_rows], drop_idx)
        parts.append(_scale_down(P, w[:lv - 1], list(range(lv - 1)), None, r, D))
    return Ciphertext(parts, lv - 1)


def automorphism(P, K, ct, t):
    """R15: sigma_t on (c0, c1), then key-switch sigma_t(c1) with the key for t."""
    lv = ct.level
    idx = list(range(lv))
    c0 = np.stack([P.ring.automorph_mod(ct.parts[0][r], t, P.moduli[i]) for r, i in enumerate(idx)])
    c1 = np.stack([P.ring.automorph_mod(ct.parts[1][r], t, P.moduli[i]) for r, i in enumerate(idx)])
    u0, u1 = keyswitch(P, K, c1, lv, t)
    return Ciphertext([_add(c0, u0, P, idx), u1], lv)


def automorphisms_hoisted(P, K, ct, ts):
    """R22 hoisted key switching for several automorphisms of ONE ciphertext:
    the ModUp digits x_j of c1 are lifted once; for each t: u = sum_j sigma_t(x_j) (b_j, a_j)^(t)
    (sigma_t of an integer digit, applied limb-wise: sigma_t is a ring map of Z[x]/Phi_m), ModDown,
    and the result is (sigma_t(c0) + u0', u1').  Decrypts like automorphism(); different bits
    (sigma_t(lift(c1)) instead of lift(sigma_t(c1)))."""
    lv = ct.level
    idx = list(range(lv))
    tgt = idx + P.special
    digits = modup(P, ct.parts[1], lv)
    outs = []
    for t in ts:
        sd = [(j, np.stack([P.ring.automorph_mod(xr[r], t, P.moduli[i]) for r, i in enumerate(tgt)]))
              for j, xr in digits]
        u0, u1 = moddown(P, *kip(P, K, sd, lv, t), lv)
        c0 = np.stack([P.ring.automorph_mod(ct.parts[0][r], t, P.moduli[i]) for r, i in enumerate(idx)])
        outs.append(Ciphertext([_add(c0, u0, P, idx), u1], lv))
    return outs


def rotate(P, K, ct, k):
    """slot s receives slot s+k (sigma_{g^k})."""
    return automorphism(P, K, ct, pow(P.alg.g, k, P.m))


def frobenius(P, K, ct, k):
    return automorphism(P, K, ct, pow(P.p, k, P.m))


# ----------------------------------------------------------------------------------------
# evaluation-form view (for kernel parity only)
# ----------------------------------------------------------------------------------------
def to_eval(P, arr, idx):
    """R3: E[k] = a(omega_i^{z_k}) per limb -- naive evaluation."""
    out = np.empty_like(arr)
    for r, i in enumerate(idx):
        out[r] = P.ring.to_eval(arr[r], P.omega[i], P.moduli[i])
    return out


def ct_to_eval(P, ct):
    idx = list(range(ct.level))
    return [to_eval(P, c, idx) for c in ct.parts]
