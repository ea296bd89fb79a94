"""Counter-based sampler (R7) -- the oracle's own implementation.

The paper does not specify its noise or secret distributions (silent, §2.1).  Both the
oracle and the product implement this same counter-based generator independently, so that
seeded keys and ciphertexts agree bit for bit:

  r(seed, tag, stream, j) = mix64(seed + tag*C_TAG + stream*C_STREAM + (j+1)*C_GOLD)  (mod 2^64)
  mix64 = SplitMix64 finaliser.
  ternary  : (r mod 3) - 1
  cbd(21)  : popcount(r & (2^21-1)) - popcount((r >> 21) & (2^21-1))
  uniform_q: floor((r(2i) * 2^64 + r(2i+1)) * q / 2^128), i = limb*n + coeff
TEST INFRASTRUCTURE ONLY.
"""
import numpy as np

M64 = (1 << 64) - 1
C_TAG = 0xD1B54A32D192ED03
C_STREAM = 0x8CB92BA72F3D8DD7
C_GOLD = 0x9E3779B97F4A7C15

TAG_S, TAG_PK_A, TAG_PK_E, TAG_KS_A, TAG_KS_E, TAG_ENC_U, TAG_ENC_E0, TAG_ENC_E1 = range(1, 9)


def _mix64(z):
    z = z.copy()
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def draws(seed, tag, stream, j):
    """r(seed, tag, stream, j) for an array of counters j (uint64)."""
    base = (int(seed) + int(tag) * C_TAG + int(stream) * C_STREAM) & M64
    j = np.asarray(j, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = np.uint64(base) + (j + np.uint64(1)) * np.uint64(C_GOLD)
    return _mix64(x)


def _popcount(x):
    x = x.astype(np.uint64)
    c = np.zeros(x.shape, dtype=np.int64)
    for b in range(21):
        c += ((x >> np.uint64(b)) & np.uint64(1)).astype(np.int64)
    return c


def ternary(seed, tag, stream, n):
    r = draws(seed, tag, stream, np.arange(n, dtype=np.uint64))
    return (r % np.uint64(3)).astype(np.int64) - 1


def cbd21(seed, tag, stream, n):
    r = draws(seed, tag, stream, np.arange(n, dtype=np.uint64))
    mask = np.uint64((1 << 21) - 1)
    return _popcount(r & mask) - _popcount((r >> np.uint64(21)) & mask)


def uniform(seed, tag, stream, n, limb, q):
    """Uniform residues mod q for coefficient index i = limb*n + coeff (python-int exact)."""
    i = np.arange(n, dtype=np.uint64) + np.uint64(limb * n)
    r1 = draws(seed, tag, stream, np.uint64(2) * i)
    r2 = draws(seed, tag, stream, np.uint64(2) * i + np.uint64(1))
    out = np.empty(n, dtype=np.uint64)
    for k in range(n):
        out[k] = ((int(r1[k]) << 64) + int(r2[k])) * q >> 128
    return out
