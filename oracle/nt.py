"""Elementary number theory for the oracle (TEST INFRASTRUCTURE ONLY).

Readings: R1 prime chain, R2 root of unity.  Plain Python ints.
"""
from functools import reduce
from math import gcd

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def is_prime(n):
    """Deterministic Miller-Rabin for n < 3.3e24 (bases 2..37)."""
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def factorize(n):
    """Trial division; returns {prime: exponent}.  Only used on small n (m, D, ...)."""
    f = {}
    d = 2
    while d * d <= n:
        while n % d == 0:
            f[d] = f.get(d, 0) + 1
            n //= d
        d += 1
    if n > 1:
        f[n] = f.get(n, 0) + 1
    return f


def lcm(*xs):
    return reduce(lambda a, b: a * b // gcd(a, b), xs, 1)


def euler_phi(m):
    r = m
    for pr in factorize(m):
        r = r // pr * (pr - 1)
    return r


def mult_order(a, m):
    """Multiplicative order of a mod m (gcd(a, m) == 1)."""
    assert gcd(a, m) == 1
    k, x = 1, a % m
    while x != 1:
        x = x * a % m
        k += 1
    return k


def bluestein_pad(m, mixed=False):
    """M = smallest power of two >= 2m - 1 ("length power of two greater than 2m-1").
    mixed (R25): the smallest length >= 2m - 1 among the powers of two and
    256 r N' with r in {3, 5, 7, 9}, N' in {32, 64, 128} (the mixed-radix lengths the transform
    supports); the convolution is exact at any length >= 2m - 1, so only the primes (R1) depend on it."""
    M = 1
    while M < 2 * m - 1:
        M *= 2
    if mixed:
        for r in (3, 5, 7, 9):
            for nn in (32, 64, 128):
                L = 256 * r * nn
                if 2 * m - 1 <= L < M:
                    M = L
    return M


def prime_chain(modulus, bits, count, after=0, exclude=()):
    """R1: the `count` smallest primes q >= max(2^(bits-1), after+1) with q = 1 (mod modulus),
    ascending, skipping `exclude`.  Primes must stay below 2^62 (word-size reading, F4)."""
    start = max(1 << (bits - 1), after + 1)
    q = start + ((1 - start) % modulus)
    out = []
    while len(out) < count:
        if q >= (1 << 62):
            raise ValueError("NotEnoughPrimes below 2^62")
        if q not in exclude and is_prime(q):
            out.append(q)
        q += modulus
    return out


def root_of_unity(m, q):
    """R2: omega = h^((q-1)/m) mod q for the smallest h >= 2 such that omega has exact order m."""
    assert (q - 1) % m == 0
    primes_m = list(factorize(m))
    h = 2
    while True:
        w = pow(h, (q - 1) // m, q)
        if all(pow(w, m // r, q) != 1 for r in primes_m):
            return w
        h += 1


def centered(x, Q):
    """[x]_Q in (-Q/2, Q/2] (Q odd: (-(Q-1)/2, (Q-1)/2])."""
    r = x % Q
    return r - Q if r > Q // 2 else r


def crt(residues, moduli):
    """Textbook CRT: x = sum r_i (Q/q_i) [(Q/q_i)^-1]_{q_i} mod Q, in [0, Q)."""
    Q = 1
    for q in moduli:
        Q *= q
    x = 0
    for r, q in zip(residues, moduli):
        Qi = Q // q
        x += int(r) * Qi * pow(Qi, -1, q)
    return x % Q, Q
