"""Seeded synthetic inputs shared by the oracle tests and the product (no method arithmetic).

Recipe: words uniform over the word capacity min(base^(d l), 2^64), mixed so the
lexicographic logic is exercised: 50% independent pairs, 12.5% a = b, 12.5% equal except the
least-significant digit, 12.5% equal above one random digit position, 12.5% |a - b| = 1.
"""
import numpy as np


def word_pairs(rng, count, base, ndigits):
    cap = min(base ** ndigits, 2 ** 64)
    a, b = [], []
    for _ in range(count):
        kind = rng.integers(0, 8)
        x = int(rng.integers(0, 2 ** 62)) * 4 % cap if cap > 2 ** 62 else int(rng.integers(0, cap))
        x = (x + int(rng.integers(0, 4))) % cap
        if kind < 4:
            y = int(rng.integers(0, 2 ** 62)) * 4 % cap if cap > 2 ** 62 else int(rng.integers(0, cap))
        elif kind == 4:
            y = x
        elif kind == 5:
            y = x - x % base + int(rng.integers(0, base))
        elif kind == 6:
            pos = int(rng.integers(0, ndigits))
            digs = [(x // base ** i) % base for i in range(ndigits)]
            digs[pos] = int(rng.integers(0, base))
            y = sum(dg * base ** i for i, dg in enumerate(digs))
            if y >= cap:
                y = x
        else:
            y = x + 1 if x + 1 < cap else x - 1
        a.append(x)
        b.append(y)
    return a, b
