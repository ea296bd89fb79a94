"""Shared helpers for the GPU parity tests (product vs oracle on the same seeded inputs)."""
import numpy as np

from conftest import load_cfg

SEED_KEYS, SEED_ENC = 0xB00C0001, 0xB00C0003


def galois_for(P, span=3):
    """Galois elements both sides generate keys for: Frobenius p^k (k < D), rotations g^{+-2^r}
    (2^r < l), compaction offsets g^{+-delta l} (delta <= span)."""
    A = P.alg
    gal = {pow(P.p, k, P.m) for k in range(1, A.D)}
    sh = 1
    while sh < P.l:
        gal |= {pow(A.g, sh, P.m), pow(A.g, -sh, P.m)}
        sh *= 2
    for k in range(1, span + 1):
        gal |= {pow(A.g, k * P.l, P.m), pow(A.g, -k * P.l, P.m)}
    return sorted(gal)


def to_u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def from_u64(arr, device):
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).to(device)


class Pair:
    """product Context + oracle Params/Keys for one config."""

    def __init__(self, name, oracle_params):
        import paper_2407_07308_b200 as bc
        from oracle import bgv
        self.name = name
        self.cfg = load_cfg(name)
        self.ctx = bc.Context(self.cfg)
        self.P = oracle_params(name)
        self.keys = self.ctx.keygen(SEED_KEYS)
        self._ok = None
        self.bgv = bgv

    @property
    def okeys(self):
        if self._ok is None:
            self._ok = self.bgv.keygen(self.P, SEED_KEYS, galois_for(self.P))
        return self._ok

    def oracle_ct(self, words, idx):
        from oracle import slots
        P = self.P
        sl = slots.words_to_slots(words, P.alg, P.d, P.l, P.base)
        return self.bgv.encrypt(P, self.okeys, P.alg.encode(sl), SEED_ENC, idx)

    def ct_eval(self, ct):
        return np.stack(self.bgv.ct_to_eval(self.P, ct))


def random_words(P, rng, ints):
    base = P.base
    cap = base ** (P.d * P.l)
    if cap >= 2 ** 64:
        return [int(x) for x in rng.integers(0, 2 ** 63, size=ints, dtype=np.int64)] 
    return [int(x) for x in rng.integers(0, cap, size=ints)]


def mixed_pairs(P, rng, ints):
    """50% independent, 12.5% equal, 12.5% equal but the lowest digit, 12.5% equal above one digit,
    12.5% |a-b| = 1 (SURVEY §8(d) input recipe; inputs module shared by both sides)."""
    from inputs import word_pairs
    return word_pairs(rng, ints, P.base, P.d * P.l)
