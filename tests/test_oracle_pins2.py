"""Pins for oracle functions that had none (round-2 VERDICT "What's weak" 2):

* prng.mix64 / draws: the SplitMix64 generator's published known-answer outputs for seed 0
  (Vigna's splitmix64.c: state += 0x9E3779B97F4A7C15, then the finaliser) -- with seed, tag and
  stream 0, R7's draw r(0, 0, 0, j) is exactly the j-th SplitMix64(0) output.
* circuits.plan_compaction / circuits.compact / block_mask_sets: the Fig. 7 example
  (4 ciphertexts at 25% utilisation -> 1 ciphertext), the destination
  count ceil(useful / capacity) and multiset preservation of the decrypted words,
  on the cyclic toy ring (c1m, m = 91) with the full oracle BGV.
"""
import math

import numpy as np

from conftest import golden
from oracle import bgv, circuits, prng, slots

SEED_KEYS, SEED_ENC = 0xB00C0001, 0xB00C0003

# SplitMix64, seed 0: the first outputs of the reference generator (published test vector)
SPLITMIX64_SEED0 = [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F,
                    0xF88BB8A8724C81EC]


def test_splitmix64_known_answer():
    got = prng.draws(0, 0, 0, np.arange(4, dtype=np.uint64))
    assert [int(x) for x in got] == SPLITMIX64_SEED0


def _fig7_useful(ints, n_in=4):
    # every 4th block useful (Fig. 7: the useful integer blocks of 4 ciphertexts interleave)
    return [[b for b in range(ints) if b % 4 == 3] for _ in range(n_in)]


def test_plan_compaction_fig7_golden():
    g = golden("spec_examples.json")["compaction"]
    for cap in (8, 12, 16, 40, 1032):
        useful = [[b for b in range(cap) if b % 4 == 3] for _ in range(g["n_in"])]
        assert abs(len(useful[0]) / cap - g["utilization"]) < 0.01
        groups, n_out, dest = circuits.plan_compaction(useful, cap, 3)
        assert n_out == g["n_out"] == math.ceil(sum(map(len, useful)) / cap)
        # a bijection of the useful blocks onto distinct output blocks
        assert len(set(dest.values())) == len(dest) == sum(map(len, useful))
        # Fig. 7: each input moves as a whole (one mask product + at most one rotation), input 0
        # stays in place, so at most 3 rotations; the last block (cap - 1) rules out offset -1
        offs = [dl for (_, _, dl, bl) in groups if bl]
        assert offs == [0, 1, 2, 3]


def test_plan_compaction_dense_inputs_need_more_outputs():
    useful = [list(range(10)), list(range(10)), [1, 5]]
    groups, n_out, dest = circuits.plan_compaction(useful, 10, 3)
    assert n_out == 3 and len(dest) == 22 and len(set(dest.values())) == 22


def test_block_mask_sets_marks_slots_of_the_blocks(oracle_params):
    P = oracle_params("c1m")
    A = P.alg
    m = circuits.block_mask_sets(A, P.l, {1, 3})
    want = np.zeros((A.S, A.D), dtype=np.int64)
    for b in (1, 3):
        w0 = A.word_slot(b, P.l)
        want[w0:w0 + P.l, 0] = 1
    assert np.array_equal(m, want) and m.sum() == 2 * P.l


def test_compact_fig7_bgv_multiset(oracle_params):
    """full oracle BGV compaction (mask product, rotations, modulus switch) of the Fig. 7 pattern:
    one output ciphertext whose decrypted blocks are exactly the useful input words."""
    P = oracle_params("c1m")
    A = P.alg
    ints = P.ints_per_ct
    gal = circuits.compaction_galois(A, P.l, 3)
    K = bgv.keygen(P, SEED_KEYS, gal)
    rng = np.random.default_rng(7)
    useful = _fig7_useful(ints)
    words = [[int(x) if b % 4 == 3 else 0 for b, x in
              enumerate(rng.integers(0, P.base ** (P.d * P.l), size=ints))] for _ in range(4)]
    cts = [bgv.encrypt(P, K, A.encode(slots.words_to_slots(w, A, P.d, P.l, P.base)), SEED_ENC, c)
           for c, w in enumerate(words)]
    outs, dest = circuits.compact(circuits.OracleEval(P, K), cts, useful, P.l, ints, 3)
    assert len(outs) == golden("spec_examples.json")["compaction"]["n_out"]
    dec = [slots.slots_to_words(A.decode(bgv.decrypt(P, K, o)), P.d, P.l, P.base, ints, A)
           for o in outs]
    got = sorted(dec[cp][b2] for (cp, b2) in dest.values())
    assert got == sorted(words[c][b] for c in range(4) for b in useful[c])
    for (c, b), (cp, b2) in dest.items():
        assert dec[cp][b2] == words[c][b]
