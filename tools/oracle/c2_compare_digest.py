"""Full-size C2 compare_lt on the CPU oracle -> tests/golden/c2_compare_digest.json.

TEST INFRASTRUCTURE: calls only `oracle/` and `inputs/` (never the CUDA path).  One ciphertext
pair of the C2 config (Table 3 p5 U: p = 13, m = 30941, (d, l) = (4, 6)), keys seed
0xB00C0001, encryption seed 0xB00C0003 (ct indices 0 and 1), words from
inputs.word_pairs(np.random.default_rng(SEED_WORDS), 1031, base, d*l).  The result ciphertext
(R15/R16 schedules) is mapped to evaluation form by naive evaluation (R3) and its
SHA-256 over the little-endian u64 array [2][level][n] is stored, with sampled coefficients for
diagnosis and the decrypted result bits checked against plaintext comparison.

    python tools/oracle/c2_compare_digest.py [c2|c2@r16] [out.json]   # 20-60 min on 6-8 host cores
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from inputs import word_pairs  # noqa: E402
from oracle import bgv, circuits, slots  # noqa: E402

SEED_KEYS, SEED_WORDS, SEED_ENC = 0xB00C0001, 0xB00C0002, 0xB00C0003
OUT = os.path.join(ROOT, "tests", "golden", "c2_compare_digest.json")


def main(cfg_name="c2", out=OUT):
    t0 = time.time()
    base, _, sched = cfg_name.partition("@")        # "c2@r16": C2 with the R16 digit circuits
    cfg = json.load(open(os.path.join(ROOT, "params", base + ".json")))
    if sched:
        cfg["schedule"] = sched
    P = bgv.Params(cfg)
    A = P.alg
    ints = P.ints_per_ct
    gal = sorted({pow(P.p, k, P.m) for k in range(1, A.D)}
                 | {pow(A.g, s, P.m) for s in (1, 2, 4) if s < P.l})
    print("params", P.n, P.L1, P.K, "ints", ints, "galois", gal, "%.0fs" % (time.time() - t0), flush=True)
    K = bgv.keygen(P, SEED_KEYS, gal)
    print("keygen %.0fs" % (time.time() - t0), flush=True)
    rng = np.random.default_rng(SEED_WORDS)
    a, b = word_pairs(rng, ints, P.base, P.d * P.l)
    oa = bgv.encrypt(P, K, A.encode(slots.words_to_slots(a, A, P.d, P.l, P.base)), SEED_ENC, 0)
    ob = bgv.encrypt(P, K, A.encode(slots.words_to_slots(b, A, P.d, P.l, P.base)), SEED_ENC, 1)
    print("encrypt %.0fs" % (time.time() - t0), flush=True)
    ev = circuits.OracleEval(P, K)
    lt, _ = circuits.compare(ev, oa, ob, P.circuit, P.d, P.l, ints)
    print("compare %.0fs counts %s level %d" % (time.time() - t0, ev.counts, lt.level), flush=True)
    dec = A.decode(bgv.decrypt(P, K, lt))
    bits = [int(dec[A.word_slot(j, P.l)][0]) for j in range(ints)]
    want = [int(x < y) for x, y in zip(a, b)]
    assert bits == want, "oracle compare_lt decrypts wrong"
    E = np.stack(bgv.ct_to_eval(P, lt))                     # [2][level][n] u64
    h = hashlib.sha256(np.ascontiguousarray(E, dtype="<u8").tobytes()).hexdigest()
    samp = [int(x) for x in E[:, :, :4].reshape(-1)]
    rec = {"config": cfg_name, "schedule": P.schedule, "what": "oracle compare_lt of one C2 pair, evaluation form (R3)",
           "seeds": {"keys": SEED_KEYS, "words": SEED_WORDS, "enc": SEED_ENC, "ct_index": [0, 1]},
           "galois": gal, "level": int(lt.level), "shape": list(E.shape), "sha256": h,
           "first4_per_limb": samp, "lt_bits_sha256": hashlib.sha256(bytes(bits)).hexdigest(),
           "ones": int(sum(bits)), "oracle_counts": ev.counts, "seconds": round(time.time() - t0)}
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    print("wrote", out, h, "%.0fs" % (time.time() - t0), flush=True)


if __name__ == "__main__":
    main(*sys.argv[1:])
