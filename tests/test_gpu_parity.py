"""GPU parity: every §8(a) row of the CUDA path vs the oracle, bit-exact, on seeded inputs.

Runs on a B200 (``-m gpu``).  Ciphertexts are compared in evaluation form: the oracle's
coefficient-form result is mapped by naive evaluation at omega_i^{z_k} (R3).
"""
import numpy as np
import pytest

from gpu_util import SEED_ENC, SEED_KEYS, Pair, from_u64, galois_for, mixed_pairs, to_u64

pytestmark = pytest.mark.gpu

_PAIRS = {}


@pytest.fixture(scope="module")
def pair(oracle_params):
    def get(name):
        if name not in _PAIRS:
            _PAIRS[name] = Pair(name, oracle_params)
        return _PAIRS[name]
    return get


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c2", "c3h", "c3s2"])
def test_tables_match_oracle(pair, cfg):
    T = pair(cfg)
    q, w = T.ctx.moduli()
    assert q == T.P.moduli
    assert w == T.P.omega
    if cfg != "c2":
        G, z, t = T.ctx.slots()
        A = T.P.alg
        assert list(G) == list(A.G)
        assert list(z) == [int(x) for x in A.zeta]
        assert list(t) == list(A.t)
        assert sorted(T.ctx.galois()) == galois_for(T.P)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_ntt_fused_cluster_matches_oracle(pair, variant):
    """a1/a2, the fused thread-block-cluster kernel (ntt4.cu; 8 x 512, 16 x 256 and 4 x 1024 CTA
    clusters) at full C2 size: forward == naive evaluation on sampled limbs, bit-identical to the three
    pass kernels on every limb of a batch (forward and inverse), and the inverse recovers the input."""
    import paper_2407_07308_b200 as bc
    T = pair("c2")
    P = T.P
    rng = np.random.default_rng(23)
    coef = np.stack([np.stack([rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.moduli]) for _ in range(3)])
    x = from_u64(coef, T.ctx.device)
    f0 = to_u64(T.ctx.ntt_fwd(x))
    i0 = to_u64(T.ctx.ntt_inv(x))
    try:
        bc.set_ntt_impl(20)
        bc._lib.bc_tune(b"nttc_variant", variant)
        f1 = to_u64(T.ctx.ntt_fwd(x))
        i1 = to_u64(T.ctx.ntt_inv(x))
        back = to_u64(T.ctx.ntt_inv(from_u64(f1, T.ctx.device)))
    finally:
        bc.set_ntt_impl(0)
        bc._lib.bc_tune(b"nttc_variant", 0)
    for b, i in ((0, 0), (2, P.L1 + P.K - 1)):
        assert np.array_equal(f1[b, i], P.ring.to_eval(coef[b, i], P.omega[i], P.moduli[i]))
    assert np.array_equal(f1, f0)
    assert np.array_equal(i1, i0)
    assert np.array_equal(back, coef)


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c3h", "c3s2"])
def test_ntt_forward_inverse(pair, cfg):
    """a1/a2: Bluestein forward == naive evaluation; inverse recovers coefficients (all limbs).
    c3h / c3s2: composite m (the inverse reduces mod Phi_m: long division on the integer path,
    Barrett division by two size-M convolutions on the binary64 path)."""
    import torch
    T = pair(cfg)
    P = T.P
    rng = np.random.default_rng(11)
    nl = P.L1 + P.K
    coef = np.stack([np.stack([rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.moduli])
                     for _ in range(3)])                              # [3, nl, n]
    x = from_u64(coef, T.ctx.device)
    ev = to_u64(T.ctx.ntt_fwd(x))
    for b in range(3):
        want = np.stack([P.ring.to_eval(coef[b, i], P.omega[i], P.moduli[i]) for i in range(nl)])
        assert np.array_equal(ev[b], want), "forward NTT mismatch (poly %d)" % b
    back = to_u64(T.ctx.ntt_inv(from_u64(ev, T.ctx.device)))
    assert np.array_equal(back, coef)
    torch.cuda.synchronize()


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_ntt_full_size_sampled(pair, cfg):
    """a1/a2 at full size (C2: n = 30940, M = 65536; C3: composite m = 52053, n = 34700, M = 131072,
    Barrett reduction mod Phi_m): two limbs vs naive evaluation, inverse recovers every limb."""
    T = pair(cfg)
    P = T.P
    rng = np.random.default_rng(12)
    coef = np.stack([rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.moduli])[None]
    ev = to_u64(T.ctx.ntt_fwd(from_u64(coef, T.ctx.device)))
    for i in (0, P.L1 + P.K - 1):
        want = P.ring.to_eval(coef[0, i], P.omega[i], P.moduli[i])
        assert np.array_equal(ev[0, i], want)
    back = to_u64(T.ctx.ntt_inv(from_u64(ev, T.ctx.device)))
    assert np.array_equal(back, coef)


def test_ntt_register_passes_match_radix2(pair):
    """the register-blocked passes (C2's 256 x 256 shape) agree with the radix-2 passes on every
    limb of a batch, forward and inverse (both are checked against the oracle elsewhere)."""
    import paper_2407_07308_b200 as bc
    T = pair("c2")
    P = T.P
    rng = np.random.default_rng(22)
    coef = np.stack([np.stack([rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.moduli]) for _ in range(5)])
    x = from_u64(coef, T.ctx.device)
    try:
        bc.set_ntt_impl(1)
        f1 = to_u64(T.ctx.ntt_fwd(x))
        i1 = to_u64(T.ctx.ntt_inv(x))
    finally:
        bc.set_ntt_impl(0)
    f2 = to_u64(T.ctx.ntt_fwd(x))
    i2 = to_u64(T.ctx.ntt_inv(x))
    assert np.array_equal(f1, f2)
    assert np.array_equal(i1, i2)
    assert np.array_equal(to_u64(T.ctx.ntt_inv(from_u64(f2, T.ctx.device))), coef)


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c3h", "c3s2"])
def test_encrypt_decrypt_match_oracle(pair, cfg):
    """R9/R10 + R7 sampler: the product's ciphertexts equal the oracle's bit for bit."""
    T = pair(cfg)
    P = T.P
    rng = np.random.default_rng(13)
    ints = T.ctx.ints_per_ct
    a, b = mixed_pairs(P, rng, ints)
    words = np.array([a, b], dtype=np.uint64)
    ct = T.ctx.encrypt(T.keys, words, SEED_ENC, ct_index0=5)
    g = to_u64(ct)
    for i in range(2):
        o = T.oracle_ct(list(words[i]), 5 + i)
        assert np.array_equal(g[i], T.ct_eval(o)), "ciphertext %d differs from oracle" % i
    dec = T.ctx.decrypt(T.keys, ct)
    assert np.array_equal(dec, words)


@pytest.mark.parametrize("cfg", ["c1", "c2s", "c3s2"])
def test_ops_match_oracle(pair, cfg):
    """a3 tensor, a4 automorphism, a5 key switching (relin / rotation / Frobenius), a6 modswitch."""
    T = pair(cfg)
    P, bgv = T.P, T.bgv
    rng = np.random.default_rng(14)
    ints = T.ctx.ints_per_ct
    a, b = mixed_pairs(P, rng, ints)
    ct = T.ctx.encrypt(T.keys, np.array([a, b], dtype=np.uint64), SEED_ENC, ct_index0=20)
    oa, ob = T.oracle_ct(a, 20), T.oracle_ct(b, 21)
    ca, cb = ct[0:1], ct[1:2]
    # tensor
    tg = to_u64(T.ctx.tensor(ca, cb))[0]
    assert np.array_equal(tg, T.ct_eval(bgv.tensor(P, oa, ob)))
    # automorphism (no key switch)
    t = pow(P.alg.g, 1, P.m)
    ag = to_u64(T.ctx.automorph(ca, t))[0]
    idx = list(range(P.L1))
    want = np.stack([bgv.to_eval(P, np.stack([P.ring.automorph_mod(c[r], t, P.moduli[r]) for r in idx]), idx)
                     for c in oa.parts])
    assert np.array_equal(ag, want)
    # modswitch
    assert np.array_equal(to_u64(T.ctx.modswitch(ca))[0], T.ct_eval(bgv.modswitch(P, oa)))
    # key switch of c1 with the relinearisation key
    d = ca[:, 1].contiguous()
    u = to_u64(T.ctx.keyswitch(T.keys, d, 0))[0]
    u0, u1 = bgv.keyswitch(P, T.okeys, oa.parts[1], P.L1, 0)
    assert np.array_equal(u, np.stack([bgv.to_eval(P, u0, idx), bgv.to_eval(P, u1, idx)]))
    # mul (tensor + relin + modswitch), rotation, Frobenius
    assert np.array_equal(to_u64(T.ctx.mul(T.keys, ca, cb))[0], T.ct_eval(bgv.mul(P, T.okeys, oa, ob)))
    assert np.array_equal(to_u64(T.ctx.rotate(T.keys, ca, 1))[0], T.ct_eval(bgv.rotate(P, T.okeys, oa, 1)))
    assert np.array_equal(to_u64(T.ctx.rotate(T.keys, ca, -1))[0], T.ct_eval(bgv.rotate(P, T.okeys, oa, -1)))
    assert np.array_equal(to_u64(T.ctx.frobenius(T.keys, ca, 1))[0], T.ct_eval(bgv.frobenius(P, T.okeys, oa, 1)))


@pytest.mark.parametrize("cfg", ["c1", "c1l2"])
def test_compare_matches_oracle(pair, cfg):
    """a7-a9 end to end: compare_lt / compare_eq ciphertexts bit-exact; decrypted bits = [a<b]; the
    EQ-only call (no LT products) returns the same EQ ciphertext."""
    from oracle import circuits
    T = pair(cfg)
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(15)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=30)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=31)
    lt, eq = T.ctx.compare(T.keys, ca, cb)
    bits = T.ctx.decrypt(T.keys, lt, as_bits=True)[0]
    ebits = T.ctx.decrypt(T.keys, eq, as_bits=True)[0]
    assert list(bits) == [int(x < y) for x, y in zip(a, b)]
    assert list(ebits) == [int(x == y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    olt, oeq = circuits.compare(ev, T.oracle_ct(a, 30), T.oracle_ct(b, 31), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(lt)[0], T.ct_eval(olt))
    assert np.array_equal(to_u64(eq)[0], T.ct_eval(oeq))
    lt2 = T.ctx.compare_lt(T.keys, ca, cb)
    assert np.array_equal(to_u64(lt2), to_u64(lt))
    eq2 = T.ctx.compare_eq(T.keys, ca, cb)          # the EQ-only schedule (no LT products)
    assert np.array_equal(to_u64(eq2), to_u64(eq))


def test_extract_matches_oracle(pair):
    from oracle import circuits
    T = pair("c1")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(16)
    a, _ = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=40)
    dg = to_u64(T.ctx.extract(T.keys, ca))[0]
    ev = circuits.OracleEval(P, T.okeys)
    od = circuits.extract_digits(ev, T.oracle_ct(a, 40), P.d)
    for i in range(P.d):
        assert np.array_equal(dg[i], T.ct_eval(od[i]))


def test_select_min_max_match_oracle(pair):
    from oracle import circuits
    T = pair("c1m")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(17)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=50)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=51)
    mn = T.ctx.min(T.keys, ca, cb)
    mx = T.ctx.max(T.keys, ca, cb)
    assert list(T.ctx.decrypt(T.keys, mn)[0]) == [min(x, y) for x, y in zip(a, b)]
    assert list(T.ctx.decrypt(T.keys, mx)[0]) == [max(x, y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    omn = circuits.vmin(ev, T.oracle_ct(a, 50), T.oracle_ct(b, 51), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(mn)[0], T.ct_eval(omn))


@pytest.mark.parametrize("cfg", ["c1m", "c3s2"])
def test_compaction_fig7(pair, cfg):
    """a10: 4 ciphertexts at 25% block utilisation (every 4th block, Fig. 7) -> 1 ciphertext, bit-exact
    vs the oracle: c1m (59-bit primes, integer kernels) and c3s2 (C3's slot structure: p = 31, composite
    m = 1851, 56 x 2 hypercube with row-aligned blocks, 50-bit primes, binary64 kernels)."""
    from oracle import circuits
    T = pair(cfg)
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(18)
    cap = min(P.base ** (P.d * P.l), 2 ** 63)
    words = [[int(x) for x in rng.integers(0, cap, size=ints)] for _ in range(4)]
    useful = np.zeros((4, ints), dtype=np.uint8)
    useful[:, 3::4] = 1
    for c in range(4):
        for j in range(ints):
            if not useful[c, j]:
                words[c][j] = 0
    cts = T.ctx.encrypt(T.keys, np.array(words, dtype=np.uint64), SEED_ENC, ct_index0=60)
    out, dest = T.ctx.compact(T.keys, cts, useful)
    wpr = P.alg.S1 // P.l            # blocks move within their row only (R6 / R17): per-row capacity wpr
    rows = -(-ints // wpr)
    per_row = [int(useful[:, r * wpr:(r + 1) * wpr].sum()) for r in range(rows)]
    assert out.shape[0] == max(-(-k // wpr) for k in per_row) >= int(np.ceil(useful.sum() / ints))
    dec = T.ctx.decrypt(T.keys, out)
    for c in range(4):
        for j in range(ints):
            if useful[c, j]:
                ct_i, blk = divmod(int(dest[c, j]), ints)
                assert dec[ct_i][blk] == words[c][j]
    ev = circuits.OracleEval(P, T.okeys)
    oin = [T.oracle_ct(words[c], 60 + c) for c in range(4)]
    outs, _ = circuits.compact(ev, oin, [list(np.nonzero(useful[c])[0]) for c in range(4)], P.l, ints, 3)
    assert len(outs) == out.shape[0]
    for k in range(out.shape[0]):
        assert np.array_equal(to_u64(out)[k], T.ct_eval(outs[k]))


def test_non_blocking_matches_blocking(pair):
    """a11: compare on a side stream joined by an event == the blocking result; double wait fails."""
    import torch
    T = pair("c1")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(19)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=70)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=71)
    ref = T.ctx.compare_lt(T.keys, ca, cb)
    side = torch.cuda.Stream()
    ws = torch.empty(T.ctx.workspace_bytes(1), dtype=torch.uint8, device=T.ctx.device)
    out = T.ctx.ct_empty(1, ref.shape[2])
    torch.cuda.synchronize()
    h = T.ctx.compare_lt_async(T.keys, ca, cb, out, side, ws)
    main = torch.cuda.current_stream()
    busy = ca.clone() * 1                # independent main-stream work meanwhile
    assert T.ctx.wait(h, main) == 0
    assert T.ctx.wait(h, main) == 7      # BC_E_CONSUMED
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    del busy


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c2s", "c2s@r16"])
def test_compare_shadow_c2_bit_exact(pair, name):
    """C2's circuit (p=13 univariate, (d,l)=(4,6), 11+3 primes) on its shadow ring m=859:
    whole compare_lt ciphertext bit-exact vs the oracle (takes ~2 minutes of oracle time), with the
    R23 digit circuit (6 products per digit, C2's schedule) and R16's (7)."""
    from oracle import circuits
    T = pair(name)
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(20)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=80)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=81)
    lt = T.ctx.compare_lt(T.keys, ca, cb)
    assert list(T.ctx.decrypt(T.keys, lt, as_bits=True)[0]) == [int(x < y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    olt, _ = circuits.compare(ev, T.oracle_ct(a, 80), T.oracle_ct(b, 81), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(lt)[0], T.ct_eval(olt))


def test_compare_full_c2_decrypts(pair):
    """C2 at full size (n = 30940): every block of 2 ciphertext pairs decrypts to [a<b]."""
    T = pair("c2")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(21)
    A, B = [], []
    for _ in range(2):
        a, b = mixed_pairs(P, rng, ints)
        A.append(a)
        B.append(b)
    ca = T.ctx.encrypt(T.keys, np.array(A, dtype=np.uint64), SEED_ENC, ct_index0=0)
    cb = T.ctx.encrypt(T.keys, np.array(B, dtype=np.uint64), SEED_ENC, ct_index0=2)
    assert np.array_equal(T.ctx.decrypt(T.keys, ca), np.array(A, dtype=np.uint64))
    lt = T.ctx.compare_lt(T.keys, ca, cb)
    bits = T.ctx.decrypt(T.keys, lt, as_bits=True)
    for i in range(2):
        assert list(bits[i]) == [int(x < y) for x, y in zip(A[i], B[i])]


@pytest.mark.parametrize("op,T", [("min", 4), ("max", 4), ("min", 3)])
def test_tournament_matches_oracle(pair, op, T):
    """R20 fixed-tree min/max over T element batches (2 ciphertexts each): every output
    ciphertext bit-exact vs the oracle's tournament, and decrypts to the brute-force min/max."""
    from oracle import circuits
    Tp = pair("c1t")
    P = Tp.P
    ints = Tp.ctx.ints_per_ct
    rng = np.random.default_rng(30 + T)
    W = [[[int(x) for x in rng.integers(0, P.base ** (P.d * P.l), size=ints)] for _ in range(2)] for _ in range(T)]
    W[0][0][0] = W[1][0][0]                                   # a tie
    elems = [Tp.ctx.encrypt(Tp.keys, np.array(W[t], dtype=np.uint64), SEED_ENC, ct_index0=500 + 2 * t)
             for t in range(T)]
    r = Tp.ctx.max_tree(Tp.keys, elems) if op == "max" else Tp.ctx.min_tree(Tp.keys, elems)
    f = min if op == "min" else max
    dec = Tp.ctx.decrypt(Tp.keys, r)
    ev = circuits.OracleEval(P, Tp.okeys)
    for c in range(2):
        assert list(dec[c]) == [f(W[t][c][j] for t in range(T)) for j in range(ints)]
        o = circuits.tournament(ev, [Tp.oracle_ct(W[t][c], 500 + 2 * t + c) for t in range(T)], op,
                                P.circuit, P.d, P.l, ints)
        assert np.array_equal(to_u64(r)[c], Tp.ct_eval(o))


def test_sort_matches_oracle(pair):
    """R21 rank sort of T = 3 = p element batches: bit-exact vs the oracle, sorted."""
    from oracle import circuits
    Tp = pair("c1t")
    P = Tp.P
    ints = Tp.ctx.ints_per_ct
    rng = np.random.default_rng(40)
    W = [[int(x) for x in rng.integers(0, 4, size=ints)] for _ in range(3)]
    W[0][0], W[1][0], W[2][0] = 3, 1, 2
    elems = [Tp.ctx.encrypt(Tp.keys, np.array([W[t]], dtype=np.uint64), SEED_ENC, ct_index0=600 + t)
             for t in range(3)]
    outs = Tp.ctx.sort(Tp.keys, elems)
    got = [Tp.ctx.decrypt(Tp.keys, o)[0] for o in outs]
    for j in range(ints):
        assert [int(got[k][j]) for k in range(3)] == sorted(W[t][j] for t in range(3))
    ev = circuits.OracleEval(P, Tp.okeys)
    oo = circuits.sort_rank(ev, [Tp.oracle_ct(W[t], 600 + t) for t in range(3)], P.circuit, P.d, P.l, ints)
    for k in range(3):
        assert np.array_equal(to_u64(outs[k])[0], Tp.ct_eval(oo[k]))


def test_bivariate_compare_matches_oracle(pair):
    """a7 bivariate path (digits < p, base p; P:71 [Tan] 3p-5 products): compare ciphertexts
    bit-exact vs the oracle, decrypted bits = [a<b] and [a=b]."""
    from oracle import circuits
    T = pair("c1b")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(41)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=800)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=801)
    lt, eq = T.ctx.compare(T.keys, ca, cb)
    assert list(T.ctx.decrypt(T.keys, lt, as_bits=True)[0]) == [int(x < y) for x, y in zip(a, b)]
    assert list(T.ctx.decrypt(T.keys, eq, as_bits=True)[0]) == [int(x == y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    olt, oeq = circuits.compare(ev, T.oracle_ct(a, 800), T.oracle_ct(b, 801), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(lt)[0], T.ct_eval(olt))
    assert np.array_equal(to_u64(eq)[0], T.ct_eval(oeq))


def test_compare_full_c3_decrypts(pair):
    """C3 at full size (Table 3 p10 B: p = 31 bivariate, m = 52053 composite, 3470 x 2 hypercube
    slots, (d,l) = (5,3), 2312 integers): compaction of 4 sparse ciphertexts (Fig. 7 pattern, every
    4th block; 289 per row per input) to 1, then compare_lt decrypts to [a<b] in every block."""
    T = pair("c3")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(42)
    A, B = [], []
    for _ in range(4):
        a, b = mixed_pairs(P, rng, ints)
        A.append(a)
        B.append(b)
    A, B = np.array(A, dtype=np.uint64), np.array(B, dtype=np.uint64)
    useful = np.zeros((4, ints), dtype=np.uint8)
    useful[:, 3::4] = 1
    A[useful == 0] = 0
    B[useful == 0] = 0
    ca = T.ctx.encrypt(T.keys, A, SEED_ENC, ct_index0=0)
    cb = T.ctx.encrypt(T.keys, B, SEED_ENC, ct_index0=4)
    da, dest = T.ctx.compact(T.keys, ca, useful)
    db, dest2 = T.ctx.compact(T.keys, cb, useful)
    assert da.shape[0] == 1 and np.array_equal(dest, dest2)
    lt = T.ctx.compare_lt(T.keys, da, db)
    bits = T.ctx.decrypt(T.keys, lt, as_bits=True)
    for c in range(4):
        for j in range(3, ints, 4):
            ct_i, blk = divmod(int(dest[c, j]), ints)
            assert int(bits[ct_i][blk]) == int(A[c, j] < B[c, j])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3t", "c3t@r27", "c3t@r23", "c3t@r16"])
def test_compare_c3t_bivariate_p31_bit_exact(pair, name):
    """C3's p = 31 bivariate digit circuit (R26: 59 products, C3's schedule; R23: 73; R16: 88) on a small
    ring (c3t: m = 1129, (d,l) = (1,2), 9 + 4 primes): whole compare_lt ciphertext bit-exact vs the
    oracle (~4 min of oracle time), decrypted bits = [a<b]."""
    from oracle import circuits
    T = pair(name)
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(43)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=900)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=901)
    lt = T.ctx.compare_lt(T.keys, ca, cb)
    assert list(T.ctx.decrypt(T.keys, lt, as_bits=True)[0]) == [int(x < y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    olt, _ = circuits.compare(ev, T.oracle_ct(a, 900), T.oracle_ct(b, 901), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(lt)[0], T.ct_eval(olt))


def test_binary64_kernels_match_integer_kernels(pair):
    """C2 at full size: the binary64 NTT / lift / KIP / tensor kernels (default) and the 64-bit integer
    kernels (ntt impl 7, f64_elem 0) give bit-identical compare_lt ciphertexts (both exact; the
    integer path is the one the shadow-ring oracle parity tests pinned first)."""
    import paper_2407_07308_b200 as bc
    T = pair("c2")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(31)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=0)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=1)
    f = to_u64(T.ctx.compare_lt(T.keys, ca, cb))
    try:
        bc.set_ntt_impl(7)
        bc._lib.bc_tune(b"f64_elem", 0)
        g = to_u64(T.ctx.compare_lt(T.keys, ca, cb))
    finally:
        bc.set_ntt_impl(0)
        bc._lib.bc_tune(b"f64_elem", 1)
    assert np.array_equal(f, g)
    bits = T.ctx.decrypt(T.keys, T.ctx.compare_lt(T.keys, ca, cb), as_bits=True)[0]
    assert list(bits) == [int(x < y) for x, y in zip(a, b)]


@pytest.mark.parametrize("name", ["c3h", "c3h@r27"])
def test_hypercube_compare_bit_exact(pair, name):
    """C3's slot structure on the tiny hypercube ring c3h (p = 31 bivariate, m = 33 = 3 x 11,
    Z_2 x Z_2 slots, one integer per row): whole compare_lt ciphertext bit-exact vs the oracle (C3's R26
    circuit, and R27: R26 with one scale-down per sum of products)."""
    from oracle import circuits
    T = pair(name)
    P = T.P
    ints = T.ctx.ints_per_ct
    a, b = [5, 923520], [7, 923520]
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=910)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=911)
    lt = T.ctx.compare_lt(T.keys, ca, cb)
    assert list(T.ctx.decrypt(T.keys, lt, as_bits=True)[0]) == [int(x < y) for x, y in zip(a, b)]
    ev = circuits.OracleEval(P, T.okeys)
    olt, _ = circuits.compare(ev, T.oracle_ct(a, 910), T.oracle_ct(b, 911), P.circuit, P.d, P.l, ints)
    assert np.array_equal(to_u64(lt)[0], T.ct_eval(olt))


def test_hypercube_shadow_compare_decrypts(pair):
    """C3's shadow c3s2 (m = 1851 composite, 56 x 2 hypercube, (d,l) = (5,3), 36 integers): a batch
    of 3 compares decrypts to [a<b] in every block (row-aligned words, row-local lex rounds)."""
    T = pair("c3s2")
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(44)
    A, B = [], []
    for _ in range(3):
        a, b = mixed_pairs(P, rng, ints)
        A.append(a)
        B.append(b)
    ca = T.ctx.encrypt(T.keys, np.array(A, dtype=np.uint64), SEED_ENC, ct_index0=0)
    cb = T.ctx.encrypt(T.keys, np.array(B, dtype=np.uint64), SEED_ENC, ct_index0=3)
    bits = T.ctx.decrypt(T.keys, T.ctx.compare_lt(T.keys, ca, cb), as_bits=True)
    for i in range(3):
        assert list(bits[i]) == [int(x < y) for x, y in zip(A[i], B[i])]


@pytest.mark.parametrize("cfg", ["c3s2", "c3"])
def test_composite_quotient_sparse_matches_convolution(pair, cfg):
    """composite m: the Barrett quotient rev(A) Phi_m^{-1} mod x^(m-n) as a sum of shifted copies
    (Phi_m^{-1} = (1 + x + x^2)(1 - x^r2) mod x^(m-n) for m = 3 r2; default) and as a size-Mb
    convolution (bc_tune phi_conv) give identical inverse transforms (both exact; the inverse itself
    is checked against the oracle's schoolbook reduction by the NTT tests)."""
    import paper_2407_07308_b200 as bc
    T = pair(cfg)
    P = T.P
    rng = np.random.default_rng(17)
    ev = np.stack([np.stack([rng.integers(0, q, size=P.n, dtype=np.uint64) for q in P.moduli]) for _ in range(2)])
    x = from_u64(ev, T.ctx.device)
    a = to_u64(T.ctx.ntt_inv(x))
    try:
        bc._lib.bc_tune(b"phi_conv", 1)
        b = to_u64(T.ctx.ntt_inv(x))
    finally:
        bc._lib.bc_tune(b"phi_conv", 0)
    assert np.array_equal(a, b)
    assert np.array_equal(to_u64(T.ctx.ntt_fwd(from_u64(a, T.ctx.device))), ev)


@pytest.mark.slow
def test_full_size_c2_encrypt_modswitch_automorph_bit_exact(pair):
    """C2 at full size (n = 30940, 11 limbs; BASELINE's mid set): the product's encryptions (R7-R9),
    modulus switch (a6), automorphism (a4) and tensor (a3) ciphertexts equal the oracle's bit for bit
    (public key only on the oracle side: a few minutes of schoolbook products)."""
    T = pair("c2")
    P, bgv = T.P, T.bgv
    ints = T.ctx.ints_per_ct
    K = bgv.keygen(P, SEED_KEYS, (), relin=False)
    ct_o = bgv.encrypt(P, K, np.zeros(P.n, dtype=np.int64), SEED_ENC, 7)
    ct_g = T.ctx.encrypt(T.keys, np.zeros((1, ints), dtype=np.uint64), SEED_ENC, ct_index0=7)
    assert np.array_equal(to_u64(ct_g)[0], np.stack(bgv.ct_to_eval(P, ct_o)))
    assert np.array_equal(to_u64(T.ctx.modswitch(ct_g))[0], np.stack(bgv.ct_to_eval(P, bgv.modswitch(P, ct_o))))
    t = pow(P.alg.g, 1, P.m) if P.n < 5000 else 2
    idx = list(range(P.L1))
    want = np.stack([bgv.to_eval(P, np.stack([P.ring.automorph_mod(c[r], t, P.moduli[r]) for r in idx]), idx)
                     for c in ct_o.parts])
    assert np.array_equal(to_u64(T.ctx.automorph(ct_g, t))[0], want)
    # a3 tensor of two full-size ciphertexts (a second, independent encryption)
    ct_o2 = bgv.encrypt(P, K, np.zeros(P.n, dtype=np.int64), SEED_ENC, 8)
    ct_g2 = T.ctx.encrypt(T.keys, np.zeros((1, ints), dtype=np.uint64), SEED_ENC, ct_index0=8)
    assert np.array_equal(to_u64(ct_g2)[0], np.stack(bgv.ct_to_eval(P, ct_o2)))
    assert np.array_equal(to_u64(T.ctx.tensor(ct_g, ct_g2))[0], np.stack(bgv.ct_to_eval(P, bgv.tensor(P, ct_o, ct_o2))))


@pytest.mark.parametrize("name", ["c2s", "c4s", "c2"])
def test_fused_epilogue_and_column_pass_variants_identical(pair, name):
    """The scale-sub / fused-ModDown epilogues inside pass C (bc_tune ntt_epi 1, opt-in), the pass-C
    staging-tile-as-exchange variant (ntt_lean 4, default), the fused a + c x of the digit circuits'
    linear combinations (axpy 1, default) and the one-kernel kappa-weighted extraction sums (ptsum 1, default)
    give the same compare_lt words as the separate kernels and the round-2 passes (ntt_epi 0, ntt_lean 0,
    axpy 0, ptsum 0); the default words are the ones the oracle parity tests
    pin (c2s) -- here on the C2 shadow, the C4 shadow and full-size C2."""
    import paper_2407_07308_b200 as bc
    T = pair(name)
    P = T.P
    ints = T.ctx.ints_per_ct
    rng = np.random.default_rng(44)
    a, b = mixed_pairs(P, rng, ints)
    ca = T.ctx.encrypt(T.keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=40)
    cb = T.ctx.encrypt(T.keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=41)
    ref = to_u64(T.ctx.compare_lt(T.keys, ca, cb))
    try:
        for epi, lean, axpy, ptsum in [(0, 0, 0, 0), (1, 4, 1, 0), (1, 0, 0, 1), (1, 2, 1, 0)]:
            bc._lib.bc_tune(b"ntt_epi", epi)
            bc._lib.bc_tune(b"ntt_lean", lean)
            bc._lib.bc_tune(b"axpy", axpy)
            bc._lib.bc_tune(b"ptsum", ptsum)
            assert np.array_equal(to_u64(T.ctx.compare_lt(T.keys, ca, cb)), ref), (epi, lean, axpy, ptsum)
    finally:
        bc._lib.bc_tune(b"ntt_epi", 0)
        bc._lib.bc_tune(b"ntt_lean", 4)
        bc._lib.bc_tune(b"axpy", 1)
        bc._lib.bc_tune(b"ptsum", 1)
    assert list(T.ctx.decrypt(T.keys, T.ctx.compare_lt(T.keys, ca, cb), as_bits=True)[0]) == [int(x < y) for x, y in zip(a, b)]
