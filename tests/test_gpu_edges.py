"""Edge cases of the CUDA path (SURVEY §8(b) error mapping, maximum words, degenerate pairs)."""
import numpy as np
import pytest

from gpu_util import SEED_ENC, SEED_KEYS, to_u64  # noqa: F401

pytestmark = pytest.mark.gpu

_CTX = {}


def ctx_keys(name):
    import paper_2407_07308_b200 as bc
    if name not in _CTX:
        ctx = bc.Context(bc.load_params(name))
        _CTX[name] = (ctx, ctx.keygen(SEED_KEYS))
    return _CTX[name]


def boundary_pairs(cap, base, digits, ints):
    """0, the maximum word, +-1 neighbours, digit-boundary carries, equal pairs"""
    mx = cap - 1
    cands = [(0, 0), (mx, mx), (mx - 1, mx), (mx, mx - 1), (0, mx), (mx, 0), (0, 1), (1, 0)]
    top = base ** (digits - 1)
    if top < cap:
        cands += [(top, top - 1), (top - 1, top), (top, top)]
    cands += [(base, base - 1), (base - 1, base)]
    while len(cands) < ints:
        cands.append((mx // 2, mx // 2 + 1))
    return [a for a, _ in cands[:ints]], [b for _, b in cands[:ints]]


@pytest.mark.parametrize("cfg", ["c2s", "c3s2"])
def test_boundary_words_compare(cfg):
    """maximum words (2^64 - 1: 7^24 and 31^15 exceed 2^64), zero, +-1 and carry neighbours, equal pairs:
    compare_lt / compare_eq decrypt to the plaintext answer in every block"""
    ctx, keys = ctx_keys(cfg)
    ints = ctx.ints_per_ct
    cap = min(ctx.base ** (ctx.d * ctx.l), 1 << 64)
    a, b = boundary_pairs(cap, ctx.base, ctx.d * ctx.l, ints)
    ca = ctx.encrypt(keys, np.array([a], dtype=np.uint64), SEED_ENC, ct_index0=0)
    cb = ctx.encrypt(keys, np.array([b], dtype=np.uint64), SEED_ENC, ct_index0=1)
    assert [int(x) for x in ctx.decrypt(keys, ca)[0]] == a
    lt = ctx.decrypt(keys, ctx.compare_lt(keys, ca, cb), as_bits=True)[0]
    eq = ctx.decrypt(keys, ctx.compare_eq(keys, ca, cb), as_bits=True)[0]
    assert [int(x) for x in lt] == [int(x < y) for x, y in zip(a, b)]
    assert [int(x) for x in eq] == [int(x == y) for x, y in zip(a, b)]


def test_out_of_range_word_is_rejected():
    """S:333 OutOfRange -> BC_E_RANGE (3): C1 words are 2-bit (base 2, d l = 2)"""
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c1")
    words = np.zeros((1, ctx.ints_per_ct), dtype=np.uint64)
    words[0, 3] = 4
    with pytest.raises(bc.BoostComError, match=r"status 3"):
        ctx.encrypt(keys, words, SEED_ENC)


def test_empty_batch_is_rejected():
    """an empty ciphertext view is an argument error (BC_E_ARG = 1), never a silent no-op"""
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c1")
    ca = ctx.encrypt(keys, np.zeros((1, ctx.ints_per_ct), dtype=np.uint64), SEED_ENC)
    with pytest.raises(bc.BoostComError, match=r"status 1"):
        ctx.compare_lt(keys, ca[0:0], ca[0:0])


def test_out_of_levels_is_rejected():
    """S:427 OutOfLevels -> BC_E_LEVEL (4): a compare of ciphertexts switched down to level 1"""
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c1")
    ca = ctx.encrypt(keys, np.zeros((1, ctx.ints_per_ct), dtype=np.uint64), SEED_ENC)
    while ca.shape[2] > 1:
        ca = ctx.modswitch(ca)
    with pytest.raises(bc.BoostComError, match=r"status 4"):
        ctx.compare_lt(keys, ca, ca)


def test_ragged_batch_and_unequal_levels():
    """an odd batch (3 pairs) on C2's shadow ring; on c1m (spare levels) b one level below a: R12
    aligns the levels; on C2's exact chain the same misalignment is BC_E_LEVEL (no level to spare)"""
    import paper_2407_07308_b200 as bc
    from inputs import word_pairs
    for name in ("c2s", "c1m"):
        ctx, keys = ctx_keys(name)
        ints = ctx.ints_per_ct
        rng = np.random.default_rng(3)
        A, B = [], []
        for _ in range(3):
            a, b = word_pairs(rng, ints, ctx.base, ctx.d * ctx.l)
            A.append(a)
            B.append(b)
        ca = ctx.encrypt(keys, np.array(A, dtype=np.uint64), SEED_ENC, ct_index0=0)
        cb = ctx.encrypt(keys, np.array(B, dtype=np.uint64), SEED_ENC, ct_index0=3)
        if name == "c2s":
            with pytest.raises(bc.BoostComError, match=r"status 4"):
                ctx.compare_lt(keys, ca, ctx.modswitch(cb))
        else:
            cb = ctx.modswitch(cb)
        bits = ctx.decrypt(keys, ctx.compare_lt(keys, ca, cb), as_bits=True)
        for i in range(3):
            assert [int(x) for x in bits[i]] == [int(x < y) for x, y in zip(A[i], B[i])]


def test_bad_output_views_are_rejected_before_any_work():
    """an output view that is too small, at the wrong level or null is BC_E_ARG (1) /
    BC_E_LEVEL (4) from the C ABI, validated before anything is enqueued (the output is untouched)"""
    import torch
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c1m")
    lib = bc._lib
    ca = ctx.encrypt(keys, np.zeros((2, ctx.ints_per_ct), dtype=np.uint64), SEED_ENC)
    lvl = ctx.out_level(ca.shape[2], 0)
    w, wb = ctx._wsargs(None)
    st = bc._stream()
    small = ctx.ct_empty(1, lvl).fill_(7)
    wrong = ctx.ct_empty(2, lvl + 1).fill_(7)
    v = ctx.view(ca)
    assert lib.bc_compare_lt(ctx._h, keys.keys, v, v, ctx.view(small), w, wb, st) == 1
    assert lib.bc_compare_lt(ctx._h, keys.keys, v, v, ctx.view(wrong), w, wb, st) == 4
    assert lib.bc_compare_lt(ctx._h, keys.keys, v, v, bc.bc_ct(None, 2, lvl), w, wb, st) == 1
    assert lib.bc_mul(ctx._h, keys.keys, v, v, ctx.view(small), w, wb, st) in (1, 4)
    assert lib.bc_rotate(ctx._h, keys.keys, v, 1, ctx.view(small), w, wb, st) in (1, 4)
    assert lib.bc_automorph(ctx._h, v, 2, ctx.view(small), st) in (1, 4)
    torch.cuda.synchronize()
    assert bool((small == 7).all()) and bool((wrong == 7).all())


@pytest.mark.parametrize("batch,chunk", [(5, 2), (3, 0), (1, 4)])
def test_compare_lt_host_pipelined(batch, chunk):
    """bc_compare_lt_host (host buffers, H2D / compare / D2H pipelined over chunks with a ragged tail) gives
    the words of bc_compare_lt on device buffers; a short staging buffer is BC_E_ARG"""
    import torch
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c2s")
    rng = np.random.default_rng(71)
    cap = min(ctx.base ** (ctx.d * ctx.l), 1 << 64)
    w = rng.integers(0, cap, size=(2, batch, ctx.ints_per_ct), dtype=np.uint64)
    ca = ctx.encrypt(keys, w[0], SEED_ENC, ct_index0=0)
    cb = ctx.encrypt(keys, w[1], SEED_ENC, ct_index0=batch)
    ref = ctx.compare_lt(keys, ca, cb)
    ha, hb = ca.cpu().pin_memory(), cb.cpu().pin_memory()
    ho = torch.zeros(ref.shape, dtype=ref.dtype).pin_memory()
    ctx.compare_lt_host(keys, ha, hb, ho, chunk=chunk)
    torch.cuda.synchronize()
    assert torch.equal(ho, ref.cpu())
    bits = ctx.decrypt(keys, ho.cuda(), as_bits=True)
    assert np.array_equal(bits, (w[0] < w[1]).astype(np.uint64))
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(bc.BoostComError):
        ctx.compare_lt_host(keys, ha, hb, ho, chunk=chunk, stage=small)


def test_fault_injection_is_detected(monkeypatch):
    """SURVEY §5 failure detection: BC_FAULT_INJECT=<prime>:<word> corrupts one word of the forward D^ table
    at context creation; the same seeded compare then no longer decrypts to the plaintext answer and its words
    differ from the clean context's (what the parity tests and the bench's verify-in-warm-up rely on)"""
    import paper_2407_07308_b200 as bc
    ctx, keys = ctx_keys("c2s")
    rng = np.random.default_rng(72)
    cap = min(ctx.base ** (ctx.d * ctx.l), 1 << 64)
    w = rng.integers(0, cap, size=(2, 2, ctx.ints_per_ct), dtype=np.uint64)
    clean = to_u64(ctx.compare_lt(keys, ctx.encrypt(keys, w[0], SEED_ENC, 0), ctx.encrypt(keys, w[1], SEED_ENC, 2)))
    monkeypatch.setenv("BC_FAULT_INJECT", "1:17")
    bad_ctx = bc.Context(bc.load_params("c2s"))
    monkeypatch.delenv("BC_FAULT_INJECT")
    bad_keys = bad_ctx.keygen(SEED_KEYS)
    lt = bad_ctx.compare_lt(bad_keys, bad_ctx.encrypt(bad_keys, w[0], SEED_ENC, 0), bad_ctx.encrypt(bad_keys, w[1], SEED_ENC, 2))
    assert not np.array_equal(to_u64(lt), clean)
    bits = bad_ctx.decrypt(bad_keys, lt, as_bits=True)
    assert not np.array_equal(bits, (w[0] < w[1]).astype(np.uint64))
