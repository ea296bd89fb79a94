"""The C-ABI library loads and exports every symbol include/boostcom.h declares (no GPU needed)."""
import ctypes
import os
import re
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "boostcom.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bc_[a-z0-9_]+)\s*\(", src)))


def test_library_builds_and_exports_all_symbols():
    from paper_2407_07308_b200 import _build
    so = _build.build()
    lib = ctypes.CDLL(so)
    missing = [s for s in _declared() if not hasattr(lib, s)]
    assert not missing, missing
    assert len(_declared()) >= 30


def test_binding_imports_without_gpu():
    import paper_2407_07308_b200 as bc
    assert "bc_compare_lt" in bc.EXPORTS or hasattr(bc._lib, "bc_compare_lt")
    cfg = bc.load_params("c2")
    assert cfg["p"] == 13 and cfg["m"] == 30941


def test_oracle_not_imported_by_product():
    """the product package never imports the oracle (independence, no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2407_07308_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


def test_circuit_plan_matches_oracle():
    """host logic, no device: the digit circuit the library evaluates (bc_circuit_plan: R23 baby-step
    size, products per digit, depth) equals the oracle's count of its own schedule for every p <= 31,
    both circuits, R16 and R23 (R16 / R23)"""
    import paper_2407_07308_b200 as bc
    from oracle import circuits as c
    for p in [3, 5, 7, 11, 13, 17, 19, 23, 29, 31]:
        for kind in "UB":
            ev = c.CountEval(p)
            if kind == "U":
                lt, eq = c.univariate_lt_eq(ev, c.CountValue(), p)
            else:
                lt, eq = c.bivariate_lt_eq(ev, c.CountValue(), c.CountValue(), p)
            assert bc.circuit_plan(p, kind, "r16") == (0, ev.counts["mul"], max(lt.depth, eq.depth))
            k = c.r23_univariate_k(p) if kind == "U" else c.r23_bivariate_k(p)
            f = c.univariate_lt_eq_r23 if kind == "U" else c.bivariate_lt_eq_r23
            assert bc.circuit_plan(p, kind, "r23") == (k,) + c._r23_cost(f, p, k)
            if kind == "B":
                k1, k2 = c.r26_bivariate_k(p)
                assert bc.circuit_plan(p, kind, "r26") == ((k1 << 8) | k2,) + c._r26_cost(p, k1, k2)
            else:
                assert bc.circuit_plan(p, kind, "r26") == bc.circuit_plan(p, kind, "r23")
            assert bc.circuit_plan(p, kind, "r27") == bc.circuit_plan(p, kind, "r26")   # R27 regroups R26's products
    with pytest.raises(bc.BoostComError):
        bc.circuit_plan(15, "U", "r23")


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_compact_plan_matches_oracle(seed):
    """host logic, no device: bc_compact's R17 plan (bitmap implementation) equals the oracle's
    plan_compaction on random and Fig. 7 usefulness patterns, with and without row limits"""
    import numpy as np
    import paper_2407_07308_b200 as bc
    from oracle import circuits
    rng = np.random.default_rng(seed)
    for nin, ints, wpr, dens in ((9, 40, 40, 0.3), (12, 36, 12, 0.2), (20, 64, 16, 0.25), (6, 30, 10, 0.6)):
        useful = (rng.random((nin, ints)) < dens).astype(np.uint8)
        if seed == 2:
            useful[:] = 0
            useful[:, 3::4] = 1          # Fig. 7: every 4th block
        dest, n = bc.compact_plan(useful, 3, wpr)
        _, n_o, dest_o = circuits.plan_compaction([list(np.nonzero(u)[0]) for u in useful], ints, 3, wpr)
        assert n == n_o
        want = np.full((nin, ints), -1, dtype=np.int32)
        for (c, b), (cp, bp) in dest_o.items():
            want[c, b] = cp * ints + bp
        assert np.array_equal(dest, want)
