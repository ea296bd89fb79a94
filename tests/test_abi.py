"""The C-ABI library loads and exports every symbol include/boostcom.h declares (no GPU needed)."""
import ctypes
import os
import re

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
