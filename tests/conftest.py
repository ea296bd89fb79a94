import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the product kernels")
    config.addinivalue_line("markers", "slow: long-running oracle computation")


def load_cfg(name):
    """params/<name>.json; "<name>@r16" / "<name>@r23" overrides the digit-circuit schedule (R16 / R23),
    "<name>@pow2" / "<name>@mixed" the Bluestein length (R25)"""
    base, _, sched = name.partition("@")
    with open(os.path.join(ROOT, "params", base + ".json")) as f:
        cfg = json.load(f)
    if sched in ("pow2", "mixed"):         # "<name>@pow2": the power-of-two Bluestein length (R25 off)
        cfg["bluestein"] = sched
    elif sched:
        cfg["schedule"] = sched
    return cfg


def golden(name):
    with open(os.path.join(ROOT, "tests", "golden", name)) as f:
        return json.load(f)


_P = {}


@pytest.fixture(scope="session")
def oracle_params():
    from oracle import bgv

    def get(name):
        if name not in _P:
            _P[name] = bgv.Params(load_cfg(name))
        return _P[name]
    return get
