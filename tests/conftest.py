"""Shared test fixtures.

Markers: ``gpu`` -- needs a CUDA device (the driver runs ``-m gpu`` on a B200
and ``-m "not gpu"`` on the CPU-only build container).  The CPU oracle
(oracle/, test infrastructure) is the checker for the GPU path; the golden
fixtures under tests/golden/ pin both to the real reference.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
for p in (ROOT, ROOT / "tests", ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

GOLDEN = ROOT / "tests" / "golden"
STATUS = {"Success": 0, "MaxIter": 1, "MinStep": 2, "NaNDetected": 3, "Failure": 4}


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as orc

    orc.build()
    return orc


@pytest.fixture(scope="session")
def speed_arg():
    from paper_2003_02547_b200 import mode_preset

    return mode_preset("speed").with_tol(1e-8)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(GOLDEN / f"{name}.npz")
    return load


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2003_02547_b200 import build as b

    b.build()
    return torch


def rel_err(a, r):
    """||a - r||_inf / max(1, ||r||_inf) (the reference's test idiom)."""
    a = np.asarray(a, dtype=float)
    r = np.asarray(r, dtype=float)
    if r.size == 0:
        return 0.0
    return float(np.max(np.abs(a - r)) / max(1.0, float(np.max(np.abs(r)))))


def random_case_qp(seed, kw):
    import qpgen

    import paper_2003_02547_b200 as pkg

    return qpgen.build_qp(pkg, *qpgen.random_ocp_fields(seed, **kw))


def random_cases():
    """(seed, kwargs) of tests/golden/make_golden.py RANDOM_CASES."""
    sys.path.insert(0, str(GOLDEN))
    import importlib.util

    spec = importlib.util.spec_from_file_location("mg_cases", GOLDEN / "make_golden.py")
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("RANDOM_CASES = [")
    end = src.index("]\n", start) + 1
    ns = {}
    exec(src[start:end], {"dict": dict}, ns)
    del spec
    return ns["RANDOM_CASES"]


def cfg_cases():
    src = (GOLDEN / "make_golden.py").read_text()
    start = src.index("CFG_CASES = [")
    end = src.index("]\n", src.index("(4, [0], None)")) + 1
    ns = {}
    exec(src[start:end], {}, ns)
    return ns["CFG_CASES"]
