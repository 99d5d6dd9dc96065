import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C ABI)")


@pytest.fixture(scope="session")
def orc():
    from oracle import restatement
    return restatement()


@pytest.fixture(scope="session")
def ref():
    from oracle import ref_available, reference
    if not ref_available():
        pytest.skip("oracle/_ref (reference compiled unmodified) not built")
    return reference()


@pytest.fixture(scope="session")
def golden():
    return dict(np.load(ROOT / "tests" / "golden" / "golden_r01.npz"))


def rel(a, b):
    """Max-norm relative difference, the reference's metric (test_support.hpp:34-37)."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(float(np.max(np.abs(b))), 1e-300)) if b.size else 0.0


def colwise_rel(a, b):
    """Per-column max-norm relative difference (SURVEY 8(c) parity metric for factors)."""
    out = []
    for q in range(b.shape[1]):
        out.append(rel(a[:, q], b[:, q]))
    return max(out) if out else 0.0
