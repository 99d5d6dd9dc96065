"""QTT on the GPU (csrc/qtt.cu, qtt.hpp drop-in) against the numpy restatement
(oracle/qtt_numpy.py; the reference's Eigen BDCSVD is absent from this image) and the
reference's own rank laws (proj/tests/test_qtt.cpp). The C++ drop-in cases re-host those
tests in tests/cpp/dropin_tests.cpp."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1405_2270_b200 as L
    return L


def _vectors():
    rng = np.random.default_rng(7)
    x = (np.arange(4096) + 0.5) / 4096 * 10 - 5
    yield "gauss4096", np.exp(-x * x), 1e-6
    yield "random256", rng.uniform(-1, 1, 256), 1e-14
    yield "noisy1024", np.exp(-((np.arange(1024) - 512) / 150.0) ** 2) + 0.01 * rng.uniform(-1, 1, 1024), 1e-4
    yield "sin1024", np.sin(0.37 * np.arange(1024) + 0.3), 1e-10
    yield "cubic2048", (lambda t: ((t - 0.4) * t + 0.25) * t - 1.0)(np.arange(2048) / 2048.0), 1e-11


@pytest.mark.parametrize("name,v,eps", list(_vectors()), ids=[x[0] for x in _vectors()])
def test_qtt_matches_numpy_restatement(L, name, v, eps):
    from oracle.qtt_numpy import qtt_compress, qtt_reconstruct, unfolding_rank_profile
    t = L.qtt_compress(v, eps)
    cores, sig = qtt_compress(v, eps)
    want = [c.shape[1] for c in cores[:-1]]
    got = t.ranks()
    N = len(v)
    delta = eps * np.linalg.norm(v) / math.sqrt(max(int(math.log2(N)) - 1, 1))
    for k, (a, b) in enumerate(zip(got, want)):
        if a != b:  # only where numpy's singular tail sits at the threshold to rounding
            s = sig[k]
            tails = np.sqrt(np.cumsum((s[::-1] ** 2)))[::-1]
            assert np.min(np.abs(tails - delta)) <= 1e-10 * max(delta, 1e-300) + 1e-14 * s[0], (name, k, a, b)
    rec = L.qtt_reconstruct(t)
    bound = max(eps, 5e-14) * np.linalg.norm(v)  # the error contract, or rounding when nothing is truncated
    assert np.linalg.norm(rec - v) <= bound
    assert np.linalg.norm(qtt_reconstruct(cores) - v) <= bound
    assert L.unfolding_rank_profile(v, eps) == unfolding_rank_profile(v, eps)


def test_qtt_batch_equals_single_and_is_deterministic(L):
    rng = np.random.default_rng(3)
    V = np.asfortranarray(np.cumsum(rng.normal(size=(1024, 9)), axis=0))
    batch = L.qtt_compress_columns(V, 1e-6)
    for c in range(V.shape[1]):
        one = L.qtt_compress(V[:, c], 1e-6)
        assert one.ranks() == batch[c].ranks()
        for a, b in zip(one.cores, batch[c].cores):
            assert np.array_equal(a, b)


def test_qtt_of_assembled_lattice_columns(L):
    """The study the reference runs on assembled box sums (qtt.hpp:219-269): every column of a
    cfg0-shaped lattice (n = 64, L = 4: N = 256) compresses within eps and the ranks follow the
    restatement."""
    from oracle.qtt_numpy import qtt_compress
    spec = L.LatticeSpec((4, 4, 4), L.GridSpec(10.0, 64), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3.0) * 40.0, 20, 1.0)
    res = L.assembled_box_sum(spec, L.build_lattice_master(spec, rule))
    A = res.tensor.factor(0)
    trains = L.qtt_compress_columns(A, 1e-8)
    mism = 0
    for q, t in enumerate(trains):
        v = A[:, q]
        rec = L.qtt_reconstruct(t)
        assert np.linalg.norm(rec - v) <= 1e-8 * np.linalg.norm(v) * (1 + 1e-9)
        want = [c.shape[1] for c in qtt_compress(v, 1e-8)[0][:-1]]
        mism += sum(a != b for a, b in zip(t.ranks(), want))
    assert mism <= 2  # borderline singular values only
