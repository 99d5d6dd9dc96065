"""K2 soak on the GPU: random lattices (up to 40 cells per axis, n up to 64, up to 8 charges on
random vertices, box and periodic) assembled from an oracle master and compared BITWISE with the
C oracle's ascending-k adds (lattice.hpp:220-274). Covers both assembly kernels (box: eight
chains per thread on a sliding register window; periodic: prefetching chains) far beyond the
per-config cases."""
import ctypes as C
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1405_2270_b200 as lat
    return lat


def _lattices(n_cases=120, seed=3):
    rng = np.random.default_rng(seed)
    for c in range(n_cases):
        Lc = tuple(int(x) for x in rng.integers(1, 41, 3))
        periodic = bool(rng.integers(0, 2))
        if periodic and rng.integers(0, 2):
            Lc = tuple(2 * ((x + 1) // 2) for x in Lc)
        n = int(2 * rng.integers(1, 33))
        M0 = int(rng.integers(1, 9))
        idx = rng.integers(0, n + 1, (M0, 3))
        M = int(rng.integers(2, 12))
        yield pytest.param(Lc, periodic, n, idx, M, id=f"c{c}-L{Lc}-n{n}-M0{M0}-{'per' if periodic else 'box'}")


@pytest.mark.parametrize("Lc,periodic,n,idx,M", list(_lattices()))
def test_assembly_soak_bitwise(L, orc, Lc, periodic, n, idx, M):
    b = 10.0
    h = b / n
    spec = L.LatticeSpec(Lc, L.GridSpec(b, n), [L.Charge(tuple(float(i) * h - b / 2 for i in idx[m]), 1.0 + m)
                                                for m in range(len(idx))])
    rule = L.sinc_quadrature(1e-6, h, math.sqrt(3.0) * max(Lc) * b, M, 1.0)
    R, M0 = rule.node_count(), len(idx)
    m = orc.lattice_master(0, list(Lc), n, b, rule.exponents)
    got = (L.assembled_periodic_sum if periodic else L.assembled_box_sum)(
        spec, L.CanonicalTensor3(m, rule.weights, trusted=True))
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    for l in range(3):
        ia = np.array([spec.charge_grid_index(l, nu) for nu in range(M0)], dtype=np.int64)
        want = np.zeros((n if periodic else Lc[l] * n, M0 * R), order="F")
        assert orc._assembled_axis(dp(np.asfortranarray(m[l])), R, M0, ia.ctypes.data_as(C.POINTER(C.c_int64)), n,
                                   Lc[l], int(periodic), dp(want)) == 0
        assert np.array_equal(got.tensor.factor(l), want), l
