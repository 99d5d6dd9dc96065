"""CPU oracle pinning (no GPU): the C restatement (oracle/latsum_oracle.c) against
the reference's own headers compiled unmodified (oracle/_ref), against the
committed golden vectors from those headers, and against the reference's
known-answer tests (proj/tests/*.cpp)."""
import ctypes as C
import math

import numpy as np
import pytest

from conftest import colwise_rel, rel

dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
i64p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731


def adaptive_simpson(f, a, b, tol=1e-14, depth=40):
    # Independent cell-integral oracle, as test_newton.cpp:11-30.
    def rec(a, b, fa, fm, fb, whole, tol, depth):
        m = 0.5 * (a + b)
        lm, rm = 0.5 * (a + m), 0.5 * (m + b)
        flm, frm = f(lm), f(rm)
        left = (m - a) / 6.0 * (fa + 4.0 * flm + fm)
        right = (b - m) / 6.0 * (fm + 4.0 * frm + fb)
        if depth <= 0 or abs(left + right - whole) < 15.0 * tol:
            return left + right + (left + right - whole) / 15.0
        return rec(a, m, fa, flm, fm, left, 0.5 * tol, depth - 1) + rec(m, b, fm, frm, fb, right, 0.5 * tol, depth - 1)
    m = 0.5 * (a + b)
    fa, fm, fb = f(a), f(m), f(b)
    return rec(a, b, fa, fm, fb, (b - a) / 6.0 * (fa + 4.0 * fm + fb), tol, depth)


# ------------------------------------------------------------------ KATs (restatement)
def test_zero_exponent_gives_cell_widths(orc):  # test_newton.cpp:32-40
    v = orc.gaussian_moment_vector(4.0, 8, 0.0, False)
    assert v.shape == (8,) and np.all(v == 0.5)
    d = orc.gaussian_moment_vector(4.0, 8, 0.0, True)
    assert d.shape == (16,) and np.all(d == 0.5)


def test_unit_cell_matches_erf_integral(orc):  # test_newton.cpp:42-52
    v = orc.gaussian_moment_vector(2.0, 2, 1.0, False)
    want = 0.5 * math.sqrt(math.pi) * math.erf(1.0)
    assert abs(v[0] - want) <= 1e-15 and abs(v[1] - want) <= 1e-15
    assert abs(v[1] - adaptive_simpson(lambda x: math.exp(-x * x), 0.0, 1.0)) <= 1e-12


@pytest.mark.parametrize("doubled", [False, True])
def test_moment_matches_adaptive_quadrature_per_cell(orc, doubled):  # test_newton.cpp:54-69
    t, h = 0.7, 0.5
    v = orc.gaussian_moment_vector(3.0, 6, t, doubled)
    length = 12 if doubled else 6
    for i in range(length):
        lo = (i - length // 2) * h
        want = adaptive_simpson(lambda x: math.exp(-t * t * x * x), lo, lo + h)
        assert abs(v[i] - want) <= 1e-12


def test_moment_even_symmetry_is_exact(orc):  # test_newton.cpp:71-77
    for t in (0.3, 1.0, 4.5):
        v = orc.gaussian_moment_vector(5.0, 10, t, False)
        assert np.array_equal(v, v[::-1])


def test_gaussian_samples_match_midpoint_values(orc):  # test_newton.cpp:86-96
    v = orc.gaussian_sample_vector(6, 0.5, 1.3)
    for i in range(6):
        x = (i + 0.5 - 3.0) * 0.5
        assert v[i] == pytest.approx(math.exp(-1.3 * 1.3 * x * x), rel=4e-16)
        assert v[i] == v[5 - i]
    with pytest.raises(RuntimeError):
        orc.gaussian_sample_vector(5, 0.5, 1.3)


def test_sinc_quadrature_layout_and_positivity(orc):  # test_newton.cpp:98-113
    nodes, tau, w, step = orc.sinc_quadrature(1e-6, 0.01, 10.0, 20, 1.0)
    assert len(tau) == 41 and step > 0
    assert np.all(w > 0) and np.all(tau >= 0)
    assert np.all(np.diff(nodes) > 0) and np.all(np.diff(tau) > 0)
    for bad in [(1e-6, 0.01, 10.0, 0, 1.0), (0.0, 0.01, 10.0, 5, 1.0), (1e-6, 1.0, 0.5, 5, 1.0)]:
        with pytest.raises(RuntimeError):
            orc.sinc_quadrature(*bad)


def test_sinc_quadrature_approximates_inverse_radius(orc):  # test_newton.cpp:115-123
    a_min, a_max, eps = 0.05, 4.0, 1e-6
    _, tau, w, _ = orc.sinc_quadrature(eps, a_min, a_max, 40, 2.0)
    for i in range(51):
        r = a_min * (a_max / a_min) ** (i / 50.0)
        assert abs(orc.quadrature_value(tau, w, r) * r - 1.0) < eps


def test_newton_entry_equals_quadrature_value_at_radius(orc):  # test_newton.cpp:143-158
    b, n = 2.0, 16
    h = b / n
    _, tau, w, _ = orc.sinc_quadrature(1e-5, h, 4.0, 25, 2.0)
    f = orc.gaussian_sample_vector  # build_newton_tensor = midpoint master on the n grid
    A = np.asfortranarray(np.stack([f(n, h, t) for t in tau], axis=1))
    mid = lambda i: (i + 0.5 - n / 2) * h  # noqa: E731
    for i in (0, 3, 8, 11):
        for j in (1, 8, 14):
            k = 5
            r = math.sqrt(mid(i) ** 2 + mid(j) ** 2 + mid(k) ** 2)
            want = orc.quadrature_value(tau, w, r)
            assert abs(orc.eval_point(A, A, A, w, i, j, k) - want) <= 1e-12 * want


def test_windows_stay_inside_doubled_master(orc):  # test_lattice.cpp:84-101
    n = 8
    for L in (1, 2, 3, 5):
        N = L * n
        for ia in range(n + 1):
            for k in range(L):
                s = orc._window_start_box(N, n, ia, k)
                assert 0 <= s and s + N <= 2 * N
                p = orc._window_start_periodic(N, n, ia, k, L)
                assert 0 <= p and p + n <= 2 * N
    assert orc._window_start_box(16, 8, 8, 0) == orc._window_start_box(16, 8, 0, 1)  # test_lattice.cpp:174-187


def test_charge_snapping(orc):  # test_lattice.cpp:111-123
    assert orc._charge_grid_index(2.0, 8, 0.25) == 5
    assert orc._charge_grid_index(2.0, 8, -1.0) == 0
    assert orc._charge_grid_index(2.0, 8, 1.0) == 8
    assert orc._charge_grid_index(2.0, 8, 0.1) == -1
    assert orc._charge_grid_index(2.0, 8, 1.25) == -1


def _physical_potential(tau, w, L, n, b, charges, idx, periodic):
    # test_lattice.cpp:16-54: exponential-sum kernel at exact offsets, explicit loops.
    h = b / n
    N = [L[l] * n for l in range(3)]
    total = 0.0
    for (px, py, pz, Z) in charges:
        for k1 in range(L[0]):
            for k2 in range(L[1]):
                for k3 in range(L[2]):
                    d2 = 0.0
                    for l, (cell, p) in enumerate(zip((k1, k2, k3), (px, py, pz))):
                        off = (L[l] // 2) * n if periodic else 0
                        x = (idx[l] + off + 0.5 - N[l] / 2.0) * h
                        y = -L[l] * b / 2.0 + cell * b + p + b / 2.0
                        d2 += (x - y) * (x - y)
                    total += Z * float(np.sum(w * np.exp(-tau * tau * d2)))
    return total


def _orc_assembled(orc, L, n, b, charges, tau, w, periodic, mode=0):
    f = orc.lattice_master(mode, L, n, b, tau)
    R = len(tau)
    M0 = len(charges)
    out = []
    for l in range(3):
        ia = np.array([orc._charge_grid_index(b, n, c[l]) for c in charges], dtype=np.int64)
        ol = n if periodic else L[l] * n
        o = np.zeros((ol, M0 * R), order="F")
        assert orc._assembled_axis(dp(f[l]), R, M0, i64p(ia), n, L[l], int(periodic), dp(o)) == 0
        out.append(o)
    wout = np.zeros(M0 * R)
    Z = np.array([c[3] for c in charges])
    orc._assembled_weights(dp(Z), M0, dp(np.ascontiguousarray(w)), R, dp(wout))
    return out, wout, f


@pytest.mark.parametrize("periodic", [False, True])
def test_assembled_sum_matches_physical_oracle(orc, periodic):  # test_lattice.cpp:139-155, 266-283
    L, n, b = (4, 2, 1), 8, 2.0
    charges = [(0.0, 0.0, 0.0, 1.0), (0.25, 0.5, -0.25, 1.5)]
    _, tau, w, _ = orc.sinc_quadrature(1e-4, b / n, math.sqrt(3) * 4 * b, 12, 1.0)
    f, wout, _ = _orc_assembled(orc, L, n, b, charges, tau, w, periodic)
    V = orc.densify_slabs(f[0], f[1], f[2], wout)
    rng = np.random.default_rng(3)
    worst = 0.0
    for _ in range(40):
        idx = [int(rng.integers(0, V.shape[l])) for l in range(3)]
        want = _physical_potential(tau, w, L, n, b, charges, idx, periodic)
        worst = max(worst, abs(V[tuple(idx)] - want) / abs(want))
    assert worst < 1e-12


def test_assembled_matches_direct_sum_across_shapes(orc):  # test_lattice.cpp:218-241
    cases = [((2, 2, 2), 16, [(0, 0, 0, 1.0)]),
             ((4, 2, 1), 8, [(0, 0, 0, 1.0), (0.5, -0.25, 0.25, 2.0)]),
             ((3, 1, 2), 8, [(-0.75, 0.5, 0.0, 0.5)])]
    b = 2.0
    for L, n, charges in cases:
        _, tau, w, _ = orc.sinc_quadrature(1e-4, b / n, math.sqrt(3) * max(L) * b, 10, 1.0)
        f, wout, m = _orc_assembled(orc, L, n, b, charges, tau, w, False)
        R, M0 = len(tau), len(charges)
        cells = L[0] * L[1] * L[2]
        N = [L[l] * n for l in range(3)]
        d = [np.zeros((N[l], M0 * cells * R), order="F") for l in range(3)]
        wd = np.zeros(M0 * cells * R)
        ia = np.array([[orc._charge_grid_index(b, n, c[l]) for l in range(3)] for c in charges], dtype=np.int64)
        Z = np.array([c[3] for c in charges])
        La = np.array(L, dtype=np.int64)
        orc._direct_sum(i64p(La), n, i64p(ia), dp(Z), M0, dp(m[0]), dp(m[1]), dp(m[2]), dp(np.ascontiguousarray(w)),
                        R, dp(d[0]), dp(d[1]), dp(d[2]), dp(wd))
        Va = orc.densify_slabs(f[0], f[1], f[2], wout)
        Vd = orc.densify_slabs(d[0], d[1], d[2], wd)
        assert rel(Va, Vd) < 1e-12


def test_densify_matches_scalar_loops(orc):  # test_canonical.cpp:63-69
    rng = np.random.default_rng(7)
    for _ in range(10):
        dims = rng.integers(2, 9, 3)
        f = [np.asfortranarray(rng.uniform(-1, 1, (d, 3))) for d in dims]
        w = rng.uniform(-1, 1, 3)
        V = orc.densify_slabs(f[0], f[1], f[2], w)
        want = np.einsum("iq,jq,kq,q->ijk", f[0], f[1], f[2], w)
        assert rel(V, want) < 1e-13


def test_scalar_product_all_ones_counts_entries(orc):  # test_canonical.cpp:100-103
    ones = [np.ones((2, 1), order="F")] * 3
    assert orc.scalar_product(ones, np.ones(1), ones, np.ones(1)) == 8.0


# ------------------------------------------------------- restatement vs _ref (pinning)
def test_rule_matches_reference(orc, ref):
    for args in [(1e-6, 10 / 64, math.sqrt(3) * 40, 20, 1.0), (1e-4, 0.25, 4.0, 10, 2.0), (1e-6, 10 / 256,
                                                                                           math.sqrt(3) * 2560, 20, 1.0)]:
        a, b = orc.sinc_quadrature(*args), ref.sinc_quadrature(*args)
        for x, y in zip(a[:3], b[:3]):
            assert rel(x, y) <= 4e-16 * 8  # host FMA contraction in the -march build: a few ulp


@pytest.mark.parametrize("mode", [0, 1])
def test_master_bitwise_matches_reference(orc, ref, mode):
    _, tau, w, _ = ref.sinc_quadrature(1e-6, 10 / 64, math.sqrt(3) * 40, 20, 1.0)
    for L in ([4, 4, 4], [3, 2, 5]):
        a = orc.lattice_master(mode, L, 64, 10.0, tau)
        b = ref.lattice_master(mode, L, 64, 10.0, tau, w)
        for l in range(3):
            assert np.array_equal(a[l], b[l])


def test_assembly_bitwise_matches_reference(orc, ref, golden):
    g = golden
    ch = g["mc_charges"]
    L = [int(x) for x in g["mc_L"]]
    for periodic, key in ((False, "mc_box"), (True, "mc_per")):
        f, wout, _ = _orc_assembled(orc, L, 8, 2.0, [tuple(c) for c in ch], g["mc_tau"], g["mc_w"], periodic)
        for l in range(3):
            assert np.array_equal(f[l], g[f"{key}_{l}"])


def test_densify_and_functionals_match_reference(orc, ref):
    rng = np.random.default_rng(5)
    for dims, R in [((5, 7, 3), 3), ((16, 12, 9), 41)]:
        f = [np.asfortranarray(rng.uniform(-1, 1, (d, R))) for d in dims]
        w = rng.uniform(-1, 1, R)
        assert rel(orc.densify_slabs(*f, w), ref.densify_slabs(*f, w)) < 1e-14
        assert abs(orc.scalar_product(f, w, f, w) - ref.scalar_product(f, w, f, w)) <= 1e-13 * abs(
            ref.scalar_product(f, w, f, w))
        for p in [(0, 0, 0), (dims[0] - 1, 1, dims[2] - 1)]:
            assert orc.eval_point(*f, w, *p) == pytest.approx(ref.eval_point(*f, w, *p), rel=1e-14, abs=1e-15)


# ------------------------------------------------------------ restatement vs golden
def test_restatement_matches_golden(orc, golden):
    g = golden
    nodes, tau, w, step = orc.sinc_quadrature(1e-6, 10 / 64, math.sqrt(3) * 40, 20, 1.0)
    assert rel(tau, g["cfg0_tau"]) <= 4e-15 and rel(w, g["cfg0_w"]) <= 4e-15
    for mode, name in ((0, "mid"), (1, "erf")):
        m = orc.lattice_master(mode, [4, 4, 4], 64, 10.0, g["cfg0_tau"])
        assert np.array_equal(m[0], g[f"cfg0_master_{name}"])
        f, wout, _ = _orc_assembled(orc, [4, 4, 4], 64, 10.0, [(0, 0, 0, 1.0)], g["cfg0_tau"], g["cfg0_w"], False,
                                    mode)
        assert np.array_equal(f[0], g[f"cfg0_asm_{name}"])
        A = f[0]
        for s, k in enumerate(g["cfg0_slab_ids"]):
            got = orc.densify_slabs(A, A, A, wout, int(k), int(k) + 1)[:, :, 0]
            assert rel(got, g[f"cfg0_slabs_{name}"][:, :, s]) < 1e-14
    assert np.array_equal(orc.gaussian_moment_vector(3.0, 6, 0.7, False), g["moment_b3_n6_t07"])
    assert np.array_equal(orc.gaussian_moment_vector(3.0, 6, 0.7, True), g["moment_b3_n6_t07_doubled"])
    # multi-charge box dense grid and potential matrix
    d = [g[f"mc_box_{l}"] for l in range(3)]
    assert rel(orc.densify_slabs(*d, g["mc_box_w"]), g["mc_box_dense"]) < 1e-14
