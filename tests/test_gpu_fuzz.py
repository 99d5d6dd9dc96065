"""Randomized K3 sweep on the GPU against the C oracle (fixed seed).

Every expansion plan is reachable from some case: the two TMEM shapes (with the zero DFMA rank
and the padded 2-rank remainder), the shared-memory tiles, the 256-rank chunks that accumulate,
odd and padded output strides, partial z ranges, and the fused functional epilogue. Factors are
positive, so there is no cancellation and the bar is the north-star 1e-13 on relative max-norm.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_1405_2270_b200 import _abi
    return torch, _abi


def _cases(n=120, seed=20261019):
    rng = np.random.default_rng(seed)
    ranks = [1, 2, 3, 4, 5, 8, 40, 41, 42, 43, 45, 46, 57, 58, 61, 70, 73, 82, 89, 93, 94, 105, 113, 121, 123, 164,
             178, 181, 199, 240, 257, 300, 520]
    for c in range(n):
        R = int(rng.choice(ranks))
        big = rng.integers(0, 4) == 0  # some cases span several 128-row i-chunks and j-chunks
        n1 = int(rng.integers(1, 700 if big else 260))
        n2 = int(rng.integers(1, 600 if big else 200))
        n3 = int(rng.integers(1, 5))
        k0 = int(rng.integers(0, n3))
        k1 = int(rng.integers(k0 + 1, n3 + 1))
        pad_y = int(rng.choice([0, 0, 1, 3]))
        pad_z = int(rng.choice([0, 0, 2, 8]))
        func = bool(rng.integers(0, 2))
        yield pytest.param(c, R, (n1, n2, n3), k0, k1, pad_y, pad_z, func, id=f"c{c}-R{R}-{n1}x{n2}x{n3}")


@pytest.mark.parametrize("case,R,dims,k0,k1,pad_y,pad_z,func", list(_cases()))
def test_expand_fuzz(env, orc, case, R, dims, k0, k1, pad_y, pad_z, func):
    torch, _abi = env
    rng = np.random.default_rng(1000 + case)
    n1, n2, n3 = dims
    f = [np.asfortranarray(rng.uniform(0.05, 1.0, (d, R))) for d in dims]
    w = rng.uniform(0.05, 1.0, R)
    want = orc.densify_slabs(f[0], f[1], f[2], w, k0, k1)
    dev = torch.device("cuda")
    fac = [torch.as_tensor(x.T.copy(), device=dev) for x in f]  # (R, n) rows = column-major (n, R)
    wd = torch.as_tensor(w, device=dev)
    ldy = n1 + pad_y
    ldz = ldy * n2 + pad_z
    nk = k1 - k0
    buf = torch.full((nk * ldz + 8,), float("nan"), dtype=torch.float64, device=dev)
    lib = _abi.load()
    p = lambda x: C.c_void_p(x.data_ptr()) if x is not None else None  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    rho = part = None
    if func:
        rho = [torch.as_tensor(rng.uniform(0.1, 1.0, d), device=dev) for d in dims]
        npart = lib.ls_expand_partial_count(n1, n2, R, k0, k1)
        assert npart >= 0
        part = torch.zeros(max(npart, 1), dtype=torch.float64, device=dev)
    rc = lib.ls_expand(p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(wd), n1, n2, n3, R, k0, k1, p(buf), ldy, ldz,
                       p(rho[0]) if func else None, p(rho[1]) if func else None, p(rho[2]) if func else None,
                       p(part), s)
    assert rc == 0, lib.ls_last_error()
    torch.cuda.synchronize()
    got_flat = buf.cpu().numpy()
    got = np.empty((n1, n2, nk))
    for kk in range(nk):
        for j in range(n2):
            got[:, j, kk] = got_flat[kk * ldz + j * ldy: kk * ldz + j * ldy + n1]
    assert not np.isnan(got).any()
    assert float(np.max(np.abs(got - want)) / np.max(np.abs(want))) <= 1e-13
    # nothing outside the grid is written: row and slab padding and the 8 trailing guard elements
    # stay NaN
    written = np.zeros(got_flat.shape, dtype=bool)
    for kk in range(nk):
        for j in range(n2):
            written[kk * ldz + j * ldy: kk * ldz + j * ldy + n1] = True
    assert np.isnan(got_flat[~written]).all()
    # run to run: the same launch again gives the same bits (K3 has no atomics or races)
    if case % 4 == 0:
        again = torch.full_like(buf, float("nan"))
        rc = lib.ls_expand(p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(wd), n1, n2, n3, R, k0, k1, p(again), ldy,
                           ldz, None, None, None, None, s)
        assert rc == 0, lib.ls_last_error()
        torch.cuda.synchronize()
        assert np.array_equal(again.cpu().numpy()[written], got_flat[written])
    if func:
        e = torch.zeros(1, dtype=torch.float64, device=dev)
        assert lib.ls_sum_partials(p(part), int(lib.ls_expand_partial_count(n1, n2, R, k0, k1)), p(e), s) == 0
        r = [x.cpu().numpy() for x in rho]
        e_want = float(np.einsum("ijk,i,j,k->", want, r[0], r[1], r[2][k0:k1]))
        assert abs(float(e.cpu()) - e_want) <= 1e-13 * abs(e_want)


# Split-K at its edges (ranks >= 250): R mod 4 = 0 / 1 / 2 / 3 (zero rank, one or two DFMA
# ranks, a zero-padded k-step), odd and even KD (which half runs the remainder), and the largest
# single-launch ranks, where the halves fill all 512 TMEM columns and no zero rank fits (512:
# KD 128; a fuzz soak found the r02 zero rank overflowing TMEM there). 513+ chunks by 256 ranks.
SPLITK_EDGES = [250, 251, 253, 256, 301, 333, 479, 480, 481, 495, 508, 509, 510, 511, 512, 513]


@pytest.mark.parametrize("R", SPLITK_EDGES)
@pytest.mark.parametrize("func", [False, True])
def test_expand_splitk_edges(env, orc, R, func):
    test_expand_fuzz(env, orc, 7000 + R, R, (150, 170, 3), 0, 3, 3, 8, func)
    test_expand_fuzz(env, orc, 8000 + R, R, (70, 33, 4), 2, 4, 0, 0, func)


def _lattices(n=40, seed=7):
    rng = np.random.default_rng(seed)
    for c in range(n):
        Lc = tuple(int(x) for x in rng.integers(1, 7, 3))
        if rng.integers(0, 3) == 0:
            Lc = tuple(2 * ((x + 1) // 2) for x in Lc)  # even L: the periodic reference cell is L/2
        nn = int(2 * rng.integers(1, 17))
        M0 = int(rng.integers(1, 4))
        idx = rng.integers(0, nn + 1, (M0, 3))
        Z = rng.uniform(0.5, 4.0, M0)
        periodic = bool(rng.integers(0, 2))
        mode = "erf" if rng.integers(0, 2) else "midpoint"
        M = int(rng.integers(3, 12))
        yield pytest.param(c, Lc, nn, idx, Z, periodic, mode, M, id=f"c{c}-L{Lc}-n{nn}-M0{M0}-{mode}")


# LS_LATTICE_SOAK=N runs N lattices instead of 40 (a longer soak, e.g. after kernel changes)
@pytest.mark.parametrize("case,Lc,nn,idx,Z,periodic,mode,M",
                         list(_lattices(n=int(__import__("os").environ.get("LS_LATTICE_SOAK", "40")))))
def test_lattice_fuzz(env, orc, case, Lc, nn, idx, Z, periodic, mode, M):
    """Random lattices (shape, cells per axis, charges on random vertices, box or periodic, both
    generators): the device pipeline's assembled factors are bit-identical to the oracle's
    assembly of the same master (K2 is bitwise); the master itself is bit-identical to the
    oracle's in both generator modes, and the expanded grid agrees to 1e-13."""
    torch, _abi = env
    import paper_1405_2270_b200 as L
    b = 2.0
    h = b / nn
    spec = L.LatticeSpec(Lc, L.GridSpec(b, nn), [L.Charge(tuple(float(i) * h - b / 2 for i in idx[c]), float(Z[c]))
                                                 for c in range(len(Z))])
    rule = L.sinc_quadrature(1e-4, h, np.sqrt(3.0) * max(Lc) * b, M, 1.0)
    master = L.build_lattice_master(spec, rule, mode=mode)
    res = (L.assembled_periodic_sum if periodic else L.assembled_box_sum)(spec, master)
    import ctypes as Cc
    dp = lambda a: a.ctypes.data_as(Cc.POINTER(Cc.c_double))  # noqa: E731
    R, M0 = rule.node_count(), spec.charge_count()
    for l in range(3):
        ia = np.array([spec.charge_grid_index(l, nu) for nu in range(M0)], dtype=np.int64)
        ol = nn if periodic else spec.L[l] * nn
        want = np.zeros((ol, M0 * R), order="F")
        m = np.asfortranarray(master.factor(l))
        assert orc._assembled_axis(dp(m), R, M0, ia.ctypes.data_as(Cc.POINTER(Cc.c_int64)), nn, spec.L[l],
                                   int(periodic), dp(want)) == 0
        assert np.array_equal(res.tensor.factor(l), want), l
    om = orc.lattice_master(0 if mode == "midpoint" else 1, list(spec.L), nn, b, rule.exponents)
    for l in range(3):
        assert np.array_equal(master.factor(l), om[l]), l  # glibc erf / exp, bit for bit
    # the single-call device path (generate -> assemble -> expand) lands on the same grid
    V, t = L.lattice_potential(spec, rule, mode=mode, periodic=periodic, return_factors=True)
    for l in range(3):
        assert np.array_equal(t.factor(l), res.tensor.factor(l)), l
    f = [np.asfortranarray(res.tensor.factor(l)) for l in range(3)]
    want_grid = orc.densify_slabs(f[0], f[1], f[2], np.ascontiguousarray(res.tensor.weights()))
    assert float(np.max(np.abs(V - want_grid)) / np.max(np.abs(want_grid))) <= 1e-13


@pytest.mark.parametrize("R", [9, 41])
def test_split_tail_schedule(env, orc, R):
    """A store-only TMEM launch whose last round of units is split at stage granularity:
    600 units (2 i-chunks x 300 slabs) of 20 stages on 296 CTAs. Checked against the oracle."""
    torch, _abi = env
    rng = np.random.default_rng(300 + R)
    dims = (256, 1280, 300)
    f = [np.asfortranarray(rng.uniform(0.05, 1.0, (d, R))) for d in dims]
    w = rng.uniform(0.05, 1.0, R)
    dev = torch.device("cuda")
    fac = [torch.as_tensor(x.T.copy(), device=dev) for x in f]
    wd = torch.as_tensor(w, device=dev)
    out = torch.empty((dims[2], dims[1], dims[0]), dtype=torch.float64, device=dev)
    lib = _abi.load()
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.ls_expand(p(fac[0]), dims[0], p(fac[1]), dims[1], p(fac[2]), dims[2], p(wd), *dims, R, 0, dims[2],
                         p(out), 0, 0, None, None, None, None, s) == 0, lib.ls_last_error()
    got = out.cpu().numpy()
    for k in list(range(0, 300, 37)) + [299]:
        want = orc.densify_slabs(f[0], f[1], f[2], w, k, k + 1)[:, :, 0]
        assert float(np.max(np.abs(got[k].T - want)) / np.max(np.abs(want))) <= 1e-13, k


@pytest.mark.parametrize("R", [1, 4, 5])
def test_single_kstep_ranks_multi_unit(env, orc, R):
    """Ranks with one DMMA k-step (KD = 1) on a grid where every CTA runs many units: the warps
    without a fill share must still hand the next A1k buffer over (regression: a hang)."""
    torch, _abi = env
    rng = np.random.default_rng(500 + R)
    dims = (1024, 64, 1200)  # 8 i-chunks x 1200 slabs = 9600 units of one stage
    f = [np.asfortranarray(rng.uniform(0.05, 1.0, (d, R))) for d in dims]
    w = rng.uniform(0.05, 1.0, R)
    dev = torch.device("cuda")
    fac = [torch.as_tensor(x.T.copy(), device=dev) for x in f]
    wd = torch.as_tensor(w, device=dev)
    out = torch.empty((dims[2], dims[1], dims[0]), dtype=torch.float64, device=dev)
    lib = _abi.load()
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.ls_expand(p(fac[0]), dims[0], p(fac[1]), dims[1], p(fac[2]), dims[2], p(wd), *dims, R, 0, dims[2],
                         p(out), 0, 0, None, None, None, None, s) == 0, lib.ls_last_error()
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    for k in (0, 599, 1199):
        want = orc.densify_slabs(f[0], f[1], f[2], w, k, k + 1)[:, :, 0]
        assert float(np.max(np.abs(got[k].T - want)) / np.max(np.abs(want))) <= 1e-13, k


@pytest.mark.parametrize("n_charges", [1, 3, 8])
def test_pipeline_bitwise_run_to_run(env, n_charges):
    """generator, assembly and expansion are deterministic. Two device-pipeline
    steps give the same grid bit for bit, and two fused energies the same double. Ranks 41, 123
    and 328 take the 8-warp TMEM, shared-memory and split-K plans."""
    torch, _abi = env
    import paper_1405_2270_b200 as L
    rng = np.random.default_rng(40 + n_charges)
    b, nn = 10.0, 32
    h = b / nn
    idx = rng.integers(3, nn - 3, (n_charges, 3))
    spec = L.LatticeSpec((8, 8, 4), L.GridSpec(b, nn), [L.Charge(tuple(float(i) * h - b / 2 for i in idx[c]),
                                                                 float(c + 1)) for c in range(n_charges)])
    rule = L.sinc_quadrature(1e-6, h, np.sqrt(3.0) * 8 * b, 20, 1.0)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    N = spec.target_dims()
    a = torch.full((N[2], N[1], N[0]), float("nan"), dtype=torch.float64, device="cuda")
    c = torch.full_like(a, float("nan"))
    pipe.step(a)
    pipe.step(c)
    rho = [torch.as_tensor(np.exp(-((np.arange(N[l]) + 0.5 - N[l] / 2) * h) ** 2 / 2), device="cuda")
           for l in range(3)]
    e1 = pipe.grid_functional(rho).item()
    e2 = pipe.grid_functional(rho).item()
    torch.cuda.synchronize()
    assert not torch.isnan(a).any()
    assert torch.equal(a, c)
    assert e1 == e2


@pytest.mark.parametrize("R,dims,plan", [
    (122, (256, 200, 300), "single A1k buffer"), (164, (300, 256, 200), "single A1k buffer"),
    (199, (256, 130, 260), "single A1k buffer"), (249, (128, 256, 300), "single A1k buffer"),
    (5, (256, 256, 300), None), (21, (200, 256, 300), None), (54, (256, 128, 300), None),
    (57, (256, 250, 300), None), (41, (256, 512, 200), None), (57, (200, 384, 160), None),
    (9, (136, 500, 150), None)])
def test_expand_many_units_per_cta(env, orc, R, dims, plan):
    """Launches with several units per CTA: the single-buffer TMEM plan's unit-boundary refill
    (ranks 122-249) and the A2-in-TMEM plan's ring reuse and next-unit scaling (N2 <= 512, 256 or 512 TMEM columns), which
    the small fuzz shapes above never reach. Sampled slabs (first, last, in between) against the
    oracle, and the fused functional against the stored grid."""
    torch, _abi = env
    import paper_1405_2270_b200 as L
    if plan:
        assert plan in L.expansion_plan(R)
    rng = np.random.default_rng(R)
    n1, n2, n3 = dims
    f = [np.asfortranarray(rng.uniform(0.05, 1.0, (d, R))) for d in dims]
    w = rng.uniform(0.05, 1.0, R)
    dev = torch.device("cuda")
    fac = [torch.as_tensor(x.T.copy(), device=dev) for x in f]
    wd = torch.as_tensor(w, device=dev)
    from paper_1405_2270_b200.latsum import _expand_device
    out = torch.empty((n3, n2, n1), dtype=torch.float64, device=dev)
    _expand_device(fac, wd, dims, 0, n3, out)
    torch.cuda.synchronize()
    for k in (0, 1, n3 // 3, n3 // 2 + 1, n3 - 2, n3 - 1):
        want = orc.densify_slabs(f[0], f[1], f[2], w, k, k + 1)[:, :, 0]
        got = out[k].cpu().numpy().T
        assert np.max(np.abs(got - want)) <= 1e-13 * np.max(np.abs(want)), k
    # fused functional (ls_expand with rho, partials, fixed-order sum) against the stored grid
    rho = [torch.as_tensor(rng.uniform(0.1, 1.0, d), device=dev) for d in dims]
    np_ = int(_abi.load().ls_expand_partial_count(n1, n2, R, 0, n3))
    part = torch.zeros(max(np_, 1), dtype=torch.float64, device=dev)
    e = torch.zeros(1, dtype=torch.float64, device=dev)
    lib = _abi.load()
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.ls_expand(p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(wd), n1, n2, n3, R, 0, n3, None, 0, 0,
                         p(rho[0]), p(rho[1]), p(rho[2]), p(part), s) == 0
    assert lib.ls_sum_partials(p(part), np_, p(e), s) == 0
    e_stored = float(torch.einsum("kji,i,j,k->", out, rho[0], rho[1], rho[2]))
    assert abs(float(e.cpu()) - e_stored) <= 1e-12 * abs(e_stored)
