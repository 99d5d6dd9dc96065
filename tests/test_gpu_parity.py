"""GPU parity: the CUDA path (through liblatsum_cuda.so's C ABI) against the CPU
oracles on the same inputs, the committed golden vectors from the reference's
own code, and size-independent properties at the BASELINE sizes.

Tolerances (BASELINE.json north_star):
  * generator masters, both modes: BITWISE. The device evaluates glibc 2.39's own erf and
    exp algorithms operation for operation (csrc/glibc_math.cuh), so every column equals
    the reference's std::erf / std::exp column bit for bit, at every config (cfg0-cfg4);
  * assembled canonical vectors: bitwise (ascending-k adds, no FMA, on a bitwise master),
    which is stricter than north_star's 1e-13;
  * full-grid values and functionals: 1e-12 relative max-norm.
"""
import math

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu



@pytest.fixture(scope="module")
def L():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1405_2270_b200 as L
    return L


def cfg(L, Lc, n=64, b=10.0, charges=((0.0, 0.0, 0.0, 1.0),), M=20, L_rule=None):
    spec = L.LatticeSpec(tuple(Lc) if isinstance(Lc, (tuple, list)) else (Lc,) * 3, L.GridSpec(b, n),
                         [L.Charge(tuple(c[:3]), c[3]) for c in charges])
    Lmax = L_rule or max(spec.L)
    rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3.0) * Lmax * b, M, 1.0)
    return spec, rule


def oracle_assembled(orc, spec, rule, mode, periodic):
    import ctypes as C
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    m = orc.lattice_master(0 if mode == "midpoint" else 1, list(spec.L), spec.unit.n, spec.unit.b, rule.exponents)
    R, M0, n = rule.node_count(), spec.charge_count(), spec.unit.n
    out = []
    for l in range(3):
        ia = np.array([spec.charge_grid_index(l, nu) for nu in range(M0)], dtype=np.int64)
        ol = n if periodic else spec.L[l] * n
        o = np.zeros((ol, M0 * R), order="F")
        assert orc._assembled_axis(dp(m[l]), R, M0, ia.ctypes.data_as(C.POINTER(C.c_int64)), n, spec.L[l],
                                   int(periodic), dp(o)) == 0
        out.append(o)
    w = np.array([c.Z * wq for c in spec.charges for wq in rule.weights])
    return m, out, w


# ------------------------------------------------------------------ K1 generator
# (L, n): cfg0-cfg3 masters (n = 64, L = 4/16/32) and the cfg4 periodic masters (n = 256,
# L = 64/128/256: 32768-131072 entries per column).
MASTER_CASES = [(4, 64), (16, 64), (32, 64), (64, 256), (128, 256), (256, 256)]


@pytest.mark.parametrize("Lc,n", MASTER_CASES)
@pytest.mark.parametrize("mode", ["midpoint", "erf"])
def test_master_bitwise_equals_oracle(L, orc, Lc, n, mode):
    spec, rule = cfg(L, Lc, n=n)
    m = L.build_lattice_master(spec, rule, mode)
    o = orc.lattice_master(0 if mode == "midpoint" else 1, list(spec.L), n, 10.0, rule.exponents)
    for l in range(3):
        f = m.factor(l)
        bad = np.flatnonzero((f != o[l]).any(axis=0))
        assert bad.size == 0, f"{mode} L={Lc} n={n} axis {l}: columns {bad[:8]} differ"
        assert np.array_equal(f, f[::-1])  # exact evenness (test_newton.cpp:71-77, :93)


def test_master_matches_golden_bitwise(L, golden):
    spec, _ = cfg(L, 4)
    rule = L.QuadratureRule(20, 1.0, 0.0, None, golden["cfg0_tau"], golden["cfg0_w"])
    assert np.array_equal(L.build_lattice_master(spec, rule, "midpoint").factor(0), golden["cfg0_master_mid"])
    assert np.array_equal(L.build_lattice_master(spec, rule, "erf").factor(0), golden["cfg0_master_erf"])


def _libm_sweep_args(rng, n):
    """Arguments over every branch of erf and exp, plus raw bit patterns."""
    u = lambda lo, hi: rng.uniform(lo, hi, n)  # noqa: E731
    sgn = lambda a: np.where(rng.integers(0, 2, a.size) == 1, -a, a)  # noqa: E731
    parts = [
        rng.integers(0, 2**64, n, dtype=np.uint64).view(np.float64),
        sgn(np.ldexp(u(1.0, 2.0), -29 - rng.integers(0, 1000, n))),
        sgn(u(2.0**-28, 0.84375)), sgn(u(0.84375, 1.25)), sgn(u(1.25, 1 / 0.35)),
        sgn(u(1 / 0.35, 6.0)), sgn(u(6.0, 8.0)), sgn(np.exp(u(-690.0, 6.9))),
        u(-746.0, -707.0), u(-1100.0, 710.0), u(-40.0, 0.0),
        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.0**-1022, 1e308, -1e308]),
    ]
    return np.concatenate(parts)


def test_device_libm_bitwise_equals_host_libm(L, orc):
    """ls_libm_eval (device erf / exp) against the host libm over ~3.3M arguments covering every
    branch, including subnormal exp results, erf's tiny-argument path, +-inf and NaN."""
    import torch
    lib = L._abi.load()
    x = _libm_sweep_args(np.random.default_rng(1405), 300_000)
    xd = torch.as_tensor(x, device="cuda")
    for fn in (0, 1):
        yd = torch.empty_like(xd)
        assert lib.ls_libm_eval(fn, xd.data_ptr(), yd.data_ptr(), xd.numel(), None) == 0
        torch.cuda.synchronize()
        got, want = yd.cpu().numpy(), orc.libm_eval(fn, x)
        same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
        assert same.all(), f"fn {fn}: {np.count_nonzero(~same)} mismatches, first x={x[~same][:4]}"


def test_generator_kats(L):  # test_newton.cpp:32-52, 71-96
    v = L.gaussian_moment_vector(L.GridSpec(4.0, 8), 0.0, False)
    assert np.all(v == 0.5)
    v = L.gaussian_moment_vector(L.GridSpec(2.0, 2), 1.0, False)
    want = 0.5 * math.sqrt(math.pi) * math.erf(1.0)
    assert abs(v[0] - want) <= 1e-15 and abs(v[1] - want) <= 1e-15
    for t in (0.3, 1.0, 4.5):
        v = L.gaussian_moment_vector(L.GridSpec(5.0, 10), t, False)
        assert np.array_equal(v, v[::-1])
    s = L.gaussian_sample_vector(6, 0.5, 1.3)
    for i in range(6):
        x = (i + 0.5 - 3.0) * 0.5
        assert s[i] == pytest.approx(math.exp(-1.3 * 1.3 * x * x), rel=4e-16)
    with pytest.raises(L.ValidationError):
        L.gaussian_sample_vector(5, 0.5, 1.3)
    with pytest.raises(L.ValidationError):
        L.gaussian_moment_vector(L.GridSpec(2.0, 4), -1.0, False)


# ------------------------------------------------------------------- K2 assembly
@pytest.mark.parametrize("periodic", [False, True])
def test_assembly_bitwise_on_oracle_master(L, orc, periodic):
    cases = [((4, 4, 4), 64, [(0, 0, 0, 1.0)]),
             ((3, 2, 5), 8, [(0, 0, 0, 1.0), (0.5, -0.25, 0.25, 2.0), (-0.75, 0.5, 0.0, 0.5)]),
             ((16, 16, 16), 64, [(0, 0, 0, 1.0)]),
             ((9, 1, 2), 16, [(1.0, -1.0, 0.25, 3.0)])]
    for Lc, n, charges in cases:
        b = 10.0 if n == 64 else 2.0
        spec, rule = cfg(L, Lc, n=n, b=b, charges=charges, M=10)
        m, want, w = oracle_assembled(orc, spec, rule, "midpoint", periodic)
        master = L.CanonicalTensor3(m, rule.weights, trusted=True)
        got = (L.assembled_periodic_sum if periodic else L.assembled_box_sum)(spec, master)
        for l in range(3):
            assert np.array_equal(got.tensor.factor(l), want[l]), (Lc, l)
        assert np.array_equal(got.tensor.weights(), w)
        assert got.rank == spec.charge_count() * rule.node_count()


@pytest.mark.parametrize("Lc,n,M0,periodic", [(32, 64, 8, False), (32, 64, 8, True), (13, 64, 8, False),
                                              (21, 16, 3, False), (256, 256, 1, True), (9, 8, 8, False)])
def test_assembly_bitwise_at_config_scale(L, orc, Lc, n, M0, periodic):
    """K2 at the BASELINE scales (cfg3: L = 32 with 8 charges; cfg4: periodic L = 256, n = 256)
    and at L not a multiple of the box kernel's 8-shift blocks: bit-identical to the oracle's
    ascending-k adds on the same master."""
    rng = np.random.default_rng(100 + Lc + M0)
    b = 10.0
    h = b / n
    ia = rng.integers(0, n + 1, size=(M0, 3))
    charges = [(*(ia[c] * h - b / 2), float(c + 1)) for c in range(M0)]
    spec, rule = cfg(L, Lc, n=n, b=b, charges=charges, M=20)
    m, want, w = oracle_assembled(orc, spec, rule, "midpoint", periodic)
    master = L.CanonicalTensor3(m, rule.weights, trusted=True)
    got = (L.assembled_periodic_sum if periodic else L.assembled_box_sum)(spec, master)
    for l in range(3):
        assert np.array_equal(got.tensor.factor(l), want[l]), l
    assert np.array_equal(got.tensor.weights(), w)


FUSED_CASES = [  # (L, n, charges, periodic, mode): the fused generator + assembly launch and its fallback
    ((4, 4, 4), 64, [(0, 0, 0, 1.0)], False, "erf"),                                 # cfg0
    ((16, 16, 16), 64, [(0, 0, 0, 1.0)], False, "erf"),                              # cfg1
    ((16, 16, 16), 64, [(0, 0, 0, 1.0)], False, "midpoint"),
    ((3, 2, 5), 8, [(0, 0, 0, 1.0), (0.5, -0.25, 0.25, 2.0), (-0.75, 0.5, 0.0, 0.5)], False, "erf"),
    ((3, 2, 5), 8, [(0, 0, 0, 1.0), (0.5, -0.25, 0.25, 2.0), (-0.75, 0.5, 0.0, 0.5)], True, "midpoint"),
    ((1, 1, 1), 16, [(0.25, 0.0, -0.5, 1.0)], False, "erf"),                          # L = 1: no adds
    ((9, 1, 2), 16, [(1.0, -1.0, 0.25, 3.0)], True, "erf"),
    ((32, 32, 32), 64, "cfg3", False, "erf"),                                         # 8 charges x 2048
    ((32, 32, 32), 64, "cfg3", True, "erf"),
    ((64, 64, 64), 256, [(0, 0, 0, 1.0)], True, "erf"),         # periodic, one charge, L >= 32: master never written
    ((32, 48, 40), 64, [(1.25, -0.3125, 2.5, 1.5)], True, "erf"),
    ((32, 32, 32), 64, [(0.46875, 0.0, -1.5625, 1.0)], True, "midpoint"),
    ((40, 3, 36), 16, [(0.0, 0.0, 0.0, 1.0)], True, "erf"),    # one short axis: the per-block kernels
]


@pytest.mark.parametrize("case", FUSED_CASES, ids=[f"{c[0][0]}x{c[0][1]}x{c[0][2]}-n{c[1]}-{'p' if c[3] else 'b'}-{c[4]}"
                                                   for c in FUSED_CASES])
def test_prepare_fused_generator_assembly_bitwise(L, orc, case):
    """ls_pipeline_prepare (generator + assembled sum in one launch where the master column fits
    shared memory) gives factors bit-identical to the oracle's ascending-k assembly of the
    reference master and to the two-launch generate() + assemble() path."""
    import torch
    Lc, n, charges, periodic, mode = case
    b = 10.0 if n >= 64 else 2.0
    if charges == "cfg3":
        rng = np.random.default_rng(20241019)
        ia = rng.integers(7, 58, size=(8, 3))
        charges = [(*(ia[c] * (b / n) - b / 2), float(c + 1)) for c in range(8)]
    spec, rule = cfg(L, Lc, n=n, b=b, charges=charges, M=20 if n >= 64 else 10)
    _, want, w = oracle_assembled(orc, spec, rule, mode, periodic)
    pipe = L.DevicePipeline(spec, rule, mode=mode, periodic=periodic)
    pipe.prepare()
    torch.cuda.synchronize()
    fused = [pipe.factor(l).cpu().numpy().T.copy() for l in range(3)]
    pipe.generate()
    pipe.assemble()
    torch.cuda.synchronize()
    split = [pipe.factor(l).cpu().numpy().T.copy() for l in range(3)]
    # assemble() right after a prepare() that may have left the master unwritten (periodic fused
    # path) rebuilds the master first
    pipe2 = L.DevicePipeline(spec, rule, mode=mode, periodic=periodic)
    pipe2.prepare()
    pipe2.assemble()
    torch.cuda.synchronize()
    again = [pipe2.factor(l).cpu().numpy().T.copy() for l in range(3)]
    for l in range(3):
        assert np.array_equal(fused[l], want[l]), ("fused vs oracle", l)
        assert np.array_equal(split[l], want[l]), ("two launches vs oracle", l)
        assert np.array_equal(again[l], want[l]), ("assemble after prepare", l)


def test_assembly_matches_golden_bitwise(L, golden):
    g = golden
    ch = g["mc_charges"]
    spec = L.LatticeSpec(tuple(int(x) for x in g["mc_L"]), L.GridSpec(2.0, 8), [L.Charge(tuple(c[:3]), c[3]) for c in ch])
    master = L.CanonicalTensor3([g[f"mc_master_{l}"] for l in range(3)], g["mc_w"], trusted=True)
    box = L.assembled_box_sum(spec, master)
    per = L.assembled_periodic_sum(spec, master)
    for l in range(3):
        assert np.array_equal(box.tensor.factor(l), g[f"mc_box_{l}"])
        assert np.array_equal(per.tensor.factor(l), g[f"mc_per_{l}"])
    assert np.array_equal(box.tensor.weights(), g["mc_box_w"])
    assert rel(L.densify(box.tensor), g["mc_box_dense"]) <= 1e-13
    assert rel(L.densify(per.tensor), g["mc_per_dense"]) <= 1e-13


def test_assembled_single_cell_restrictions(L):  # test_lattice.cpp:205-216, 255-264
    spec, rule = cfg(L, 1, n=16, b=2.0, M=8)
    master = L.build_lattice_master(spec, rule)
    box = L.assembled_box_sum(spec, master)
    per = L.assembled_periodic_sum(spec, master)
    for l in range(3):
        assert np.array_equal(box.tensor.factor(l), master.factor(l)[8:24])
        assert np.array_equal(per.tensor.factor(l), box.tensor.factor(l))
    assert box.grid_dims == (16, 16, 16)


def test_assembly_rejects_mismatched_master(L):  # test_lattice.cpp:196-203
    spec, rule = cfg(L, (2, 1, 1), n=8, b=2.0, M=8)
    wrong = L.CanonicalTensor3([np.ones((16, rule.node_count()))] * 3, rule.weights)
    with pytest.raises(L.ValidationError):
        L.assembled_box_sum(spec, wrong)


# ----------------------------------------------------------------- K3 expansion
@pytest.mark.parametrize("dims,R", [((5, 7, 3), 3), ((33, 17, 9), 41), ((130, 66, 4), 45), ((64, 64, 4), 328),
                                    ((2, 2, 2), 1), ((257, 129, 3), 8), ((4, 5, 6), 2), ((200, 3, 2), 43),
                                    ((1, 9, 2), 5), ((130, 66, 4), 61), ((257, 129, 3), 82), ((64, 200, 5), 73),
                                    ((70, 33, 3), 42), ((129, 64, 2), 90), ((100, 70, 3), 40), ((33, 129, 4), 44)])
def test_expansion_matches_oracle_random(L, orc, dims, R):  # test_canonical.cpp:63-69
    rng = np.random.default_rng(R * 1000 + dims[0])
    f = [np.asfortranarray(rng.uniform(-1, 1, (d, R))) for d in dims]
    w = rng.uniform(-1, 1, R)
    t = L.CanonicalTensor3(f, w)
    V = L.densify(t)
    Vo = orc.densify_slabs(f[0], f[1], f[2], w)
    assert rel(V, Vo) <= 1e-13
    # slab sub-ranges land on the same values
    if dims[2] > 1:
        part = L.expand_slabs(t, 1, dims[2])
        assert np.array_equal(part, V[:, :, 1:])


def test_expansion_edge_cases(L):
    zero = L.CanonicalTensor3([np.zeros((3, 0)), np.zeros((4, 0)), np.zeros((5, 0))], np.zeros(0))
    assert np.all(L.densify(zero) == 0.0)  # rank 0 is the zero tensor (canonical.hpp:243)
    ones = L.CanonicalTensor3([np.ones((2, 1))] * 3, np.ones(1))
    assert np.all(L.densify(ones) == 1.0)
    empty = L.expand_slabs(ones, 1, 1)
    assert empty.shape == (2, 2, 0)
    with pytest.raises(L.ValidationError):
        L.expand_slabs(ones, 1, 3)
    with pytest.raises(L.ResourceGuardError):
        L.densify(L.CanonicalTensor3([np.ones((8, 1))] * 3, np.ones(1)), guard=100)


def test_cfg0_full_grid_matches_oracle(L, orc, golden):
    spec, rule = cfg(L, 4)
    for mode in ("midpoint", "erf"):
        V, t = L.lattice_potential(spec, rule, mode=mode, return_factors=True)
        _, fo, wo = oracle_assembled(orc, spec, rule, mode, False)
        for l in range(3):
            assert np.array_equal(t.factor(l), fo[l])
        # full grid against the oracle expansion of the oracle's own assembled vectors
        Vo = orc.densify_slabs(fo[0], fo[1], fo[2], wo)
        assert rel(V, Vo) <= 1e-12
        key = "mid" if mode == "midpoint" else "erf"
        for s, k in enumerate(golden["cfg0_slab_ids"]):
            assert rel(V[:, :, int(k)], golden[f"cfg0_slabs_{key}"][:, :, s]) <= 1e-12
        pts = golden["cfg0_point_idx"]
        assert rel(np.array([V[tuple(p)] for p in pts]), golden[f"cfg0_points_{key}"]) <= 1e-12
        assert rel(L.eval_points(t, pts), golden[f"cfg0_points_{key}"]) <= 1e-12


def test_cfg1_sampled_slabs_match_oracle(L, orc):
    import torch
    spec, rule = cfg(L, 16)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    N = spec.target_dims()
    out = torch.empty((N[2], N[1], N[0]), dtype=torch.float64, device="cuda")
    pipe.step(out)
    torch.cuda.synchronize()
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", False)
    for l in range(3):
        assert np.array_equal(pipe.factor(l).T.cpu().numpy(), fo[l])
    for k in (0, 511, 1023):
        got = out[k].cpu().numpy().T
        want = orc.densify_slabs(fo[0], fo[1], fo[2], wo, k, k + 1)[:, :, 0]
        assert rel(got, want) <= 1e-12
    # size-independent checks over the whole 1024^3 grid: mirror and transposition symmetry of
    # the cubic centred lattice (to rounding: the ascending-k sums are not mirror-ordered) and
    # positivity.
    v = out[::97]
    assert bool(torch.all(v > 0))
    scale = float(v.abs().max())
    assert float((v - torch.flip(v, dims=[2])).abs().max()) <= 1e-13 * scale
    assert float((out[100] - out[100].T).abs().max()) <= 1e-13 * scale
    # every slab, including the last round's units that the store-only schedule splits at stage
    # granularity: z-mirror symmetry of the whole grid, chunk by chunk
    for k0 in range(0, N[2] // 2, 128):
        lo = out[k0:k0 + 128]
        hi = torch.flip(out[N[2] - k0 - 128:N[2] - k0], dims=[0])
        assert float((lo - hi).abs().max()) <= 1e-13 * scale, k0


def test_cfg2_functional_and_slabs(L, orc):
    """2048^3 (64 GiB) is not stored: sampled slabs through the device pipeline, and the fused
    full-grid energy <V, rho> against the 1D rank-term form (canonical.hpp:126-136)."""
    import torch
    spec, rule = cfg(L, 32)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    pipe.generate()
    pipe.assemble()
    N = spec.target_dims()
    out = torch.empty((2, N[1], N[0]), dtype=torch.float64, device="cuda")
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", False)
    for k in (0, 1024):
        pipe.expand(out, k, k + 2)
        torch.cuda.synchronize()
        want = orc.densify_slabs(fo[0], fo[1], fo[2], wo, k, k + 2)
        assert rel(out.cpu().numpy().transpose(2, 1, 0), want) <= 1e-12
    # separable Gaussian density, centre = box centre, sigma = 1 bohr (recorded choice)
    h = spec.unit.h
    x = (np.arange(N[0]) + 0.5 - N[0] / 2) * h
    r1 = np.exp(-x * x / 2.0)
    rho = [torch.as_tensor(r1, device="cuda")] * 3
    e_grid = float(pipe.grid_functional(rho).cpu())
    e_grid2 = float(pipe.grid_functional(rho).cpu())
    assert e_grid == e_grid2  # deterministic reduction
    r = np.asfortranarray(r1.reshape(-1, 1))
    e_1d = orc.scalar_product(fo, wo, [r, r, r], np.ones(1))
    assert abs(e_grid - e_1d) <= 1e-12 * abs(e_1d)
    e_batch = L.functional_batch(L.CanonicalTensor3(fo, wo, trusted=True), [r, r, r])[0]
    assert abs(e_batch - e_1d) <= 1e-12 * abs(e_1d)


def test_cfg2_whole_grid_one_gpu(L, orc):
    """The whole 2048^3 grid (8.6e9 points, 64 GiB) in one device buffer: element offsets pass
    2^32, so any 32-bit index in the store path would land in the wrong slab or fault. The last
    slabs are checked against the oracle, the grid against its z-mirror, and the fused energy of
    the stored grid against the streamed functional."""
    import torch
    free, _ = torch.cuda.mem_get_info()
    if free < 72 * 2**30:
        pytest.skip("needs 72 GiB of free HBM")
    spec, rule = cfg(L, 32)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    N = spec.target_dims()
    out = torch.empty((N[2], N[1], N[0]), dtype=torch.float64, device="cuda")
    pipe.step(out)
    torch.cuda.synchronize()
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", False)
    for k in (N[2] - 1, N[2] // 2 + 3):
        want = orc.densify_slabs(fo[0], fo[1], fo[2], wo, k, k + 1)[:, :, 0]
        assert rel(out[k].cpu().numpy().T, want) <= 1e-12, k
    scale = float(out[N[2] // 2].abs().max())
    for k0 in range(0, N[2] // 2, 128):
        lo = out[k0:k0 + 128]
        hi = torch.flip(out[N[2] - k0 - 128:N[2] - k0], dims=[0])
        assert float((lo - hi).abs().max()) <= 1e-13 * scale, k0
    h = spec.unit.h
    x = (np.arange(N[0]) + 0.5 - N[0] / 2) * h
    r1 = torch.as_tensor(np.exp(-x * x / 2.0), device="cuda")
    e_stored = float(torch.einsum("kji,i->kj", out, r1).mul_(r1).sum(dim=1).dot(r1))
    e_fused = float(pipe.grid_functional([r1] * 3).cpu())
    assert abs(e_stored - e_fused) <= 1e-12 * abs(e_fused)


def test_cfg3_multi_atom_rank_328(L, orc):
    import torch
    rng = np.random.default_rng(20241019)
    n, b = 64, 10.0
    h = b / n
    ia = rng.integers(7, 58, size=(8, 3))       # snapped to vertices in [0.1 n, 0.9 n]
    Z = rng.integers(1, 9, size=8).astype(float)
    charges = [(*(ia[c] * h - b / 2), Z[c]) for c in range(8)]
    spec, rule = cfg(L, 32, charges=charges)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    assert pipe.Rt == 328
    pipe.generate()
    pipe.assemble()
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", False)
    for l in range(3):
        assert np.array_equal(pipe.factor(l).T.cpu().numpy(), fo[l])
    N = spec.target_dims()
    out = torch.empty((1, N[1], N[0]), dtype=torch.float64, device="cuda")
    k = 777
    pipe.expand(out, k, k + 1)
    torch.cuda.synchronize()
    want = orc.densify_slabs(fo[0], fo[1], fo[2], wo, k, k + 1)
    assert rel(out[0].cpu().numpy().T, want[:, :, 0]) <= 1e-12


@pytest.mark.parametrize("Lc", [64, 128, 256])
def test_cfg4_periodic_and_functional_batch(L, orc, Lc):
    import torch
    spec, rule = cfg(L, Lc, n=256)
    V, t = L.lattice_potential(spec, rule, mode="erf", periodic=True, k0=0, k1=4, return_factors=True)
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", True)
    for l in range(3):
        assert np.array_equal(t.factor(l), fo[l])
    want = orc.densify_slabs(fo[0], fo[1], fo[2], wo, 0, 4)
    assert rel(V, want) <= 1e-12
    # batch of 1024 separable Gaussian test functions (alpha log-uniform in [0.1, 10])
    rng = np.random.default_rng(4)
    F = 1024
    alpha = 10 ** rng.uniform(-1, 1, F)
    sigma = 1 / np.sqrt(2 * alpha)
    centres = rng.uniform(-5.0, 5.0, (F, 3))
    mids = (np.arange(256) + 0.5 - 128) * spec.unit.h
    G = [np.asfortranarray(np.exp(-(mids[:, None] - centres[None, :, l]) ** 2 / (2 * sigma ** 2))) for l in range(3)]
    got = L.functional_batch(t, G)
    P = L.CanonicalTensor3(fo, wo, trusted=True)
    for f in rng.integers(0, F, 16):
        want = orc.scalar_product(fo, wo, [np.asfortranarray(G[l][:, [f]]) for l in range(3)], np.ones(1))
        assert abs(got[f] - want) <= 1e-12 * abs(want)
    del P


@pytest.mark.parametrize("dims,R,F", [((5, 7, 3), 3, 5), ((33, 17, 9), 41, 70), ((130, 66, 4), 6, 129),
                                      ((64, 64, 64), 41, 64), ((1, 1, 1), 1, 1), ((200, 3, 2), 2, 200)])
def test_grid_functional_batch_random(L, orc, dims, R, F):
    """Full-grid functional batch (fused DMMA GEMM) vs the dense grid contracted on the host.
    Odd N1 takes the 8-byte copy path; F and N2*N3 not multiples of the 64 x 128 tiles."""
    rng = np.random.default_rng(7 * R + F)
    f = [np.asfortranarray(rng.uniform(-1, 1, (d, R))) for d in dims]
    w = rng.uniform(-1, 1, R)
    t = L.CanonicalTensor3(f, w)
    V = orc.densify_slabs(f[0], f[1], f[2], w)
    G = [np.asfortranarray(rng.uniform(-1, 1, (d, F))) for d in dims]
    got = L.grid_functional_batch(t, G, scale=0.5)
    want = 0.5 * np.einsum("ijk,if,jf,kf->f", V, *G)
    mag = 0.5 * np.einsum("ijk,if,jf,kf->f", np.abs(V), *[np.abs(g) for g in G])
    assert np.all(np.abs(got - want) <= 1e-13 * mag + 1e-300)
    # slab-chunked evaluation (accumulating launches) agrees to rounding
    chunked = L.grid_functional_batch(t, G, scale=0.5, max_chunk_points=dims[0] * dims[1])
    assert np.all(np.abs(chunked - want) <= 1e-13 * mag + 1e-300)


@pytest.mark.parametrize("pad_y,pad_z", [(0, 0), (2, 0), (2, 6), (0, 2)])
def test_grid_functional_batch_strides(pad_y, pad_z):
    """ls_grid_functional_batch on a padded device grid: one row stride (pad_z = 0) takes the
    tensor-map feed, whose row stride is then ldy, not N1; padded slabs take the cp.async feed.
    N1 = 50 is not a multiple of the 16-wide K chunk (the TMA box's tail arrives as zeros)."""
    import ctypes as C
    import torch
    from paper_1405_2270_b200 import _abi
    rng = np.random.default_rng(11 + pad_y + 10 * pad_z)
    N1, N2, N3, F = 50, 37, 9, 77
    V = rng.uniform(-1, 1, (N1, N2, N3))
    G = [rng.uniform(-1, 1, (d, F)) for d in (N1, N2, N3)]
    ldy = N1 + pad_y
    ldz = ldy * N2 + pad_z
    buf = np.full(N3 * ldz, np.nan)
    for k in range(N3):
        for j in range(N2):
            buf[k * ldz + j * ldy: k * ldz + j * ldy + N1] = V[:, j, k]
    dev = torch.device("cuda")
    Vd = torch.as_tensor(buf, device=dev)
    Gd = [torch.as_tensor(np.asfortranarray(g).T.copy(), device=dev) for g in G]  # column f at f * ld
    out = torch.zeros(F, dtype=torch.float64, device=dev)
    lib = _abi.load()
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert lib.ls_grid_functional_batch(p(Vd), N1, N2, N3, ldy, ldz, p(Gd[0]), N1, p(Gd[1]), N2, p(Gd[2]), N3, F,
                                        C.c_double(1.0), 0, p(out), s) == 0, lib.ls_last_error()
    got = out.cpu().numpy()
    want = np.einsum("ijk,if,jf,kf->f", V, *G)
    mag = np.einsum("ijk,if,jf,kf->f", np.abs(V), *[np.abs(g) for g in G])
    assert np.all(np.abs(got - want) <= 1e-13 * mag)


def test_cfg4_grid_functional_batch_matches_1d_form(L):
    """cfg4: 1024 separable Gaussian test functions over the whole 256^3 periodic potential,
    full-grid form (expansion + fused GEMM) vs the 1D rank-term form (scalar_product)."""
    import torch
    spec, rule = cfg(L, 64, n=256)
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=True)
    pipe.generate()
    pipe.assemble()
    rng = np.random.default_rng(11)
    F = 1024
    alpha = 10 ** rng.uniform(-1, 1, F)
    sigma = 1 / np.sqrt(2 * alpha)
    centres = rng.uniform(-5.0, 5.0, (F, 3))
    mids = (np.arange(256) + 0.5 - 128) * spec.unit.h
    G = [torch.as_tensor(np.exp(-(mids[:, None] - centres[None, :, l]) ** 2 / (2 * sigma ** 2)), device="cuda")
         for l in range(3)]
    full = pipe.grid_functional_batch(G).cpu().numpy()
    one_d = L.DevicePipeline.functional_batch_device([pipe.factor(l).T for l in range(3)], pipe.w, G).cpu().numpy()
    assert np.max(np.abs(full - one_d) / np.abs(one_d)) <= 1e-12
    again = pipe.grid_functional_batch(G).cpu().numpy()
    assert np.array_equal(full, again)  # fixed-order reductions: bitwise run to run


@pytest.mark.parametrize("charges,periodic", [
    (((0.0, 0.0, 0.0, 1.0), (1.25, -0.625, 2.5, 2.0)), False),                       # rank 82: 16-warp TMEM plan
    (((0.0, 0.0, 0.0, 1.0), (1.25, -0.625, 2.5, 2.0), (-2.5, 1.25, 0.3125, 3.0)), True),  # rank 123: smem plan 9
])
def test_fused_energy_matches_1d_form_multi_charge(L, charges, periodic):
    """The fused full-grid <V, rho> (per-warp or per-unit partials, fixed-order sum) against the 1D
    rank-term form, on multi-charge lattices whose ranks take the other expansion plans."""
    import torch
    spec, rule = cfg(L, 4, charges=charges)
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=periodic)
    pipe.generate()
    pipe.assemble()
    N = pipe.dims
    rho = []
    for l in range(3):
        x = (np.arange(N[l]) + 0.5 - N[l] / 2) * spec.unit.h
        rho.append(torch.as_tensor(np.exp(-x * x / (2.0 + l)), device="cuda"))
    e = float(pipe.grid_functional(rho).cpu())
    one_d = L.DevicePipeline.functional_batch_device([pipe.factor(l).T for l in range(3)], pipe.w,
                                                    [r.reshape(-1, 1) for r in rho]).cpu().numpy()[0]
    assert abs(e - one_d) <= 1e-12 * abs(one_d)
    # and the stored grid contracted on the host agrees
    out = torch.empty((N[2], N[1], N[0]), dtype=torch.float64, device="cuda")
    pipe.expand(out)
    V = out.cpu().numpy()
    r = [x.cpu().numpy() for x in rho]
    host = float(np.einsum("kji,i,j,k->", V, r[0], r[1], r[2]))
    assert abs(host - one_d) <= 1e-12 * abs(one_d)


def test_eval_points_and_scalar_product(L, orc):  # test_canonical.cpp:88-139
    rng = np.random.default_rng(9)
    f = [np.asfortranarray(rng.uniform(-1, 1, (d, 3))) for d in (4, 5, 6)]
    w = rng.uniform(-1, 1, 3)
    t = L.CanonicalTensor3(f, w)
    d = orc.densify_slabs(*f, w)
    idx = np.array([[i, j, k] for i in range(4) for j in range(5) for k in range(6)])
    assert np.max(np.abs(L.eval_points(t, idx) - d[idx[:, 0], idx[:, 1], idx[:, 2]])) <= 1e-13
    with pytest.raises(L.ValidationError):
        L.eval_point(t, 4, 0, 0)
    ones = L.CanonicalTensor3([np.ones((2, 1))] * 3, np.ones(1))
    assert L.scalar_product(ones, ones) == 8.0
    for trial in range(10):
        dims = rng.integers(2, 9, 3)
        fa = [np.asfortranarray(rng.uniform(-1, 1, (x, 3))) for x in dims]
        fb = [np.asfortranarray(rng.uniform(-1, 1, (x, 4))) for x in dims]
        wa, wb = rng.uniform(-1, 1, 3), rng.uniform(-1, 1, 4)
        a, b = L.CanonicalTensor3(fa, wa), L.CanonicalTensor3(fb, wb)
        want = float(np.sum(orc.densify_slabs(*fa, wa) * orc.densify_slabs(*fb, wb)))
        got = L.scalar_product(a, b)
        assert abs(got - want) <= 1e-11 * max(1.0, abs(want))
        assert all(L.scalar_product(a, b) == got for _ in range(3))


def test_potential_matrix_via_functional_batch(L, golden):
    """potential_matrix(basis, P, h^3) (project.hpp:65-97) = h^3 <G_k.*G_m, P> from the batched
    kernel, against the reference's matrix (golden)."""
    g = golden
    P = L.CanonicalTensor3([g[f"mc_per_{l}"] for l in range(3)],
                           np.array([c[3] * wq for c in g["mc_charges"] for wq in g["mc_w"]]), trusted=True)
    basis = L.sample_gaussian_basis(L.GridSpec(2.0, 8), [L.GaussianBasisSpec(tuple(c), s)
                                                         for c, s in zip(g["pm_centers"], g["pm_sigmas"])])
    nb = len(basis)
    pairs = [(k, m) for k in range(nb) for m in range(k, nb)]
    cols = [np.asfortranarray(np.stack([basis[k][l] * basis[m][l] for k, m in pairs], axis=1)) for l in range(3)]
    vals = L.functional_batch(P, cols, scale=0.25 ** 3)
    V = np.zeros((nb, nb))
    for (k, m), v in zip(pairs, vals):
        V[k, m] = V[m, k] = v
    assert rel(V, g["pm_V"]) <= 1e-12


def test_determinism_bitwise(L):
    spec, rule = cfg(L, 4)
    a = L.lattice_potential(spec, rule, mode="erf")
    b = L.lattice_potential(spec, rule, mode="erf")
    assert np.array_equal(a, b)


def test_off_grid_charge_rejected(L):
    spec, rule = cfg(L, 2, n=8, b=2.0, charges=((0.1, 0, 0, 1.0),), M=8)
    with pytest.raises(L.ValidationError):
        L.lattice_potential(spec, rule)


# ------------------------------------------------- size-independent properties at BASELINE sizes
def _grid(L, spec, rule, mode="erf", k0=0, k1=None):
    import torch
    pipe = L.DevicePipeline(spec, rule, mode=mode)
    N = pipe.dims
    k1 = N[2] if k1 is None else k1
    out = torch.empty((k1 - k0, N[1], N[0]), dtype=torch.float64, device="cuda")
    pipe.step(out, k0, k1)
    torch.cuda.synchronize()
    return pipe, out


def test_cfg1_charge_scaling_is_exact(L):
    """Z enters only through the weights Z*w_q (lattice.hpp:284-287): doubling Z doubles every grid
    value bit for bit over the full 1024^3 grid."""
    import torch
    spec1, rule = cfg(L, 16)
    spec2, _ = cfg(L, 16, charges=((0.0, 0.0, 0.0, 2.0),))
    _, v1 = _grid(L, spec1, rule)
    _, v2 = _grid(L, spec2, rule)
    assert torch.equal(v2, 2.0 * v1)


def test_cfg1_superposition_of_charges(L):
    """Linearity in the charges (test_lattice.cpp:157-172 at full size): the two-charge potential
    equals the sum of the single-charge potentials to rounding."""
    import torch
    a = (0.0, 0.0, 0.0, 1.0)
    b = (1.25, -2.5, 3.75, 3.0)
    spec_ab, rule = cfg(L, 16, charges=(a, b))
    spec_a, _ = cfg(L, 16, charges=(a,))
    spec_b, _ = cfg(L, 16, charges=(b,))
    _, vab = _grid(L, spec_ab, rule)
    _, va = _grid(L, spec_a, rule)
    va.add_(_grid(L, spec_b, rule)[1])
    scale = float(vab.abs().max())
    assert float((vab - va).abs().max()) <= 1e-13 * scale


def test_cfg1_shards_and_determinism(L):
    """z-slab shards reproduce the single-GPU grid bit for bit, and repeated runs are identical."""
    import torch
    spec, rule = cfg(L, 16)
    pipe, full = _grid(L, spec, rule)
    again = torch.empty_like(full)
    pipe.step(again)
    torch.cuda.synchronize()
    assert torch.equal(full, again)
    from paper_1405_2270_b200.distributed import slab_range
    N3 = pipe.dims[2]
    for world in (2, 3, 8):
        for r in range(world):
            k0, k1 = slab_range(N3, r, world)
            part = torch.empty((k1 - k0, pipe.dims[1], pipe.dims[0]), dtype=torch.float64, device="cuda")
            pipe.expand(part, k0, k1)
            torch.cuda.synchronize()
            assert torch.equal(part, full[k0:k1])
    del again


def test_cfg2_sharded_energy_matches_whole(L):
    """The per-shard fused energies summed (what the NCCL all_reduce does) equal the single-pass
    2048^3 energy to rounding, and both match the 1D rank-term form."""
    import torch
    spec, rule = cfg(L, 32)
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    pipe.generate()
    pipe.assemble()
    N = pipe.dims
    x = (np.arange(N[0]) + 0.5 - N[0] / 2) * spec.unit.h
    r1 = torch.as_tensor(np.exp(-x * x / 8.0), device="cuda")  # sigma = 2 bohr
    rho = [r1, r1, r1]
    whole = float(pipe.grid_functional(rho)[0])
    from paper_1405_2270_b200.distributed import slab_range
    parts = [float(pipe.grid_functional(rho, *slab_range(N[2], r, 8))[0]) for r in range(8)]
    assert abs(sum(parts) - whole) <= 1e-13 * abs(whole)
    X = [r1.reshape(-1, 1)] * 3
    one_d = float(L.DevicePipeline.functional_batch_device([pipe.factor(l).T for l in range(3)], pipe.w, X)[0])
    assert abs(whole - one_d) <= 1e-12 * abs(one_d)


def test_cfg4_periodic_mirror_symmetry(L):
    """A unit charge at the cell centre of a periodic block with odd L (reference cell (L-1)/2, so
    the images sit symmetrically, lattice.hpp:100-106): the unit-cell potential at the cfg4 grid
    (n = 256) is symmetric under i -> n-1-i on every axis, to rounding of the ascending-k sums.
    (For the even-L BASELINE blocks the image set is one cell longer on one side.)"""
    import torch
    spec, rule = cfg(L, 63, n=256)
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=True)
    out = torch.empty((256, 256, 256), dtype=torch.float64, device="cuda")
    pipe.step(out)
    torch.cuda.synchronize()
    scale = float(out.abs().max())
    for d in range(3):
        assert float((out - torch.flip(out, dims=[d])).abs().max()) <= 1e-13 * scale


def test_calibration_matches_reference(L, ref):
    """calibrate_quadrature / calibrate_for_lattice (newton.hpp:161-189, lattice.hpp:118-126) with
    every candidate's probes evaluated on the GPU pick the same (M, C0) as the reference."""
    import ctypes as C
    ref.lib.ref_calibrate_quadrature.restype = C.c_int
    ref.lib.ref_calibrate_quadrature.argtypes = [C.c_double, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_int,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int)]
    for b, n, eps in ((2.0, 16, 1e-4), (2.0, 16, 1e-6), (2.0, 32, 1e-5)):
        grid = L.GridSpec(b, n)
        tol = L.default_tolerance(grid, eps)
        trace = []
        rule = L.calibrate_quadrature(grid, tol, trace)
        c0 = C.c_double(0)
        tl = C.c_int(0)
        M = ref.lib.ref_calibrate_quadrature(b, n, eps, tol.a_min, tol.a_max, 128, C.byref(c0), C.byref(tl))
        assert (rule.M, rule.C0) == (M, c0.value)
        assert len(trace) == tl.value
        assert L.measure_probe_error(L.build_newton_master([n] * 3, grid.h, rule), L.kernel_probe_set(grid, tol)) <= eps
    ref.lib.ref_calibrate_for_lattice.restype = C.c_int
    ref.lib.ref_calibrate_for_lattice.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_double, C.c_double,
                                                  C.POINTER(C.c_double)]
    spec = L.LatticeSpec((4, 2, 1), L.GridSpec(2.0, 8), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.calibrate_for_lattice(spec, 1e-4)
    Lx = np.array(spec.L, dtype=np.int64)
    c0 = C.c_double(0)
    M = ref.lib.ref_calibrate_for_lattice(Lx.ctypes.data_as(C.POINTER(C.c_int64)), 8, 2.0, 1e-4, C.byref(c0))
    assert (rule.M, rule.C0) == (M, c0.value)


# ------------------------------------------------------------ large ranks / caller buffers
@pytest.mark.parametrize("R,F", [(2200, 600), (9000, 40), (3, 700)])
def test_functional_batch_any_rank(L, orc, R, F):
    """functional_batch beyond the shared-memory Gram kernels: F >= 4 * SMs with R > 2133 used
    to be refused; now the 4-density kernel falls back to the single one, and
    ranks beyond that take the global-scratch Gram path, with the same rank-ordered sum."""
    rng = np.random.default_rng(R + F)
    dims = (12, 10, 9)
    fac = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], R))) for l in range(3)]
    w = rng.uniform(0.5, 1.5, R)
    G = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], F))) for l in range(3)]
    got = L.functional_batch(L.CanonicalTensor3(fac, w, trusted=True), G)
    for f in rng.integers(0, F, 6):
        want = orc.scalar_product(fac, w, [np.asfortranarray(G[l][:, [f]]) for l in range(3)], np.ones(1))
        assert abs(got[f] - want) <= 1e-12 * abs(want), (R, F, f)


def test_functional_batch_paths_agree_bitwise(L):
    """The same density through the 4-density kernel (large batch) and the single-density
    kernel (small batch) gives bit-identical results."""
    rng = np.random.default_rng(5)
    dims = (16, 8, 8)
    R = 100
    fac = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], R))) for l in range(3)]
    w = rng.uniform(0.5, 1.5, R)
    t = L.CanonicalTensor3(fac, w, trusted=True)
    G = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], 700))) for l in range(3)]
    big = L.functional_batch(t, G)      # F >= 4 * SMs: four densities per block
    small = L.functional_batch(t, [np.asfortranarray(g[:, :3]) for g in G])
    assert np.array_equal(big[:3], small)


def test_caller_buffers_are_validated(L):
    import torch
    spec, rule = cfg(L, 2, n=8)
    pipe = L.DevicePipeline(spec, rule)
    N = pipe.dims
    with pytest.raises(L.ValidationError):
        pipe.expand(torch.empty((N[2], N[1], N[0] - 1), dtype=torch.float64, device="cuda"))
    with pytest.raises(L.ValidationError):
        pipe.expand(torch.empty((N[2], N[1], N[0]), dtype=torch.float32, device="cuda"))
    with pytest.raises(L.ValidationError):
        pipe.step(torch.empty((N[0], N[1], N[2]), dtype=torch.float64, device="cuda").transpose(0, 2))
    with pytest.raises(L.ValidationError):
        pipe.grid_functional([torch.ones(N[0] + 1, dtype=torch.float64, device="cuda")] * 3)
    with pytest.raises(L.ValidationError):
        L.lattice_potential(spec, rule, out=np.empty((N[0], N[1], N[2])))  # C order
    with pytest.raises(L.ValidationError):
        L.lattice_potential(spec, rule, out=np.empty((N[0], N[1], N[2] - 1), order="F"))
    t = L.CanonicalTensor3([np.ones((N[l], 1)) for l in range(3)], np.ones(1))
    with pytest.raises(L.ValidationError):
        L.grid_functional(t, [np.ones(N[0]), np.ones(N[1]), np.ones(N[2] - 1)])
    with pytest.raises(L.ValidationError):
        L.expand_slabs(t, 0, 2, out=np.empty((N[0], N[1], 3), order="F"))
    # square factors (n_l == R) keep their meaning: no shape-based transposition
    R = 6
    rng = np.random.default_rng(9)
    fac = [np.asfortranarray(rng.uniform(0.1, 1.0, (R, R))) for _ in range(3)]
    w = rng.uniform(0.5, 1.5, R)
    X = [np.asfortranarray(rng.uniform(0.1, 1.0, (R, 2))) for _ in range(3)]
    got = L.functional_batch(L.CanonicalTensor3(fac, w, trusted=True), X)
    want = np.einsum("q,iq,jq,kq,i,j,k->", w, *fac, X[0][:, 0], X[1][:, 0], X[2][:, 0])
    assert abs(got[0] - want) <= 1e-13 * abs(want)


def test_watchdog_clear_and_product_build(L):
    lib = L._abi.load()
    assert lib.ls_dev_knobs_enabled() == 0
    spec, rule = cfg(L, 2, n=8)
    L.lattice_potential(spec, rule)
    assert lib.ls_fault_status(0) == 0


@pytest.mark.parametrize("Lc,periodic", [(4, False), (16, False), (64, True)])
def test_lattice_energy_end_to_end(L, orc, Lc, periodic):
    """ls_h_lattice_energy (host inputs, scalar out, V never stored) against the 1D rank-term form
    of the oracle's own assembled tensor (scalar_product, canonical.hpp:126-136)."""
    n = 256 if periodic else 64
    spec, rule = cfg(L, Lc, n=n)
    N = (n,) * 3 if periodic else spec.target_dims()
    sigma = (spec.unit.b if periodic else Lc * spec.unit.b) / 4
    rho = [np.exp(-((np.arange(N[l]) + 0.5 - N[l] / 2) * spec.unit.h) ** 2 / (2 * sigma ** 2)) for l in range(3)]
    e = L.lattice_energy(spec, rule, rho, periodic=periodic)
    _, fo, wo = oracle_assembled(orc, spec, rule, "erf", periodic)
    want = orc.scalar_product(fo, wo, [np.asfortranarray(r.reshape(-1, 1)) for r in rho], np.ones(1))
    assert abs(e - want) <= 1e-12 * abs(want)
    with pytest.raises(L.ValidationError):
        L.lattice_energy(spec, rule, [rho[0], rho[1], rho[2][:-1]], periodic=periodic)
