"""Python mirror of the reference latsum hot-path API (arXiv 1405.2270).

Same names, argument meaning and error behaviour as the reference's C++
headers (/root/reference/proj/include/latsum/*.hpp, cited per function), so
parity tests read like the reference's own tests. Every numeric stage runs in
liblatsum_cuda.so on the GPU; this module only validates, converts layouts
and calls the C ABI. Factor matrices are numpy arrays of shape (n_l, R) in
Fortran (column-major) order, exactly Eigen::MatrixXd's layout.

Host-level functions (numpy in, numpy out) go through the synchronous
``ls_h_*`` entry points. :class:`DevicePipeline` keeps every stage resident in
HBM (torch tensors as device memory and streams) for the benchmark path.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _abi
from ._abi import GEN_ERF, GEN_MIDPOINT, ResourceGuardError, ValidationError, call

DEFAULT_DENSIFY_GUARD = 1 << 27  # canonical.hpp:237
MODES = {"midpoint": GEN_MIDPOINT, "erf": GEN_ERF}


def _p(a: np.ndarray | None):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a, order="F"):
    return np.require(np.asarray(a, dtype=np.float64), requirements=[order, "A"])


def _check_host_out(out, shape, what):
    """A caller-supplied host grid goes to native code as a raw pointer: it must be exactly the
    Fortran-ordered float64 (n1, n2, k1 - k0) block the call writes."""
    shape = tuple(int(x) for x in shape)
    if not isinstance(out, np.ndarray) or out.dtype != np.float64 or out.shape != shape \
            or not out.flags["F_CONTIGUOUS"] or not out.flags["WRITEABLE"]:
        got = (getattr(out, "shape", None), getattr(out, "dtype", None))
        raise ValidationError(f"{what}: out must be a writeable Fortran-ordered float64 array of shape {shape}, "
                              f"got shape/dtype {got}")


def _check_lengths(vecs, dims, what):
    if len(vecs) != 3:
        raise ValidationError(f"{what}: need three density factors")
    for l in range(3):
        if vecs[l].shape[0] != dims[l]:
            raise ValidationError(f"{what}: density factor {l} has length {vecs[l].shape[0]}, grid axis has {dims[l]}")


def _check_device_tensor(x, shape, dev, what):
    """A caller-supplied device tensor: float64, contiguous, on the pipeline's device, exact shape."""
    import torch
    shape = tuple(int(v) for v in shape)
    if not isinstance(x, torch.Tensor) or x.dtype != torch.float64 or tuple(x.shape) != shape \
            or not x.is_contiguous() or x.device != dev:
        got = (tuple(getattr(x, "shape", ())), getattr(x, "dtype", None), getattr(x, "device", None))
        raise ValidationError(f"{what}: need a contiguous float64 tensor of shape {shape} on {dev}, got {got}")


# --------------------------------------------------------------------- grid.hpp
@dataclass(frozen=True)
class GridSpec:
    """grid.hpp:14-36: n x n x n cells over [-b/2, b/2]^3, mesh h = b/n."""
    b: float
    n: int

    def __post_init__(self):
        # grid.hpp:21-27 through the library's one implementation (ls_validate_grid)
        _abi.check(_abi.load().ls_validate_grid(float(self.b), int(self.n)))

    @property
    def h(self) -> float:
        return self.b / float(self.n)

    @staticmethod
    def midpoint_of(i: int, length: int, h: float) -> float:
        return (float(i) + 0.5 - float(length) / 2.0) * h

    def midpoint(self, i: int) -> float:
        return self.midpoint_of(i, self.n, self.h)


# --------------------------------------------------------------- quadrature.hpp
@dataclass
class QuadratureRule:
    """quadrature.hpp:20-29."""
    M: int
    C0: float
    step: float
    nodes: np.ndarray
    exponents: np.ndarray
    weights: np.ndarray

    def node_count(self) -> int:
        return 2 * self.M + 1


def sinc_quadrature(eps: float, a_min: float, a_max: float, M: int, C0: float = 1.0) -> QuadratureRule:
    """quadrature.hpp:50-89 (computed by the library's host code)."""
    R = 2 * M + 1 if M >= 1 else 1
    nodes, tau, w = np.zeros(R), np.zeros(R), np.zeros(R)
    step = C.c_double(0.0)
    call("ls_sinc_quadrature", eps, a_min, a_max, M, C0, _p(nodes), _p(tau), _p(w), C.byref(step))
    return QuadratureRule(M, C0, step.value, nodes, tau, w)


def quadrature_value(rule: QuadratureRule, r: float) -> float:
    """quadrature.hpp:93-100 (host scalar; sequential accumulation)."""
    s = 0.0
    for t, w in zip(rule.exponents, rule.weights):
        tr = t * r
        s += w * math.exp(-tr * tr)
    return s


# --------------------------------------------------------------- canonical.hpp
class CanonicalTensor3:
    """canonical.hpp:33-82: entry (i,j,k) = sum_q w_q A1(i,q) A2(j,q) A3(k,q)."""

    def __init__(self, factors: Sequence[np.ndarray], weights: np.ndarray, trusted: bool = False):
        fs = [_f64(f) for f in factors]
        w = _f64(weights).ravel()
        if len(fs) != 3:
            raise ValidationError("canonical tensor: need three factor matrices")
        r = w.shape[0]
        for l, f in enumerate(fs):
            if f.ndim != 2 or f.shape[1] != r:
                raise ValidationError(f"canonical tensor: factor {l} has {f.shape[1] if f.ndim == 2 else '?'} "
                                      f"columns, expected rank {r}")
            if not trusted and not np.all(np.isfinite(f)):
                raise ValidationError(f"canonical tensor: factor {l} contains a non-finite value")
        if not trusted and not np.all(np.isfinite(w)):
            raise ValidationError("canonical tensor: weights contain a non-finite value")
        self._f = fs
        self._w = w

    def rank(self) -> int:
        return int(self._w.shape[0])

    def dim(self, axis: int) -> int:
        return int(self._f[axis].shape[0])

    def dims(self) -> tuple[int, int, int]:
        return (self.dim(0), self.dim(1), self.dim(2))

    def factor(self, axis: int) -> np.ndarray:
        return self._f[axis]

    def weights(self) -> np.ndarray:
        return self._w


def _dims_arr(t: CanonicalTensor3) -> np.ndarray:
    return np.array(t.dims(), dtype=np.int64)


def densify(t: CanonicalTensor3, guard: int = DEFAULT_DENSIFY_GUARD) -> np.ndarray:
    """canonical.hpp:251-266: dense (n1, n2, n3) Fortran-ordered grid, computed on the GPU."""
    d = t.dims()
    total = d[0] * d[1] * d[2]
    if total > guard:
        raise ResourceGuardError(f"densify: {total} entries exceed the guard of {guard}")
    return expand_slabs(t, 0, d[2])


def expand_slabs(t: CanonicalTensor3, k0: int, k1: int, out: np.ndarray | None = None) -> np.ndarray:
    """densify_slab over slabs [k0, k1) (canonical.hpp:241-246) into host memory (no guard)."""
    d = t.dims()
    if not (0 <= k0 <= k1 <= d[2]):
        raise ValidationError("expand: slab range outside [0, N3]")
    if out is None:
        out = np.empty((d[0], d[1], k1 - k0), order="F")
    _check_host_out(out, (d[0], d[1], k1 - k0), "expand_slabs")
    call("ls_h_expand", _p(_dims_arr(t)), t.rank(), _p(t.factor(0)), _p(t.factor(1)), _p(t.factor(2)),
         _p(t.weights()), k0, k1, _p(out))
    return out


def eval_points(t: CanonicalTensor3, idx: np.ndarray) -> np.ndarray:
    """eval_point (canonical.hpp:304-314) for a (P, 3) array of indices."""
    idx = np.ascontiguousarray(idx, dtype=np.int64).reshape(-1, 3)
    out = np.zeros(idx.shape[0])
    call("ls_h_eval_points", _p(_dims_arr(t)), t.rank(), _p(t.factor(0)), _p(t.factor(1)), _p(t.factor(2)),
         _p(t.weights()), _p(idx), idx.shape[0], _p(out))
    return out


def eval_point(t: CanonicalTensor3, i: int, j: int, k: int) -> float:
    return float(eval_points(t, np.array([[i, j, k]]))[0])


def scalar_product(a: CanonicalTensor3, b: CanonicalTensor3) -> float:
    """canonical.hpp:126-136."""
    if a.dims() != b.dims():
        raise ValidationError(f"scalar_product: dimension mismatch {a.dims()} vs {b.dims()}")
    out = np.zeros(1)
    call("ls_h_scalar_product", _p(_dims_arr(a)), a.rank(), _p(a.factor(0)), _p(a.factor(1)), _p(a.factor(2)),
         _p(a.weights()), b.rank(), _p(b.factor(0)), _p(b.factor(1)), _p(b.factor(2)), _p(b.weights()), _p(out))
    return float(out[0])


def grid_functional(t: CanonicalTensor3, rho: Sequence[np.ndarray], k0: int = 0, k1: int | None = None) -> float:
    """Full-grid sum_{ijk} V(i,j,k) rho1(i) rho2(j) rho3(k) over slabs [k0, k1), V never stored."""
    k1 = t.dim(2) if k1 is None else k1
    r = [_f64(x).ravel() for x in rho]
    _check_lengths(r, t.dims(), "grid_functional")
    out = np.zeros(1)
    call("ls_h_grid_functional", _p(_dims_arr(t)), t.rank(), _p(t.factor(0)), _p(t.factor(1)), _p(t.factor(2)),
         _p(t.weights()), _p(r[0]), _p(r[1]), _p(r[2]), k0, k1, _p(out))
    return float(out[0])


# ------------------------------------------------------------------ newton.hpp
def gaussian_sample_vector(length: int, h: float, t: float) -> np.ndarray:
    """newton.hpp:43-52 (midpoint samples), one GPU column."""
    if length < 2 or length % 2 != 0:
        raise ValidationError("gaussian_sample_vector: length must be even and >= 2")
    out = np.zeros(length)
    call("ls_h_gen_column", GEN_MIDPOINT, t, length, h, _p(out))
    return out


def gaussian_moment_vector(grid: GridSpec, t: float, doubled: bool) -> np.ndarray:
    """newton.hpp:21-37 (erf-difference cell integrals), one GPU column."""
    if not (t >= 0.0) or not math.isfinite(t):
        raise ValidationError("gaussian_moment_vector: t must be finite and >= 0")
    length = 2 * grid.n if doubled else grid.n
    out = np.zeros(length)
    call("ls_h_gen_column", GEN_ERF, t, length, grid.h, _p(out))
    return out


def build_newton_master(lens: Sequence[int], h: float, rule: QuadratureRule,
                        mode: str = "midpoint") -> CanonicalTensor3:
    """newton.hpp:57-75: rank-R master, axes of equal length share factors."""
    factors: list[np.ndarray] = []
    for l, n_l in enumerate(lens):
        for m in range(l):
            if lens[m] == n_l:
                factors.append(factors[m].copy(order="F"))
                break
        else:
            f = np.zeros((n_l, rule.node_count()), order="F")
            for q, t in enumerate(rule.exponents):
                f[:, q] = (gaussian_sample_vector(n_l, h, float(t)) if mode == "midpoint"
                           else gaussian_moment_vector(GridSpec(n_l * h, n_l), float(t), False))
            factors.append(f)
    return CanonicalTensor3(factors, rule.weights.copy())


# ------------------------------------------------------- probes and calibration (newton.hpp)
@dataclass(frozen=True)
class KernelTolerance:
    """grid.hpp:41-60."""
    eps: float
    a_min: float
    a_max: float

    def __post_init__(self):
        if not (0.0 < self.eps < 1.0):
            raise ValidationError(f"tolerance: eps must lie in (0, 1), got {self.eps}")
        if not (0.0 < self.a_min < self.a_max):
            raise ValidationError(f"tolerance: need 0 < a_min < a_max, got a_min = {self.a_min}, "
                                  f"a_max = {self.a_max}")


def default_tolerance(grid: GridSpec, eps: float) -> KernelTolerance:
    """grid.hpp:62-64."""
    return KernelTolerance(eps, grid.h, math.sqrt(3.0) * grid.b)


def kernel_probe_set(grid: GridSpec, tol: KernelTolerance) -> np.ndarray:
    """newton.hpp:97-132: (P, 4) array of (i, j, k, r) probes in ascending (i, j, k) order."""
    n = grid.n
    c, sh = n // 2, min(8, n // 2)
    keys = set()
    rng = range(c - sh, c + sh)
    for i in rng:
        for j in rng:
            for k in rng:
                keys.add((i * n + j) * n + k)
    for i in range(n):
        keys.update({(i * n + c) * n + c, (i * n + i) * n + c, (i * n + i) * n + i})
    stride = max(1, n // 16)
    for i in range(0, n, stride):
        for j in range(0, n, stride):
            for k in range(0, n, stride):
                keys.add((i * n + j) * n + k)
    key = np.array(sorted(keys), dtype=np.int64)
    i, j, k = key // (n * n), (key // n) % n, key % n
    mid = lambda a: (a.astype(np.float64) + 0.5 - n / 2.0) * grid.h  # noqa: E731
    x, y, z = mid(i), mid(j), mid(k)
    r = np.sqrt(x * x + y * y + z * z)
    keep = (r >= tol.a_min) & (r <= tol.a_max)
    return np.stack([i[keep], j[keep], k[keep], r[keep]], axis=1)


def measure_probe_error(kernel: CanonicalTensor3, probes: np.ndarray) -> float:
    """newton.hpp:136-144: max |T(p) r - 1| over the probes, all evaluated in one GPU batch."""
    v = eval_points(kernel, probes[:, :3].astype(np.int64))
    return float(np.max(np.abs(v * probes[:, 3] - 1.0))) if len(v) else 0.0


def calibrate_quadrature(grid: GridSpec, tol: KernelTolerance, trace: list | None = None,
                         m_cap: int = 128) -> QuadratureRule:
    """newton.hpp:161-189: smallest M (best C0 in {1,2,3,4} at that M) meeting eps on the probes;
    the whole scan runs natively (ls_h_calibrate_quadrature) with every candidate's probes
    evaluated by one fused GPU kernel."""
    cap = 4 * max(m_cap, 2)
    tM = np.zeros(cap, dtype=np.int32)
    tC = np.zeros(cap)
    tE = np.zeros(cap)
    M, C0, n_tr = C.c_int(0), C.c_double(0.0), C.c_int(0)
    rc = _abi.load().ls_h_calibrate_quadrature(grid.b, grid.n, tol.eps, tol.a_min, tol.a_max, m_cap, C.byref(M),
                                               C.byref(C0), C.byref(n_tr), _p(tM), _p(tC), _p(tE), cap)
    if trace is not None:
        trace.extend((int(tM[e]), float(tC[e]), float(tE[e])) for e in range(min(n_tr.value, cap)))
    _abi.check(rc, "calibrate_quadrature")
    return sinc_quadrature(tol.eps, tol.a_min, tol.a_max, M.value, C0.value)


# ----------------------------------------------------------------- lattice.hpp
@dataclass
class Charge:
    """lattice.hpp:21-24."""
    pos: tuple[float, float, float] = (0.0, 0.0, 0.0)
    Z: float = 1.0


@dataclass
class LatticeSpec:
    """lattice.hpp:28-69."""
    L: tuple[int, int, int] = (1, 1, 1)
    unit: GridSpec = field(default_factory=lambda: GridSpec(1.0, 2))
    charges: list[Charge] = field(default_factory=list)

    def validate(self) -> None:
        """lattice.hpp:33-45 through the library's one implementation (ls_validate_lattice)."""
        L = np.array(self.L, dtype=np.int64)
        ch = np.array([[*c.pos, c.Z] for c in self.charges], dtype=np.float64).reshape(-1, 4)
        _abi.check(_abi.load().ls_validate_lattice(_p(L), int(self.unit.n), float(self.unit.b), _p(ch),
                                                   len(self.charges), None))

    def target_cells(self, axis: int) -> int:
        return self.L[axis] * self.unit.n

    def target_dims(self) -> tuple[int, int, int]:
        return (self.target_cells(0), self.target_cells(1), self.target_cells(2))

    def charge_count(self) -> int:
        return len(self.charges)

    def cell_count(self) -> int:
        return self.L[0] * self.L[1] * self.L[2]

    def charge_grid_index(self, axis: int, nu: int) -> int:
        """lattice.hpp:57-68 (ls_charge_grid_index): off-grid positions are rejected."""
        out = C.c_int64(0)
        _abi.check(_abi.load().ls_charge_grid_index(float(self.unit.b), int(self.unit.n),
                                                    float(self.charges[nu].pos[axis]), int(axis), int(nu),
                                                    C.byref(out)))
        return int(out.value)


def calibrate_for_lattice(spec: "LatticeSpec", eps: float, trace: list | None = None) -> QuadratureRule:
    """lattice.hpp:118-126: probes drawn from the doubled target extent."""
    spec.validate()
    Lm = max(spec.L)
    grid = GridSpec(2.0 * Lm * spec.unit.b, 2 * Lm * spec.unit.n)
    return calibrate_quadrature(grid, KernelTolerance(eps, spec.unit.h, math.sqrt(3.0) * Lm * spec.unit.b), trace)


def window_start_box(N: int, n: int, i_a: int, k: int) -> int:
    """lattice.hpp:98."""
    return N - i_a - k * n


def window_start_periodic(N: int, n: int, i_a: int, k: int, L: int) -> int:
    """lattice.hpp:104-106."""
    return N + (L // 2 - k) * n - i_a


def build_lattice_master(spec: LatticeSpec, rule: QuadratureRule, mode: str = "midpoint") -> CanonicalTensor3:
    """lattice.hpp:109-113 (mode='midpoint', the reference); mode='erf' is the BASELINE
    erf-difference generator on the same doubled target grid."""
    spec.validate()
    L = np.array(spec.L, dtype=np.int64)
    R = rule.node_count()
    f = [np.zeros((2 * spec.target_cells(l), R), order="F") for l in range(3)]
    tau = _f64(rule.exponents).ravel()
    call("ls_h_lattice_master", MODES[mode], _p(L), spec.unit.n, spec.unit.b, _p(tau), R, _p(f[0]), _p(f[1]),
         _p(f[2]))
    return CanonicalTensor3(f, rule.weights.copy(), trusted=True)


@dataclass
class SumResult:
    """lattice.hpp:130-135."""
    tensor: CanonicalTensor3
    grid_dims: tuple[int, int, int]
    rank: int
    time_ms: float


def _require_master_matches(spec: LatticeSpec, master: CanonicalTensor3) -> None:
    """lattice.hpp:139-148."""
    N = spec.target_dims()
    for l in range(3):
        if master.dim(l) != 2 * N[l]:
            raise ValidationError(f"lattice: master axis {l} has {master.dim(l)} cells, expected doubled target "
                                  f"grid {2 * N[l]}")
    if master.rank() < 1:
        raise ValidationError("lattice: master tensor has rank 0")


def assembled_axis_columns(spec: LatticeSpec, master: CanonicalTensor3, axis: int, periodic: bool) -> np.ndarray:
    """lattice.hpp:220-274 on the GPU (bit-identical ascending-k adds)."""
    n = spec.unit.n
    Ll = spec.L[axis]
    out_len = n if periodic else Ll * n
    R = master.rank()
    ia = np.array([spec.charge_grid_index(axis, nu) for nu in range(spec.charge_count())], dtype=np.int64)
    out = np.zeros((out_len, spec.charge_count() * R), order="F")
    call("ls_h_assemble_axis", _p(master.factor(axis)), master.dim(axis), R, spec.charge_count(), _p(ia), n, Ll,
         int(periodic), _p(out))
    return out


def _assembled_sum(spec: LatticeSpec, master: CanonicalTensor3, periodic: bool) -> SumResult:
    """lattice.hpp:276-296."""
    import time
    t0 = time.perf_counter()
    spec.validate()
    _require_master_matches(spec, master)
    R = master.rank()
    factors = [assembled_axis_columns(spec, master, l, periodic) for l in range(3)]
    w = np.array([c.Z * wq for c in spec.charges for wq in master.weights()])
    t = CanonicalTensor3(factors, w, trusted=True)
    n = spec.unit.n
    dims = (n, n, n) if periodic else spec.target_dims()
    return SumResult(t, dims, t.rank(), (time.perf_counter() - t0) * 1e3)


def assembled_box_sum(spec: LatticeSpec, master: CanonicalTensor3) -> SumResult:
    """lattice.hpp:303-305."""
    return _assembled_sum(spec, master, False)


def assembled_periodic_sum(spec: LatticeSpec, master: CanonicalTensor3) -> SumResult:
    """lattice.hpp:310-312."""
    return _assembled_sum(spec, master, True)


def lattice_potential(spec: LatticeSpec, rule: QuadratureRule, mode: str = "erf", periodic: bool = False,
                      k0: int = 0, k1: int | None = None, out: np.ndarray | None = None,
                      return_factors: bool = False):
    """End-to-end: generator -> assembled sum -> expansion of slabs [k0, k1) into host memory,
    one C-ABI call (ls_h_lattice_potential). `out` may be a pinned buffer."""
    spec.validate()
    n = spec.unit.n
    dims = (n, n, n) if periodic else spec.target_dims()
    k1 = dims[2] if k1 is None else k1
    if not (0 <= k0 <= k1 <= dims[2]):
        raise ValidationError("lattice_potential: slab range outside [0, N3]")
    if out is None:
        out = np.empty((dims[0], dims[1], k1 - k0), order="F")
    _check_host_out(out, (dims[0], dims[1], k1 - k0), "lattice_potential")
    M0, R = spec.charge_count(), rule.node_count()
    ch = np.array([[*c.pos, c.Z] for c in spec.charges], dtype=np.float64)
    L = np.array(spec.L, dtype=np.int64)
    f = [np.zeros((dims[l], M0 * R), order="F") for l in range(3)] if return_factors else [None] * 3
    wout = np.zeros(M0 * R)
    call("ls_h_lattice_potential", MODES[mode], _p(L), n, spec.unit.b, _p(_f64(rule.exponents).ravel()),
         _p(_f64(rule.weights).ravel()), R, _p(ch), M0, int(periodic), k0, k1, _p(out), _p(f[0]), _p(f[1]),
         _p(f[2]), _p(wout))
    if return_factors:
        return out, CanonicalTensor3(f, wout, trusted=True)
    return out


def lattice_energy(spec: LatticeSpec, rule: QuadratureRule, rho: Sequence[np.ndarray], mode: str = "erf",
                   periodic: bool = False, k0: int = 0, k1: int | None = None) -> float:
    """End-to-end <V, rho> (BASELINE configs[2]'s energy) in one C-ABI call
    (ls_h_lattice_energy): host rule, charges and separable density in, the scalar out; the
    grid is evaluated point by point on the device, fused with the reduction, and never stored."""
    spec.validate()
    n = spec.unit.n
    dims = (n, n, n) if periodic else spec.target_dims()
    k1 = dims[2] if k1 is None else k1
    if not (0 <= k0 <= k1 <= dims[2]):
        raise ValidationError("lattice_energy: slab range outside [0, N3]")
    r = [_f64(x).ravel() for x in rho]
    _check_lengths(r, dims, "lattice_energy")
    ch = np.array([[*c.pos, c.Z] for c in spec.charges], dtype=np.float64)
    L = np.array(spec.L, dtype=np.int64)
    out = np.zeros(1)
    call("ls_h_lattice_energy", MODES[mode], _p(L), n, spec.unit.b, _p(_f64(rule.exponents).ravel()),
         _p(_f64(rule.weights).ravel()), rule.node_count(), _p(ch), spec.charge_count(), int(periodic), k0, k1,
         _p(r[0]), _p(r[1]), _p(r[2]), _p(out))
    return float(out[0])


# --------------------------------------------------------------------- qtt.hpp
QTT_RANK_CAP = 64


@dataclass
class QTTVector:
    """qtt.hpp:25-44: cores[k] is (2 r_{k-1}) x r_k (Fortran order)."""
    cores: list
    eps_used: float = 0.0

    def levels(self) -> int:
        return len(self.cores)

    def ranks(self) -> list[int]:
        return [int(c.shape[1]) for c in self.cores[:-1]]


def qtt_compress_columns(V: np.ndarray, eps: float) -> list[QTTVector]:
    """qtt_compress (qtt.hpp:49-86) of every column of V (N x ncols, N a power of two), one
    batched GPU sweep (ls_h_qtt_compress)."""
    V = _f64(V if np.ndim(V) == 2 else np.reshape(V, (-1, 1)))
    N, ncols = V.shape
    if N < 2 or N & (N - 1):
        raise ValidationError(f"qtt_compress: length {N} is not a power of two >= 2")
    if not eps > 0:
        raise ValidationError("qtt_compress: eps must be positive")
    L = N.bit_length() - 1
    lib = _abi.load()
    stride = int(lib.ls_qtt_core_stride(N, QTT_RANK_CAP))
    cores = np.zeros(stride * max(ncols, 1))
    ranks = np.zeros((L + 1) * max(ncols, 1), dtype=np.int32)
    capped = np.zeros(max(ncols, 1), dtype=np.int32)
    call("ls_h_qtt_compress", _p(V), N, ncols, float(eps), QTT_RANK_CAP, _p(cores), stride, _p(ranks), _p(capped))
    out = []
    for c in range(ncols):
        if capped[c]:
            raise ResourceGuardError(f"qtt_compress: a quantized rank exceeds the cap of {QTT_RANK_CAP}")
        rk = ranks[(L + 1) * c:(L + 1) * (c + 1)]
        off, cs = stride * c, []
        for k in range(L):
            rows, cols = 2 * int(rk[k]), int(rk[k + 1])
            cs.append(cores[off:off + rows * cols].reshape((rows, cols), order="F").copy())
            off += rows * cols
        out.append(QTTVector(cs, eps))
    return out


def qtt_compress(v: np.ndarray, eps: float) -> QTTVector:
    return qtt_compress_columns(np.asarray(v, dtype=np.float64).reshape(-1, 1), eps)[0]


def qtt_reconstruct(t: QTTVector) -> np.ndarray:
    """qtt.hpp:89-107 (host contraction)."""
    if not t.cores:
        raise ValidationError("qtt_reconstruct: empty train")
    w = t.cores[0]
    for k, core in enumerate(t.cores[1:], 1):
        r = core.shape[0] // 2
        if w.shape[1] != r:
            raise ValidationError(f"qtt_reconstruct: rank profile mismatch at core {k}")
        w = np.vstack([w @ core[:r], w @ core[r:]])
    if t.cores[-1].shape[1] != 1:
        raise ValidationError("qtt_reconstruct: boundary rank is not 1")
    return w[:, 0]


def unfolding_rank_profile(v: np.ndarray, eps: float) -> list[int]:
    """qtt.hpp:131-152 on the GPU (ls_h_qtt_unfolding_ranks)."""
    v = _f64(v).ravel()
    N = v.size
    if N < 2 or N & (N - 1):
        raise ValidationError("unfolding_rank_profile: length is not a power of two >= 2")
    if not eps > 0:
        raise ValidationError("unfolding_rank_profile: eps must be positive")
    L = N.bit_length() - 1
    out = np.zeros(max(L - 1, 1), dtype=np.int32)
    call("ls_h_qtt_unfolding_ranks", _p(v), N, 1, float(eps), _p(out))
    return [int(x) for x in out[:L - 1]]


# ----------------------------------------------------------------- project.hpp
@dataclass
class GaussianBasisSpec:
    """project.hpp:15-18."""
    center: tuple[float, float, float] = (0.0, 0.0, 0.0)
    sigma: float = 1.0


def sample_gaussian_basis(grid: GridSpec, specs: Sequence[GaussianBasisSpec]) -> list[list[np.ndarray]]:
    """project.hpp:30-57 (host; n samples per axis per function)."""
    if not specs:
        raise ValidationError("basis: at least one function required")
    mids = (np.arange(grid.n, dtype=np.float64) + 0.5 - grid.n / 2.0) * grid.h
    out = []
    for f, s in enumerate(specs):
        if not (s.sigma > 0.0) or not math.isfinite(s.sigma):
            raise ValidationError(f"basis: function {f} needs positive finite sigma")
        axes = []
        for l in range(3):
            if not math.isfinite(s.center[l]):
                raise ValidationError(f"basis: function {f} has a non-finite center")
            d = mids - s.center[l]
            axes.append(np.exp(-d * d / (2.0 * s.sigma * s.sigma)))
        out.append(axes)
    return out


def functional_batch(P: CanonicalTensor3, rho: Sequence[np.ndarray], scale: float = 1.0) -> np.ndarray:
    """scale * scalar_product(P, rho_f) for F rank-1 densities; rho = (X, Y, Z) each (n_l, F)."""
    import torch
    dev = torch.device("cuda")
    X, Y, Z = (torch.as_tensor(_f64(r), device=dev) for r in rho)
    F = X.shape[1]
    out = DevicePipeline.functional_batch_device(
        [torch.as_tensor(P.factor(l), device=dev) for l in range(3)],
        torch.as_tensor(P.weights(), device=dev), [X, Y, Z], scale)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:F]


def expansion_plan(R: int) -> str:
    """The expansion plan the device path takes for rank R (ls_expand_plan_name)."""
    buf = C.create_string_buffer(256)
    call("ls_expand_plan_name", int(R), buf, 256)
    return buf.value.decode()


def grid_functional_batch(P: CanonicalTensor3, rho: Sequence[np.ndarray], scale: float = 1.0,
                          max_chunk_points: int = 1 << 28) -> np.ndarray:
    """Full-grid form of functional_batch: P is expanded on the device in
    z-slab chunks of at most max_chunk_points and every chunk is contracted against the F
    separable densities by one fused DMMA GEMM (ls_grid_functional_batch). Agrees with the
    1D rank-term form (scalar_product, canonical.hpp:126-136) to rounding."""
    import torch
    dev = torch.device("cuda")
    fac = [torch.as_tensor(P.factor(l), device=dev).T.contiguous() for l in range(3)]  # (R, n_l)
    w = torch.as_tensor(P.weights(), device=dev)
    X, Y, Z = (torch.as_tensor(_f64(r), device=dev) for r in rho)
    out = DevicePipeline.grid_functional_batch_device(
        lambda buf, k0, k1: _expand_device(fac, w, P.dims(), k0, k1, buf), P.dims(), [X, Y, Z], scale,
        max_chunk_points)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _expand_device(fac, w, dims, k0, k1, buf):
    """ls_expand of slabs [k0, k1) of the device factors fac[l] ((R, n_l) row-major) into buf."""
    import torch
    n1, n2, n3 = dims
    R = w.shape[0]
    s = torch.cuda.current_stream(buf.device)
    p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
    call("ls_expand", p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(w), n1, n2, n3, R, k0, k1,
         C.c_void_p(buf.data_ptr()), buf.stride(1), buf.stride(0), None, None, None, None,
         C.c_void_p(s.cuda_stream))


# ---------------------------------------------------------- device pipeline
class _DeviceView:
    """Zero-copy torch view of device memory owned by the native pipeline (CUDA array interface)."""

    def __init__(self, ptr: int, shape: tuple[int, ...]):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<f8", "data": (ptr, False), "version": 2,
                                         "strides": None}


class DevicePipeline:
    """Generator -> assembly -> expansion -> functional, every stage resident in HBM.

    A thin handle on the native pipeline object of liblatsum_cuda.so
    (``ls_pipeline_*``, csrc/pipeline.cu), which owns the master, the assembled
    factors and the weights. torch provides output buffers and streams only;
    factors are exposed as zero-copy (R, N_l) views, i.e. column-major
    (N_l x R) matrices with leading dimension N_l.
    """

    def __init__(self, spec: LatticeSpec, rule: QuadratureRule, mode: str = "erf", periodic: bool = False,
                 device=None):
        import torch
        spec.validate()
        self.torch = torch
        self.spec, self.rule, self.mode, self.periodic = spec, rule, mode, periodic
        self.dev = torch.device("cuda") if device is None else torch.device(device)
        self._devc = torch.device("cuda", self.dev.index if self.dev.index is not None else torch.cuda.current_device())
        self._lib = _abi.load()
        L = np.array(spec.L, dtype=np.int64)
        ch = np.array([[*c.pos, c.Z] for c in spec.charges], dtype=np.float64)
        tau = _f64(rule.exponents).ravel()
        w = _f64(rule.weights).ravel()
        handle = C.c_void_p()
        with torch.cuda.device(self.dev):
            call("ls_pipeline_create", MODES[mode], _p(L), spec.unit.n, spec.unit.b, _p(tau), _p(w),
                 rule.node_count(), _p(ch), len(ch), int(periodic), C.byref(handle))
        self._h = handle
        dims = np.zeros(3, dtype=np.int64)
        rt = C.c_int(0)
        ptrs = [C.c_void_p() for _ in range(4)]
        call("ls_pipeline_info", self._h, _p(dims), C.byref(rt), *(C.byref(q) for q in ptrs))
        self.dims = tuple(int(d) for d in dims)
        self.Rt = rt.value
        self.R = rule.node_count()
        self.M0 = spec.charge_count()
        self._fac = [torch.as_tensor(_DeviceView(ptrs[l].value, (self.Rt, self.dims[l])), device=self.dev)
                     for l in range(3)]
        self.w = torch.as_tensor(_DeviceView(ptrs[3].value, (self.Rt,)), device=self.dev)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.ls_pipeline_destroy(h)
            self._h = None

    @staticmethod
    def _ptr(x):
        return C.c_void_p(x.data_ptr()) if x is not None else None

    def factor(self, l):
        return self._fac[l]

    def _stream(self, stream):
        s = stream if stream is not None else self.torch.cuda.current_stream(self.dev)
        return C.c_void_p(s.cuda_stream)

    def generate(self, stream=None):
        call("ls_pipeline_generate", self._h, self._stream(stream))

    def assemble(self, stream=None):
        call("ls_pipeline_assemble", self._h, self._stream(stream))

    def prepare(self, stream=None):
        """generate + assemble (one launch on small lattices, bit-identical); step() runs it."""
        call("ls_pipeline_prepare", self._h, self._stream(stream))

    def _check_out(self, out, k0, k1):
        if not (0 <= k0 <= k1 <= self.dims[2]):
            raise ValidationError("expand: slab range outside [0, N3]")
        _check_device_tensor(out, (k1 - k0, self.dims[1], self.dims[0]), self._devc, "expand")

    def expand(self, out, k0=0, k1=None, stream=None):
        """Writes slabs [k0, k1) into `out` (a contiguous (k1-k0, N2, N1) float64 tensor)."""
        k1 = self.dims[2] if k1 is None else k1
        self._check_out(out, k0, k1)
        call("ls_pipeline_expand", self._h, k0, k1, self._ptr(out), self._stream(stream))

    def step(self, out, k0=0, k1=None, stream=None):
        """One pass of the hot path: generate, assemble, expand into `out`."""
        k1 = self.dims[2] if k1 is None else k1
        self._check_out(out, k0, k1)
        call("ls_pipeline_step", self._h, k0, k1, self._ptr(out), self._stream(stream))

    def partial_count(self, k0=0, k1=None):
        k1 = self.dims[2] if k1 is None else k1
        return int(self._lib.ls_expand_partial_count(self.dims[0], self.dims[1], self.Rt, k0, k1))

    def grid_functional(self, rho, k0=0, k1=None, stream=None):
        """sum V*rho over slabs [k0, k1) fused into the expansion (V not stored); returns a
        1-element device tensor."""
        k1 = self.dims[2] if k1 is None else k1
        if not (0 <= k0 <= k1 <= self.dims[2]):
            raise ValidationError("grid_functional: slab range outside [0, N3]")
        r = [x.contiguous() for x in rho]
        for l in range(3):
            _check_device_tensor(r[l], (self.dims[l],), self._devc, f"grid_functional: density factor {l}")
        s = stream if stream is not None else self.torch.cuda.current_stream(self.dev)
        with self.torch.cuda.stream(s):
            out = self.torch.zeros(1, dtype=self.torch.float64, device=self.dev)
        call("ls_pipeline_energy", self._h, self._ptr(r[0]), self._ptr(r[1]), self._ptr(r[2]), k0, k1,
             self._ptr(out), self._stream(stream))
        return out

    @staticmethod
    def grid_functional_batch_device(expand, dims, rho, scale=1.0, max_chunk_points=1 << 28):
        """Full-grid functionals sum V * rho_f for F separable rho = (X, Y, Z) (device (n_l, F)
        tensors): expand(buf, k0, k1) writes slabs [k0, k1) into buf ((k1-k0, n2, n1) float64),
        which is contracted chunk by chunk (ls_grid_functional_batch, accumulate in slab order)."""
        import torch
        n1, n2, n3 = dims
        X, Y, Z = rho
        F = X.shape[1]
        Xt, Yt, Zt = (r.T.contiguous() for r in (X, Y, Z))  # (F, n) rows = column-major (n, F)
        out = torch.zeros(F, dtype=torch.float64, device=X.device)
        kc = max(1, min(n3, max_chunk_points // max(1, n1 * n2)))
        buf = torch.empty((kc, n2, n1), dtype=torch.float64, device=X.device)
        s = torch.cuda.current_stream(X.device)
        p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
        for k0 in range(0, n3, kc):
            k1 = min(n3, k0 + kc)
            expand(buf, k0, k1)
            call("ls_grid_functional_batch", p(buf), n1, n2, k1 - k0, buf.stride(1), buf.stride(0), p(Xt), n1,
                 p(Yt), n2, C.c_void_p(Zt.data_ptr() + 8 * k0), n3, F, float(scale), int(k0 > 0), p(out),
                 C.c_void_p(s.cuda_stream))
        return out

    def grid_functional_batch(self, rho, scale=1.0, max_chunk_points=1 << 28):
        """Full-grid form of functional_batch on this pipeline's potential (cfg4's 1024 test
        functions over the whole grid); rho = (X, Y, Z) device (n_l, F) tensors."""
        return DevicePipeline.grid_functional_batch_device(
            lambda buf, k0, k1: self.expand(buf, k0, k1), self.dims, rho, scale, max_chunk_points)

    @staticmethod
    def functional_batch_device(factors, w, rho, scale=1.0, stream=None):
        """scale * scalar_product(P, rho_f) for every column f of rho = (X, Y, Z).

        Every matrix is given in its logical (Eigen) shape, whatever its memory layout:
        factors[l] is (n_l, R) (e.g. ``pipe.factor(l).T``), rho[l] is (n_l, F); the rank-major
        and density-major buffers the kernel reads are built here with ``.T.contiguous()``."""
        import torch
        X, Y, Z = rho
        R = w.shape[0]
        F = X.shape[1]
        if len(factors) != 3 or any(f.dim() != 2 or f.shape[1] != R for f in factors):
            raise ValidationError(f"functional_batch: factors must be three (n_l, R={R}) matrices")
        if any(r.dim() != 2 or r.shape[1] != F or r.shape[0] != f.shape[0] for r, f in zip(rho, factors)):
            raise ValidationError("functional_batch: rho[l] must be (n_l, F) with the factor's n_l")
        Xt, Yt, Zt = (r.T.contiguous() for r in (X, Y, Z))  # (F, n) rows = columns
        ft = [f.T.contiguous() for f in factors]  # (R, n) rows = rank columns
        n = [ft[l].shape[1] for l in range(3)]
        out = torch.zeros(F, dtype=torch.float64, device=w.device)
        s = stream if stream is not None else torch.cuda.current_stream(w.device)
        p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
        call("ls_functional_batch", p(ft[0]), n[0], p(ft[1]), n[1], p(ft[2]), n[2], p(w), R, n[0], n[1], n[2],
             p(Xt), n[0], p(Yt), n[1], p(Zt), n[2], F, float(scale), p(out), C.c_void_p(s.cuda_stream))
        return out
