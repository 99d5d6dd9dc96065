"""ctypes bindings for the two CPU oracles (TEST INFRASTRUCTURE ONLY)."""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["F_CONTIGUOUS"] or a.ndim == 1, "need contiguous f64"
    return a.ctypes.data_as(_dp)


def _host_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            return "avx512f" in f.read()
    except OSError:
        return False


class _Lib:
    """Thin numpy-facing wrapper; `prefix` is 'orc_' or 'ref_'."""

    def __init__(self, path: Path, prefix: str):
        self.path = path
        self.lib = C.CDLL(str(path))
        self.p = prefix
        self.is_ref = prefix == "ref_"
        L = self.lib
        f = self._f
        f("sinc_quadrature", C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int, C.c_double, _dp, _dp, _dp, _dp])
        f("gaussian_sample_vector", C.c_int, [C.c_int64, C.c_double, C.c_double, _dp])
        f("gaussian_moment_vector", C.c_int, [C.c_double, C.c_int64, C.c_double, C.c_int, _dp])
        f("densify_slabs", C.c_int, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_int64] * 2 + [_dp])
        f("eval_point", C.c_double, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_int64] * 3)
        f("scalar_product", C.c_double, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_int] + [_dp] * 4)
        if self.is_ref:
            f("lattice_master", C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, _dp, _dp, C.c_int, _dp, C.c_int, _dp, _dp, _dp, _dp])
            f("assembled_sum", C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, _dp, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp, _dp])
            f("direct_sum", C.c_int, [_i64p, C.c_int64, C.c_double, _dp, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp])
            f("densify", C.c_int, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_uint64, _dp])
            f("stream_functional", C.c_double, [C.c_int64] * 3 + [C.c_int] + [_dp] * 7 + [C.c_int64] * 2 + [_dp])
            f("expand_into", C.c_int, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_int64] * 2 + [_dp, _dp])
            f("max_norm_diff_canonical", C.c_int, [C.c_int64] * 3 + [C.c_int] + [_dp] * 4 + [C.c_int] + [_dp] * 4 + [_dp, _dp])
            f("sample_gaussian_basis", C.c_int, [C.c_double, C.c_int64, C.c_int, _dp, _dp, _dp])
            f("potential_matrix", C.c_int, [C.c_double, C.c_int64, C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp])
            f("quadrature_value", C.c_double, [_dp, _dp, C.c_int, C.c_double])
            f("set_threads", None, [C.c_int])
            f("max_threads", C.c_int, [])
            f("last_error", C.c_char_p, [])
        else:
            f("lattice_master", C.c_int, [C.c_int, _i64p, C.c_int64, C.c_double, _dp, C.c_int, _dp, _dp, _dp])
            f("assembled_axis", C.c_int, [_dp, C.c_int, C.c_int, _i64p, C.c_int64, C.c_int64, C.c_int, _dp])
            f("assembled_weights", None, [_dp, C.c_int, _dp, C.c_int, _dp])
            f("charge_grid_index", C.c_int64, [C.c_double, C.c_int64, C.c_double])
            f("window_start_box", C.c_int64, [C.c_int64] * 4)
            f("window_start_periodic", C.c_int64, [C.c_int64] * 5)
            f("direct_sum", C.c_int, [_i64p, C.c_int64, _i64p, _dp, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp, _dp, _dp, _dp])
            f("sample_gaussian", C.c_int, [C.c_double, C.c_int64, _dp, C.c_double, _dp])
            f("potential_matrix", C.c_int, [C.c_int64, C.c_double, C.c_int, _dp, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp])
            f("grid_functional", C.c_double, [C.c_int64] * 3 + [C.c_int] + [_dp] * 7 + [C.c_int64] * 2)
            f("quadrature_value", C.c_double, [_dp, _dp, C.c_int, C.c_double])
            f("libm_eval", C.c_int, [C.c_int, _dp, _dp, C.c_int64])

    def _f(self, name, res, args):
        fn = getattr(self.lib, self.p + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    def _check(self, rc, what):
        if rc != 0:
            msg = self._last_error().decode() if self.is_ref else ""
            raise RuntimeError(f"{self.p}{what} failed rc={rc} {msg}")

    # ---- quadrature / generator ----
    def sinc_quadrature(self, eps, a_min, a_max, M, C0=1.0):
        R = 2 * M + 1
        nodes, tau, w = (np.zeros(R) for _ in range(3))
        step = C.c_double(0)
        self._check(self._sinc_quadrature(eps, a_min, a_max, M, C0, _ptr(nodes), _ptr(tau), _ptr(w), C.byref(step)), "sinc_quadrature")
        return nodes, tau, w, step.value

    def quadrature_value(self, tau, w, r):
        return self._quadrature_value(_ptr(tau), _ptr(w), len(tau), r)

    def gaussian_sample_vector(self, length, h, t):
        out = np.zeros(length)
        self._check(self._gaussian_sample_vector(length, h, t, _ptr(out)), "gaussian_sample_vector")
        return out

    def gaussian_moment_vector(self, b, n, t, doubled):
        out = np.zeros(2 * n if doubled else n)
        self._check(self._gaussian_moment_vector(b, n, t, int(doubled), _ptr(out)), "gaussian_moment_vector")
        return out

    def lattice_master(self, mode, L, n, b, tau, w=None, charges=None):
        """Master factors [f0, f1, f2], each (2*L_l*n, R) Fortran-ordered."""
        L = np.asarray(L, dtype=np.int64)
        R = len(tau)
        f = [np.zeros((2 * int(L[l]) * n, R), order="F") for l in range(3)]
        if self.is_ref:
            ch = np.asarray(charges if charges is not None else [[0, 0, 0, 1.0]], dtype=np.float64)
            t = C.c_double(0)
            rc = self._lattice_master(mode, L.ctypes.data_as(_i64p), n, b, _ptr(tau), _ptr(np.asarray(w)), R,
                                      _ptr(ch.ravel()), len(ch), _ptr(f[0]), _ptr(f[1]), _ptr(f[2]), C.byref(t))
        else:
            rc = self._lattice_master(mode, L.ctypes.data_as(_i64p), n, b, _ptr(tau), R, _ptr(f[0]), _ptr(f[1]), _ptr(f[2]))
        self._check(rc, "lattice_master")
        return f

    def libm_eval(self, fn, x):
        """Host libm erf (fn 0) / exp (fn 1) of every element of x."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty_like(x)
        self._check(self._libm_eval(fn, _ptr(x), _ptr(y), x.size), "libm_eval")
        return y

    # ---- tensors ----
    def densify_slabs(self, A, B, Cf, w, k0=0, k1=None):
        n1, n2, n3 = A.shape[0], B.shape[0], Cf.shape[0]
        R = len(w)
        k1 = n3 if k1 is None else k1
        out = np.zeros((n1, n2, k1 - k0), order="F")
        self._check(self._densify_slabs(n1, n2, n3, R, _ptr(A), _ptr(B), _ptr(Cf), _ptr(w), k0, k1, _ptr(out)), "densify_slabs")
        return out

    def eval_point(self, A, B, Cf, w, i, j, k):
        return self._eval_point(A.shape[0], B.shape[0], Cf.shape[0], len(w), _ptr(A), _ptr(B), _ptr(Cf), _ptr(w), i, j, k)

    def scalar_product(self, fa, wa, fb, wb):
        return self._scalar_product(fa[0].shape[0], fa[1].shape[0], fa[2].shape[0], len(wa), _ptr(fa[0]), _ptr(fa[1]),
                                    _ptr(fa[2]), _ptr(wa), len(wb), _ptr(fb[0]), _ptr(fb[1]), _ptr(fb[2]), _ptr(wb))


def _load(name):
    p = HERE / name
    return p if p.exists() else None


_cache: dict = {}


def restatement() -> _Lib:
    if "orc" not in _cache:
        p = _load("liblatsum_oracle.so")
        if p is None:
            raise FileNotFoundError("oracle/liblatsum_oracle.so not built (run `make -C oracle`)")
        _cache["orc"] = _Lib(p, "orc_")
    return _cache["orc"]


def ref_available() -> bool:
    return _load("_ref/libref_latsum_v3.so") is not None


def reference() -> _Lib:
    if "ref" not in _cache:
        v4 = _load("_ref/libref_latsum_v4.so")
        v3 = _load("_ref/libref_latsum_v3.so")
        p = v4 if (v4 is not None and _host_has_avx512()) else v3
        if p is None:
            raise FileNotFoundError("oracle/_ref not built (needs /root/reference; run `make -C oracle ref`)")
        _cache["ref"] = _Lib(p, "ref_")
    return _cache["ref"]
