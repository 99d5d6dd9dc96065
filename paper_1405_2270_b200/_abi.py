"""ctypes binding of liblatsum_cuda.so (declared in include/latsum_cuda.h).

Loads the in-tree library and fails loudly if it is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "liblatsum_cuda.so"

LS_OK, LS_EVALIDATION, LS_EGUARD, LS_ECUDA = 0, 2, 4, 5
GEN_MIDPOINT, GEN_ERF = 0, 1


class ValidationError(ValueError):
    """Mirror of latsum::validation_error (reference errors.hpp:9-12)."""


class ResourceGuardError(RuntimeError):
    """Mirror of latsum::resource_guard_error (reference errors.hpp:17-20)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure inside liblatsum_cuda.so."""


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p
_i64 = C.c_int64
_d = C.c_double
_i = C.c_int

# name -> (restype, argtypes); mirrors include/latsum_cuda.h
SIGNATURES = {
    "ls_abi_version": (_i, []),
    "ls_last_error": (C.c_char_p, []),
    "ls_set_device": (_i, [_i]),
    "ls_launch_count": (_i64, []),
    "ls_sinc_quadrature": (_i, [_d, _d, _d, _i, _d, _vp, _vp, _vp, _dp]),
    "ls_gen_master": (_i, [_i, _vp, _i, _i64, _d, _vp, _i64, _vp]),
    "ls_libm_eval": (_i, [_i, _vp, _vp, _i64, _vp]),
    "ls_fault_status": (_i, [_i]),
    "ls_validate_grid": (_i, [_d, _i64]),
    "ls_charge_grid_index": (_i, [_d, _i64, _d, _i, _i, _vp]),
    "ls_validate_lattice": (_i, [_vp, _i64, _d, _vp, _i, _vp]),
    "ls_dev_knobs_enabled": (_i, []),
    "ls_set_host_threads": (_i, [_i]),
    "ls_comm_unique_id": (_i, [_vp, _i]),
    "ls_comm_init": (_i, [_i, _i, _vp, _i, _vp]),
    "ls_comm_destroy": (_i, [_vp]),
    "ls_comm_info": (_i, [_vp, _vp, _vp]),
    "ls_comm_allreduce_f64": (_i, [_vp, _vp, _i64, _i, _vp]),
    "ls_pipeline_energy_allreduce": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp]),
    "ls_assemble_axis": (_i, [_vp, _i64, _i, _i, _vp, _i64, _i64, _i, _vp, _i64, _vp]),
    "ls_expand": (_i, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i64, _i64, _i, _i64, _i64, _vp, _i64, _i64,
                       _vp, _vp, _vp, _vp, _vp]),
    "ls_expand_partial_count": (_i64, [_i64, _i64, _i, _i64, _i64]),
    "ls_sum_partials": (_i, [_vp, _i64, _vp, _vp]),
    "ls_eval_points": (_i, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i, _vp, _i64, _vp, _vp]),
    "ls_gram": (_i, [_vp, _i64, _i, _vp, _i64, _i, _i64, _vp, _vp]),
    "ls_gram_reduce": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _vp, _vp]),
    "ls_functional_batch": (_i, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i, _i64, _i64, _i64, _vp, _i64, _vp, _i64,
                                 _vp, _i64, _i, _d, _vp, _vp]),
    "ls_maxdiff_accumulate": (_i, [_vp, _vp, _i64, _vp, _i, _vp]),
    "ls_expand_plan_name": (_i, [_i, C.c_char_p, _i]),
    "ls_grid_functional_batch": (_i, [_vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _i, _d,
                                      _i, _vp, _vp]),
    "ls_probe_error": (_i, [_vp, _vp, _i, _i64, _d, _vp, _vp, _i64, _vp, _vp]),
    "ls_h_calibrate_quadrature": (_i, [_d, _i64, _d, _d, _d, _i, C.POINTER(_i), C.POINTER(_d), C.POINTER(_i), _vp, _vp,
                                       _vp, _i]),
    "ls_h_newton_master": (_i, [_i, _vp, _d, _vp, _i, _vp, _vp, _vp]),
    "ls_h_functional_batch": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _d, _vp]),
    "ls_h_max_norm_diff": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ls_pipeline_create": (_i, [_i, _vp, _i64, _d, _vp, _vp, _i, _vp, _i, _i, C.POINTER(_vp)]),
    "ls_pipeline_destroy": (_i, [_vp]),
    "ls_pipeline_info": (_i, [_vp, _vp, C.POINTER(_i), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "ls_pipeline_generate": (_i, [_vp, _vp]),
    "ls_pipeline_assemble": (_i, [_vp, _vp]),
    "ls_pipeline_prepare": (_i, [_vp, _vp]),
    "ls_pipeline_expand": (_i, [_vp, _i64, _i64, _vp, _vp]),
    "ls_pipeline_step": (_i, [_vp, _i64, _i64, _vp, _vp]),
    "ls_pipeline_energy": (_i, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp]),
    "ls_device_malloc": (_i, [C.c_size_t, C.POINTER(_vp)]),
    "ls_device_free": (_i, [_vp]),
    "ls_memcpy": (_i, [_vp, _vp, C.c_size_t, _vp]),
    "ls_synchronize": (_i, [_vp]),
    "ls_h_lattice_master": (_i, [_i, _vp, _i64, _d, _vp, _i, _vp, _vp, _vp]),
    "ls_h_gen_column": (_i, [_i, _d, _i64, _d, _vp]),
    "ls_h_assemble_axis": (_i, [_vp, _i64, _i, _i, _vp, _i64, _i64, _i, _vp]),
    "ls_h_expand": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "ls_h_eval_points": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "ls_h_scalar_product": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp]),
    "ls_h_grid_functional": (_i, [_vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]),
    "ls_h_lattice_potential": (_i, [_i, _vp, _i64, _d, _vp, _vp, _i, _vp, _i, _i, _i64, _i64, _vp, _vp, _vp, _vp,
                                    _vp]),
    "ls_h_lattice_energy": (_i, [_i, _vp, _i64, _d, _vp, _vp, _i, _vp, _i, _i, _i64, _i64, _vp, _vp, _vp, _vp]),
    "ls_qtt_core_stride": (_i64, [_i64, _i]),
    "ls_qtt_compress": (_i, [_vp, _i64, _i64, _i, _d, _i, _vp, _i64, _vp, _vp, _vp]),
    "ls_qtt_unfolding_ranks": (_i, [_vp, _i64, _i64, _i, _d, _vp, _vp]),
    "ls_h_qtt_compress": (_i, [_vp, _i64, _i, _d, _i, _vp, _i64, _vp, _vp]),
    "ls_h_qtt_unfolding_ranks": (_i, [_vp, _i64, _i, _d, _vp]),
}

_lib = None


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA extension is required, there is no CPU fallback)")
        lib = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def check(rc: int, what: str = "") -> None:
    if rc == LS_OK:
        return
    msg = load().ls_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == LS_EVALIDATION:
        raise ValidationError(text)
    if rc == LS_EGUARD:
        raise ResourceGuardError(text)
    raise CudaError(f"{text} (status {rc})")


def call(name: str, *args):
    """Calls an int-status entry point and raises the mirrored exception."""
    rc = getattr(load(), name)(*args)
    check(rc, name)
    return rc
