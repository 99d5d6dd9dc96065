"""C-ABI checks that need no GPU: the library loads, exports every entry point
include/latsum_cuda.h declares, the host-side quadrature matches the oracle,
and argument validation fails loudly (mirrored exception types) before any
device work."""
import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, rel

import paper_1405_2270_b200 as L
from paper_1405_2270_b200 import _abi


def declared_symbols():
    text = (ROOT / "include" / "latsum_cuda.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ls_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_abi.exported_symbols())
    assert lib.ls_abi_version() == 1


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_abi.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_quadrature_matches_oracle(orc):
    for args in [(1e-6, 10 / 64, math.sqrt(3) * 40, 20, 1.0), (1e-4, 0.25, 4.0, 10, 2.0)]:
        r = L.sinc_quadrature(*args)
        _, tau, w, step = orc.sinc_quadrature(*args)
        assert r.node_count() == 2 * args[3] + 1
        assert rel(r.exponents, tau) <= 1e-15 and rel(r.weights, w) <= 1e-15
        assert r.step == pytest.approx(step, rel=1e-15)


@pytest.mark.parametrize("bad", [(1e-6, 0.01, 10.0, 0, 1.0), (0.0, 0.01, 10.0, 5, 1.0), (1e-6, 1.0, 0.5, 5, 1.0)])
def test_quadrature_validation(bad):  # test_newton.cpp:110-112
    with pytest.raises(L.ValidationError):
        L.sinc_quadrature(*bad)


def test_device_entry_points_validate_before_device_work():
    lib = _abi.load()
    # odd length, non-positive mesh, bad mode: LS_EVALIDATION without touching the GPU
    assert lib.ls_gen_master(0, None, 3, 5, 0.1, None, 5, None) == _abi.LS_EVALIDATION
    assert lib.ls_gen_master(0, None, 3, 6, 0.0, None, 6, None) == _abi.LS_EVALIDATION
    assert lib.ls_gen_master(7, None, 3, 6, 0.1, None, 6, None) == _abi.LS_EVALIDATION
    assert b"length" in lib.ls_last_error() or b"mode" in lib.ls_last_error()
    assert lib.ls_expand(None, 4, None, 4, None, 4, None, 4, 4, 4, 3, 2, 5, None, 0, 0, None, None, None, None,
                         None) == _abi.LS_EVALIDATION
    assert lib.ls_assemble_axis(None, 16, 3, 1, None, 8, 1, 0, None, 4, None) == _abi.LS_EVALIDATION
    # pipeline entry points reject a null handle; shape errors of the grid batch come first
    assert lib.ls_pipeline_generate(None, None) == _abi.LS_EVALIDATION
    assert lib.ls_pipeline_energy(None, None, None, None, 0, 1, None, None) == _abi.LS_EVALIDATION
    assert b"null handle" in lib.ls_last_error()
    assert lib.ls_grid_functional_batch(None, 4, 4, 4, 3, 16, None, 4, None, 4, None, 4, 2, 1.0, 0, None,
                                        None) == _abi.LS_EVALIDATION


def test_device_work_without_a_gpu_fails_loudly():
    """No CPU fallback: a valid call that needs the device returns LS_ECUDA (the headers throw
    device_error, the Python mirror raises CudaError) when no CUDA device is usable."""
    import ctypes as C
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    lib = _abi.load()
    dims = np.array([2, 2, 2], dtype=np.int64)
    f, w = np.ones((2, 1)), np.ones(1)
    idx, out = np.zeros(3, dtype=np.int64), np.zeros(1)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    assert lib.ls_h_eval_points(p(dims), 1, p(f), p(f), p(f), p(w), p(idx), 1, p(out)) == _abi.LS_ECUDA
    assert lib.ls_last_error()
    import paper_1405_2270_b200 as L
    with pytest.raises(L.CudaError):
        L.densify(L.CanonicalTensor3([np.ones((2, 1))] * 3, np.ones(1)))


def test_expansion_plan_names():
    """Plan selection is host logic (no device needed): BASELINE rank 41 takes the 8-warp TMEM
    kernel compiled for KD 10; 2-charge rank 82 the 16-warp TMEM one; 122-160 the single-buffer
    16-warp TMEM one; cfg3's 328 the split-K TMEM plan."""
    assert L.expansion_plan(41).startswith("expand_tmem_kernel, 8 warps x 2 CTAs/SM")
    assert "KD 10 (compiled)" in L.expansion_plan(41)
    assert L.expansion_plan(82).startswith("expand_tmem_kernel, 16 warps x 1 CTA/SM")
    assert "two stages per tile" in L.expansion_plan(113)
    assert "single A1k buffer" in L.expansion_plan(122)
    assert "single A1k buffer" in L.expansion_plan(160)
    assert L.expansion_plan(328).startswith("expand_splitk_kernel")
    assert "256-rank chunks" in L.expansion_plan(600)
    with pytest.raises(L.ValidationError):
        L.expansion_plan(-1)


def test_python_mirror_validation():  # lattice.hpp:57-68, grid.hpp:21-27, canonical.hpp:42-56
    with pytest.raises(L.ValidationError):
        L.GridSpec(2.0, 3)
    with pytest.raises(L.ValidationError):
        L.GridSpec(-1.0, 4)
    spec = L.LatticeSpec((1, 1, 1), L.GridSpec(2.0, 8), [L.Charge((0.1, 0.0, 0.0), 1.0)])
    with pytest.raises(L.ValidationError):
        spec.validate()
    spec = L.LatticeSpec((1, 1, 1), L.GridSpec(2.0, 8), [L.Charge((0.25, -1.0, 1.0), 1.0)])
    spec.validate()
    assert [spec.charge_grid_index(l, 0) for l in range(3)] == [5, 0, 8]
    with pytest.raises(L.ValidationError):
        L.LatticeSpec((0, 2, 2), L.GridSpec(2.0, 8), [L.Charge()]).validate()
    with pytest.raises(L.ValidationError):
        L.LatticeSpec((2, 2, 2), L.GridSpec(2.0, 8), []).validate()
    with pytest.raises(L.ValidationError):
        L.LatticeSpec((2, 2, 2), L.GridSpec(2.0, 8), [L.Charge((0, 0, 0), -1.0)]).validate()
    with pytest.raises(L.ValidationError):
        L.CanonicalTensor3([np.ones((2, 1)), np.ones((2, 2)), np.ones((2, 1))], np.ones(1))
    with pytest.raises(L.ValidationError):
        L.CanonicalTensor3([np.ones((2, 1))] * 3, np.array([np.inf]))
    with pytest.raises(L.ResourceGuardError):
        L.densify(L.CanonicalTensor3([np.ones((8, 1))] * 3, np.ones(1)), guard=100)


def test_windows_match_reference_formulae(orc):
    for N, n, ia, k, Lc in [(16, 8, 8, 0, 2), (64, 8, 3, 5, 8), (32768, 256, 128, 0, 128)]:
        assert L.window_start_box(N, n, ia, k) == orc._window_start_box(N, n, ia, k)
        assert L.window_start_periodic(N, n, ia, k, Lc) == orc._window_start_periodic(N, n, ia, k, Lc)
