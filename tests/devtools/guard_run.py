"""Guard-page run of the CUDA entry points (test_gpu_guard.py runs it in a subprocess).

compute-sanitizer is closed on the GPU pool, so out-of-bounds device accesses are caught here by
the MMU instead: every input and output buffer of a call gets its own virtual-address range
(cuMemAddressReserve) with only the pages the buffer needs mapped (cuMemCreate/cuMemMap) and an
unmapped guard granule on each side. The buffer is placed flush against the upper guard
("end": an access one element past the last one faults) or the lower guard ("start": an access
one element before the first faults). A stray read or write then ends in an illegal-address
error instead of silently touching a neighbour, and this process exits non-zero.

  python tests/devtools/guard_run.py end|start|control
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch
from cuda.bindings import driver as drv

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_1405_2270_b200 import _abi  # noqa: E402


def _ok(res):
    err = res[0] if isinstance(res, tuple) else res
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"driver call failed: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class Arena:
    """Guarded device buffers, each alone in its own reserved range."""

    def __init__(self, placement: str):
        self.placement = placement
        self.prop = drv.CUmemAllocationProp()
        self.prop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        self.prop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        self.prop.location.id = torch.cuda.current_device()
        self.gran = int(_ok(drv.cuMemGetAllocationGranularity(
            self.prop, drv.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM)))
        self.live = []

    def alloc(self, arr: np.ndarray) -> int:
        """Copies the float64/int64 array into a guarded buffer; returns its device address."""
        nbytes = max(arr.nbytes, 8)
        g = self.gran
        mapped = (nbytes + g - 1) // g * g
        va = int(_ok(drv.cuMemAddressReserve(mapped + 2 * g, 0, 0, 0)))
        h = _ok(drv.cuMemCreate(mapped, self.prop, 0))
        _ok(drv.cuMemMap(drv.CUdeviceptr(va + g), mapped, 0, h, 0))
        desc = drv.CUmemAccessDesc()
        desc.location = self.prop.location
        desc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        _ok(drv.cuMemSetAccess(drv.CUdeviceptr(va + g), mapped, [desc], 1))
        ptr = va + g + (mapped - nbytes if self.placement == "end" else 0)
        if arr.nbytes:
            src = np.ascontiguousarray(arr)
            _ok(drv.cuMemcpyHtoD(drv.CUdeviceptr(ptr), src.ctypes.data, arr.nbytes))
        self.live.append((va, mapped, h))
        return ptr

    def read(self, ptr: int, n: int, dtype=np.float64) -> np.ndarray:
        out = np.empty(n, dtype=dtype)
        _ok(drv.cuMemcpyDtoH(out.ctypes.data, drv.CUdeviceptr(ptr), out.nbytes))
        return out

    def free(self):
        for va, mapped, h in self.live:
            _ok(drv.cuMemUnmap(drv.CUdeviceptr(va + self.gran), mapped))
            _ok(drv.cuMemRelease(h))
            _ok(drv.cuMemAddressFree(drv.CUdeviceptr(va), mapped + 2 * self.gran))
        self.live = []


def _check(lib, rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: status {rc}: {lib.ls_last_error().decode()}")
    torch.cuda.synchronize()
    if lib.ls_fault_status(1) != 0:
        raise RuntimeError(f"{what}: device watchdog fired")


# (N1, N2, N3, R, k0, k1, pad_y, pad_z): every expansion plan with ragged edges -- A2-in-TMEM
# (N2 <= 256), the 8- and 16-warp TMEM plans, the single-buffer TMEM plan, split-K, tiny ranks.
EXPAND = [(200, 256, 9, 41, 0, 9, 0, 0), (256, 130, 7, 57, 2, 7, 3, 8), (130, 77, 5, 9, 1, 4, 0, 2),
          (300, 300, 4, 41, 0, 4, 1, 0), (257, 129, 3, 70, 0, 3, 0, 0), (129, 257, 3, 164, 1, 3, 0, 4),
          (130, 140, 2, 300, 0, 2, 0, 0), (61, 33, 3, 1, 0, 3, 1, 1), (70, 70, 3, 3, 0, 3, 0, 0),
          (128, 1, 2, 54, 0, 2, 0, 0), (1, 128, 2, 5, 0, 2, 0, 0)]


def control() -> int:
    """Negative control: an A factor one element short of what the call is told (N1 x R with the
    last element missing) must fault against the guard, proving the harness catches overruns."""
    torch.zeros(1, device="cuda")
    lib = _abi.load()
    rng = np.random.default_rng(6)
    arena = Arena("end")
    n1, n2, n3, R = 200, 256, 4, 41
    f = [rng.uniform(0.05, 1.0, (R, d)) for d in (n1, n2, n3)]
    pa = arena.alloc(f[0].reshape(-1)[:-1])  # short by one element
    pb, pc, pw = (arena.alloc(x) for x in (f[1], f[2], rng.uniform(0.05, 1.0, R)))
    po = arena.alloc(np.zeros(n1 * n2 * n3))
    rc = lib.ls_expand(C.c_void_p(pa), n1, C.c_void_p(pb), n2, C.c_void_p(pc), n3, C.c_void_p(pw), n1, n2, n3, R, 0,
                       n3, C.c_void_p(po), n1, n1 * n2, None, None, None, None, None)
    try:
        torch.cuda.synchronize()
    except RuntimeError as e:  # the expected illegal-address error
        print(f"fault caught: {str(e).splitlines()[0]}")
        return 3
    print(f"no fault (rc {rc})")
    return 0


def main(placement: str) -> int:
    if placement == "control":
        return control()
    torch.zeros(1, device="cuda")  # primary context current on this thread
    lib = _abi.load()
    rng = np.random.default_rng(5)
    arena = Arena(placement)
    n_calls = 0
    V = C.c_void_p
    for (n1, n2, n3, R, k0, k1, py, pz) in EXPAND:
        f = [rng.uniform(0.05, 1.0, (R, d)) for d in (n1, n2, n3)]  # (R, N) rows = column-major N x R
        w = rng.uniform(0.05, 1.0, R)
        ldy, nk = n1 + py, k1 - k0
        ldz = ldy * n2 + pz
        pa, pb, pc, pw = (arena.alloc(x) for x in (*f, w))
        po = arena.alloc(np.full(nk * ldz, np.nan))
        _check(lib, lib.ls_expand(V(pa), n1, V(pb), n2, V(pc), n3, V(pw), n1, n2, n3, R, k0, k1, V(po), ldy, ldz,
                                  None, None, None, None, None), f"expand {n1}x{n2}x{n3} R={R}")
        got = arena.read(po, nk * ldz)
        want = np.einsum("qi,qj,qk,q->kji", f[0], f[1], f[2][:, k0:k1], w)
        for kk in range(nk):
            sl = got[kk * ldz: kk * ldz + n2 * ldy].reshape(n2, ldy)[:, :n1]
            assert np.max(np.abs(sl - want[kk])) <= 1e-12 * np.max(np.abs(want)), (n1, n2, n3, R)
        # fused functional: rho vectors and the partials guarded too
        rho = [rng.uniform(0.1, 1.0, d) for d in (n1, n2, n3)]
        pr = [arena.alloc(x) for x in rho]
        npart = int(lib.ls_expand_partial_count(n1, n2, R, k0, k1))
        pp = arena.alloc(np.zeros(max(npart, 1)))
        pe = arena.alloc(np.zeros(1))
        _check(lib, lib.ls_expand(V(pa), n1, V(pb), n2, V(pc), n3, V(pw), n1, n2, n3, R, k0, k1, None, 0, 0,
                                  V(pr[0]), V(pr[1]), V(pr[2]), V(pp), None), f"energy R={R}")
        _check(lib, lib.ls_sum_partials(V(pp), npart, V(pe), None), "sum_partials")
        e = arena.read(pe, 1)[0]
        e_want = float(np.einsum("kji,i,j,k->", want, rho[0], rho[1], rho[2][k0:k1]))
        assert abs(e - e_want) <= 1e-12 * abs(e_want), (e, e_want)
        # batch of F functionals over the stored grid (the grid itself is the guarded output above)
        F = 5
        X, Y, Z = (rng.uniform(0.1, 1.0, (F, d)) for d in (n1, n2, nk))
        px, py_, pz_ = (arena.alloc(x) for x in (X, Y, Z))
        pf = arena.alloc(np.zeros(F))
        _check(lib, lib.ls_grid_functional_batch(V(po), n1, n2, nk, ldy, ldz, V(px), n1, V(py_), n2, V(pz_), nk, F,
                                                 1.0, 0, V(pf), None), "grid_functional_batch")
        fb = arena.read(pf, F)
        fb_want = np.einsum("kji,fi,fj,fk->f", want, X, Y, Z)
        assert np.max(np.abs(fb - fb_want) / np.abs(fb_want)) <= 1e-12
        n_calls += 4
        arena.free()
    # K1 + K2: generator masters and the assembled axis, guarded
    tau = rng.uniform(0.5, 40.0, 9)
    for mode in (0, 1):
        for (L, n, M0, periodic) in ((4, 16, 1, 0), (6, 10, 3, 1), (1, 8, 2, 0)):
            R = tau.size
            ln = 2 * L * n
            pt = arena.alloc(tau)
            pm = arena.alloc(np.full(ln * R, np.nan))
            _check(lib, lib.ls_gen_master(mode, V(pt), R, ln, 0.25, V(pm), ln, None), "gen_master")
            master = arena.read(pm, ln * R)
            assert np.isfinite(master).all()
            ia = rng.integers(0, n + 1, M0).astype(np.int64)
            pia = arena.alloc(ia)
            dim = L * n if not periodic else n
            pf_ = arena.alloc(np.full(dim * M0 * R, np.nan))  # dim x M0*R, column nu*R + q
            _check(lib, lib.ls_assemble_axis(V(pm), ln, R, M0, V(pia), n, L, periodic, V(pf_), dim, None),
                   "assemble_axis")
            assert np.isfinite(arena.read(pf_, dim * M0 * R)).all()
            n_calls += 2
            arena.free()
    print(f"ok {n_calls} guarded calls ({placement})")
    return 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1] if len(sys.argv) > 1 else "end"))
