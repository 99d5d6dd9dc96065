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
    ranks = [1, 2, 3, 4, 5, 8, 40, 41, 42, 43, 45, 46, 57, 58, 61, 70, 73, 82, 89, 93, 94, 123, 164, 257, 300, 520]
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
    # padding between rows / slabs is never written
    if pad_y:
        assert np.isnan(got_flat[n1:ldy]).all()
    if func:
        e = torch.zeros(1, dtype=torch.float64, device=dev)
        assert lib.ls_sum_partials(p(part), int(lib.ls_expand_partial_count(n1, n2, R, k0, k1)), p(e), s) == 0
        r = [x.cpu().numpy() for x in rho]
        e_want = float(np.einsum("ijk,i,j,k->", want, r[0], r[1], r[2][k0:k1]))
        assert abs(float(e.cpu()) - e_want) <= 1e-13 * abs(e_want)
