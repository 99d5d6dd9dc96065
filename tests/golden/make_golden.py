"""Generates tests/golden/golden_r01.npz from the reference's OWN code.

Run in the build container (needs oracle/_ref, i.e. /root/reference compiled
unmodified by `make -C oracle ref`):  python tests/golden/make_golden.py

Every array is produced by the reference headers (oracle/ref_capi.cpp); the
fixture travels with the repo so GPU-box tests can pin both the C
restatement and the CUDA path without /root/reference.
"""
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle import reference  # noqa: E402

import ctypes as C  # noqa: E402

dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
i64p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731


def assembled(r, periodic, L, n, b, charges, master, w):
    L = np.asarray(L, dtype=np.int64)
    ch = np.asarray(charges, dtype=np.float64)
    M0, R = len(ch), len(w)
    dims = [n if periodic else int(L[l]) * n for l in range(3)]
    f = [np.zeros((dims[l], M0 * R), order="F") for l in range(3)]
    wout = np.zeros(M0 * R)
    r._check(r._assembled_sum(int(periodic), i64p(L), n, b, dp(ch.ravel()), M0, dp(master[0]), dp(master[1]),
                              dp(master[2]), dp(np.ascontiguousarray(w)), R, dp(f[0]), dp(f[1]), dp(f[2]), dp(wout),
                              None), "assembled_sum")
    return f, wout


def main():
    r = reference()
    g = {}
    # cfg0: n=64, L=4, b=10, one unit charge at the cell centre, M=20.
    n, L, b = 64, 4, 10.0
    h = b / n
    nodes, tau, w, step = r.sinc_quadrature(1e-6, h, math.sqrt(3) * L * b, 20, 1.0)
    g.update(cfg0_nodes=nodes, cfg0_tau=tau, cfg0_w=w, cfg0_step=np.array([step]))
    for mode, name in ((0, "mid"), (1, "erf")):
        m = r.lattice_master(mode, [L, L, L], n, b, tau, w)
        g[f"cfg0_master_{name}"] = m[0]  # cubic: all three axes identical
        f, wout = assembled(r, False, [L, L, L], n, b, [[0, 0, 0, 1.0]], m, w)
        g[f"cfg0_asm_{name}"] = f[0]
        g["cfg0_asm_w"] = wout
        # sampled grid values of the assembled tensor (densify_slab over a few slabs)
        slabs = [37, 128]
        vals = np.stack([r.densify_slabs(f[0], f[1], f[2], wout, k, k + 1)[:, :, 0] for k in slabs], axis=-1)
        g[f"cfg0_slabs_{name}"] = vals
        g["cfg0_slab_ids"] = np.array(slabs)
        pts = np.array([[128, 128, 128], [0, 0, 0], [255, 3, 77], [17, 200, 255], [64, 64, 64]], dtype=np.int64)
        g[f"cfg0_points_{name}"] = np.array([r.eval_point(f[0], f[1], f[2], wout, *p) for p in pts])
        g["cfg0_point_idx"] = pts
    # multi-charge non-cubic box and periodic sums (b=2, n=8), rule M=10
    ch = np.array([[0.0, 0.0, 0.0, 1.0], [0.5, -0.25, 0.25, 2.0], [-0.75, 0.5, 0.0, 0.5]])
    Lm = [3, 2, 2]
    nodes, tau, w, step = r.sinc_quadrature(1e-4, 0.25, math.sqrt(3) * 3 * 2.0, 10, 1.0)
    g.update(mc_tau=tau, mc_w=w, mc_charges=ch, mc_L=np.array(Lm))
    m = r.lattice_master(0, Lm, 8, 2.0, tau, w, ch)
    for l in range(3):
        g[f"mc_master_{l}"] = m[l]
    f, wout = assembled(r, False, Lm, 8, 2.0, ch, m, w)
    for l in range(3):
        g[f"mc_box_{l}"] = f[l]
    g["mc_box_w"] = wout
    d = np.zeros((24, 16, 16), order="F")
    r._check(r._densify(24, 16, 16, len(wout), dp(f[0]), dp(f[1]), dp(f[2]), dp(wout), 1 << 27, dp(d)), "densify")
    g["mc_box_dense"] = d
    fp, wp = assembled(r, True, Lm, 8, 2.0, ch, m, w)
    for l in range(3):
        g[f"mc_per_{l}"] = fp[l]
    dpd = np.zeros((8, 8, 8), order="F")
    r._check(r._densify(8, 8, 8, len(wp), dp(fp[0]), dp(fp[1]), dp(fp[2]), dp(wp), 1 << 27, dp(dpd)), "densify")
    g["mc_per_dense"] = dpd
    # scalar products and a potential matrix on the periodic tensor
    centers = np.array([[0.0, 0.0, 0.0], [0.25, -0.5, 0.5], [-0.5, 0.25, 0.0]])
    sig = np.array([0.4, 0.7, 0.3])
    V = np.zeros((3, 3), order="F")
    r._check(r._potential_matrix(2.0, 8, 3, dp(centers.ravel()), dp(sig), len(wp), dp(fp[0]), dp(fp[1]), dp(fp[2]),
                                 dp(wp), 1, dp(V)), "potential_matrix")
    g.update(pm_centers=centers, pm_sigmas=sig, pm_V=V)
    g["mc_box_selfdot"] = np.array([r.scalar_product(f, wout, f, wout)])
    # erf moment KAT columns (newton.hpp:21-37): b=3, n=6, t=0.7, both lengths
    g["moment_b3_n6_t07"] = r.gaussian_moment_vector(3.0, 6, 0.7, False)
    g["moment_b3_n6_t07_doubled"] = r.gaussian_moment_vector(3.0, 6, 0.7, True)
    # a bundle file written by the reference's own save_bundle (bundle.hpp:33-54)
    r.lib.ref_save_bundle.restype = C.c_int
    r.lib.ref_save_bundle.argtypes = [C.c_char_p] + [C.c_int64] * 3 + [C.c_int] + [C.POINTER(C.c_double)] * 4 + \
        [C.c_double] * 4
    bpath = ROOT / "tests" / "golden" / "ref_bundle_mc_box.bin"
    r._check(r.lib.ref_save_bundle(str(bpath).encode(), 24, 16, 16, len(wout), dp(f[0]), dp(f[1]), dp(f[2]),
                                   dp(wout), 0.25, -2.875, -1.875, -1.875), "save_bundle")
    out = ROOT / "tests" / "golden" / "golden_r01.npz"
    np.savez_compressed(out, **g)
    print(out, out.stat().st_size, "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
