"""Times calibrate_for_lattice (the reference CLI's dominant cost) on the GPU vs the reference."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_1405_2270_b200 as L  # noqa: E402
from oracle import reference  # noqa: E402

r = reference()
r.lib.ref_calibrate_for_lattice.restype = C.c_int
r.lib.ref_calibrate_for_lattice.argtypes = [C.POINTER(C.c_int64), C.c_int64, C.c_double, C.c_double,
                                            C.POINTER(C.c_double)]
for Lc, n, eps in ((8, 16, 1e-6), (16, 64, 1e-6), (32, 64, 1e-6)):
    spec = L.LatticeSpec((Lc,) * 3, L.GridSpec(10.0, n), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    L.calibrate_for_lattice(spec, eps)  # warm-up
    t0 = time.perf_counter()
    rule = L.calibrate_for_lattice(spec, eps)
    tg = time.perf_counter() - t0
    Lx = np.array(spec.L, dtype=np.int64)
    c0 = C.c_double(0)
    t0 = time.perf_counter()
    M = r.lib.ref_calibrate_for_lattice(Lx.ctypes.data_as(C.POINTER(C.c_int64)), n, 10.0, eps, C.byref(c0))
    tr = time.perf_counter() - t0
    print(f"L={Lc} n={n} eps={eps}: gpu M={rule.M} C0={rule.C0} {tg*1e3:.1f} ms | ref M={M} C0={c0.value} "
          f"{tr*1e3:.1f} ms ({r._max_threads()} threads)")
