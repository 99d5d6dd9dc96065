"""Quick GPU-vs-oracle parity probe used during development (not a test)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1405_2270_b200 as L
from oracle import restatement, reference, ref_available

o = restatement()
r = reference() if ref_available() else None
def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))

n, Lc, b = 64, 4, 10.0
spec = L.LatticeSpec((Lc, Lc, Lc), L.GridSpec(b, n), [L.Charge((0, 0, 0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, 3**0.5 * Lc * b, 20, 1.0)
for mode in ("midpoint", "erf"):
    m = L.build_lattice_master(spec, rule, mode)
    fo = o.lattice_master(0 if mode == "midpoint" else 1, [Lc] * 3, n, b, rule.exponents)
    print(mode, "master rel", max(rel(m.factor(l), fo[l]) for l in range(3)),
          "bitwise", all(np.array_equal(m.factor(l), fo[l]) for l in range(3)),
          "ulp-mismatch frac", np.mean(m.factor(0) != fo[0]))
    s = L.assembled_box_sum(spec, m)
    ia = np.array([n // 2], dtype=np.int64)
    import ctypes as C
    ao = np.zeros((Lc * n, rule.node_count()), order="F")
    o._assembled_axis(fo[0].ctypes.data_as(C.POINTER(C.c_double)), rule.node_count(), 1,
                      ia.ctypes.data_as(C.POINTER(C.c_int64)), n, Lc, 0, ao.ctypes.data_as(C.POINTER(C.c_double)))
    # assemble the oracle master with the GPU to check bitwise adds
    s_or = L.assembled_box_sum(spec, L.CanonicalTensor3(fo, rule.weights, trusted=True))
    print("  assembly: gpu(oracle master) bitwise vs oracle:", np.array_equal(s_or.tensor.factor(0), ao),
          " gpu vs oracle rel:", rel(s.tensor.factor(0), ao))
    t = s.tensor
    t0 = time.time(); V = L.densify(t); t1 = time.time()
    Vo = o.densify_slabs(t.factor(0), t.factor(1), t.factor(2), t.weights(), 0, 8)
    print("  densify first 8 slabs rel", rel(V[:, :, :8], Vo), "time", t1 - t0)
    pts = np.array([[128, 128, 128], [0, 0, 0], [255, 3, 77], [17, 200, 255]])
    ev = L.eval_points(t, pts)
    evo = [o.eval_point(t.factor(0), t.factor(1), t.factor(2), t.weights(), *p) for p in pts]
    print("  eval_points", ev, evo, "dense", [V[tuple(p)] for p in pts])
# random small tensors, odd sizes, various ranks
rng = np.random.default_rng(0)
for dims, R in [((5, 7, 3), 3), ((33, 17, 9), 41), ((130, 66, 4), 45), ((64, 64, 8), 328), ((2, 2, 2), 1), ((257, 129, 3), 8)]:
    f = [np.asfortranarray(rng.uniform(-1, 1, (d, R))) for d in dims]
    w = rng.uniform(-1, 1, R)
    t = L.CanonicalTensor3(f, w)
    V = L.expand_slabs(t, 0, dims[2])
    Vo = o.densify_slabs(f[0], f[1], f[2], w)
    rho = [rng.uniform(0, 1, d) for d in dims]
    g = L.grid_functional(t, rho)
    go = float(np.einsum("ijk,i,j,k->", Vo, *rho))
    sp = L.scalar_product(t, t)
    spo = o.scalar_product(f, w, f, w)
    print(dims, R, "densify rel", rel(V, Vo), "functional rel", abs(g - go) / abs(go), "sp rel", abs(sp - spo) / abs(spo))
