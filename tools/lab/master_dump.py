"""Dumps generator masters (both modes) for an A/B bitwise comparison between two builds:

  LS_LAB_ROOT=<build A> python tools/lab/master_dump.py a.npz
  python tools/lab/master_dump.py b.npz && python tools/lab/master_dump.py --compare a.npz b.npz
"""
import math
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print(f"{len(a.files)} masters compared, {len(bad)} differ: {bad[:5]}")
    sys.exit(1 if bad else 0)

import paper_1405_2270_b200 as L  # noqa: E402

out = {}
for Lc, n in ((4, 64), (16, 64), (32, 64), (64, 256), (256, 256), (3, 6), (1, 2)):
    b = 10.0
    spec = L.LatticeSpec((Lc, Lc, Lc), L.GridSpec(b, n), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.sinc_quadrature(1e-6, b / n, math.sqrt(3.0) * Lc * b, 20, 1.0)
    tau = np.concatenate([[0.0], rule.exponents[:-1]])  # include a t = 0 column, keep 2M+1
    rule0 = L.QuadratureRule(rule.M, rule.C0, rule.step, None, tau, np.ones(len(tau)))
    for mode in ("erf", "midpoint"):
        out[f"{mode}_{Lc}_{n}"] = L.build_lattice_master(spec, rule0, mode).factor(0)
np.savez(sys.argv[1], **out)
print("saved", len(out))
