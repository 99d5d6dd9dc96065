"""Randomized soak of the functional entry points (K4) against numpy: functional_batch (the 1D
rank-term form, every Gram path: 4-density and single-density shared-memory kernels and the
global-scratch path for large ranks) and grid_functional_batch (the full-grid form fused into the
expansion), random ranks, batch sizes and shapes, positive factors (no cancellation), bar 1e-12.

  python tools/lab/fuzz_functionals.py [--cases 400] [--seed 5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=400)
ap.add_argument("--seed", type=int, default=5)
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
t0, fails, worst = time.time(), 0, 0.0
for c in range(args.cases):
    grid = rng.integers(0, 3) == 0  # every third case: the full-grid form too
    R = int(rng.choice([rng.integers(1, 64), rng.integers(64, 700), rng.integers(700, 3000)], p=[0.5, 0.35, 0.15]))
    if grid:
        R = min(R, 600)
    F = int(rng.choice([rng.integers(1, 16), rng.integers(16, 900)]))
    dims = tuple(int(x) for x in rng.integers(1, 40 if grid else 70, 3))
    fac = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], R))) for l in range(3)]
    w = rng.uniform(0.5, 1.5, R)
    G = [np.asfortranarray(rng.uniform(0.1, 1.0, (dims[l], F))) for l in range(3)]
    t = L.CanonicalTensor3(fac, w, trusted=True)
    gram = [fac[l].T @ G[l] for l in range(3)]  # (R, F)
    want = np.einsum("q,qf,qf,qf->f", w, gram[0], gram[1], gram[2])
    got = np.asarray(L.functional_batch(t, G))
    err = float(np.max(np.abs(got - want) / np.abs(want)))
    if grid:
        gg = np.asarray(L.grid_functional_batch(t, G))
        err = max(err, float(np.max(np.abs(gg - want) / np.abs(want))))
    worst = max(worst, err)
    if not err <= 1e-12:
        fails += 1
        print(f"FAIL case {c}: R={R} F={F} dims={dims} grid={grid}: rel {err:.2e}", flush=True)
print(f"{args.cases} cases, {fails} failures, worst rel {worst:.2e}, {time.time() - t0:.0f} s")
