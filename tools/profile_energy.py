"""Times the fused full-grid functional <V, rho> at cfg1 (store-free expansion) for A/B runs.

  python tools/profile_energy.py [--reps 10] [--L 16]
"""
import argparse
import math
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--L", type=int, default=16)
args = ap.parse_args()
spec = L.LatticeSpec((args.L,) * 3, L.GridSpec(10.0, 64), [L.Charge((0, 0, 0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3) * args.L * 10.0, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode="erf")
pipe.generate()
pipe.assemble()
N = pipe.dims
rho = [torch.as_tensor(np.exp(-((np.arange(n) + 0.5 - n / 2) * spec.unit.h) ** 2 / 2), device="cuda") for n in N]
e = pipe.grid_functional(rho)
ts = []
for _ in range(args.reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    e = pipe.grid_functional(rho)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
print(f"energy {N[0]}x{N[1]}x{N[2]}: {ts[0]:.3f} ms (median {ts[len(ts) // 2]:.3f}), value {float(e.cpu()):.15g}")
