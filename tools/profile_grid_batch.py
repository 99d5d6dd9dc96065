"""Times the cfg4 full-grid functional batch (256^3 periodic, F = 1024) for ncu / A-B runs.

  python tools/profile_grid_batch.py [--reps 10] [--F 1024]
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
ap.add_argument("--F", type=int, default=1024)
args = ap.parse_args()
spec = L.LatticeSpec((256,) * 3, L.GridSpec(10.0, 256), [L.Charge((0, 0, 0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3) * 256 * 10.0, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=True)
pipe.generate()
pipe.assemble()
rng = np.random.default_rng(4)
G = [torch.as_tensor(rng.uniform(0, 1, (256, args.F)), device="cuda") for _ in range(3)]
ts = []
for r in range(args.reps + 1):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    pipe.grid_functional_batch(G)
    e[1].record()
    torch.cuda.synchronize()
    ts.append(e[0].elapsed_time(e[1]))
ts = sorted(ts[1:])
flop = 2.0 * 256 ** 3 * args.F
print(f"grid functional batch F={args.F}: {ts[0]:.3f} ms (median {ts[len(ts) // 2]:.3f}), "
      f"{flop / ts[0] / 1e9:.1f} TF/s incl. expansion")
