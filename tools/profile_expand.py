"""Runs the cfg1 hot path a few times so ncu can capture the expansion kernel.

  python tools/profile_expand.py [--steps S] [--L 16] [--charges 1]
"""
import argparse
import math
import sys

import os  # noqa: E402
sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--L", type=int, default=16)
ap.add_argument("--slabs", type=int, default=0, help="expand only this many slabs (0 = all)")
ap.add_argument("--mode", default="erf")
ap.add_argument("--reps", type=int, default=1)
args = ap.parse_args()
spec = L.LatticeSpec((args.L,) * 3, L.GridSpec(10.0, 64), [L.Charge((0, 0, 0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3) * args.L * 10.0, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode=args.mode)
N1, N2, N3 = spec.target_dims()
k1 = args.slabs or N3
out = torch.empty((k1, N2, N1), dtype=torch.float64, device="cuda")
for s in range(args.steps):
    pipe.step(out, 0, k1)
torch.cuda.synchronize()
ts = []
for r in range(args.reps):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    pipe.expand(out, 0, k1)
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
print(f"expand {N1}x{N2}x{k1} R={pipe.Rt}: {ts[0]:.3f} ms (median {ts[len(ts) // 2]:.3f} of {len(ts)})")
