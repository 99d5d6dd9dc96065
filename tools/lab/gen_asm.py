"""Device time of the generator and the assembly per call (cfg4 periodic L = 64/128/256 with
n = 256, cfg1 box L = 16, cfg3 box L = 32 with 8 charges), back-to-back launches.

  python tools/lab/gen_asm.py [--reps 50]
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
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()
B = 10.0


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / args.reps)
    return best * 1e3


cases = [("cfg4 L=64", 64, 256, 1, True), ("cfg4 L=128", 128, 256, 1, True), ("cfg4 L=256", 256, 256, 1, True),
         ("cfg1", 16, 64, 1, False), ("cfg3", 32, 64, 8, False)]
rng = np.random.default_rng(20241019)
for name, Lc, n, M0, periodic in cases:
    h = B / n
    if M0 == 1:
        charges = [L.Charge((0.0, 0.0, 0.0), 1.0)]
    else:
        ia = rng.integers(7, 58, size=(M0, 3))
        charges = [L.Charge(tuple(ia[c] * h - B / 2), float(c + 1)) for c in range(M0)]
    spec = L.LatticeSpec((Lc, Lc, Lc), L.GridSpec(B, n), charges)
    rule = L.sinc_quadrature(1e-6, h, math.sqrt(3.0) * Lc * B, 20, 1.0)
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=periodic)
    tg = timed(pipe.generate)
    ta = timed(pipe.assemble)
    tp = timed(pipe.prepare)
    print(f"{name}: master {2 * Lc * n} x {rule.node_count()}: generate {tg:.1f} us, assemble {ta:.1f} us, "
          f"prepare {tp:.1f} us "
          f"({pipe.Rt} columns of {n if periodic else Lc * n})", flush=True)
