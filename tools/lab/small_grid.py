"""Device time per ls_expand call on small grids, back-to-back launches (host overhead hidden
behind the queue), R = 41 random factors.

  python tools/lab/small_grid.py [--shapes 256x256x256,512x512x512] [--reps 50]
"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shapes", default="256x256x256,512x512x512")
ap.add_argument("--R", type=int, default=41)
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(1)
R = args.R
for s in args.shapes.split(","):
    n1, n2, ks = map(int, s.split("x"))
    out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
    fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, ks)]
    w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
    for _ in range(5):
        _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(args.reps):
            _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
        e[1].record()
        torch.cuda.synchronize()
        best = min(best, e[0].elapsed_time(e[1]) / args.reps)
    print(f"{s} R={R}: {best * 1e3:.1f} us/call, {2.0 * R * n1 * n2 * ks / best / 1e9:.2f} TF/s", flush=True)
