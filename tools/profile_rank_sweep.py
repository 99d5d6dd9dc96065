"""Times ls_expand over a rank sweep on random factors (plan selection study).

  python tools/profile_rank_sweep.py [--n 1024] [--slabs 64] [--ranks 60,82,164,328]
Set LS_EXPAND_PLAN / LS_EXPAND_KC in the environment to force a plan (needs the dev build:
`python -m paper_1405_2270_b200.build --dev`; the product library ignores them).
"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--slabs", type=int, default=64)
ap.add_argument("--ranks", default="60,82,123,164,246,328")
ap.add_argument("--n1", type=int, default=0, help="rows along i (default --n)")
ap.add_argument("--n2", type=int, default=0, help="rows along j (default --n)")
args = ap.parse_args()
n, ks = args.n, args.slabs
n1, n2 = args.n1 or n, args.n2 or n
out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
g = torch.Generator(device="cuda").manual_seed(1)
for R in map(int, args.ranks.split(",")):
    fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, max(ks, 1))]
    w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
        e[1].record()
        torch.cuda.synchronize()
        best = min(best, e[0].elapsed_time(e[1]))
    print(f"{n1}x{n2}x{ks} R={R:4d}: {best:.3f} ms, {2.0 * R * n1 * n2 * ks / best / 1e9:.2f} TF/s")
