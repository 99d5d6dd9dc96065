"""A/B of small-grid expansion builds: device time per ls_expand call (back-to-back launches)
and a hash of every output grid, so variants can be compared for speed and bitwise equality
in one GPU call.

  for v in o0 o7; do LS_LAB_ROOT=/root/repo/labx/$v python tools/lab/a2t_ab.py --tag $v; done
"""
import argparse
import hashlib
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="")
ap.add_argument("--cases", default="256x256x256:41,256x256x256:57,256x256x256:21,256x128x256:41,"
                                   "200x250x37:41,256x256x512:9,130x97x300:53")
ap.add_argument("--reps", type=int, default=50)
args = ap.parse_args()
for case in args.cases.split(","):
    s, r = case.split(":")
    n1, n2, ks = map(int, s.split("x"))
    R = int(r)
    g = torch.Generator(device="cuda").manual_seed(1000 + R + n1 + 7 * n2 + 13 * ks)
    out = torch.full((ks, n2, n1), float("nan"), dtype=torch.float64, device="cuda")
    fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) - 0.5 for m in (n1, n2, ks)]
    w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    torch.cuda.synchronize()
    h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()[:12]
    for _ in range(5):
        _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        for _ in range(args.reps):
            _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
        e[1].record()
        torch.cuda.synchronize()
        best = min(best, e[0].elapsed_time(e[1]) / args.reps)
    print(f"{args.tag:6s} {s:>12s} R={R:3d}: {best * 1e3:7.2f} us/call {2.0 * R * n1 * n2 * ks / best / 1e9:6.2f} TF/s "
          f"hash {h}", flush=True)
