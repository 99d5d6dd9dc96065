"""Per-warp event timeline of one TMEM expansion launch (lab build with -DLS_TIMELINE, see
k3.cuh): where a CTA's time goes on small grids.

  LAB_DIR=labx tools/lab/build_lab.sh tl "-DLS_DEV_KNOBS -DLS_TIMELINE"
  LS_LAB_ROOT=/root/repo/labx/tl python tools/lab/timeline.py --shape 256x256x256
Events: 1 set-up done, 2 prologue fill published, 3 unit A1k ready, 7 stage loop top,
4 stage landed, 5 DMMAs issued, 6 slot released + fill tasks done, 8 all units done.
"""
import argparse
import os
import statistics
import sys
from collections import defaultdict

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

os.environ["LS_TIMELINE"] = "1"
from paper_1405_2270_b200 import _abi  # noqa: E402
from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="256x256x256")
ap.add_argument("--R", type=int, default=41)
ap.add_argument("--save", default="", help="also save the raw event buffer (.npy)")
args = ap.parse_args()
n1, n2, ks = map(int, args.shape.split("x"))
g = torch.Generator(device="cuda").manual_seed(1)
R = args.R
out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, ks)]
w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
torch.cuda.synchronize()
lib = _abi.load()
lib.ls_lab_timeline.argtypes = [C.c_void_p, C.c_int64]
n = 148 * 2 * 16 * 128
buf = np.zeros(n, dtype=np.uint64)
lib.ls_lab_timeline(buf.ctypes.data, n)
buf = buf.reshape(-1, 128)
if args.save:
    np.save(args.save, buf)
warps = []
for row in buf:
    cnt = int(row[0] & 0xFFFFFFFF)
    if cnt <= 1:
        continue
    sm = int(row[0] >> 32)
    ev = [(int(x >> 8), int(x & 0xFF)) for x in row[1:cnt]]
    warps.append((sm, ev))
print(f"{len(warps)} warps logged")
by_sm = defaultdict(list)
for sm, ev in warps:
    by_sm[sm].append(ev)
clk_ghz = 1.965
ph = defaultdict(list)
ends, starts = [], []
for sm, wl in by_sm.items():
    t0 = min(ev[0][0] for ev in wl)
    for ev in wl:
        d = {}
        last = {}
        for t, e in ev:
            if e in last:
                pass
            last[e] = t
        seq = ev
        starts.append((seq[0][0] - t0) / clk_ghz / 1e3)
        ends.append((seq[-1][0] - t0) / clk_ghz / 1e3)
        ph["prologue"].append((next(t for t, e in seq if e == 2) - seq[0][0]) / clk_ghz / 1e3)
        prev = None
        for i, (t, e) in enumerate(seq):
            if prev is not None:
                pt, pe = prev
                key = f"{pe}->{e}"
                ph[key].append((t - pt) / clk_ghz / 1e3)
            prev = (t, e)
for k in sorted(ph):
    v = ph[k]
    print(f"{k:10s} n={len(v):6d} mean={statistics.mean(v):8.3f} us  p50={statistics.median(v):8.3f}  max={max(v):8.3f}  sum/warp={sum(v)/len(warps):8.3f}")
print(f"warp end (us after its SM's first set-up): mean {statistics.mean(ends):.2f} max {max(ends):.2f} min {min(ends):.2f}")
