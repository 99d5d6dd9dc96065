"""Per-warp phase breakdown of one A2-in-TMEM expansion launch (256^3 by default), from a
-DLS_TIMELINE lab build (see timeline.py for the build line). Times are per SM (clock64), in
us at 1.965 GHz. Events of expand_a2t_kernel: 1 set-up done, 2 A2 in TMEM, 3 unit operands
scaled (chunk 0), 5 item DMMAs issued, 6 next unit's share handed over, 9 slot released, 8 end.
"""
import argparse
import os
import statistics as st
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
args = ap.parse_args()
n1, n2, ks = map(int, args.shape.split("x"))
g = torch.Generator(device="cuda").manual_seed(1)
R = args.R
out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, ks)]
w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
for _ in range(5):
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
torch.cuda.synchronize()
lib = _abi.load()
lib.ls_lab_timeline.argtypes = [C.c_void_p, C.c_int64]
n = 148 * 2 * 16 * 128
buf = np.zeros(n, dtype=np.uint64)
lib.ls_lab_timeline(buf.ctypes.data, n)
buf = buf.reshape(-1, 128)
ghz = 1.965
warps = []
for row in buf:
    cnt = int(row[0] & 0xFFFFFFFF)
    if cnt <= 1:
        continue
    warps.append((int(row[0] >> 32), [(int(x >> 8), int(x & 0xFF)) for x in row[1:cnt]]))
by_sm = defaultdict(list)
for sm, ev in warps:
    by_sm[sm].append(ev)
us = lambda c: c / ghz / 1e3  # noqa: E731
ph = defaultdict(list)
for sm, wl in by_sm.items():
    t0 = min(ev[0][0] for ev in wl)
    tend = max(ev[-1][0] for ev in wl)
    ph["sm span (first set-up .. last end)"].append(us(tend - t0))
    for ev in wl:
        t = {}
        for c, e in ev:
            t.setdefault(e, []).append(c)
        ph["set-up skew vs SM's first warp"].append(us(ev[0][0] - t0))
        ph["A2 load (1->2)"].append(us(t[2][0] - t[1][0]))
        if 3 in t:
            ph["first unit wait (2->3)"].append(us(t[3][0] - t[2][0]))
        fives = t.get(5, [])
        prev = t[3][0] if 3 in t else None
        for i, c in enumerate(fives):
            if prev is not None:
                ph["item c=%d (prev event -> 5)" % (i % 2)].append(us(c - prev))
            prev = c
        for a, b in zip(t.get(9, []), t.get(3, [])[1:]):
            ph["release -> next unit scaled (9->3)"].append(us(b - a))
        if fives:
            ph["last item 5 -> end 8"].append(us(t[8][0] - fives[-1]))
            ph["items per warp"].append(len(fives))
        ph["warp total (1->8)"].append(us(t[8][0] - t[1][0]))
        ph["warp end vs SM's last end"].append(us(tend - ev[-1][0]))
for k, v in ph.items():
    print(f"{k:40s} n={len(v):6d} mean={st.mean(v):8.3f} p50={st.median(v):8.3f} min={min(v):8.3f} max={max(v):8.3f}")
