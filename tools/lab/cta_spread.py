"""Per-CTA start/end spread of one expansion launch on the device's global timer (lab build with
-DLS_TIMELINE: slots 126/127 of each warp's log hold %globaltimer at warp start/end).

  LAB_DIR=labx tools/lab/build_lab.sh tl "-DLS_DEV_KNOBS -DLS_TIMELINE"
  LS_LAB_ROOT=/root/repo/labx/tl python tools/lab/cta_spread.py --shape 1024x1024x1024
Answers: how far apart do the CTAs of the static schedule finish (tail imbalance), and how long
is the launch's span against the sum of its parts.
"""
import argparse
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

os.environ["LS_TIMELINE"] = "1"
from paper_1405_2270_b200 import _abi  # noqa: E402
from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="1024x1024x1024")
ap.add_argument("--R", type=int, default=41)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
n1, n2, ks = map(int, args.shape.split("x"))
g = torch.Generator(device="cuda").manual_seed(1)
R = args.R
out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, ks)]
w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
lib = _abi.load()
lib.ls_lab_timeline.argtypes = [C.c_void_p, C.c_int64]
n = 148 * 2 * 16 * 128
for rep in range(args.reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    e1.record()
    torch.cuda.synchronize()
    if rep < 2:
        continue
    buf = np.zeros(n, dtype=np.uint64)
    lib.ls_lab_timeline(buf.ctypes.data, n)
    buf = buf.reshape(-1, 128)
    rows = [r for r in buf if int(r[0] & 0xFFFFFFFF) > 1]
    sm = np.array([int(r[0] >> 32) for r in rows])
    st = np.array([int(r[126]) for r in rows], dtype=np.float64)
    en = np.array([int(r[127]) for r in rows], dtype=np.float64)
    t0 = st.min()
    st = (st - t0) / 1e3
    en = (en - t0) / 1e3
    # per SM: the last warp's end
    sm_end = {s: en[sm == s].max() for s in np.unique(sm)}
    ends = np.array(sorted(sm_end.values()))
    print(f"rep {rep - 2}: event time {e0.elapsed_time(e1) * 1e3:.1f} us; {len(rows)} warps on {len(sm_end)} SMs; "
          f"warp start max {st.max():.1f} us; SM end min {ends[0]:.1f} p10 {np.percentile(ends, 10):.1f} "
          f"p50 {np.percentile(ends, 50):.1f} p90 {np.percentile(ends, 90):.1f} max {ends[-1]:.1f} us; "
          f"mean idle before the last SM ends {np.mean(ends[-1] - ends):.1f} us")
    by = sorted(sm_end.items(), key=lambda kv: kv[1])
    print("   earliest SMs:", [(s, round(t, 1)) for s, t in by[:6]], " latest:", [(s, round(t, 1)) for s, t in by[-6:]])
