"""Is the cfg0 step (256^3, 55 us of device time) host-bound? Times 400 back-to-back
DevicePipeline.step calls: host enqueue time per call (wall clock, no sync inside) against the
device time per call (CUDA events around the whole batch).

  python tools/lab/step_host_bound.py
"""
import math
import os
import sys
import time

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
sys.path.insert(0, "/root/repo")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1405_2270_b200 import latsum as L  # noqa: E402

spec = L.LatticeSpec((4, 4, 4), L.GridSpec(bench.B, bench.n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule = L.sinc_quadrature(bench.EPS, spec.unit.h, math.sqrt(3.0) * 4 * bench.B, bench.M_QUAD, bench.C0)
pipe = L.DevicePipeline(spec, rule, mode="erf")
grid = torch.empty(tuple(reversed(pipe.dims)), dtype=torch.float64, device="cuda")
for _ in range(20):
    pipe.step(grid)
torch.cuda.synchronize()
n = 400
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
t0 = time.perf_counter()
for _ in range(n):
    pipe.step(grid)
t_host = (time.perf_counter() - t0) / n * 1e6
e1.record()
torch.cuda.synchronize()
t_dev = e0.elapsed_time(e1) / n * 1e3
print(f"cfg0 step: host enqueue {t_host:.1f} us/call, device {t_dev:.1f} us/call "
      f"({'host-bound' if t_host > 0.9 * t_dev else 'device-bound'})")
