"""cfg0 (256^3, one charge, R = 41) step broken into its launches: device time per call of the
full step (eager and CUDA-graph replay), generator, assembly and expansion alone.

  python tools/lab/cfg0_step.py
"""
import math
import os
import sys

sys.path.insert(0, "/root/repo")  # bench.py
sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))  # the package under test comes first
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1405_2270_b200 import latsum as L  # noqa: E402

dev = torch.device("cuda:0")
spec = L.LatticeSpec((4, 4, 4), L.GridSpec(bench.B, bench.n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule = L.sinc_quadrature(bench.EPS, spec.unit.h, math.sqrt(3.0) * 4 * bench.B, bench.M_QUAD, bench.C0)
pipe = L.DevicePipeline(spec, rule, mode="erf", device=dev)
grid = torch.empty(tuple(reversed(pipe.dims)), dtype=torch.float64, device=dev)
pipe.step(grid)
torch.cuda.synchronize()
for name, fn in (("step", lambda: pipe.step(grid)), ("generate", pipe.generate), ("assemble", pipe.assemble),
                 ("prepare", pipe.prepare),
                 ("expand", lambda: pipe.expand(grid))):
    eager = bench._ev_ms(fn) * 1e3
    graph, how = bench._graph_ms(fn)
    print(f"{name:9s} eager {eager:7.1f} us/call   {how} {graph * 1e3:7.1f} us/call", flush=True)
