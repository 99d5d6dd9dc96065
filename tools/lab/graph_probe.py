"""Checks that the side-config calls of bench.py can be captured in CUDA graphs, and compares the
graph-replay time with eager back-to-back time."""
import math
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1405_2270_b200 as L  # noqa: E402

dev = torch.device("cuda", 0)
B = 10.0
spec = L.LatticeSpec((4, 4, 4), L.GridSpec(B, 64), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3.0) * 4 * B, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode="erf", device=dev)
grid = torch.empty(tuple(reversed(pipe.dims)), dtype=torch.float64, device=dev)
ref = torch.empty_like(grid)
pipe.step(ref)
torch.cuda.synchronize()
for name, fn in [("cfg0 step", lambda: pipe.step(grid)), ("gen+asm", lambda: (pipe.generate(), pipe.assemble())),
                 ("expand", lambda: pipe.expand(grid))]:
    e = bench._ev_ms(fn)
    gm, how = bench._graph_ms(fn)
    print(f"{name}: eager {e * 1e3:.1f} us, {how} {gm * 1e3:.1f} us", flush=True)
torch.cuda.synchronize()
assert torch.equal(grid, ref), "graph replay changed the grid"
spec4 = L.LatticeSpec((256, 256, 256), L.GridSpec(B, 256), [L.Charge((0.0, 0.0, 0.0), 1.0)])
rule4 = L.sinc_quadrature(1e-6, spec4.unit.h, math.sqrt(3.0) * 256 * B, 20, 1.0)
p4 = L.DevicePipeline(spec4, rule4, mode="erf", periodic=True, device=dev)
rng = np.random.default_rng(4)
G = [torch.as_tensor(rng.uniform(size=(256, 1024)), device=dev) for _ in range(3)]
fb = lambda: L.DevicePipeline.functional_batch_device([p4.factor(l).T for l in range(3)], p4.w, G)  # noqa: E731
p4.generate(); p4.assemble()
want = fb().clone()
for name, fn in [("cfg4 gen+asm", lambda: (p4.generate(), p4.assemble())), ("functionals 1D", fb),
                 ("functionals full grid", lambda: p4.grid_functional_batch(G))]:
    e = bench._ev_ms(fn)
    gm, how = bench._graph_ms(fn)
    print(f"{name}: eager {e * 1e3:.1f} us, {how} {gm * 1e3:.1f} us", flush=True)
assert torch.equal(fb(), want)
print("graph probe ok")
