"""Times one 8-GPU z-shard of the cfg3 expansion (8 atoms, rank 328, 2048^2 x 256 slabs)."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").environ.get("LS_LAB_ROOT", "/root/repo"))
import paper_1405_2270_b200 as L  # noqa: E402

rng = np.random.default_rng(20241019)
n, B = 64, 10.0
h = B / n
ia = rng.integers(7, 58, size=(8, 3))
Z = rng.integers(1, 9, size=8).astype(float)
spec = L.LatticeSpec((32, 32, 32), L.GridSpec(B, n), [L.Charge(tuple(ia[c] * h - B / 2), Z[c]) for c in range(8)])
rule = L.sinc_quadrature(1e-6, h, math.sqrt(3) * 32 * B, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode="erf")
N = pipe.dims
k1 = int(sys.argv[1]) if len(sys.argv) > 1 else N[2] // 8
out = torch.empty((k1, N[1], N[0]), dtype=torch.float64, device="cuda")
pipe.step(out, 0, k1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record()
    pipe.expand(out, 0, k1)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
flops = 2 * pipe.Rt * N[0] * N[1] * k1
print(f"rank {pipe.Rt} shard {N[0]}x{N[1]}x{k1}: {best:.3f} ms, {flops / best / 1e9:.2f} TF/s")
