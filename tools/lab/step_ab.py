"""Back-to-back cfg1 steps (generator + assembly + prep + expansion), one event pair around the
batch: the bench's timing, for A/B builds (LS_LAB_ROOT)."""
import math
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import torch  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402

Lc = int(sys.argv[1]) if len(sys.argv) > 1 else 16
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
spec = L.LatticeSpec((Lc,) * 3, L.GridSpec(10.0, 64), [L.Charge((0, 0, 0), 1.0)])
rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3) * Lc * 10.0, 20, 1.0)
pipe = L.DevicePipeline(spec, rule, mode="erf")
N1, N2, N3 = spec.target_dims()
out = torch.empty((N3, N2, N1), dtype=torch.float64, device="cuda")
for _ in range(5):
    pipe.step(out)
torch.cuda.synchronize()
best = 1e9
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        pipe.step(out)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / steps)
print(f"{os.environ.get('LS_LAB_ROOT', 'product'):>24s} L={Lc}: {best:.4f} ms/step, {N1 * N2 * N3 / best / 1e6:.1f} Gpts/s")
