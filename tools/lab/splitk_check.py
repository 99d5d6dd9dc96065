"""Split-K parity spot check against a float64 einsum on a small random shard (ranks >= 176)."""
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1405_2270_b200.latsum import _expand_device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(3)
for R in (176, 200, 240, 250, 251, 253, 255, 301, 328, 331, 332, 350):
    n1, n2, ks = 200, 136, 3
    fac = [torch.rand((R, m), dtype=torch.float64, device="cuda", generator=g) for m in (n1, n2, ks)]
    w = torch.rand(R, dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty((ks, n2, n1), dtype=torch.float64, device="cuda")
    _expand_device(fac, w, (n1, n2, ks), 0, ks, out)
    want = torch.einsum("q,qi,qj,qk->kji", w, fac[0], fac[1], fac[2])
    err = float((out - want).abs().max() / want.abs().max())
    print(f"R={R}: rel {err:.2e}", "OK" if err < 1e-13 else "FAIL", flush=True)
