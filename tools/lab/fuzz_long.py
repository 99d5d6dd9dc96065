"""Long randomized K3 sweep (a soak test beyond tests/test_gpu_fuzz.py): random shapes, ranks
(every plan), slab ranges and padded output strides, checked against a float64 torch einsum of
the same factors (a different summation algorithm) at 1e-13 relative max-norm, with NaN canaries
around every written row, and bitwise run-to-run.

  python tools/lab/fuzz_long.py [--cases 2000] [--seed 7]
"""
import argparse
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1405_2270_b200 import _abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cases", type=int, default=2000)
ap.add_argument("--seed", type=int, default=7)
ap.add_argument("--trace", action="store_true", help="print every case before running it (triage)")
args = ap.parse_args()
rng = np.random.default_rng(args.seed)
lib = _abi.load()
dev = torch.device("cuda")
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
p = lambda x: C.c_void_p(x.data_ptr())  # noqa: E731
worst, t0, fails = 0.0, time.time(), 0
plans = {}
for c in range(args.cases):
    R = int(rng.choice([int(rng.integers(1, 130)), int(rng.integers(130, 600))], p=[0.8, 0.2]))
    big = rng.integers(0, 5) == 0
    n1 = int(rng.integers(1, 900 if big else 300))
    n2 = int(rng.integers(1, 700 if big else 260))
    n3 = int(rng.integers(1, 6))
    k0 = int(rng.integers(0, n3))
    k1 = int(rng.integers(k0 + 1, n3 + 1))
    pad_y, pad_z = int(rng.choice([0, 0, 1, 2, 5])), int(rng.choice([0, 0, 2, 7]))
    if args.trace:
        print(f"case {c}: {R},{n1},{n2},{n3},{k0},{k1},{pad_y},{pad_z}", flush=True)
    fac = [torch.rand((R, m), dtype=torch.float64, device=dev) * 0.95 + 0.05 for m in (n1, n2, n3)]
    w = torch.rand(R, dtype=torch.float64, device=dev) * 0.95 + 0.05
    ldy, nk = n1 + pad_y, k1 - k0
    ldz = ldy * n2 + pad_z
    outs = []
    for _ in range(2):
        buf = torch.full((nk * ldz + 8,), float("nan"), dtype=torch.float64, device=dev)
        rc = lib.ls_expand(p(fac[0]), n1, p(fac[1]), n2, p(fac[2]), n3, p(w), n1, n2, n3, R, k0, k1, p(buf), ldy, ldz,
                           None, None, None, None, s)
        assert rc == 0, lib.ls_last_error()
        outs.append(buf)
    torch.cuda.synchronize()
    a = outs[0]
    written = torch.zeros_like(a, dtype=torch.bool)
    v = written[: nk * ldz].view(nk, ldz)[:, : ldy * n2].reshape(nk, n2, ldy)[:, :, :n1]
    v.fill_(True)
    got = a[: nk * ldz].view(nk, ldz)[:, : ldy * n2].reshape(nk, n2, ldy)[:, :, :n1]
    want = torch.einsum("q,qi,qj,qk->kji", w, fac[0], fac[1], fac[2][:, k0:k1])
    err = float((got - want).abs().max() / want.abs().max())
    ok = err <= 1e-13 and not torch.isnan(got).any() and bool(torch.isnan(a[~written]).all()) \
        and torch.equal(a[written], outs[1][written])
    worst = max(worst, err)
    key = lib.ls_expand_plan_name  # plan family per rank, for the coverage summary
    buf_name = C.create_string_buffer(256)
    key(R, buf_name, 256)
    fam = buf_name.value.decode().split(";")[0]
    plans[fam] = plans.get(fam, 0) + 1
    if not ok:
        fails += 1
        print(f"FAIL case {c}: R={R} {n1}x{n2}x{n3} [{k0},{k1}) pad {pad_y},{pad_z}: rel {err:.2e}", flush=True)
print(f"{args.cases} cases, {fails} failures, worst rel {worst:.2e}, {time.time() - t0:.0f} s")
for fam, n in sorted(plans.items(), key=lambda x: -x[1]):
    print(f"  {n:5d}  {fam}")
