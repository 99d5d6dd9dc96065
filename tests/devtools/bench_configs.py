"""Per-config measurements for every BASELINE.json config (cfg0..cfg4) on one B200.

Writes one JSON object per line to stdout (and --out):
  cfg0  n=64, L=4   (256^3)      : full step GPU vs the reference (oracle/_ref) densify on all cores
  cfg1  n=64, L=16  (1024^3)     : see bench.py (headline)
  cfg2  n=64, L=32  (2048^3)     : whole 64 GiB grid on one GPU, one 8-GPU z-shard, energy <V,rho>
  cfg3  8 atoms, rank 328, L=32  : assembly GPU vs reference, one 8-GPU z-shard of the expansion
  cfg4  periodic n=256, L=64/128/256 : assembly, 256^3 expansion, batch of 1024 functionals
Timing: CUDA events around device work after warm-up (inputs resident in HBM); the reference
arm is timed on the host with its own time_ms / wall clock, all host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402
from oracle import ref_available, reference  # noqa: E402

dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
i64p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
B, EPS, M = 10.0, 1e-6, 20


def ev_time(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def make(Lc, n=64, charges=((0.0, 0.0, 0.0, 1.0),), periodic_L=None):
    spec = L.LatticeSpec(tuple(Lc), L.GridSpec(B, n), [L.Charge(tuple(c[:3]), c[3]) for c in charges])
    rule = L.sinc_quadrature(EPS, spec.unit.h, math.sqrt(3.0) * max(spec.L) * B, M, 1.0)
    return spec, rule


def ref_assembly(spec, rule, periodic):
    """Reference: erf master (gaussian_moment_vector columns) + assembled sum, all host cores."""
    r = reference()
    r._set_threads(os.cpu_count() or 1)
    Lx = np.array(spec.L, dtype=np.int64)
    ch = np.array([[*c.pos, c.Z] for c in spec.charges])
    t0 = time.perf_counter()
    f = r.lattice_master(1, Lx, spec.unit.n, spec.unit.b, rule.exponents, rule.weights, ch)
    t_master = time.perf_counter() - t0
    R, M0 = rule.node_count(), spec.charge_count()
    dims = [spec.unit.n if periodic else spec.L[l] * spec.unit.n for l in range(3)]
    out = [np.zeros((dims[l], M0 * R), order="F") for l in range(3)]
    wout = np.zeros(M0 * R)
    ms = C.c_double(0)
    r._check(r._assembled_sum(int(periodic), i64p(Lx), spec.unit.n, spec.unit.b, dp(ch.ravel()), M0, dp(f[0]),
                              dp(f[1]), dp(f[2]), dp(np.ascontiguousarray(rule.weights)), R, dp(out[0]), dp(out[1]),
                              dp(out[2]), dp(wout), C.byref(ms)), "assembled_sum")
    return t_master * 1e3, ms.value, out, wout


def ref_expand_rate(fac, w, dims, slabs):
    """Reference densify_slab streamed over `slabs` z-slabs (all cores): points per second."""
    r = reference()
    buf = np.empty((dims[0], dims[1], slabs), order="F")
    ms = C.c_double(0)
    r._check(r._expand_into(dims[0], dims[1], dims[2], len(w), dp(fac[0]), dp(fac[1]), dp(fac[2]),
                            dp(np.ascontiguousarray(w)), 0, slabs, dp(buf), C.byref(ms)), "expand_into")
    return dims[0] * dims[1] * slabs / (ms.value * 1e-3)


def gpu_pipeline_times(spec, rule, periodic=False, k0=0, k1=None, store=True):
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=periodic)
    N = pipe.dims
    k1 = N[2] if k1 is None else k1
    out = torch.empty((k1 - k0, N[1], N[0]), dtype=torch.float64, device="cuda") if store else None
    t_gen = ev_time(pipe.generate)
    t_asm = ev_time(pipe.assemble)
    t_exp = ev_time(lambda: pipe.expand(out, k0, k1), reps=3) if store else None
    return pipe, out, t_gen, t_asm, t_exp


def cfg0(emit):
    spec, rule = make((4, 4, 4))
    pipe, out, tg, ta, te = gpu_pipeline_times(spec, rule)
    N = pipe.dims
    pts = float(np.prod(N))
    line = {"config": "cfg0", "grid": list(N), "rank": pipe.Rt, "gpu_gen_ms": tg, "gpu_assembly_ms": ta,
            "gpu_expand_ms": te, "gpu_step_gpts": pts / ((tg + ta + te) * 1e-3) / 1e9}
    if ref_available():
        tm, tasm, fac, w = ref_assembly(spec, rule, False)
        rate = ref_expand_rate(fac, w, N, N[2])
        line.update({"ref_master_ms": tm, "ref_assembly_ms": tasm, "ref_expand_gpts": rate / 1e9,
                     "ref_cores": os.cpu_count()})
    emit(line)


def cfg2(emit):
    spec, rule = make((32, 32, 32))
    N = spec.target_dims()
    free = torch.cuda.mem_get_info()[0]
    line = {"config": "cfg2", "grid": list(N), "rank": rule.node_count()}
    # one 8-GPU z-shard (256 slabs of 2048^2)
    pipe, out, tg, ta, te = gpu_pipeline_times(spec, rule, k0=0, k1=N[2] // 8)
    line.update({"gpu_gen_ms": tg, "gpu_assembly_ms": ta, "shard8_expand_ms": te,
                 "shard8_gpts": N[0] * N[1] * (N[2] // 8) / (te * 1e-3) / 1e9})
    del out
    torch.cuda.empty_cache()
    # whole grid on one GPU (64 GiB) when it fits
    if free > 8 * np.prod(N) * 1.05:
        out = torch.empty((N[2], N[1], N[0]), dtype=torch.float64, device="cuda")
        t_full = ev_time(lambda: pipe.expand(out), reps=2, warm=1)
        line.update({"full_1gpu_expand_ms": t_full, "full_1gpu_gpts": float(np.prod(N)) / (t_full * 1e-3) / 1e9})
        del out
        torch.cuda.empty_cache()
    # energy <V, rho>: fused full-grid reduction vs the 1D rank-term form
    x = (np.arange(N[0]) + 0.5 - N[0] / 2) * spec.unit.h
    r1 = torch.as_tensor(np.exp(-x * x / 2.0), device="cuda")
    rho = [r1, r1, r1]
    holder = {}
    t_e = ev_time(lambda: holder.__setitem__("e", pipe.grid_functional(rho)), reps=2, warm=1)
    X = [r1.reshape(-1, 1)] * 3
    t_1d = ev_time(lambda: holder.__setitem__("e1", L.DevicePipeline.functional_batch_device(
        [pipe.factor(l).T for l in range(3)], pipe.w, X)))
    e, e1 = float(holder["e"][0]), float(holder["e1"][0])
    line.update({"energy_full_grid": e, "energy_1d": e1, "energy_rel_diff": abs(e - e1) / abs(e1),
                 "energy_full_grid_ms": t_e, "energy_1d_ms": t_1d})
    emit(line)


def cfg3(emit):
    rng = np.random.default_rng(20241019)
    n = 64
    h = B / n
    ia = rng.integers(7, 58, size=(8, 3))
    Z = rng.integers(1, 9, size=8).astype(float)
    charges = [(*(ia[c] * h - B / 2), Z[c]) for c in range(8)]
    spec, rule = make((32, 32, 32), charges=charges)
    N = spec.target_dims()
    pipe, out, tg, ta, te = gpu_pipeline_times(spec, rule, k0=0, k1=N[2] // 8)
    line = {"config": "cfg3", "grid": list(N), "rank": pipe.Rt, "charges": 8, "gpu_gen_ms": tg, "gpu_assembly_ms": ta,
            "shard8_expand_ms": te, "shard8_gpts": N[0] * N[1] * (N[2] // 8) / (te * 1e-3) / 1e9,
            "shard8_tflops": 2 * pipe.Rt * N[0] * N[1] * (N[2] // 8) / (te * 1e-3) / 1e12}
    if ref_available():
        tm, tasm, fac, w = ref_assembly(spec, rule, False)
        line.update({"ref_master_ms": tm, "ref_assembly_ms": tasm, "ref_cores": os.cpu_count(),
                     "ref_expand_gpts_4slabs": ref_expand_rate(fac, w, N, 4) / 1e9})
    emit(line)


def cfg4(emit):
    for Lc in (64, 128, 256):
        spec, rule = make((Lc, Lc, Lc), n=256)
        pipe, out, tg, ta, te = gpu_pipeline_times(spec, rule, periodic=True)
        line = {"config": f"cfg4_L{Lc}", "grid": list(pipe.dims), "rank": pipe.Rt, "master_len": 2 * Lc * 256,
                "gpu_gen_ms": tg, "gpu_assembly_ms": ta, "gpu_expand_ms": te,
                "gpu_expand_gpts": float(np.prod(pipe.dims)) / (te * 1e-3) / 1e9}
        # batch of 1024 separable Gaussian test functions, alpha log-uniform in [0.1, 10]
        rng = np.random.default_rng(4)
        F = 1024
        alpha = 10 ** rng.uniform(-1, 1, F)
        sigma = 1 / np.sqrt(2 * alpha)
        centres = rng.uniform(-B / 2, B / 2, (F, 3))
        mids = (np.arange(256) + 0.5 - 128) * spec.unit.h
        G = [torch.as_tensor(np.exp(-(mids[:, None] - centres[None, :, l]) ** 2 / (2 * sigma ** 2)), device="cuda")
             for l in range(3)]
        holder = {}
        t_b = ev_time(lambda: holder.__setitem__("v", L.DevicePipeline.functional_batch_device(
            [pipe.factor(l).T for l in range(3)], pipe.w, G)))
        # full-grid form for a sample of 16 test functions (fused expansion-reduction each)
        t_f = ev_time(lambda: [pipe.grid_functional([G[0][:, f].contiguous(), G[1][:, f].contiguous(),
                                                      G[2][:, f].contiguous()]) for f in range(16)], reps=2, warm=1)
        v1 = holder["v"][:16].cpu().numpy()
        vf = np.array([float(pipe.grid_functional([G[l][:, f].contiguous() for l in range(3)])[0]) for f in range(16)])
        line.update({"batch1024_1d_ms": t_b, "full_grid_16_ms": t_f,
                     "full_vs_1d_max_rel": float(np.max(np.abs(vf - v1) / np.abs(v1)))})
        if ref_available():
            tm, tasm, fac, w = ref_assembly(spec, rule, True)
            line.update({"ref_master_ms": tm, "ref_assembly_ms": tasm, "ref_cores": os.cpu_count(),
                         "ref_expand_gpts": ref_expand_rate(fac, w, pipe.dims, 16) / 1e9})
        emit(line)
        del out
        torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="cfg0,cfg2,cfg3,cfg4")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    fh = open(a.out, "w") if a.out else None

    def emit(d):
        s = json.dumps({k: (float(f"{v:.7g}") if isinstance(v, float) else v) for k, v in d.items()})
        print(s, flush=True)
        if fh:
            fh.write(s + "\n")
            fh.flush()
    for name in a.only.split(","):
        {"cfg0": cfg0, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}[name](emit)


if __name__ == "__main__":
    main()
