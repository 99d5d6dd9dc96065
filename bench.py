#!/usr/bin/env python
"""Benchmark of the latsum hot path on B200 (arXiv 1405.2270, BASELINE.json).

One "step" = one pass of the hot path over the lattice: the rank-R erf
generator (K1) for every distinct axis, the assembled O(N L R) lattice sum
(K2) and the FP64 rank-R expansion of this rank's z-slabs onto the full grid
in HBM (K3).

  * N = 1: configs[1] (1024^3) through the Python mirror of the device pipeline,
    plus the other configs as side measurements and configs[2] on one GPU through
    the C++ runner (the strong-scaling anchor).
  * N > 1 (torchrun, one process per GPU): configs[2] STRONG scaling -- one
    2048^3 grid, 2048/N z-slabs per GPU -- run by the C++ runner
    (paper_1405_2270_b200/bin/latsum_shard_runner: include/latsum/sharded.hpp,
    NCCL through the C ABI for the one scalar all-reduce of the energy); the
    weak-scaling variant (1024^3 points per GPU) is an extra key.

Prints ONE JSON line (rank 0). `value` = grid points/s of the whole job with
inputs in HBM; `e2e` = the same metric through the host-level C-ABI call
(ls_h_lattice_potential: host rule/charges in, full grid out into pinned host
memory, every copy inside the timed region); `roofline` = the expansion
kernel's achieved FP64 rate against the measured DMMA peak; `cpu_baseline` =
the reference's own code (oracle/_ref, compiled unmodified) on the host cores.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "lattice potential Gpts/s (rank-R N^3 eval)"
UNIT = "Gpts/s"
B = 10.0          # unit-cell edge, bohr (BASELINE configs)
n_CELL = 64       # grid points per cell per axis
M_QUAD = 20       # R = 2M+1 = 41
EPS = 1e-6        # sinc_quadrature(eps, h, sqrt(3) L b, M, C0) -- SURVEY 8(d)
C0 = 1.0


def lattice_for(world: int) -> tuple[int, int, int]:
    """Weak-scaling lattice: 1024^3 points (L = 16^3) per rank, grown along z, then y, then x."""
    from paper_1405_2270_b200.distributed import weak_scaling_lattice
    return weak_scaling_lattice(world)


def fp64_peak_tflops() -> tuple[float, str]:
    """Measured FP64 DMMA peak (tools/microbench/fp64_peak.cu on this pool's B200)."""
    p = ROOT / "profiles" / "r01_fp64_peak_microbench.jsonl"
    best = 0.0
    if p.exists():
        for line in p.read_text().splitlines():
            try:
                d = json.loads(line)
            except json.JSONDecodeError:
                continue
            if str(d.get("bench", "")).startswith("dmma"):
                best = max(best, float(d.get("tflops", 0.0)))
    if best > 0:
        return best, "measured (DMMA m8n8k4 microbench, profiles/r01_fp64_peak_microbench.jsonl)"
    return 37.2, "nominal (148 SM x 64 FMA/clk x 1965 MHz)"


def hbm_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = Path(f"/tmp/latsum_clocks_{os.getpid()}.csv")

    def __enter__(self):
        # device index, None for every GPU of the node, -1 for no sampling (non-zero ranks)
        sel = [] if self.dev is None else ["-i", str(self.dev)]
        try:
            if self.dev == -1:
                raise OSError("sampling disabled")
            self.proc = subprocess.Popen(
                ["nvidia-smi", *sel, f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        # nvidia-smi needs a moment to start; wait for its first sample (bounded).
        t0 = time.time()
        while self.proc is not None and time.time() - t0 < 5.0:
            if self.path.exists() and self.path.stat().st_size > 0:
                break
            time.sleep(0.02)
        self.t_start = time.time()
        return self

    def mark(self):
        """Restrict the summary to samples taken after this call (the timed region)."""
        self.skip = 0
        if self.path.exists():
            self.skip = len(self.path.read_text().splitlines())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        if self.path.exists():
            for line in self.path.read_text().splitlines()[getattr(self, "skip", 0):]:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[0]) for r in rows if num(r[0]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for name, v in zip(names, r[3:7]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        power = [num(r[7]) for r in rows if num(r[7]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": num(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows),
                "power_w_max": max(power) if power else None}


def make_problem(world: int):
    import paper_1405_2270_b200 as L
    Lx = lattice_for(world)
    spec = L.LatticeSpec(Lx, L.GridSpec(B, n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    Lmax = max(Lx)
    rule = L.sinc_quadrature(EPS, spec.unit.h, math.sqrt(3.0) * Lmax * B, M_QUAD, C0)
    return L, spec, rule


def slab_range(N3: int, rank: int, world: int) -> tuple[int, int]:
    from paper_1405_2270_b200.distributed import slab_range as sr
    return sr(N3, rank, world)


def workload_config(spec, world, rule) -> dict:
    N = spec.target_dims()
    return {
        "workload": ("cfg1: n=64, L=16^3, N=1024 (1024^3 FP64 grid, 8 GiB) on 1 GPU" if world == 1 else
                     f"weak z-slab scaling: lattice L={spec.L}, grid {N[0]}x{N[1]}x{N[2]}, 1024^3 points per GPU"
                     + (" (= cfg2, 2048^3 sharded 8-way)" if world == 8 else "")),
        "grid": list(N), "rank_R": rule.node_count(), "charges_per_cell": 1, "generator": "erf (newton.hpp:21-37)",
        "box_b_bohr": B, "n_per_cell": n_CELL, "quadrature": f"sinc_quadrature({EPS}, h, sqrt(3)*L*b, M=20, C0=1)",
        "parallelism": f"z-slab x{world}, no collective in the timed region",
        "l2_policy": "output 8 GiB per GPU per step >> 126 MB L2; factors regenerated every step",
    }


# --------------------------------------------------------------------------- ours
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_1405_2270_b200.distributed import ShardedPotential
    L, spec, rule = make_problem(world)
    dev_idx = local_rank % torch.cuda.device_count()  # one GPU per rank; see main() for the plumbing test
    dev = torch.device("cuda", dev_idx)
    torch.cuda.set_device(dev)
    lib = L.load_library()
    lib.ls_set_device(dev_idx)
    if lib.ls_dev_knobs_enabled():
        raise SystemExit("bench.py: liblatsum_cuda.so is a dev build (-DLS_DEV_KNOBS); rebuild the product library")
    N1, N2, N3 = spec.target_dims()
    shard = ShardedPotential(spec, rule, mode="erf", device=dev)
    pipe, k0, k1 = shard.pipe, shard.k0, shard.k1
    out = shard.allocate()
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_idx) as clk:
        for _ in range(args.warmup):
            shard.step(out, stream)
        torch.cuda.synchronize()
        # Timed region: K steps, events around each expansion launch for the roofline.
        launches0 = lib.ls_launch_count()
        barrier()
        torch.cuda.synchronize()
        clk.mark()
        t_start.record(stream)
        for s in range(args.steps):
            pipe.prepare(stream)  # generator + assembly (one launch on small lattices)
            ev[s][0].record(stream)
            pipe.expand(out, k0, k1, stream)
            ev[s][1].record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
        barrier()
        launches = lib.ls_launch_count() - launches0
    ms_total = t_start.elapsed_time(t_end)
    exp_ms = [a.elapsed_time(b) for a, b in ev]
    exp_mean = statistics.mean(exp_ms)
    if world > 1:
        tt = torch.tensor([ms_total, exp_mean], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_total, exp_mean = float(tt[0]), float(tt[1])
    ms_step = ms_total / args.steps
    pts_total = float(N1) * N2 * N3
    value = pts_total / (ms_step * 1e-3) / 1e9

    # Roofline of the expansion kernel (per launch, this rank's slabs).
    pts_rank = float(N1) * N2 * (k1 - k0)
    flops = 2.0 * pipe.Rt * pts_rank
    peak_tf, peak_src = fp64_peak_tflops()
    achieved_tf = flops / (exp_mean * 1e-3) / 1e12
    hbm_gbs, hbm_src = hbm_peak_gbs()
    out_gbs = 8.0 * pts_rank / (exp_mean * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "ncu_expand_traffic.json"
    if tp.exists():
        try:
            tj = json.loads(tp.read_text())
            if tj.get("grid") == [N1, N2, k1 - k0]:
                traffic = tj.get("dram_bytes_per_launch")
        except (ValueError, KeyError):
            traffic = None
    roofline = {
        "bound": "tensor", "pipe": "fp64 DMMA (mma.sync m8n8k4.f64)", "achieved": round(achieved_tf, 3),
        "peak": round(peak_tf, 3), "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4),
        "peak_source": peak_src, "traffic": traffic,
        "algorithmic": f"2*R*points FLOP = {flops:.4e} per launch (R={pipe.Rt}), 8 B/point written",
        "kernel_ms": round(exp_mean, 4),
        "kernel": expand_plan_name(lib, pipe.Rt),
        "hbm_leg": {"achieved_gbs": round(out_gbs, 1), "peak_gbs": hbm_gbs, "frac": round(out_gbs / hbm_gbs, 4),
                    "peak_source": hbm_src},
        "share_of_step": round(exp_mean / ms_step, 4),
    }

    # Energy functional <V, rho> (BASELINE cfg2): fused expansion-reduction over this rank's slabs
    # + one scalar all_reduce, checked against the 1D rank-term form.
    energy = e2e = None
    if not args.step_only:
        energy = run_energy(L, shard, spec, world, dev)
    del out
    torch.cuda.empty_cache()

    # e2e through the host-level C-ABI call: host rule/charges in, pinned host grid out.
    e2e_energy = None
    if not args.step_only:
        e2e = run_e2e(L, spec, rule, k0, k1, args, world, dev)
        if world == 1:
            e2e_energy = run_e2e_energy(L, spec, rule, args)

    cpu = None
    if rank == 0 and world == 1 and not (args.no_cpu_baseline or args.step_only):
        cpu = cpu_baseline(spec, rule, budget_s=args.cpu_seconds)
        one = cpu_baseline(spec, rule, budget_s=min(3.0, args.cpu_seconds), threads=1)  # also 1 thread
        cpu["single_thread"] = {"value": one["value"], "unit": one["unit"], "cores": 1, "sample": one["sample"]}

    configs = None
    if rank == 0 and world == 1 and not (args.no_configs or args.step_only):
        configs = run_other_configs(L, dev)
        torch.cuda.empty_cache()
        configs["cfg2_runner_1gpu"] = run_cfg2_runner_1gpu(dev_idx)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE configs; "
            "unit charge at each cell centre; quadrature rule computed on the host)",
            "config": workload_config(spec, world, rule), "roofline": roofline, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk.summary(), "cpu_baseline": cpu, "energy": energy,
            "e2e_energy": e2e_energy,
            "other_configs": configs,
            "assembly_note": "generator + assembly are inside every step (replicated per rank)",
        }
        print(json.dumps(line), flush=True)


def expand_plan_name(lib, R):
    import ctypes as C
    buf = C.create_string_buffer(256)
    return buf.value.decode() if lib.ls_expand_plan_name(R, buf, 256) == 0 else None


def _ev_ms(fn, reps=3, batch_ms=10.0):
    """Device ms per call: best of `reps` batches of back-to-back calls between two events, each
    batch at least `batch_ms` long (up to 200 calls), so a short call's host launch cost stays
    behind the queue and the first call's enqueue delay after the start event is amortized (the
    same convention as the K-step headline)."""
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    inner = max(1, min(200, int(batch_ms / max(e0.elapsed_time(e1), 1e-3))))
    best = float("inf")
    for _ in range(reps):
        e0.record()
        for _ in range(inner):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / inner)
    return best


def _graph_ms(fn, reps=3, batch_ms=2.0):
    """Device ms per call from back-to-back replays of a CUDA graph of `fn` (the host launch cost
    of a short call is then outside the measurement); falls back to _ev_ms when the call cannot
    be captured. Returns (ms, how)."""
    import torch
    fn()
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g, stream=side, capture_error_mode="relaxed"):
            fn()
        torch.cuda.synchronize()
    except Exception:  # noqa: BLE001 -- not capturable: eager timing
        torch.cuda.synchronize()
        return _ev_ms(fn, reps, batch_ms), "eager"
    return _ev_ms(g.replay, reps, batch_ms), "graph"


def run_other_configs(L, dev):
    """The other BASELINE configs, measured live on this GPU (device time, inputs in HBM):
    cfg0 full step; cfg2 (2048^3, 64 GiB) full step and energy on one GPU (its 8-way z-sharded
    form is the N=8 point of the scaling run); cfg3 (8 atoms, rank 328) assembly and one 8-GPU
    z-shard of the expansion; cfg4 (periodic n=256, L=256) assembly, 256^3 expansion and the
    batch of 1024 functionals."""
    import torch
    out = {}
    # cfg0
    spec = L.LatticeSpec((4, 4, 4), L.GridSpec(B, n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.sinc_quadrature(EPS, spec.unit.h, math.sqrt(3.0) * 4 * B, M_QUAD, C0)
    pipe = L.DevicePipeline(spec, rule, mode="erf", device=dev)
    grid = torch.empty(tuple(reversed(pipe.dims)), dtype=torch.float64, device=dev)
    t = _ev_ms(lambda: pipe.step(grid))
    out["cfg0"] = {"grid": list(pipe.dims), "rank": pipe.Rt, "step_ms": round(t, 4),
                   "gpts": round(float(np.prod(pipe.dims)) / (t * 1e-3) / 1e9, 2)}
    del grid
    torch.cuda.empty_cache()
    # cfg2 on one GPU: the whole 2048^3 grid (64 GiB) resident in HBM -- full step -- and the
    # energy <V, rho> in its full-grid (fused, V not stored) and 1D rank-term forms
    spec2 = L.LatticeSpec((32, 32, 32), L.GridSpec(B, n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule2 = L.sinc_quadrature(EPS, spec2.unit.h, math.sqrt(3.0) * 32 * B, M_QUAD, C0)
    pipe2 = L.DevicePipeline(spec2, rule2, mode="erf", device=dev)
    N2d = pipe2.dims
    pts2 = float(np.prod(N2d))
    if torch.cuda.mem_get_info(dev)[0] > 8 * pts2 + (4 << 30):
        grid = torch.empty(tuple(reversed(N2d)), dtype=torch.float64, device=dev)
        t2 = _ev_ms(lambda: pipe2.step(grid))
        del grid
        torch.cuda.empty_cache()
        out["cfg2_1gpu"] = {"grid": list(N2d), "rank": pipe2.Rt, "step_ms": round(t2, 3),
                            "gpts": round(pts2 / (t2 * 1e-3) / 1e9, 1),
                            "tflops": round(2 * pipe2.Rt * pts2 / (t2 * 1e-3) / 1e12, 2)}
    else:
        out["cfg2_1gpu"] = {"skipped": "less than 68 GiB of free HBM"}
    x2 = [(np.arange(N2d[l]) + 0.5 - N2d[l] / 2.0) * spec2.unit.h for l in range(3)]
    sig2 = energy_sigma(spec2)
    r2 = [np.exp(-x * x / (2.0 * sig2 * sig2)) for x in x2]  # as run_energy: sigma = L*b/4, box centre
    rho2 = [torch.as_tensor(r, device=dev) for r in r2]
    X2 = [torch.as_tensor(r.reshape(-1, 1), device=dev) for r in r2]
    one_d = lambda: L.DevicePipeline.functional_batch_device([pipe2.factor(l).T for l in range(3)], pipe2.w, X2)  # noqa: E731
    t_full = _ev_ms(lambda: pipe2.grid_functional(rho2))
    t_1d = _ev_ms(one_d)
    e_full = float(pipe2.grid_functional(rho2)[0])
    e_1d = float(one_d()[0])
    out["cfg2_1gpu"].update({"energy_full_grid_ms": round(t_full, 3), "energy_1d_ms": round(t_1d, 4),
                             "energy": e_full, "energy_rel_diff_vs_1d": abs(e_full - e_1d) / abs(e_1d)})
    del pipe2, rho2, X2
    # calibration of the cfg1 lattice (the reference CLI's dominant cost): GPU-evaluated probes
    spec1 = L.LatticeSpec((16, 16, 16), L.GridSpec(B, n_CELL), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    L.calibrate_for_lattice(spec1, EPS)
    t0 = time.perf_counter()
    cal = L.calibrate_for_lattice(spec1, EPS)
    out["calibration_cfg1"] = {"eps": EPS, "M": cal.M, "C0": cal.C0,
                               "ms": round((time.perf_counter() - t0) * 1e3, 3),
                               "note": "calibrate_for_lattice, host-timed; picks the BASELINE M=20"}
    # cfg3: 8 atoms at seeded vertices in [0.1b, 0.9b]^3, Z in 1..8, L = 32
    rng = np.random.default_rng(20241019)
    h = B / n_CELL
    ia = rng.integers(7, 58, size=(8, 3))
    Z = rng.integers(1, 9, size=8).astype(float)
    spec = L.LatticeSpec((32, 32, 32), L.GridSpec(B, n_CELL), [L.Charge(tuple(ia[c] * h - B / 2), Z[c]) for c in range(8)])
    rule = L.sinc_quadrature(EPS, h, math.sqrt(3.0) * 32 * B, M_QUAD, C0)
    pipe = L.DevicePipeline(spec, rule, mode="erf", device=dev)
    N = pipe.dims
    k1 = N[2] // 8
    shard = torch.empty((k1, N[1], N[0]), dtype=torch.float64, device=dev)
    t_asm, how_asm = _graph_ms(pipe.prepare)
    t_exp = _ev_ms(lambda: pipe.expand(shard, 0, k1))
    out["cfg3"] = {"grid": list(N), "rank": pipe.Rt, "generator_plus_assembly_ms": round(t_asm, 4),
                   "shard8_expand_ms": round(t_exp, 3),
                   "shard8_tflops": round(2 * pipe.Rt * N[0] * N[1] * k1 / (t_exp * 1e-3) / 1e12, 2),
                   "full_grid_at_8_gpus_gpts": round(8 * N[0] * N[1] * k1 / (t_exp * 1e-3) / 1e9, 1)}
    del shard
    torch.cuda.empty_cache()
    # cfg4: periodic, L = 256, n = 256 (master 131072 per axis), 1024 Gaussian test functions
    spec = L.LatticeSpec((256, 256, 256), L.GridSpec(B, 256), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.sinc_quadrature(EPS, spec.unit.h, math.sqrt(3.0) * 256 * B, M_QUAD, C0)
    pipe = L.DevicePipeline(spec, rule, mode="erf", periodic=True, device=dev)
    grid = torch.empty(tuple(reversed(pipe.dims)), dtype=torch.float64, device=dev)
    t_asm, how_asm = _graph_ms(pipe.prepare)
    t_exp = _ev_ms(lambda: pipe.expand(grid))
    rng = np.random.default_rng(4)
    F = 1024
    alpha = 10 ** rng.uniform(-1, 1, F)
    sigma = 1 / np.sqrt(2 * alpha)
    centres = rng.uniform(-B / 2, B / 2, (F, 3))
    mids = (np.arange(256) + 0.5 - 128) * spec.unit.h
    G = [torch.as_tensor(np.exp(-(mids[:, None] - centres[None, :, l]) ** 2 / (2 * sigma ** 2)), device=dev)
         for l in range(3)]
    t_f, how_f = _graph_ms(lambda: L.DevicePipeline.functional_batch_device([pipe.factor(l).T for l in range(3)], pipe.w, G))
    # full-grid form: expansion + fused DMMA GEMM (2 * 256^3 * 1024 FLOP) + fixed-order reduction
    t_fg = _ev_ms(lambda: pipe.grid_functional_batch(G))
    fg_flop = 2.0 * float(np.prod(pipe.dims)) * F
    out["cfg4_L256"] = {"grid": list(pipe.dims), "rank": pipe.Rt, "master_len": 2 * 256 * 256,
                        "generator_plus_assembly_ms": round(t_asm, 4), "expand_ms": round(t_exp, 4),
                        "expand_gpts": round(float(np.prod(pipe.dims)) / (t_exp * 1e-3) / 1e9, 1),
                        "functionals_1024_ms": round(t_f, 4),
                        "functionals_1024_full_grid_ms": round(t_fg, 4),
                        "functionals_1024_full_grid_tflops": round(fg_flop / (t_fg * 1e-3) / 1e12, 2)}
    del grid
    torch.cuda.empty_cache()
    out["timing"] = ("CUDA events around back-to-back calls (batches >= 2 ms, best of 3); inputs in HBM. "
                     f"cfg3/cfg4 generator_plus_assembly and cfg4 functionals_1024 (short calls whose host "
                     f"launch cost would dominate) time back-to-back replays of a CUDA graph of the call: "
                     f"{how_asm}/{how_f}")
    return out


def energy_sigma(spec) -> float:
    """Width of the energy density: a quarter of the box edge, so the density is >= e^-2 of its
    peak on every box face and the fused functional epilogue weighs every grid point."""
    return max(spec.L) * spec.unit.b / 4.0


def run_cfg2_runner_1gpu(dev_idx: int) -> dict:
    """configs[2] (one 2048^3 grid, 64 GiB) on this GPU through the C++ runner at world 1 (NCCL
    world-1 communicator): the N = 1 anchor of the strong-scaling curve, measured on the same
    host path the N > 1 lines use."""
    from paper_1405_2270_b200.distributed import run_runner
    try:
        res = run_runner(["--L", CFG2_L, "--n", n_CELL, "--b", B, "--M", M_QUAD, "--eps", EPS, "--world", 1,
                          "--rank", 0, "--device", dev_idx, "--steps", 5, "--warmup", 3, "--energy"],
                         {"NCCL_DEBUG": "WARN"})
    except (RuntimeError, FileNotFoundError) as e:  # report, do not sink the N = 1 line
        return {"error": str(e)[-500:]}
    keep = ("grid", "rank_R", "steps", "ms_per_step_max", "expand_ms_mean_max", "value_gpts", "plan", "energy")
    out = {k: res[k] for k in keep if k in res}
    out["tflops"] = round(res["flops_per_launch_rank0"] / (res["expand_ms_mean_max"] * 1e-3) / 1e12, 2)
    return out


def run_energy(L, shard, spec, world, dev):
    import torch
    N = spec.target_dims()
    h = spec.unit.h
    rho_np = []
    sigma = energy_sigma(spec)
    for l in range(3):
        x = (np.arange(N[l]) + 0.5 - N[l] / 2.0) * h
        rho_np.append(np.exp(-x * x / (2.0 * sigma * sigma)))  # rank-1 Gaussian, centre = box centre
    rho = [torch.as_tensor(r, device=dev) for r in rho_np]
    shard.energy(rho)  # warm-up
    torch.cuda.synchronize()
    # device time of the fused expansion-reduction + fixed-order partial sum (CUDA events, median
    # of 5), and the host wall time of the whole call incl. the all_reduce and the scalar readback
    dev_ms = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        shard.pipe.grid_functional(rho, shard.k0, shard.k1)
        e1.record()
        torch.cuda.synchronize()
        dev_ms.append(e0.elapsed_time(e1))
    t0 = time.perf_counter()
    e = shard.energy(rho)
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - t0) * 1e3
    ms = statistics.median(dev_ms)
    pipe = shard.pipe
    X = [torch.as_tensor(r.reshape(-1, 1), device=dev) for r in rho_np]
    e1d = float(L.DevicePipeline.functional_batch_device([pipe.factor(l).T for l in range(3)], pipe.w, X)[0])
    return {"value": e, "one_d_value": e1d, "rel_diff_vs_1d": abs(e - e1d) / abs(e1d), "ms": round(ms, 3),
            "wall_ms": round(wall_ms, 3),
            "density": f"rho(x)=exp(-|x|^2/(2 sigma^2)) separable, centre = box centre, sigma = L*b/4 = {sigma} bohr "
                       "(rho >= e^-2 of its peak at every box face, so every grid point carries weight)",
            "path": "fused expansion-reduction over own z-slabs + scalar all_reduce (NCCL)"}


def run_e2e(L, spec, rule, k0, k1, args, world, dev):
    import torch
    import torch.distributed as dist
    N1, N2, N3 = spec.target_dims()
    steps = max(1, min(args.steps, args.e2e_steps))
    pts = float(N1) * N2 * N3
    h2d = 8 * rule.node_count() * 2 + 8 * 4 * spec.charge_count()
    d2h = 8 * N1 * N2 * (k1 - k0)

    def timed(buf):
        L.lattice_potential(spec, rule, mode="erf", k0=k0, k1=k1, out=buf)  # warm-up (pool, module load)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(steps):
            L.lattice_potential(spec, rule, mode="erf", k0=k0, k1=k1, out=buf)
        el = time.perf_counter() - t0
        if world > 1:
            tt = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el = float(tt[0])
        return el / steps

    # (a) an ordinary numpy array: the library stages through its bounded pinned ring
    page = np.empty((N1, N2, k1 - k0), order="F")
    page.fill(0.0)  # fault the pages in outside the timed region
    t_page = timed(page)
    del page
    # (b) a pinned destination (what a throughput-minded caller passes): direct D2H
    t_pin = None
    try:
        host = torch.empty((k1 - k0) * N2 * N1, dtype=torch.float64, pin_memory=True)
        t_pin = timed(host.numpy().reshape((N1, N2, k1 - k0), order="F"))
        del host
    except RuntimeError:  # pinned-memory limit of the host
        pass
    best = min(t for t in (t_pin, t_page) if t is not None)
    return {"value": round(pts / best / 1e9, 4), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": steps,
            "d2h_gbs": round(d2h / best / 1e9, 1),
            "pinned_dest_gpts": None if t_pin is None else round(pts / t_pin / 1e9, 4),
            "pageable_dest_gpts": round(pts / t_page / 1e9, 4),
            "bound": "PCIe device-to-host (the 8 B/point grid leaves the GPU every step)",
            "api": "ls_h_lattice_potential (host tau/w/charges in; full grid out to host memory; value = the "
                   "faster of a pinned destination and an ordinary numpy array, which goes through the "
                   "library's bounded 256 MiB pinned ring)"}


def run_e2e_energy(L, spec, rule, args):
    """The energy <V, rho> end to end through one host-level call (ls_h_lattice_energy): host
    rule, charges and separable density in, the scalar out; every grid point is evaluated on
    the device, fused with the reduction. Same Gpts/s metric; informational beside `e2e`, whose
    result is the whole grid in host memory."""
    N = spec.target_dims()
    sigma = energy_sigma(spec)
    rho = [np.exp(-((np.arange(N[l]) + 0.5 - N[l] / 2.0) * spec.unit.h) ** 2 / (2 * sigma * sigma)) for l in range(3)]
    L.lattice_energy(spec, rule, rho)  # warm-up
    steps = max(3, min(args.steps, 20))
    t0 = time.perf_counter()
    for _ in range(steps):
        e = L.lattice_energy(spec, rule, rho)
    el = (time.perf_counter() - t0) / steps
    pts = float(N[0]) * N[1] * N[2]
    h2d = 8 * (2 * rule.node_count() + 4 * spec.charge_count() + sum(N))
    return {"value": round(pts / el / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8,
            "steps": steps, "energy": e, "ms": round(el * 1e3, 3),
            "api": "lattice_energy -> ls_h_lattice_energy (host rule/charges/rho in, scalar out; host-timed)"}


# ---------------------------------------------------------------- CPU reference
def cpu_baseline(spec, rule, budget_s: float = 15.0, threads: int | None = None, sample_slabs: int | None = None):
    """The reference's own code (oracle/_ref, headers compiled unmodified) on the host cores:
    erf master + assembled_box_sum + densify_slab streamed over z-slabs into a reused slab buffer.
    Bounded sample: slabs until `budget_s` of expansion time; reported per grid point."""
    import ctypes as C
    from oracle import ref_available, reference, restatement
    kind = "reference" if ref_available() else "port"
    lib = reference() if kind == "reference" else restatement()
    cores = threads or os.cpu_count() or 1
    if kind == "reference":
        lib._set_threads(cores)
    else:
        cores = 1
    N = spec.target_dims()
    R = rule.node_count()
    Lx = np.array(spec.L, dtype=np.int64)
    tau = np.ascontiguousarray(rule.exponents)
    w = np.ascontiguousarray(rule.weights)
    t0 = time.perf_counter()
    if kind == "reference":
        f = lib.lattice_master(1, Lx, spec.unit.n, spec.unit.b, tau, w)
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        fac = [np.zeros((N[l], R), order="F") for l in range(3)]
        wout = np.zeros(R)
        ch = np.array([0.0, 0.0, 0.0, 1.0])
        lib._check(lib._assembled_sum(0, Lx.ctypes.data_as(C.POINTER(C.c_int64)), spec.unit.n, spec.unit.b, dp(ch), 1,
                                      dp(f[0]), dp(f[1]), dp(f[2]), dp(w), R, dp(fac[0]), dp(fac[1]), dp(fac[2]),
                                      dp(wout), None), "assembled_sum")
    else:
        raise RuntimeError("oracle/_ref not built; cpu baseline needs the compiled reference")
    t_asm = time.perf_counter() - t0
    chunk = max(1, min(N[2], cores * 2))
    buf = np.empty((N[0], N[1], chunk), order="F")
    done = 0
    t_exp = 0.0
    limit = sample_slabs if sample_slabs is not None else N[2]
    while done < limit:
        k1 = min(N[2], done + chunk, limit)
        ms = C.c_double(0)
        lib._check(lib._expand_into(N[0], N[1], N[2], R, dp(fac[0]), dp(fac[1]), dp(fac[2]), dp(wout), done, k1,
                                    dp(buf), C.byref(ms)), "expand_into")
        t_exp += ms.value * 1e-3
        done = k1
        if sample_slabs is None and t_exp > budget_s:
            break
    pts = float(N[0]) * N[1] * done
    # per-point cost of the sampled slabs plus the (whole) generator+assembly, scaled to the full grid
    full_s = t_exp * (N[2] / done) + t_asm
    return {"value": round(float(N[0]) * N[1] * N[2] / full_s / 1e9, 5), "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"erf master + assembled_box_sum + densify_slab over {done}/{N[2]} z-slabs "
                      f"({pts:.3e} points, {t_exp:.2f} s expansion, {t_asm * 1e3:.1f} ms master+assembly) "
                      f"via oracle/_ref (reference headers + eigen_compat shim GEMM), LATSUM_THREADS={cores}",
            "expansion_s_sampled": round(t_exp, 3), "assembly_ms": round(t_asm * 1e3, 3)}


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on the host cores (rank 0 only)."""
    if rank != 0:
        return
    from types import SimpleNamespace
    from oracle import reference
    Lx = lattice_for(1) if world == 1 else (CFG2_L,) * 3  # our arm's workload: cfg1, or cfg2 strong
    spec = SimpleNamespace(L=Lx, unit=SimpleNamespace(n=n_CELL, b=B, h=B / n_CELL), charges=[None],
                           target_dims=lambda: tuple(l * n_CELL for l in Lx), charge_count=lambda: 1)
    # The reference's own sinc_quadrature (quadrature.hpp:50-89) builds the rule on this arm.
    _, tau, w, _ = reference().sinc_quadrature(EPS, B / n_CELL, math.sqrt(3.0) * max(Lx) * B, M_QUAD, C0)
    rule = SimpleNamespace(exponents=tau, weights=w, node_count=lambda: len(tau))
    vals = []
    t_all = time.perf_counter()
    for s in range(args.warmup + args.steps):
        cb = cpu_baseline(spec, rule, budget_s=args.cpu_seconds / max(1, args.steps + args.warmup))
        if s >= args.warmup:
            vals.append(cb)
    value = statistics.median(v["value"] for v in vals)
    cb = dict(vals[-1])
    cb["value"] = value
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(float(np.prod(spec.target_dims())) / (value * 1e9) * 1e3, 3),
        "higher_is_better": True, "scaling": "weak" if world == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (same inputs as the GPU arm)",
        "config": workload_config(spec, world, rule) if world == 1 else strong_config(world),
        "impl": "reference", "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_all, 2),
        "sampling": "each step is a bounded sample of the workload's z-slabs (cpu_baseline.sample); value is the "
                    "sampled rate and ms_per_step that rate extrapolated to the whole grid; "
                    "ms_per_step_sampled is the wall time a step actually took",
        "ms_per_step_sampled": round((time.perf_counter() - t_all) * 1e3 / max(1, args.steps + args.warmup), 3),
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ N > 1 (C++)
CFG2_L = 32


def strong_config(world: int) -> dict:
    N = CFG2_L * n_CELL
    return {
        "workload": f"cfg2 strong z-slab scaling: n=64, L=32^3, one 2048^3 FP64 grid (64 GiB), "
                    f"{N // world} slabs (2048^2 x {N // world}) per GPU",
        "grid": [N, N, N], "rank_R": 2 * M_QUAD + 1, "charges_per_cell": 1, "generator": "erf (newton.hpp:21-37)",
        "box_b_bohr": B, "n_per_cell": n_CELL, "quadrature": f"sinc_quadrature({EPS}, h, sqrt(3)*L*b, M=20, C0=1)",
        "parallelism": f"z-slab x{world}, one process per GPU; only collective: ncclAllReduce of the energy",
        "host": "C++ (paper_1405_2270_b200/bin/latsum_shard_runner over include/latsum/sharded.hpp)",
        "l2_policy": "output >= 8 GiB per GPU per step >> 126 MB L2; factors regenerated every step",
        "n1_anchor": "other_configs.cfg2_1gpu / cfg2_runner_1gpu of the N=1 line (same grid on one GPU)",
    }


def run_sharded(args, rank, world, local_rank):
    """configs[2] strong scaling through the C++ runner, one process per GPU. The NCCL id is
    made by rank 0's runner and handed to every rank over a CPU-only gloo group; the runner
    does all device work, takes every timing as the max over ranks (NCCL all-reduce) and rank
    0's Python composes the JSON line."""
    import torch.distributed as dist
    import secrets
    from paper_1405_2270_b200.distributed import run_runner, weak_scaling_lattice
    import paper_1405_2270_b200 as L
    L.load_library()  # the product library is mapped in this process too (the runner links it)
    dist.init_process_group("gloo")

    def id_file():
        # rank 0's runner creates the NCCL id (its bootstrap root lives in that process) and
        # writes it to this fresh path; the other ranks' runners wait for the file
        box = [f"/tmp/latsum_nccl_{secrets.token_hex(8)}.id" if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        return box[0]
    ncores = os.cpu_count() or 1
    common = ["--n", n_CELL, "--b", B, "--M", M_QUAD, "--eps", EPS, "--world", world, "--rank", rank,
              "--device", local_rank, "--host-threads", max(1, ncores // world)]
    env = {"NCCL_DEBUG": os.environ.get("NCCL_DEBUG", "INFO")}
    with ClockSampler(None if rank == 0 else -1) as clk:
        dist.barrier()
        clk.mark()
        res = run_runner(["--L", CFG2_L, "--id-file", id_file(), "--steps", args.steps, "--warmup", args.warmup,
                          "--energy", "--e2e-steps", 0 if args.step_only else max(1, min(args.e2e_steps, 2)),
                          *common], env)
        clocks = clk.summary()
    weak = None
    if not args.step_only:
        Lw = weak_scaling_lattice(world)
        weak = run_runner(["--L", ",".join(map(str, Lw)), "--id-file", id_file(), "--steps", max(3, args.steps // 4),
                           "--warmup", 3, *common], env)
    dist.barrier()
    dist.destroy_process_group()
    if rank != 0:
        return
    N = res["grid"]
    peak_tf, peak_src = fp64_peak_tflops()
    hbm_gbs, hbm_src = hbm_peak_gbs()
    exp_ms = res["expand_ms_mean_max"]
    flops = res["flops_per_launch_rank0"]
    achieved = flops / (exp_ms * 1e-3) / 1e12
    pts_rank = flops / (2.0 * res["rank_R"])
    out_gbs = 8.0 * pts_rank / (exp_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(res["value_gpts"], 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(res["ms_per_step_max"], 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (BASELINE configs[2]; unit charge at each cell centre; rule computed on the host)",
        "config": strong_config(world),
        "roofline": {
            "bound": "tensor", "pipe": "fp64 DMMA (mma.sync m8n8k4.f64)", "achieved": round(achieved, 3),
            "peak": round(peak_tf, 3), "unit": "TFLOP/s", "frac": round(achieved / peak_tf, 4),
            "peak_source": peak_src, "traffic": None,
            "algorithmic": f"2*R*points FLOP = {flops:.4e} per launch (rank 0's slabs), 8 B/point written",
            "kernel_ms": round(exp_ms, 4), "kernel": res["plan"],
            "hbm_leg": {"achieved_gbs": round(out_gbs, 1), "peak_gbs": hbm_gbs, "frac": round(out_gbs / hbm_gbs, 4),
                        "peak_source": hbm_src},
            "share_of_step": round(exp_ms / res["ms_per_step_max"], 4),
        },
        "e2e": res["e2e"], "gpu_launches": res["launches_rank0"], "clocks": clocks, "cpu_baseline": None,
        "energy": res["energy"], "weak_scaling": weak, "nccl_comm_init_s": res["comm_init_s"],
        "assembly_note": "generator + assembly are inside every step (replicated per rank, nothing sent)",
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the cfg0/cfg3/cfg4 side measurements")
    ap.add_argument("--step-only", action="store_true",
                    help="only the timed step (for ncu launch lists): no energy, e2e, CPU baseline or configs")
    ap.add_argument("--sharded", action="store_true",
                    help="use the N > 1 path (cfg2 strong scaling through the C++ runner) at any N; under torchrun")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"note: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if (world > 1 and os.environ.get("LS_BENCH_BACKEND") != "gloo") or args.sharded:
        run_sharded(args, rank, world, local_rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # NCCL, one GPU per rank. LS_BENCH_BACKEND=gloo exists only to exercise the N>1 plumbing
        # on a single GPU (ranks then share it, so such a run's numbers are not measurements).
        backend = os.environ.get("LS_BENCH_BACKEND", "nccl")
        dev_idx = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(dev_idx)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
