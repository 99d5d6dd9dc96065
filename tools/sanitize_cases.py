"""Small cases that launch every kernel of liblatsum_cuda.so once or more, for compute-sanitizer
(one tool per gpurun call, as the profiling recipe asks):

  compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py
  compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_cases.py

Covered: generator (erf, midpoint), assembly (box, periodic), every expansion plan (TMEM 8-warp,
TMEM 16-warp, 16-warp two-stage, shared-memory, split-K, 256-rank chunks) on grids with ragged
edges, the fused functional epilogue, eval_points, Gram / scalar product, the functional batch,
the full-grid functional batch (TMA and cp.async feeds), calibration and the device pipeline.
Sizes are tiny: the tools slow kernels by 10-100x.
"""
import math
import os
import sys

sys.path.insert(0, os.environ.get("LS_LAB_ROOT", "/root/repo"))
import numpy as np  # noqa: E402

import paper_1405_2270_b200 as L  # noqa: E402

rng = np.random.default_rng(7)


def rand_tensor(dims, R):
    return L.CanonicalTensor3([np.asfortranarray(rng.uniform(0.1, 1.0, (n, R))) for n in dims],
                              rng.uniform(0.1, 1.0, R))


def main():
    only = set(sys.argv[1:])
    n_cases = 0

    def case(name):
        nonlocal n_cases
        n_cases += 1
        print(f"case {name}", flush=True)
        return not only or name in only

    # expansion plans (expansion_plan names the kernel each rank takes)
    for R in (41, 42, 70, 100, 130, 200, 300):
        if case(f"expand_R{R}"):
            t = rand_tensor((136, 72, 3), R)  # ragged i-chunk and j-stage edges
            V = L.expand_slabs(t, 0, 3)
            assert np.isfinite(V).all()
            print(f"  {L.expansion_plan(R)}")
    if case("expand_chunked_R600"):
        t = rand_tensor((40, 24, 2), 600)
        L.expand_slabs(t, 0, 2)
    if case("grid_functional"):
        t = rand_tensor((136, 72, 3), 41)
        L.grid_functional(t, [rng.uniform(size=136), rng.uniform(size=72), rng.uniform(size=3)])
    if case("eval_points"):
        t = rand_tensor((16, 16, 16), 41)
        L.eval_points(t, rng.integers(0, 16, (100, 3)).astype(np.int64))
    if case("scalar_product"):
        L.scalar_product(rand_tensor((16, 16, 16), 41), rand_tensor((16, 16, 16), 5))
    if case("functional_batch"):
        t = rand_tensor((32, 32, 32), 41)
        L.functional_batch(t, [np.asfortranarray(rng.uniform(size=(32, 70))) for _ in range(3)])
    if case("grid_functional_batch"):
        t = rand_tensor((64, 40, 6), 41)  # even N1: TMA tensor-map feed
        L.grid_functional_batch(t, [np.asfortranarray(rng.uniform(size=(n, 70))) for n in (64, 40, 6)])
        t = rand_tensor((33, 20, 3), 41)  # odd N1: cp.async feed
        L.grid_functional_batch(t, [np.asfortranarray(rng.uniform(size=(n, 9))) for n in (33, 20, 3)])
    # generator + assembly + expansion through the host e2e call and the device pipeline
    b, n = 10.0, 16
    spec = L.LatticeSpec((2, 2, 2), L.GridSpec(b, n), [L.Charge((0.0, 0.0, 0.0), 1.0)])
    rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3.0) * 2 * b, 20, 1.0)
    if case("lattice_potential_box_erf"):
        L.lattice_potential(spec, rule, mode="erf")
    if case("lattice_potential_periodic_midpoint"):
        L.lattice_potential(spec, rule, mode="midpoint", periodic=True)
    if case("assembled_sums"):
        m = L.build_lattice_master(spec, rule)
        L.assembled_box_sum(spec, m)
        L.assembled_periodic_sum(spec, m)
    if case("calibrate"):
        L.calibrate_for_lattice(spec, 1e-4)
    if case("device_pipeline"):
        import torch
        pipe = L.DevicePipeline(spec, rule, mode="erf")
        N = spec.target_dims()
        out = torch.empty((N[2], N[1], N[0]), dtype=torch.float64, device="cuda")
        pipe.step(out)
        rho = [torch.ones(N[l], dtype=torch.float64, device="cuda") for l in range(3)]
        pipe.grid_functional(rho)
        torch.cuda.synchronize()
    print(f"sanitize_cases: {n_cases} cases done", flush=True)


if __name__ == "__main__":
    main()
