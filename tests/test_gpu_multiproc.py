"""The Python sharded path with the product kernels: two ranks (gloo for the one scalar
all-reduce, so no collective ever waits inside a kernel) each run the generator, assembly and
expansion of their own z-slabs on cuda:0 through ShardedPotential, and the fused energy of their
slabs plus the all-reduce. Against one unsharded process: every rank's slabs bit-identical to
the same slabs of the whole grid, and the all-reduced energy equal to the whole-grid energy
within the summation-order tolerance (the reference's k-slab parallel_for, canonical.hpp:251-266,
spread over processes)."""
import hashlib
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

LC, NCELL, B = (4, 4, 6), 64, 10.0  # 256 x 256 x 384 grid: 384 slabs, 192 per rank
CHARGES = [(0.0, 0.0, 0.0, 1.0), (1.25, -0.3125, 2.5, 2.0)]  # on grid vertices (h = 0.15625)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    import paper_1405_2270_b200 as L
    spec = L.LatticeSpec(LC, L.GridSpec(B, NCELL), [L.Charge(c[:3], c[3]) for c in CHARGES])
    rule = L.sinc_quadrature(1e-6, spec.unit.h, math.sqrt(3.0) * max(LC) * B, 20, 1.0)
    return L, spec, rule


def _rho(torch, dims, h):
    out = []
    for l, N in enumerate(dims):
        x = (np.arange(N) + 0.5 - N / 2) * h
        sigma = N * h / 4
        out.append(torch.as_tensor(np.exp(-x * x / (2 * sigma * sigma)) * (1.0 + 0.1 * l), device="cuda"))
    return out


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_1405_2270_b200.distributed import ShardedPotential
        L, spec, rule = _setup()
        sp = ShardedPotential(spec, rule, mode="erf", device=torch.device("cuda:0"))
        out = sp.allocate()
        sp.step(out)
        e = sp.energy(_rho(torch, sp.pipe.dims, spec.unit.h))
        torch.cuda.synchronize()
        h = hashlib.sha1(out.cpu().numpy().tobytes()).hexdigest()
        q.put((rank, sp.k0, sp.k1, h, e, L.load_library().ls_launch_count()))
    finally:
        dist.destroy_process_group()


def test_two_ranks_product_kernels_match_unsharded():
    import torch
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0

    L, spec, rule = _setup()
    pipe = L.DevicePipeline(spec, rule, mode="erf")
    N1, N2, N3 = pipe.dims
    whole = torch.empty((N3, N2, N1), dtype=torch.float64, device="cuda")
    pipe.step(whole)
    e_whole = float(pipe.grid_functional(_rho(torch, pipe.dims, spec.unit.h)).cpu())
    torch.cuda.synchronize()
    assert res[0][1] == 0 and res[-1][2] == N3 and res[0][2] == res[1][1]
    for rank, k0, k1, h, e, launches in res:
        assert launches > 0  # the product kernels ran in every rank
        assert hashlib.sha1(whole[k0:k1].cpu().numpy().tobytes()).hexdigest() == h, rank
        assert abs(e - e_whole) <= 1e-13 * abs(e_whole), (e, e_whole)
    assert res[0][4] == res[1][4]  # every rank holds the same reduced energy
