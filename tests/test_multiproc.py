"""Multi-rank host logic on CPU (gloo, world_size 2): the z-slab partition covers
the grid exactly once, and the energy functional summed per shard and
all-reduced equals the unsharded value (oracle arithmetic stands in for the
per-rank GPU functional, which uses the same partition and reduction)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1405_2270_b200.distributed import all_reduce_sum, slab_range, weak_scaling_lattice


def test_slab_partition_covers_once():
    for N3 in (1, 7, 256, 1024, 2048, 2049):
        for world in (1, 2, 3, 4, 8):
            ranges = [slab_range(N3, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == N3
            for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1


def test_weak_scaling_lattice_points_per_gpu():
    for world in (1, 2, 4, 8):
        L = weak_scaling_lattice(world)
        assert np.prod([l * 64 for l in L]) == world * 1024 ** 3
    assert weak_scaling_lattice(8) == (32, 32, 32)  # BASELINE configs[2]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import torch.distributed as dist
    from oracle import restatement
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = restatement()
        rng = np.random.default_rng(5)
        dims, R = (12, 10, 9), 7
        f = [np.asfortranarray(rng.uniform(0.1, 1.0, (d, R))) for d in dims]
        w = rng.uniform(0.1, 1.0, R)
        rho = [rng.uniform(0.0, 1.0, d) for d in dims]
        k0, k1 = slab_range(dims[2], rank, world)
        import ctypes as C
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
        local = orc._grid_functional(dims[0], dims[1], dims[2], R, dp(f[0]), dp(f[1]), dp(f[2]), dp(w),
                                     dp(rho[0]), dp(rho[1]), dp(rho[2]), k0, k1)
        total = all_reduce_sum(local)
        full = orc._grid_functional(dims[0], dims[1], dims[2], R, dp(f[0]), dp(f[1]), dp(f[2]), dp(w),
                                    dp(rho[0]), dp(rho[1]), dp(rho[2]), 0, dims[2])
        result_q.put((rank, total, full, k0, k1))
    finally:
        dist.destroy_process_group()


def test_sharded_energy_allreduce_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert res[0][3] == 0 and res[-1][4] == 9 and res[0][4] == res[1][3]
    for _, total, full, _, _ in res:
        assert abs(total - full) <= 1e-13 * abs(full)
    assert res[0][1] == res[1][1]  # every rank holds the same reduced value


def test_bench_sharded_path_world2_gloo(tmp_path):
    """bench.py --gpus 2 under torchrun on CPU, with a stand-in for the C++ runner: the ranks agree
    on a fresh NCCL-id file over gloo, rank 0's runner writes it and the other waits for it, and
    rank 0 prints one JSON line for cfg2 strong scaling (the N > 1 path of the driver's run)."""
    import json
    import subprocess
    import sys
    from conftest import ROOT
    env = dict(os.environ, LS_SHARD_RUNNER=str(ROOT / "tests" / "devtools" / "fake_shard_runner.py"),
               CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(ROOT / "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3"], capture_output=True, text=True, env=env,
                       timeout=300, cwd=str(tmp_path))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["metric"].startswith("lattice potential")
    assert d["config"]["grid"] == [2048, 2048, 2048] and "cfg2 strong" in d["config"]["workload"]
    assert d["value"] > 0 and d["roofline"]["frac"] > 0 and d["e2e"]["value"] > 0
    assert d["weak_scaling"]["grid"] == [1024, 1024, 2048] and d["energy"] is not None
