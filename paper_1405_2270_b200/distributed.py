"""Multi-GPU z-slab sharding of the expansion.

One process per GPU (torchrun), torch.distributed for the plumbing. The
expansion shards with no data-path exchange: rank r owns the contiguous slab
range slab_range(N3, r, world) of the i-fastest grid (one contiguous block of
HBM per rank) and recomputes the microsecond-scale generator and assembly
locally. The only collective is the scalar all_reduce(SUM) of the energy
functional <V, rho> (NCCL over NVLink on GPUs; gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Sequence


def slab_range(N3: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous partition of [0, N3): the first N3 % world ranks get one extra slab."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(N3, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def weak_scaling_lattice(world: int) -> tuple[int, int, int]:
    """Lattice (cells per axis, n = 64) holding 1024^3 grid points per GPU: world 1 is
    BASELINE configs[1] (1024^3), world 8 is configs[2] (2048^3), grown z, then y, then x."""
    table = {1: (16, 16, 16), 2: (16, 16, 32), 4: (16, 32, 32), 8: (32, 32, 32)}
    return table.get(world, (16, 16, 16 * world))


def all_reduce_sum(value, group=None):
    """Sums a scalar (python float or 1-element tensor) over the process group; returns a float."""
    import torch
    import torch.distributed as dist
    t = value if isinstance(value, torch.Tensor) else torch.tensor([float(value)], dtype=torch.float64)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.reshape(-1)[0].item())


class ShardedPotential:
    """This rank's z-slabs of the lattice potential, device resident, plus the
    all-reduced energy functional."""

    def __init__(self, spec, rule, mode: str = "erf", periodic: bool = False, group=None, device=None):
        import torch
        import torch.distributed as dist
        from .latsum import DevicePipeline
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.pipe = DevicePipeline(spec, rule, mode=mode, periodic=periodic, device=device)
        N1, N2, N3 = self.pipe.dims
        self.k0, self.k1 = slab_range(N3, self.rank, self.world)
        self.shape = (self.k1 - self.k0, N2, N1)
        self.torch = torch

    def allocate(self):
        return self.torch.empty(self.shape, dtype=self.torch.float64, device=self.pipe.dev)

    def step(self, out, stream=None):
        """Generator + assembly (replicated) + expansion of this rank's slabs into `out`."""
        self.pipe.step(out, self.k0, self.k1, stream)

    def energy(self, rho: Sequence, stream=None) -> float:
        """<V, rho> over the whole grid for a separable rho = (rho1, rho2, rho3) (device tensors
        of length N1, N2, N3): fused expansion-reduction over this rank's slabs, then one
        scalar all_reduce."""
        local = self.pipe.grid_functional(rho, self.k0, self.k1, stream)
        return all_reduce_sum(local, self.group)


# ------------------------------------------------------------- the C++ runner
def runner_path():
    """The C++ multi-GPU runner (paper_1405_2270_b200/bin/latsum_shard_runner, built by
    ``python -m paper_1405_2270_b200.build``): one process per GPU, DevicePotential +
    Communicator (include/latsum/sharded.hpp), NCCL all-reduce through the C ABI."""
    import os
    from pathlib import Path
    # LS_SHARD_RUNNER: another executable with the same command line (the CPU tests' stand-in).
    p = Path(os.environ.get("LS_SHARD_RUNNER") or Path(__file__).resolve().parent / "bin" / "latsum_shard_runner")
    if not p.exists():
        raise FileNotFoundError(f"{p} not built (python -m paper_1405_2270_b200.build)")
    return p


def run_runner(args: Sequence[str], env: dict | None = None, timeout: float = 1800.0) -> dict | None:
    """Runs one rank of the C++ runner; returns its JSON line (rank 0) or None (other ranks).
    The runner's stderr (NCCL INFO lines included) passes through."""
    import json
    import os
    import subprocess
    import sys
    e = dict(os.environ)
    if env:
        e.update(env)
    r = subprocess.run([str(runner_path()), *map(str, args)], stdout=subprocess.PIPE, stderr=sys.stderr,
                       text=True, env=e, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"latsum_shard_runner exited with {r.returncode}: {r.stdout[-2000:]}")
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    return json.loads(lines[-1]) if lines else None
