#!/usr/bin/env python
"""CPU stand-in for bin/latsum_shard_runner with the same command line (tests/test_multiproc.py):
rank 0 writes the id file (temporary + rename), the other ranks wait for it, then rank 0 prints
a JSON line shaped like the runner's. No GPU, no NCCL; it exercises bench.py's N > 1 plumbing."""
import argparse
import json
import os
import sys
import time

ap = argparse.ArgumentParser()
for k in ("--L", "--n", "--b", "--M", "--eps", "--world", "--rank", "--device", "--id-file", "--id-hex",
          "--steps", "--warmup", "--e2e-steps", "--host-threads"):
    ap.add_argument(k)
ap.add_argument("--energy", action="store_true")
a = ap.parse_args()
world, rank = int(a.world), int(a.rank)
if a.id_file:
    if rank == 0:
        with open(a.id_file + ".tmp", "wb") as f:
            f.write(os.urandom(128))
        os.replace(a.id_file + ".tmp", a.id_file)
    else:
        t0 = time.time()
        while not os.path.exists(a.id_file):
            if time.time() - t0 > 60:
                sys.exit("no id file")
            time.sleep(0.02)
L = [int(x) for x in a.L.split(",")] if "," in a.L else [int(a.L)] * 3
N = [l * int(a.n) for l in L]
k1 = N[2] // world
if rank == 0:
    pts = float(N[0] * N[1] * N[2])
    ms = 2.5 * (k1 / 1024.0)
    print(json.dumps({
        "runner": "fake", "world": world, "grid": N, "rank_R": 41, "slabs_rank0": [0, k1], "steps": int(a.steps),
        "warmup": int(a.warmup), "ms_per_step_max": ms, "expand_ms_mean_max": ms * 0.99,
        "value_gpts": pts / (ms * 1e-3) / 1e9, "flops_per_launch_rank0": 82.0 * N[0] * N[1] * k1,
        "launches_rank0": 4 * int(a.steps), "plan": "fake", "comm_init_s": 0.0,
        "energy": {"value": 1.0, "fused_ms_max": ms, "allreduce_ms_max": 0.01} if a.energy else None,
        "e2e": {"value": 1.0, "unit": "Gpts/s", "h2d_bytes_per_step": 688, "d2h_bytes_per_step": 8 * N[0] * N[1] * k1}
        if a.e2e_steps and int(a.e2e_steps) > 0 else None}))
