"""Builds liblatsum_cuda.so in-tree for sm_100a (nvcc cross-compiles; no GPU needed).

Every CUDA translation unit under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` and linked into
``paper_1405_2270_b200/liblatsum_cuda.so`` (git-ignored, but it travels to the
GPU box with the gpurun snapshot).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OUT = PKG / "liblatsum_cuda.so"
OBJ = ROOT / "build" / "obj"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{ROOT / 'include'}", "-Xptxas", "-v"]
# `--dev` (or LS_BUILD_DEV=1) compiles in the development A/B knobs (LS_EXPAND_PLAN, ...) that
# the lab scripts under tools/ use; the product build ignores the environment.
DEV = "--dev" in sys.argv or os.environ.get("LS_BUILD_DEV") == "1"
if DEV:
    FLAGS.append("-DLS_DEV_KNOBS")
    OBJ = ROOT / "build" / "obj_dev"


def sources():
    return sorted(CSRC.glob("*.cu"))


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src, *CSRC.glob("*.cuh"), ROOT / "include" / "latsum_cuda.h"]
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def _compile(src: Path) -> tuple[Path, str]:
    obj = OBJ / (src.stem + ".o")
    if not _stale(obj, src):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    marker = OUT.with_suffix(".dev")
    if OUT.exists() and marker.exists() != DEV:
        OUT.unlink()  # switching between the product and the dev build: relink from this OBJ dir
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        results = list(ex.map(_compile, sources()))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not OUT.exists() or any(o.stat().st_mtime > OUT.stat().st_mtime for o in objs):
        tmp = OUT.with_suffix(".so.tmp")
        cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        tmp.replace(OUT)
        if DEV:
            marker.touch()
        elif marker.exists():
            marker.unlink()
    return OUT


RUNNER_SRC = PKG / "runner" / "latsum_shard_runner.cpp"
RUNNER = PKG / "bin" / "latsum_shard_runner"
CLI_SRC = PKG / "runner" / "latsum_cli.cpp"
CLI = PKG / "bin" / "latsum"
CUDA_HOME = Path(os.environ.get("CUDA_HOME", "/usr/local/cuda"))


def _host_tool(src: Path, out: Path) -> Path:
    deps = [src, OUT, *(ROOT / "include" / "latsum").glob("*.hpp"), ROOT / "include" / "latsum_cuda.h"]
    if out.exists() and all(d.stat().st_mtime <= out.stat().st_mtime for d in deps):
        return out
    out.parent.mkdir(exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'include' / 'eigen_compat'}", f"-I{CUDA_HOME / 'include'}", str(src), "-o",
           str(out), f"-L{PKG}", "-llatsum_cuda", f"-L{CUDA_HOME / 'lib64'}", "-lcudart", "-pthread",
           "-Wl,-rpath,$ORIGIN/.."]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"{out.name} build failed:\n{r.stderr}")
    return out


def build_runner() -> Path:
    """The C++ host tools, linked against the in-tree liblatsum_cuda.so (rpath $ORIGIN/..): the
    multi-GPU runner (one process per GPU, NCCL all-reduce through the C ABI) and the `latsum`
    command line (the reference CLI's kernel / sum-box / sum-periodic / series / project)."""
    build()
    _host_tool(CLI_SRC, CLI)
    return _host_tool(RUNNER_SRC, RUNNER)


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
    print(build_runner())
