"""The C++ multi-GPU host (paper_1405_2270_b200/bin/latsum_shard_runner over
include/latsum/sharded.hpp): one process per GPU, NCCL all-reduce through the C ABI
(ls_comm_*). CPU: it builds and rejects bad arguments; GPU: a world-1 NCCL run on one
B200 whose energy matches the 1D rank-term form and whose e2e pass completes. The
world-2 plumbing (slab split, scalar all-reduce) is covered on CPU with gloo in
tests/test_multiproc.py; this environment has one GPU per job."""
import json
import subprocess

import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def runner():
    from paper_1405_2270_b200.build import build_runner
    return build_runner()


def test_runner_builds_and_links_the_product_library(runner):
    out = subprocess.run(["ldd", str(runner)], capture_output=True, text=True).stdout
    assert "liblatsum_cuda.so" in out and str(ROOT / "paper_1405_2270_b200") in out


def test_runner_rejects_bad_arguments(runner):
    r = subprocess.run([str(runner), "--bogus"], capture_output=True, text=True)
    assert r.returncode == 2 and "unknown argument" in r.stderr
    r = subprocess.run([str(runner), "--world", "2", "--rank", "1", "--steps", "0"], capture_output=True, text=True)
    assert r.returncode == 2


def test_sharded_header_compiles(tmp_path):
    src = tmp_path / "s.cpp"
    src.write_text('#include "latsum/sharded.hpp"\nint main() { return latsum::slab_range(10, 1, 3).first == 4 ? 0 : 1; }\n')
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
                        f"-I{ROOT / 'include' / 'eigen_compat'}", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_runner_world1_nccl(runner):
    r = subprocess.run([str(runner), "--L", "4", "--n", "32", "--world", "1", "--rank", "0", "--device", "0",
                        "--steps", "3", "--warmup", "3", "--energy", "--e2e-steps", "1"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["world"] == 1 and res["grid"] == [128, 128, 128] and res["rank_R"] == 41
    assert res["slabs_rank0"] == [0, 128]
    assert res["value_gpts"] > 0 and res["launches_rank0"] >= 3 * 3
    e = res["energy"]
    assert e["rel_diff_vs_1d"] <= 1e-12 and e["value"] == e["api_value"]
    assert res["e2e"]["value"] > 0


@pytest.mark.gpu
def test_runner_id_file_rendezvous(runner, tmp_path):
    """Communicator::from_id_file (rank 0 writes the id, others read it) at world 1."""
    idf = tmp_path / "job.id"
    r = subprocess.run([str(runner), "--L", "2", "--n", "16", "--world", "1", "--id-file", str(idf), "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert idf.exists() and idf.stat().st_size == 128


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [["--periodic", "--L", "64", "--n", "16"],
                                   ["--charges", "CSV", "--L", "6", "--n", "32"]])
def test_runner_periodic_and_multi_charge(runner, tmp_path, extra):
    """The runner's step and energy on the other prepare paths: a periodic lattice with one charge
    and L >= 32 (generator fused into the assembly, master never written) and a box cell with
    several charges from the reference's CSV format; the fused energy matches the 1D form."""
    if "CSV" in extra:
        csv = tmp_path / "cell.csv"
        csv.write_text("x,y,z,Z\n0,0,0,1\n1.25,-0.3125,2.5,2\n-2.5,1.875,0.625,0.5\n")
        extra = [str(csv) if a == "CSV" else a for a in extra]
    r = subprocess.run([str(runner), *extra, "--world", "1", "--rank", "0", "--device", "0", "--steps", "2",
                        "--warmup", "1", "--energy"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    res = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert res["value_gpts"] > 0
    assert res["energy"]["rel_diff_vs_1d"] <= 1e-12
