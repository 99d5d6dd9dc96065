"""The `latsum` command line (paper_1405_2270_b200/bin/latsum, runner/latsum_cli.cpp): the
reference CLI's kernel / sum-box / sum-periodic / series / project subcommands
(proj/tools/latsum.cpp) over the drop-in headers. CPU: argument and validation errors map to
the reference's exit codes. GPU: the bundles, reports and run configurations it writes match
the Python mirror of the same calls bit for bit (test_cli.cpp's checks, re-hosted)."""
import json
import math
import subprocess

import numpy as np
import pytest

from conftest import ROOT


@pytest.fixture(scope="module")
def cli():
    from paper_1405_2270_b200.build import CLI, build_runner
    build_runner()
    return CLI


def run(cli, *args, cwd=None):
    return subprocess.run([str(cli), *map(str, args)], capture_output=True, text=True, timeout=600, cwd=cwd)


def read_bundle(path):
    """LATSUMB1 (bundle.hpp:18-94): magic, dims + rank (int64), h + origin, weights, factors."""
    raw = open(path, "rb").read()
    assert raw[:8] == b"LATSUMB1"
    hdr = np.frombuffer(raw, dtype=np.int64, count=4, offset=8)
    geom = np.frombuffer(raw, dtype=np.float64, count=4, offset=40)
    R = int(hdr[3])
    off = 72
    w = np.frombuffer(raw, dtype=np.float64, count=R, offset=off)
    off += 8 * R
    f = []
    for l in range(3):
        n = int(hdr[l])
        f.append(np.frombuffer(raw, dtype=np.float64, count=n * R, offset=off).reshape((n, R), order="F"))
        off += 8 * n * R
    assert off == len(raw)
    return f, w, geom


def test_cli_usage_errors_exit_2(cli, tmp_path):
    assert run(cli).returncode == 2
    r = run(cli, "sum-box", "--L", "2", "--n", "7", "--b", "2", "--out", tmp_path / "x.bin")
    assert r.returncode == 2 and "n must be even" in r.stderr
    r = run(cli, "sum-box", "--L", "2,3", "--n", "8", "--b", "2", "--out", tmp_path / "x.bin")
    assert r.returncode == 2 and "--L expects" in r.stderr
    assert run(cli, "bench", "--L", "2").returncode == 2  # harness subcommands are out of scope
    assert run(cli, "qtt-gauss", "--levels", 30, cwd=tmp_path).returncode == 2  # writes qtt-gauss.run.json there
    assert run(cli, "sum-box", "--n", "8", "--b", "2", "--out", tmp_path / "x.bin").returncode == 2  # --L required
    cfg = json.loads((tmp_path / "x.bin.run.json").read_text())  # written before validation, as the reference
    assert cfg["command"] == "sum-box" and cfg["params"]["n"] == 8


@pytest.mark.gpu
@pytest.mark.parametrize("periodic", [False, True])
def test_cli_sum_matches_python_mirror(cli, tmp_path, periodic):
    import paper_1405_2270_b200 as L
    charges = tmp_path / "cell.csv"
    charges.write_text("x,y,z,Z\n0,0,0,1\n0.5,-0.25,0,2\n")
    out, rep = tmp_path / "sum.bin", tmp_path / "sum.csv"
    r = run(cli, "--threads", 3, "sum-periodic" if periodic else "sum-box", "--L", "2,2,4", "--n", 8, "--b", 2,
            "--eps", "1e-4", "--charges", charges, "--out", out, "--report", rep)
    assert r.returncode == 0, r.stderr
    f, w, geom = read_bundle(out)
    spec = L.LatticeSpec((2, 2, 4), L.GridSpec(2.0, 8), [L.Charge((0, 0, 0), 1.0), L.Charge((0.5, -0.25, 0.0), 2.0)])
    rule = L.calibrate_for_lattice(spec, 1e-4)
    master = L.build_lattice_master(spec, rule)
    res = (L.assembled_periodic_sum if periodic else L.assembled_box_sum)(spec, master)
    for l in range(3):
        assert np.array_equal(f[l], res.tensor.factor(l))
    assert np.array_equal(w, res.tensor.weights())
    assert geom[0] == spec.unit.h
    dims = res.grid_dims
    assert all(geom[1 + l] == (0.5 - dims[l] / 2) * spec.unit.h for l in range(3))
    p_center = L.eval_point(res.tensor, dims[0] // 2, dims[1] // 2, dims[2] // 2)
    rows = rep.read_text().splitlines()
    assert rows[0] == "L,rank,time_ms,p_center_au,p_hat_au"
    assert rows[1].split(",")[0] == "2x2x4" and float(rows[1].split(",")[3]) == p_center
    cfg = json.loads(out.with_name("sum.bin.run.json").read_text())
    assert cfg["command"] == ("sum-periodic" if periodic else "sum-box") and cfg["threads"] == 3
    assert cfg["params"]["L"] == [2, 2, 4] and cfg["params"]["eps"] == 1e-4
    assert ("periodic" if periodic else "box") + " sum: lattice 2x2x4" in r.stdout


@pytest.mark.gpu
def test_cli_kernel_series_project(cli, tmp_path):
    import paper_1405_2270_b200 as L
    k = tmp_path / "k.bin"
    r = run(cli, "kernel", "--n", 16, "--b", 2, "--eps", "1e-5", "--out", k, "--report", tmp_path / "k.csv")
    assert r.returncode == 0, r.stderr
    f, w, geom = read_bundle(k)
    grid = L.GridSpec(2.0, 16)
    rule = L.calibrate_quadrature(grid, L.default_tolerance(grid, 1e-5))
    assert len(w) == rule.node_count() and np.array_equal(w, np.asarray(rule.weights))
    assert (tmp_path / "k.csv").read_text().startswith("M,C0,probe_rel_err\n")
    r = run(cli, "series", "--kind", "line", "--L", "2,4", "--n", 8, "--b", 2, "--extrapolate", "linear",
            "--report", tmp_path / "s.csv")
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "s.csv").read_text().splitlines()
    assert len(rows) == 3 and rows[1].split(",")[4] != "" and rows[2].split(",")[4] == ""
    # project: a periodic sum bundle against a two-function Gaussian basis
    out = tmp_path / "p.bin"
    assert run(cli, "sum-periodic", "--L", 2, "--n", 8, "--b", 2, "--eps", "1e-4", "--out", out).returncode == 0
    basis = tmp_path / "basis.csv"
    basis.write_text("cx,cy,cz,sigma\n0,0,0,0.4\n0.25,0,0,0.3\n")
    r = run(cli, "project", "--from", out, "--basis", basis, "--out", tmp_path / "V.csv")
    assert r.returncode == 0, r.stderr
    lines = (tmp_path / "V.csv").read_text().splitlines()
    assert lines[0] == "v0_au,v1_au" and len(lines) == 3
    V = np.array([[float(x) for x in ln.split(",")] for ln in lines[1:]])
    assert V[0, 1] == V[1, 0] and np.all(V > 0)  # exactly symmetric (project.hpp:65-97)
    assert math.isfinite(V.sum())


@pytest.mark.gpu
def test_cli_qtt_subcommands(cli, tmp_path):
    out = tmp_path / "b.bin"
    assert run(cli, "sum-box", "--L", "4", "--n", 16, "--b", 2, "--eps", "1e-4", "--out", out).returncode == 0
    r = run(cli, "qtt-ranks", "--from", out, "--eps", "1e-8", "--report", tmp_path / "q.csv")
    assert r.returncode == 0, r.stderr
    rows = (tmp_path / "q.csv").read_text().splitlines()
    assert rows[0] == "axis,q,max_rank,avg_rank,err"
    f, w, _ = read_bundle(out)
    assert len(rows) == 1 + 3 * len(w)
    assert all(float(x.split(",")[4]) <= 1e-8 for x in rows[1:])
    r = run(cli, "qtt-gauss", "--p", "1,0.5", "--eps-list", "1e-3,1e-5,1e-7", "--levels", 10, "--report", tmp_path / "g.csv")
    assert r.returncode == 0, r.stderr
    g = (tmp_path / "g.csv").read_text().splitlines()
    assert g[0] == "p,eps,max_rank" and len(g) == 7
    assert "max rank vs ln(1/eps) slope" in r.stdout
