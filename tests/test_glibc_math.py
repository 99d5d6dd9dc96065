"""CPU checks of csrc/glibc_math.cuh, the erf / exp the generator runs on the device.

The header's host instantiation (same source, compiled with -ffp-contract=off) is compared
with this host's libm bit for bit: a seeded sweep over every branch of both functions, and
every argument the cfg0-cfg4 erf and midpoint masters feed to erf / exp. The device
instantiation is compared in tests/test_gpu_parity.py (test_device_libm_bitwise_equals_host_libm
and the bitwise master tests).
"""
import math
import subprocess

import numpy as np
import pytest

from conftest import ROOT

SRC = ROOT / "tools" / "glibc_math" / "check_vs_libm.cpp"


@pytest.fixture(scope="module")
def checker(tmp_path_factory):
    exe = tmp_path_factory.mktemp("gm") / "check_vs_libm"
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-mfma", "-pthread", "-o", str(exe), str(SRC)],
                   check=True)
    return exe


def _host_selects_fma_exp() -> bool:
    with open("/proc/cpuinfo") as f:
        flags = f.read()
    return " fma" in flags and " avx2" in flags


def test_random_sweep_bitwise(checker):
    if not _host_selects_fma_exp():
        pytest.skip("glibc picks its FMA exp only on FMA + AVX2 hosts")
    r = subprocess.run([str(checker), "random", "300000", "7"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("erf_mismatch=0 exp_mismatch=0") == 11, r.stdout


@pytest.mark.parametrize("Lc,n", [(4, 64), (16, 64), (32, 64), (64, 256), (256, 256)])
def test_generator_arguments_bitwise(checker, orc, tmp_path, Lc, n):
    """Every erf argument t * vertex(i) and midpoint argument t * mid(i) of the master columns
    (newton.hpp:33-34, :47-50) with the rule sinc_quadrature(1e-6, h, sqrt(3) L b, 20, 1)."""
    if not _host_selects_fma_exp():
        pytest.skip("glibc picks its FMA exp only on FMA + AVX2 hosts")
    b = 10.0
    h = b / n
    _, tau, _, _ = orc.sinc_quadrature(1e-6, h, math.sqrt(3.0) * Lc * b, 20, 1.0)
    length = 2 * Lc * n
    half = length // 2
    vertex = (np.arange(half + 1, dtype=np.int64) - half).astype(np.float64) * h
    mid = ((np.arange(half, dtype=np.float64) + 0.5) - length / 2.0) * h
    args = np.concatenate([np.multiply.outer(tau, vertex).ravel(), np.multiply.outer(tau, mid).ravel()])
    f = tmp_path / "args.f64"
    args.tofile(f)
    r = subprocess.run([str(checker), "file", str(f)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
