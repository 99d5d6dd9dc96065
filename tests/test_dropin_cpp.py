"""The drop-in C++ API (include/latsum/*.hpp): the reference's own hot-path
test cases re-hosted in tests/cpp/dropin_tests.cpp, compiled against the
drop-in headers and linked to liblatsum_cuda.so. Compilation is checked on
CPU; the cases run on the GPU."""
import os
import shutil
import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

SRC = ROOT / "tests" / "cpp" / "dropin_tests.cpp"
LIBDIR = ROOT / "paper_1405_2270_b200"


def compile_dropin(out: Path) -> subprocess.CompletedProcess:
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-Werror", f"-I{ROOT / 'include'}",
           f"-I{ROOT / 'include' / 'eigen_compat'}", str(SRC), "-o", str(out), f"-L{LIBDIR}", "-llatsum_cuda",
           f"-Wl,-rpath,{LIBDIR}"]
    return subprocess.run(cmd, capture_output=True, text=True)


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    out = tmp_path_factory.mktemp("dropin") / "dropin_tests"
    r = compile_dropin(out)
    assert r.returncode == 0, r.stderr
    return out


def test_dropin_headers_compile_cleanly(binary):
    assert binary.exists()


def test_headers_are_self_contained(tmp_path):
    # every public header compiles on its own (drop-in include hygiene)
    for h in sorted((ROOT / "include" / "latsum").glob("*.hpp")):
        src = tmp_path / f"inc_{h.stem}.cpp"
        src.write_text(f'#include "latsum/{h.name}"\nint main() {{ return 0; }}\n')
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror",
                            f"-I{ROOT / 'include'}", f"-I{ROOT / 'include' / 'eigen_compat'}", str(src)],
                           capture_output=True, text=True)
        assert r.returncode == 0, (h.name, r.stderr)


@pytest.mark.gpu
def test_dropin_cases_pass_on_gpu(binary):
    r = subprocess.run([str(binary)], capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 failed" in r.stdout
