"""Guard-page runs of the CUDA entry points (tests/devtools/guard_run.py): every buffer of every
call alone in its own virtual-address range with unmapped guard granules on both sides, placed
flush against the upper guard and then against the lower one, so any out-of-bounds device read
or write faults. compute-sanitizer is closed on the GPU pool; this is the memory-safety check
that replaces it. Each placement runs in its own process (a fault poisons the CUDA context)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("placement", ["end", "start"])
def test_guarded_buffers(placement):
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "devtools" / "guard_run.py"), placement],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"({placement})" in r.stdout and r.stdout.startswith("ok ")


def test_guard_catches_an_overrun():
    """Negative control: a factor one element short of its stated size faults against the guard."""
    r = subprocess.run([sys.executable, str(ROOT / "tests" / "devtools" / "guard_run.py"), "control"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode != 0 and "no fault" not in r.stdout, r.stdout + r.stderr[-2000:]
