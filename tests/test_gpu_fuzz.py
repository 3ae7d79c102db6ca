"""Randomised shapes / dtypes / memory layouts / reductions through the public
API against the CPU oracle (tests/fuzz_probe.py): 250 seeded cases."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", [11, 12])
def test_fuzz_against_oracle(seed):
    r = subprocess.run([sys.executable, "-W", "ignore", os.path.join(ROOT, "tests", "fuzz_probe.py"), "125", str(seed)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout


@pytest.mark.gpu
def test_fuzz_time_resolved_and_front_end_against_oracle():
    # time-resolved mode (Eq 8), analytic signal and band-pass front end: tests/fuzz_probe2.py
    r = subprocess.run([sys.executable, "-W", "ignore", os.path.join(ROOT, "tests", "fuzz_probe2.py"), "150", "7"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failures" in r.stdout
