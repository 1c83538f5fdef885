"""GPU: race stress of the TMA ring's slot release (thiim_ring.cuh).  Random
shapes / seeds / step counts through the fused, TBLOCK and table engines,
bitwise against the oracle.  Calibration: a test build without release
ordering (-DTHIIM_RING_FENCE=2) fails ~1% of these cases (19 / 1925 in
120 s on a B200); the shipped dependency-token release must fail none."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ring_release_stress():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "stress_ring.py"),
                        "--seconds", "25", "--seed", "11"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"failures": 0' in r.stdout
