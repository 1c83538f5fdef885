"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU
(runnable here), the native line on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _line(args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _line(["--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "MLUP/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_native_line():
    d = _line(["--config", "c0", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["scaling"] == "weak"
    assert d["config"]["workload"].startswith("configs[0]")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["stream"]["value"] > 0 and e["serial"]["value"] > 0
    assert e["value"] == max(e["stream"]["value"], e["serial"]["value"])
    assert e["api"] in (e["stream"]["api"], e["serial"]["api"])
    assert set(e["stream"]["device_ms_per_step"]) == {"upload", "sweep", "download"}
    assert d["gpu_launches"] >= 3
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert "traffic_bytes_per_lup" in r  # null unless this grid was captured under ncu
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1
    if cb["kind"] == "reference":
        assert cb["host_triad_gbs"] > 0  # the reference's own measure_bandwidth
    c = d["clocks"]
    assert c["sm_max_mhz"] and isinstance(c["reasons"], list)
    b = d["cpu_baseline"]
    assert b["value"] > 0 and b["unit"] == "MLUP/s" and b["cores"] >= 1
