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
    d = _line(["--impl", "reference", "--config", "c0", "--steps", "1", "--warmup", "1"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["unit"] == "MLUP/s"
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}


def test_reference_arm_loads_only_the_reference_library():
    """The reference arm generates its problem inside oracle/_ref and times the
    reference's run_naive there: no product library (and no C port) is mapped."""
    code = ("import runpy, sys\n"
            "sys.argv = ['bench.py', '--impl', 'reference', '--config', 'c0', '--steps', '1',"
            " '--warmup', '0']\n"
            "runpy.run_path('bench.py', run_name='__main__')\n"
            "print('MAPS', sorted({l.split()[-1] for l in open('/proc/self/maps')"
            " if l.rstrip().endswith('.so') and '/root' in l or 'repo' in l.split()[-1]}))\n")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    maps = eval(r.stdout.split("MAPS", 1)[1].strip())
    mine = [m for m in maps if m.startswith(ROOT)]
    from oracle import oracle as O
    if O.ref_available():
        assert mine == [os.path.join(ROOT, "oracle", "_ref", "libthiim_ref.so")], mine
    assert not any("paper_1510_05218_b200" in m for m in mine), mine


def test_default_configs():
    m = _bench_module()
    assert m.default_config(1) == "c2" and m.default_config(2) == "c4"
    assert m.default_config(8) == "c4"
    assert m.CONFIGS["c2"][:2] == ((512, 512, 512), 200)
    assert m.CONFIGS["c4"][:2] == ((1024, 1024, 128), 100)
    assert m.sample_grid((512, 512, 512)) == (512, 512, 128)
    assert m.sample_grid((64, 64, 64)) == (64, 64, 64)


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


def _bench_module():
    import importlib.util
    spec = importlib.util.spec_from_file_location("thiim_bench", os.path.join(ROOT, "bench.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_roofline_helper_keys_traffic_by_kernel_and_grid():
    """Host logic only: the roofline of a TBLOCK pass (two iterations; one launch
    per round of CTAs) uses the algorithmic 832 B per cell, reports ncu traffic
    only for a captured grid; a depth-3 pass is three iterations."""
    import paper_1510_05218_b200 as P
    B = _bench_module()
    dims = P.GridDims(256, 256, 256)
    r = B._roofline(P, dims, P.ENGINE_TBLOCK, dev_secs=0.15, launches=150, iters_total=100)
    cells = 256 ** 3
    assert r["algorithmic_bytes_per_launch"] == 832.0 * cells
    assert abs(r["achieved"] - 832.0 * cells / (0.15 / 50) / 1e9) < 0.1
    assert r["bytes_per_lup_model"] == 416.0 and r["kernel"] == "k_tblock_tm<15,6>"
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
        t = json.load(f)
    if "k_tblock_tm<15,6>@256x256x256" in t:
        assert r["traffic"] == t["k_tblock_tm<15,6>@256x256x256"]
        assert abs(r["traffic_bytes_per_lup"] - r["traffic"] / (2 * cells)) < 0.1
    if "k_tblock_tm<15,6>@512x512x512" in t:
        big = B._roofline(P, P.GridDims(512, 512, 512), P.ENGINE_TBLOCK, 1.0, 600, iters_total=200)
        assert big["traffic"] == t["k_tblock_tm<15,6>@512x512x512"]
    other = B._roofline(P, P.GridDims(384, 320, 96), P.ENGINE_TBLOCK, 1.0, 100)
    assert other["traffic"] is None and other["traffic_bytes_per_lup"] is None


def test_roofline_helper_depth3():
    import paper_1510_05218_b200 as P
    B = _bench_module()
    cells = 128 ** 3
    r = B._roofline(P, P.GridDims(128, 128, 128), P.ENGINE_TBLOCK, dev_secs=0.3, launches=99,
                    iters_total=99, depth=3)
    assert r["kernel"] == "k_tblock3_tm<15,6>" and r["bytes_per_lup_model"] == pytest.approx(832 / 3)
    assert abs(r["achieved"] - 832.0 * cells / (0.3 / 33) / 1e9) < 0.1


def test_clock_sampler_parses_reasons_and_power():
    """Host logic only: the nvidia-smi sampler's parsing (median SM clock and
    power, throttle reasons) on canned output."""
    B = _bench_module()

    class FakeProc:
        def terminate(self):
            pass

        def communicate(self, timeout=None):
            return ("0, 1530, 1965, 990.5, 0x4, Not Active, Not Active, Not Active, Active\n"
                    "0, 1545, 1965, 998.1, 0x4, Not Active, Not Active, Not Active, Active\n"
                    "0, 1560, 1965, 994.0, 0x0, Not Active, Not Active, Not Active, Not Active\n",
                    "")

    c = B.Clocks(0)
    c.proc = FakeProc()
    c.__exit__(None, None, None)
    assert c.result["sm_mhz"] == 1545.0 and c.result["sm_max_mhz"] == 1965.0
    assert c.result["reasons"] == ["sw_power_cap"] and c.result["samples"] == 3
    assert abs(c.result["power_w"] - 994.0) < 1e-9
