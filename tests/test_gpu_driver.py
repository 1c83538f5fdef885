"""The repo-local driver build/thiim-gpu-bench (adapter/thiim_gpu_bench.cpp):
`run` / `tune` with the reference CLI's semantics (tools/main.cpp:63-208) on
the reference's benchmark problem -- report line, check_against_naive,
exactly-once sanitizer, reports.jsonl/csv, trial table CSV and winner JSON."""
import csv
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "thiim-gpu-bench")
needs_exe = pytest.mark.skipif(not os.path.exists(EXE),
                               reason="build/thiim-gpu-bench not built (needs /root/reference)")


def drive(*args, cwd=None):
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=900, cwd=cwd)


@needs_exe
def test_usage_and_config_errors():
    r = drive("--help")
    assert r.returncode == 0 and "usage: thiim-gpu-bench run|tune" in r.stderr
    assert drive("run", "--bogus").returncode == 2
    assert drive("frobnicate").returncode == 2


@needs_exe
@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["gpu", "gpu-tblock", "gpu-tblock-inplace", "gpu-fused",
                                    "gpu-split"])
def test_run_checks_against_naive_and_sanitizes(tmp_path, engine):
    # TBLOCK in place is not instrumented: the sanitizer is a config error there
    san = [] if engine == "gpu-tblock-inplace" else ["--sanitize"]
    r = drive("run", "--grid", "40x36x30", "--steps", "5", "--engine", engine, "--check",
              *san, "--report-dir", str(tmp_path))
    assert r.returncode == 0, r.stdout + r.stderr
    assert "verification: bitwise-equal" in r.stdout
    if san:
        assert "sanitizer: exactly-once coverage OK" in r.stdout
    else:
        r2 = drive("run", "--grid", "40x36x30", "--steps", "5", "--engine", engine, "--sanitize",
                   "--report-dir", str(tmp_path))
        assert r2.returncode == 2, r2.stdout + r2.stderr
    line = [l for l in r.stdout.splitlines() if l.startswith("engine=")][0]
    want = {"gpu": "gpu-tblock"}.get(engine, engine)
    assert line.startswith("engine=%s grid=40x36x30 steps=5(executed 5) threads=1" % want)
    assert "mlups=" in line and "balance_model=" in line and "predicted_mlups=" in line
    rep = [json.loads(l) for l in open(tmp_path / "reports.jsonl")]
    assert rep[-1]["engine"] == want and rep[-1]["verification"] == "bitwise-equal"
    assert os.path.getsize(tmp_path / "reports.csv") > 0


@needs_exe
@pytest.mark.gpu
def test_run_multi_slab_on_one_gpu_is_rejected_or_checked(tmp_path):
    # --threads counts GPUs; with one GPU visible, 2 slabs must fail as a config error
    r = drive("run", "--grid", "32", "--steps", "2", "--threads", "2",
              "--report-dir", str(tmp_path))
    assert r.returncode in (0, 2), r.stdout + r.stderr
    if r.returncode == 0:
        assert "verification: bitwise-equal" in r.stdout


@needs_exe
@pytest.mark.gpu
def test_tune_writes_trial_table_and_verified_winner(tmp_path):
    """Model-ranked candidates (time block x tile height x z-chunk x band x
    schedule), timed; the winner is the deepest time block within 2% of the
    fastest and is verified against run_naive on the benchmark problem."""
    table, winner = tmp_path / "trials.csv", tmp_path / "winner.json"
    r = drive("tune", "--grid", "64", "--steps", "6", "--trials", "6", "--min-seconds", "0.05",
              "--table", str(table), "--winner", str(winner))
    assert r.returncode == 0, r.stdout + r.stderr
    rows = list(csv.DictReader(open(table)))
    assert 6 <= len(rows) <= 7 and all(r_["engine"] == "gpu-tblock" for r_ in rows)
    assert {r_["time_block"] for r_ in rows} == {"2", "3"}  # both depths are timed
    assert all(r_["ok"] == "1" and float(r_["mlups"]) > 0 for r_ in rows)
    assert all(float(r_["model_mlups"]) > 0 and float(r_["model_bytes_per_lup"]) > 0 for r_ in rows)
    w = json.loads(open(winner).read())
    best = max(float(r_["mlups"]) for r_ in rows)
    assert w["mlups"] >= 0.98 * best - 0.01
    assert "verification: bitwise-equal vs naive" in r.stdout
