"""Host-side coefficient compression (thiim_coeff_compress): the reference
layout's 28 coefficient arrays of a piecewise-constant medium -> material ids
+ table (the THIIM_COEFF_TABLE layout), as run_gpu(coeff_layout=COEFF_AUTO)
and thiim::run_gpu(coeff_layout = THIIM_COEFF_AUTO_HOST) use it.  CPU tests
run without a GPU (the function is host code); the gpu test runs the AUTO
path end to end against the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def interior_rows(s: P.ProblemState) -> np.ndarray:
    """(interior cells, 56) uint64 coefficient rows in linear-index order."""
    cols = [np.ascontiguousarray(s.interior(12 + k)).reshape(-1).view(np.uint64).reshape(-1, 2)
            for k in range(28)]
    return np.concatenate(cols, axis=1)


@pytest.mark.parametrize("shape,seed", [((40, 33, 24), 3), ((17, 9, 31), 8), ((64, 64, 12), 1)])
def test_layered_media_round_trip(shape, seed):
    d = P.GridDims(*shape)
    s = P.generate_problem(d, P.GEN_LAYERED, seed)
    r = P.coeff_compress(s)
    assert r is not None
    mid, tab = r
    assert mid.shape == (d.padded_cells(),) and tab.shape[1] == 28 and 1 <= len(tab) <= 16
    # interior cells get their own rows back, bit for bit
    m3 = mid.reshape(d.pz(), d.py(), d.px())
    got = tab[m3[1:-1, 1:-1, 1:-1].reshape(-1)]
    want = interior_rows(s)
    assert np.array_equal(np.ascontiguousarray(got).view(np.uint64).reshape(-1, 56), want)
    # ghost cells carry id 0
    ghost = np.ones_like(m3, dtype=bool)
    ghost[1:-1, 1:-1, 1:-1] = False
    assert (m3[ghost] == 0).all()
    # table rows in order of first appearance along the interior
    uniq, first = np.unique(want, axis=0, return_index=True)
    order = uniq[np.argsort(first)]
    assert np.array_equal(np.ascontiguousarray(tab).view(np.uint64).reshape(-1, 56), order)


def test_random_media_and_material_limit():
    d = P.GridDims(20, 18, 16)
    assert P.coeff_compress(P.generate_problem(d, P.GEN_RANDOM, 4)) is None
    layered = P.generate_problem(d, P.GEN_LAYERED, 4)
    n = len(P.coeff_compress(layered)[1])
    assert P.coeff_compress(layered, max_materials=n) is not None
    assert P.coeff_compress(layered, max_materials=n - 1) is None
    with pytest.raises(P.ConfigError):
        P.coeff_compress(layered, max_materials=17)


def test_independent_of_the_thread_count():
    code = ("import sys, hashlib; sys.path.insert(0, %r); import paper_1510_05218_b200 as P; "
            "s = P.generate_problem(P.GridDims(50, 40, 37), P.GEN_LAYERED, 9); m, t = P.coeff_compress(s); "
            "print(hashlib.sha256(m.tobytes() + t.tobytes()).hexdigest())" % ROOT)
    out = set()
    for n in ("1", "3", "8"):
        env = dict(os.environ, OMP_NUM_THREADS=n)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                           timeout=300)
        assert r.returncode == 0, r.stderr
        out.add(r.stdout.strip())
    assert len(out) == 1


def test_context_rejects_the_host_only_layout():
    with pytest.raises(P.ConfigError):
        P.GpuEngine(P.GridDims(8, 8, 8), P.GpuOptions(coeff_layout=P.COEFF_AUTO))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,table", [(P.GEN_LAYERED, True), (P.GEN_RANDOM, False)])
def test_run_gpu_auto_layout_matches_oracle(kind, table):
    d = P.GridDims(48, 37, 29)
    s = P.generate_problem(d, kind, 12)
    want = P.clone_state(s)
    O.c_step((d.nx, d.ny, d.nz), want.arrays, 7, threads=min(16, os.cpu_count() or 1))
    r = P.run_gpu(s, 7, P.GpuOptions(coeff_layout=P.COEFF_AUTO))
    assert r.engine.endswith("-table") == table, r.engine
    assert r.balance_model == (192.5 if table else 416.0)
    assert P.compare_states(s, want).bitwise_equal
