"""GPU parity of TBLOCK in place (THIIM_ENGINE_TBLOCK_INPLACE): two-step
sub-range passes on one field set whose outputs shift into a gap of L + 2
planes, alternately up and down (thiim_gpu.cu launch_tblock_inplace) -- the engine AUTO picks when
the state fits in HBM once but not twice (BASELINE config 3 in the reference
layout).  Bitwise against the C oracle (step_reference, kernels.cpp:105-113)
for sub-range lengths that split z raggedly, L = 2 (every plane through the
tail), L >= nz (one sub-range), odd step counts (split remainder), ragged x
(folded remainder tiles), the layered problem and non-zero ghost rings (the
copy-back must leave them alone)."""
import os

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _oracle(state, steps):
    out = P.clone_state(state)
    d = state.dims
    O.c_step((d.nx, d.ny, d.nz), out.arrays, steps, threads=min(16, os.cpu_count() or 1))
    return out


def _inplace(state, steps, L, monkeypatch):
    monkeypatch.setenv("THIIM_INPLACE_TB", str(L))
    out = P.clone_state(state)
    rep = P.run_gpu(out, steps, P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE))
    assert rep.engine == "gpu-tblock-inplace"
    return out


def _same(a, b):
    d = P.compare_states(a, b)
    assert d.bitwise_equal, d


@pytest.mark.parametrize("shape,L", [((33, 17, 12), 5), ((31, 29, 40), 7), ((70, 13, 37), 16),
                                     ((9, 7, 6), 2), ((40, 26, 9), 64), ((256, 24, 30), 8),
                                     ((4, 4, 4), 2),
                                     # last sub-range of exactly one plane (nz % L == 1)
                                     ((33, 17, 13), 4), ((20, 9, 9), 8)])
def test_inplace_matches_oracle(shape, L, monkeypatch):
    s = P.generate_problem(P.GridDims(*shape), P.GEN_RANDOM, seed=5)
    # 1, 2, 3 and 4 passes: odd counts end on the shifted position and move back
    for steps in (2, 3, 4, 6, 8):
        _same(_inplace(s, steps, L, monkeypatch), _oracle(s, steps))


def test_inplace_layered_and_ghost_ring(monkeypatch):
    s = P.generate_problem(P.GridDims(37, 30, 23), P.GEN_LAYERED, seed=2)
    # non-zero ghost data: read by the sweep, never written, never copied over
    rng = np.random.default_rng(0)
    d = s.dims
    px, py = d.nx + 2, d.ny + 2
    for k in range(12):
        a = s.arrays[k].reshape(d.nz + 2, py, px)
        a[:, 0, :] = rng.uniform(-1, 1, (d.nz + 2, px)) + 1j * rng.uniform(-1, 1, (d.nz + 2, px))
        a[:, :, -1] = rng.uniform(-1, 1, (d.nz + 2, py))
    for steps in (4, 5):
        _same(_inplace(s, steps, 6, monkeypatch), _oracle(s, steps))


def test_inplace_rejects_slabs_and_table():
    s = P.generate_problem(P.GridDims(8, 8, 8), P.GEN_RANDOM, seed=1)
    with pytest.raises(P.ConfigError):  # two z-slabs: in place needs one whole-z slab
        P.run_gpu(P.clone_state(s), 2, P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE, n_gpus=2,
                                                    same_device=1))
    with pytest.raises(P.ConfigError):  # the table layout has no in-place form
        P.run_gpu(P.clone_state(s), 2, P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE,
                                                    coeff_layout=P.COEFF_TABLE, n_materials=2))


def test_inplace_single_step_runs_split_and_says_so(monkeypatch):
    """One step has no two-step pass: the split remainder runs, and the report
    names the engine that ran."""
    monkeypatch.setenv("THIIM_INPLACE_TB", "4")
    s = P.generate_problem(P.GridDims(21, 11, 10), P.GEN_RANDOM, seed=3)
    out = P.clone_state(s)
    rep = P.run_gpu(out, 1, P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE))
    assert rep.engine == "gpu-split"
    _same(out, _oracle(s, 1))


@pytest.mark.parametrize("L", ["0", "1"])
def test_inplace_rejects_short_sub_ranges(L, monkeypatch):
    monkeypatch.setenv("THIIM_INPLACE_TB", L)
    with pytest.raises(P.ConfigError, match="sub-ranges"):
        P.GpuEngine(P.GridDims(16, 16, 16), P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE))


def test_inplace_rejects_the_sanitizer(monkeypatch):
    monkeypatch.setenv("THIIM_INPLACE_TB", "4")
    with P.GpuEngine(P.GridDims(16, 16, 16), P.GpuOptions(engine=P.ENGINE_TBLOCK_INPLACE)) as e:
        with pytest.raises(P.ConfigError):
            e.set_sanitize(True)
