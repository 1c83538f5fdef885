"""GPU parity of TBLOCK at time-block depth 3 (k_tblock3_tm, thiim_tblock3.cuh):
three THIIM steps per HBM pass, single-slot TMEM hand-offs between the three
levels, per-level chunk prologues and ghost planes.  Bitwise against the C
oracle (step_reference, kernels.cpp:105-113) over grids smaller than a tile,
ragged in x / y, z-chunkings that put a chunk start at every plane offset
(0, 1, 2, interior), step counts 3k, 3k+1 (fused remainder), 3k+2 (depth-2
remainder), the layered problem, non-zero ghost rings; the exactly-once
sanitizer certifies the schedule; configs[1]'s full grid equals depth 2."""
import os

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def threads():
    return min(16, os.cpu_count() or 1)


def oracle_run(state, steps):
    out = P.clone_state(state)
    d = state.dims
    O.c_step((d.nx, d.ny, d.nz), out.arrays, steps, threads=threads())
    return out


def tb3_run(state, steps, **kw):
    out = P.clone_state(state)
    rep = P.run_gpu(out, steps, P.GpuOptions(engine=P.ENGINE_TBLOCK, time_block=3, **kw))
    assert rep.engine == "gpu-tblock"
    return out


def assert_same(got, want):
    d = P.compare_states(got, want)
    assert d.bitwise_equal, d


@pytest.mark.parametrize("shape", [(4, 4, 4), (9, 7, 6), (26, 9, 10), (27, 10, 11), (33, 17, 12),
                                   (53, 19, 40), (70, 13, 37), (64, 64, 64)])
@pytest.mark.parametrize("steps", [3, 6, 7, 8])
def test_depth3_matches_oracle(shape, steps):
    s = P.generate_problem(P.GridDims(*shape), P.GEN_RANDOM, 3)
    assert_same(tb3_run(s, steps), oracle_run(s, steps))


@pytest.mark.parametrize("zc", [1, 2, 3, 4, 5, 7, 13])
def test_depth3_chunk_starts(zc):
    """Every chunk start re-runs three level prologues; chunk lengths from 1
    (every plane a chunk start) to ragged."""
    s = P.generate_problem(P.GridDims(40, 25, 29), P.GEN_RANDOM, 5)
    assert_same(tb3_run(s, 6, z_chunk=zc), oracle_run(s, 6))


def test_depth3_one_launch_schedule_and_bands():
    s = P.generate_problem(P.GridDims(150, 60, 18), P.GEN_RANDOM, 6)
    want = oracle_run(s, 9)
    assert_same(tb3_run(s, 9, schedule=1), want)
    assert_same(tb3_run(s, 9, band=2), want)
    assert_same(tb3_run(s, 9, band=1), want)


def test_depth3_layered_and_ghost_rings():
    d = P.GridDims(45, 31, 36)
    s = P.generate_problem(d, P.GEN_LAYERED, 2)
    rng = np.random.default_rng(1)
    for k in range(12):  # non-zero ghost values must be read, never written
        v = s.view3d(k)
        v[0], v[-1] = rng.standard_normal(v[0].shape), rng.standard_normal(v[-1].shape)
        v[:, 0], v[:, -1] = rng.standard_normal(v[:, 0].shape), rng.standard_normal(v[:, -1].shape)
        v[:, :, 0], v[:, :, -1] = (rng.standard_normal(v[:, :, 0].shape),
                                   rng.standard_normal(v[:, :, -1].shape))
    assert_same(tb3_run(s, 12), oracle_run(s, 12))


def test_depth3_exactly_once():
    d = P.GridDims(60, 33, 27)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK, time_block=3, z_chunk=7)) as e:
        e.generate(P.GEN_RANDOM, 5)
        e.set_sanitize(True)
        e.step(9)
        assert e.coverage() == (3, 0)


def test_depth3_config1_grid_vs_depth2():
    d = P.GridDims(256, 256, 256)
    n = d.padded_cells()
    ref = [np.empty(n, np.complex128) for _ in range(12)]
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK)) as a:
        a.generate(P.GEN_RANDOM, 1)
        a.step(12)
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK, time_block=3)) as b:
        b.generate(P.GEN_RANDOM, 1)
        st = b.step(12)
        assert st.balance_model == pytest.approx(832 / 3)
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff


def test_depth3_rejected_where_unsupported():
    with pytest.raises(P.ConfigError):
        P.GpuEngine(P.GridDims(16, 16, 16), P.GpuOptions(time_block=4))
    with pytest.raises(P.ConfigError):
        P.GpuEngine(P.GridDims(16, 16, 16), P.GpuOptions(time_block=3, n_gpus=2, same_device=1))


def test_python_tuner_on_a_small_grid():
    """paper_1510_05218_b200.tune: model-ranked candidates timed, the winner
    verified bitwise against the fused engine."""
    r = P.tune(P.GridDims(40, 30, 24), steps=6, min_seconds=0.02, max_trials=6)
    assert r.winner_verification == "bitwise-equal vs gpu-fused"
    assert 6 <= len(r.table) <= 7 and all(t["ok"] and t["mlups"] > 0 for t in r.table)
    # the best candidate of every (time block, tile height) is among the trials
    assert {(t["time_block"], t["tile_y"]) for t in r.table} >= {(2, 15), (2, 14), (2, 12),
                                                                    (2, 16), (3, 15)}
    best = max(t["mlups"] for t in r.table)
    won = [t for t in r.table if t["time_block"] == r.best.time_block and
           t["tile_y"] == r.best.tile_y and t["z_chunk"] == r.best.z_chunk and
           t["band"] == r.best.band and t["schedule"] == r.best.schedule]
    assert won and won[0]["mlups"] >= 0.98 * best
    # the winner runs and is bitwise
    s = P.generate_problem(P.GridDims(40, 30, 24), P.GEN_RANDOM, 2)
    want = oracle_run(s, 5)
    got = P.clone_state(s)
    P.run_gpu(got, 5, r.best)
    assert_same(got, want)
