"""Pipelined batches (thiim_gpu_run_batch / run_gpu_batch): a stream of
independent problems, each == run_naive(problem, steps)
(reference_engines.cpp:34-67), bitwise against the C oracle, in every
engine, for explicit and in-place outputs, shared outputs and every depth."""
import os

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

DIMS = P.GridDims(40, 33, 24)


def threads():
    return min(16, os.cpu_count() or 1)


def oracle_run(state: P.ProblemState, steps: int) -> P.ProblemState:
    out = P.clone_state(state)
    d = state.dims
    O.c_step((d.nx, d.ny, d.nz), out.arrays, steps, threads=threads())
    return out


def fields_equal(got, want) -> bool:
    return all(np.array_equal(g.view(np.uint64), w.view(np.uint64)) for g, w in zip(got, want))


def test_overlap_rejected_before_any_device_work():
    """Runs without a GPU: the aliasing check precedes every CUDA call."""
    s = P.generate_problem(P.GridDims(8, 8, 8), P.GEN_RANDOM, 1)
    with pytest.raises(P.ConfigError, match="overlaps input array 0 of problem 1"):
        P.run_gpu_batch([s, s], 2)  # in place into a state another problem reads
    t = P.generate_problem(P.GridDims(8, 8, 8), P.GEN_RANDOM, 2)
    with pytest.raises(P.ConfigError, match="overlaps"):
        P.run_gpu_batch([s, t], 2, outputs=[t.fields, s.fields])
    with pytest.raises(P.ConfigError, match="same grid dims"):
        P.run_gpu_batch([s, P.generate_problem(P.GridDims(9, 8, 8), P.GEN_RANDOM, 1)], 1)
    with pytest.raises(P.ConfigError):
        P.run_gpu_batch([s], -1)
    assert P.run_gpu_batch([], 3).n_problems == 0


@pytest.mark.gpu
@pytest.mark.parametrize("engine", [P.ENGINE_TBLOCK, P.ENGINE_FUSED, P.ENGINE_SPLIT])
@pytest.mark.parametrize("depth", [1, 2, 3, 8])
def test_batch_distinct_problems(engine, depth):
    steps = 5
    kinds = [P.GEN_RANDOM, P.GEN_LAYERED, P.GEN_RANDOM, P.GEN_LAYERED, P.GEN_RANDOM]
    states = [P.generate_problem(DIMS, k, seed=11 + i) for i, k in enumerate(kinds)]
    want = [oracle_run(s, steps) for s in states]
    outs = [[np.zeros_like(a) for a in s.fields] for s in states]
    before = [[a.copy() for a in s.arrays] for s in states]
    rep = P.run_gpu_batch(states, steps, P.GpuOptions(engine=engine), outputs=outs, depth=depth)
    assert rep.n_problems == len(states) and rep.depth == min(depth, len(states))
    for i, (o, w) in enumerate(zip(outs, want)):
        assert fields_equal(o, w.fields), ("problem", i)
    for s, b in zip(states, before):  # inputs untouched
        assert fields_equal(s.arrays, b)
    n = DIMS.padded_cells() * 16
    assert rep.h2d_bytes == len(states) * 40 * n and rep.d2h_bytes == len(states) * 12 * n
    assert rep.kernel_launches > 0 and rep.seconds > 0 and rep.device_seconds > 0
    assert rep.mlups > 0


@pytest.mark.gpu
def test_batch_in_place_and_shared_output():
    steps = 4
    states = [P.generate_problem(DIMS, P.GEN_RANDOM, seed=s) for s in (3, 4, 5, 6)]
    want = [oracle_run(s, steps) for s in states]
    P.run_gpu_batch(states, steps)  # in place, like run_naive
    for s, w in zip(states, want):
        assert fields_equal(s.fields, w.fields)
    # one input streamed K times into one shared output (bench.py's e2e shape)
    src = P.generate_problem(DIMS, P.GEN_LAYERED, seed=9)
    ref = oracle_run(src, steps)
    shared = [np.zeros_like(a) for a in src.fields]
    P.run_gpu_batch([src] * 5, steps, outputs=[shared] * 5)
    assert fields_equal(shared, ref.fields)


@pytest.mark.gpu
def test_batch_zero_steps_and_odd_steps():
    states = [P.generate_problem(DIMS, P.GEN_RANDOM, seed=s) for s in (21, 22)]
    outs = [[np.full_like(a, 7.0) for a in s.fields] for s in states]
    P.run_gpu_batch(states, 0, outputs=outs)
    for s, o in zip(states, outs):
        assert fields_equal(o, s.fields)
    want = [oracle_run(s, 7) for s in states]  # graph replay + odd remainder pass
    P.run_gpu_batch(states, 7, outputs=outs)
    for o, w in zip(outs, want):
        assert fields_equal(o, w.fields)


@pytest.mark.gpu
def test_batch_pinned_large():
    """256x128x64 problems, pinned host memory: results bitwise equal to the
    one-problem API (run_gpu), which the parity suite pins to the oracle."""
    d = P.GridDims(256, 128, 64)
    steps = 6
    src = P.generate_problem(d, P.GEN_RANDOM, seed=1)
    one = P.clone_state(src)
    P.run_gpu(one, steps)
    outs = [[np.zeros_like(a) for a in src.fields] for _ in range(2)]
    L = P.lib()
    bufs = src.arrays + [a for fs in outs for a in fs]
    for a in bufs:
        assert L.thiim_gpu_pin_host(a.ctypes.data, a.nbytes) == 0
    try:
        rep = P.run_gpu_batch([src] * 4, steps, outputs=[outs[0], outs[1], outs[0], outs[1]])
    finally:
        for a in bufs:
            L.thiim_gpu_unpin_host(a.ctypes.data)
    assert fields_equal(outs[0], one.fields) and fields_equal(outs[1], one.fields)
    # pipelining: the whole batch takes less than the phases run back to back
    assert rep.device_seconds < rep.upload_seconds + rep.kernel_seconds + rep.download_seconds


@pytest.mark.gpu
def test_batch_depth_shrinks_to_fit_memory():
    """With device memory for one context only, the stream runs at depth 1
    (one problem at a time) instead of failing; results unchanged."""
    import torch

    d = P.GridDims(128, 128, 128)
    ctx_bytes = d.padded_cells() * 16 * 52  # 2 field sets + 28 coefficient arrays
    states = [P.generate_problem(d, P.GEN_RANDOM, seed=s) for s in (1, 2, 3)]
    want = [oracle_run(s, 2) for s in states]
    outs = [[np.zeros_like(a) for a in s.fields] for s in states]
    P.release_cached(0)
    free, _ = torch.cuda.mem_get_info(0)
    hog = torch.empty(free - int(1.5 * ctx_bytes), dtype=torch.uint8, device="cuda:0")
    try:
        rep = P.run_gpu_batch(states, 2, outputs=outs, depth=3)
    finally:
        del hog
        torch.cuda.empty_cache()
    assert rep.depth == 1, rep
    for o, w in zip(outs, want):
        assert fields_equal(o, w.fields)


@pytest.mark.gpu
def test_batch_auto_runs_in_place_when_ping_pong_fits_once():
    """AUTO batch plan (thiim_gpu_run_batch, batch_plan): with device memory
    for one ping-pong TBLOCK context (52 arrays) but two TBLOCK-in-place ones
    (40 arrays + a gap of sub-range planes), the stream runs two in-place
    contexts so copies overlap sweeps (configs[2] on a 180-GB B200); results
    bitwise equal to the oracle."""
    import torch

    d = P.GridDims(256, 256, 128)
    ctx_bytes = d.padded_cells() * 16 * 52
    states = [P.generate_problem(d, k, seed=s) for k, s in ((P.GEN_RANDOM, 31), (P.GEN_LAYERED, 32))]
    srcs = [states[0], states[1], states[0]]
    # 6 steps: three passes, ends on an odd pass (array moved back); 7: plus the
    # split remainder step
    want = {steps: [oracle_run(s, steps) for s in states] for steps in (6, 7)}
    outs = {steps: [[np.zeros_like(a) for a in s.fields] for s in states] for steps in (6, 7)}
    P.release_cached(0)
    free, _ = torch.cuda.mem_get_info(0)
    hog = torch.empty(free - int(1.9 * ctx_bytes), dtype=torch.uint8, device="cuda:0")
    try:
        reps = {steps: P.run_gpu_batch(srcs, steps, outputs=[outs[steps][0], outs[steps][1],
                                                             outs[steps][0]], depth=3)
                for steps in (6, 7)}
    finally:
        del hog
        torch.cuda.empty_cache()
    for steps, rep in reps.items():
        assert rep.engine == "gpu-tblock-inplace" and rep.depth == 2, rep
        for o, w in zip(outs[steps], want[steps]):
            assert fields_equal(o, w.fields), steps
