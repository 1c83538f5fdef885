"""GPU parity: the CUDA engines against the C oracle / the reference, through
the C-ABI (paper_1510_05218_b200 binds include/thiim_gpu.h with ctypes).

Bar: BITWISE equality (kernels built with -fmad=false plus explicit _rn
intrinsics, reference op order kernels.cpp:43-51).  The north-star tolerance
(max per-component relative L2 <= 1e-12) is asserted too, as the weaker
documented bound.
"""
import os

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ENGINES = [P.ENGINE_SPLIT, P.ENGINE_FUSED, P.ENGINE_TBLOCK]
REL_L2_TOL = 1e-12  # BASELINE.json north_star


def threads():
    return min(16, os.cpu_count() or 1)


def gpu_run(state: P.ProblemState, steps: int, engine: int, **kw) -> P.ProblemState:
    out = P.clone_state(state)
    P.run_gpu(out, steps, P.GpuOptions(engine=engine, **kw))
    return out


def oracle_run(state: P.ProblemState, steps: int) -> P.ProblemState:
    out = P.clone_state(state)
    d = state.dims
    O.c_step((d.nx, d.ny, d.nz), out.arrays, steps, threads=threads())
    return out


def assert_same(got: P.ProblemState, want: P.ProblemState):
    diff = P.compare_states(got, want)
    assert diff.max_rel_l2 <= REL_L2_TOL, diff
    assert diff.bitwise_equal, diff


# ---------------------------------------------------------------- equivalence matrix
SHAPES = [
    (4, 4, 4),       # minimum valid grid (grid.hpp:21)
    (9, 7, 6),       # ragged, smaller than one tile
    (33, 17, 12),    # one past a warp in x
    (31, 29, 40),    # ragged vs 30x6 fused tiles and 32x4 split tiles
    (70, 13, 37),
    (64, 64, 64),    # config 0 grid
    (96, 48, 20),
]


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", SHAPES)
def test_engine_matches_oracle(engine, shape):
    dims = P.GridDims(*shape)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed=11)
    for steps in (1, 2, 5):
        assert_same(gpu_run(s, steps, engine), oracle_run(s, steps))


@pytest.mark.parametrize("engine,tile_y", [(P.ENGINE_TBLOCK, 12), (P.ENGINE_TBLOCK, 14),
                                           (P.ENGINE_TBLOCK, 16), (P.ENGINE_FUSED, 8),
                                           (P.ENGINE_FUSED, 16)])
def test_tile_height_instances_match_oracle(engine, tile_y):
    """The alternative CTA heights `tune` times (thiim-gpu-bench tune)."""
    dims = P.GridDims(70, 45, 33)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed=13)
    for steps in (2, 3):
        assert_same(gpu_run(s, steps, engine, tile_y=tile_y), oracle_run(s, steps))


@pytest.mark.parametrize("engine", ENGINES)
@pytest.mark.parametrize("shape", [(300, 5, 4), (5, 300, 9), (4, 4, 130)])
def test_extreme_aspect_ratios(engine, shape):
    dims = P.GridDims(*shape)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed=17)
    assert_same(gpu_run(s, 3, engine), oracle_run(s, 3))


@pytest.mark.parametrize("engine", ENGINES)
def test_layered_problem_matches_oracle(engine):
    dims = P.GridDims(40, 36, 48)
    s = P.generate_problem(dims, P.GEN_LAYERED, seed=5)
    assert_same(gpu_run(s, 4, engine), oracle_run(s, 4))


@pytest.mark.parametrize("engine", ENGINES)
def test_zchunks_do_not_change_results(engine):
    dims = P.GridDims(40, 24, 50)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed=3)
    want = oracle_run(s, 2)
    for zc in (1, 4, 7, 50):
        assert_same(gpu_run(s, 2, engine, z_chunk=zc), want)


def test_config0_full_length_vs_reference():
    """BASELINE config 0: 64^3 x 50 iterations, checked against the real reference
    run_naive (oracle/_ref) when available, else the C restatement."""
    dims = P.GridDims(64, 64, 64)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed=1)
    want = P.clone_state(s)
    if O.ref_available():
        O.ref_run_naive((64, 64, 64), want.arrays, 50, threads())
    else:
        O.c_step((64, 64, 64), want.arrays, 50, threads=threads())
    for engine in ENGINES:
        assert_same(gpu_run(s, 50, engine), want)


def test_tblock_full_config1_grid_vs_fused():
    """TBLOCK (2 steps per HBM pass) == fused, bitwise, on the 256^3 grid."""
    d = P.GridDims(256, 256, 256)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_FUSED)) as a:
        a.generate(P.GEN_RANDOM, 1)
        a.step(6)
        ref = P.allocate_state(d)
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK)) as b:
        b.generate(P.GEN_RANDOM, 1)
        st = b.step(6)
        # three passes, each one launch per round of <= one CTA per SM
        assert st.kernel_launches >= 3 and st.kernel_launches % 3 == 0
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff


# ---------------------------------------------------------------- generator
@pytest.mark.parametrize("kind", [P.GEN_RANDOM, P.GEN_LAYERED])
def test_device_generator_matches_host(kind):
    dims = P.GridDims(37, 21, 30)
    host = P.generate_problem(dims, kind, seed=9)
    with P.GpuEngine(dims) as eng:
        eng.generate(kind, seed=9)
        dev = eng.download_state()
    for a in range(40):
        assert np.array_equal(dev.arrays[a].view(np.uint64), host.arrays[a].view(np.uint64)), a


# ---------------------------------------------------------------- reference KATs
# (tests/test_kernels.cpp of the reference, re-expressed on whole steps)
@pytest.mark.parametrize("engine", ENGINES)
def test_single_cell_kat(engine):
    """test_kernels.cpp:27-43: Hyz with t=0.5, F=2, c=1, dE=0.25, src=0.1 -> 1.35."""
    d = P.GridDims(4, 4, 4)
    s = P.allocate_state(d)
    c = P.Component.Hyz
    i, j = d.linear_index(1, 1, 1), d.linear_index(1, 1, 2)
    s.field(c)[i] = 2.0
    s.t_of(c)[i] = 0.5
    s.c_of(c)[i] = 1.0
    s.coeff_src[P.source_index(c)][i] = 0.1
    s.field(P.Component.Exy)[j] = 0.25  # operand_a of Hyz at +z
    out = gpu_run(s, 1, engine)
    assert abs(out.field(c)[i].real - 1.35) <= 1e-15 * 1.35
    assert out.field(c)[i].imag == 0.0
    assert_same(out, oracle_run(s, 1))


@pytest.mark.parametrize("engine", ENGINES)
def test_identity_coefficients(engine):
    """test_kernels.cpp:45-61: t = 1, c = 0 leaves fields bitwise unchanged."""
    d = P.GridDims(8, 8, 8)
    s = P.allocate_state(d)
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    for ci in range(12):
        s.interior(12 + ci)[...] = 1.0
        s.interior(ci)[...] = (0.1 * x - 0.2 * y) + 1j * (0.3 * z + 0.01 * x)
    out = gpu_run(s, 1, engine)
    assert P.compare_states(out, s).bitwise_equal


@pytest.mark.parametrize("engine", ENGINES)
def test_zero_fixed_point_and_ghosts(engine):
    """test_kernels.cpp:131-153: zero fields/sources stay zero; ghosts stay zero."""
    d = P.GridDims(8, 12, 8)
    dims = (d.nx, d.ny, d.nz)
    arrays = O.c_benchmark_problem(dims)
    s = P.ProblemState(d, arrays)
    out = gpu_run(s, 3, engine)
    for ci in range(12):
        v = out.view3d(ci).copy()
        v[1:-1, 1:-1, 1:-1] = 0
        assert not np.any(v), "ghost written"
    z = P.clone_state(s)
    for a in z.coeff_src:
        a[:] = 0
    outz = gpu_run(z, 4, engine)
    assert not any(np.any(f) for f in outz.fields)


@pytest.mark.parametrize("engine", ENGINES)
def test_power_of_two_source_scaling(engine):
    """test_kernels.cpp:155-177 / acceptance criterion 9: src x2 -> fields x2 bitwise."""
    d = P.GridDims(8, 8, 8)
    a = P.ProblemState(d, O.c_benchmark_problem((8, 8, 8)))
    b = P.clone_state(a)
    for s in b.coeff_src:
        s *= 2.0
    ra, rb = gpu_run(a, 8, engine), gpu_run(b, 8, engine)
    for ci in range(12):
        assert np.array_equal((2.0 * ra.interior(ci)).view(np.uint64), rb.interior(ci).view(np.uint64))


@pytest.mark.parametrize("engine", ENGINES)
def test_point_source_support(engine):
    """test_kernels.cpp:179-216: one step spreads a point source one H and one E shift."""
    d = P.GridDims(10, 10, 10)
    s = P.allocate_state(d)
    O.c_fill_uniform((10, 10, 10), s.arrays)
    for a in s.coeff_src:
        a[:] = 0
    seed = P.Component.Hxz
    px = py = pz = 5
    s.coeff_src[P.source_index(seed)][d.linear_index(px, py, pz)] = 1.0
    out = gpu_run(s, 1, engine)
    expect = {c: set() for c in P.Component}
    expect[seed].add((px, py, pz))
    for c, (fam, axis, _, oa, ob, _, _) in P.COMPONENT_TABLE.items():
        if fam != "E" or seed not in (oa, ob):
            continue
        expect[c].add((px, py, pz))
        p = [px, py, pz]
        p[axis] += 1
        if all(v < n for v, n in zip(p, (d.nx, d.ny, d.nz))):
            expect[c].add(tuple(p))
    for c in P.Component:
        nz = np.argwhere(out.interior(int(c)) != 0)
        got = {(int(x), int(y), int(z)) for z, y, x in nz}
        assert got == expect[c], c


# ---------------------------------------------------------------- API behaviour
def test_zero_steps_and_validation():
    d = P.GridDims(8, 8, 8)
    s = P.generate_problem(d, P.GEN_RANDOM, 2)
    out = P.clone_state(s)
    r = P.run_gpu(out, 0)
    assert P.compare_states(out, s).bitwise_equal and r.mlups is None
    with pytest.raises(P.ConfigError):
        P.run_gpu(out, -1)
    with pytest.raises(P.SetupError):
        P.GpuEngine(P.GridDims(3, 8, 8))


def test_split_vs_fused_full_config1_grid():
    """Size-independent check at BASELINE config 1 (256^3): both engines agree
    bitwise after several steps (compared on device)."""
    d = P.GridDims(256, 256, 256)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_SPLIT)) as a:
        a.generate(P.GEN_RANDOM, 1)
        a.step(4)
        ref = P.allocate_state(d)
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_FUSED)) as b:
        b.generate(P.GEN_RANDOM, 1)
        b.step(4)
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff
