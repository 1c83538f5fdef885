"""GPU: the compressed coefficient layout (THIIM_COEFF_TABLE: uint8 material
ids + a per-material table) gives results bitwise equal to
the reference-layout oracle on the equivalent full problem."""
import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def oracle_run(s, steps):
    out = P.clone_state(s)
    d = s.dims
    O.c_step((d.nx, d.ny, d.nz), out.arrays, steps, threads=8)
    return out


@pytest.mark.parametrize("engine", [P.ENGINE_FUSED, P.ENGINE_TBLOCK])
@pytest.mark.parametrize("shape,steps,zc", [((40, 36, 48), 4, 0), ((31, 29, 60), 3, 7),
                                           ((64, 64, 64), 5, 0), ((9, 7, 12), 2, 0),
                                           ((57, 30, 19), 6, 5)])
def test_table_layout_generated_matches_oracle(shape, steps, zc, engine):
    d = P.GridDims(*shape)
    host = P.generate_problem(d, P.GEN_LAYERED, seed=5)
    want = oracle_run(host, steps)
    opts = P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6, z_chunk=zc, engine=engine)
    with P.GpuEngine(d, opts) as eng:
        eng.generate(P.GEN_LAYERED, seed=5)
        mid, tab = eng.download_table(6)
        # the device generator's ids/table expand to the host generator's arrays
        full = P.expand_coefficients(d, mid, tab)
        for k in range(12, 40):
            assert np.array_equal(full.interior(k).view(np.uint64), host.interior(k).view(np.uint64))
        st = eng.step(steps)
        assert st.engine == engine
        assert st.balance_model == (192.5 if engine == P.ENGINE_TBLOCK else 385.0)
        got = P.allocate_state(d)
        eng.download_fields(got)
    diff = P.compare_states(got, want)
    assert diff.bitwise_equal, diff


@pytest.mark.parametrize("engine", [P.ENGINE_FUSED, P.ENGINE_TBLOCK])
def test_table_layout_upload_benchmark_problem(engine):
    """build_benchmark_problem (coefficients.cpp:94-111): vacuum + source plane,
    compressed to 3 coefficient rows (interior, source plane, ghosts)."""
    d = P.GridDims(24, 20, 28)
    s = P.ProblemState(d, O.c_benchmark_problem((24, 20, 28)))
    s.arrays[0][:] = P.generate_problem(d, P.GEN_RANDOM, 3).arrays[0]  # non-trivial fields
    for k in range(12):
        s.view3d(k)[0, :, :] = 0
        s.view3d(k)[-1, :, :] = 0
        s.view3d(k)[:, 0, :] = 0
        s.view3d(k)[:, -1, :] = 0
        s.view3d(k)[:, :, 0] = 0
        s.view3d(k)[:, :, -1] = 0
    mid, tab = P.compress_coefficients(s)
    assert len(tab) <= 4
    want = oracle_run(s, 6)
    with P.GpuEngine(d, P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=len(tab),
                                     engine=engine)) as eng:
        eng.upload_table(s.fields, mid, tab)
        eng.step(6)
        got = P.allocate_state(d)
        eng.download_fields(got)
    assert P.compare_states(got, want).bitwise_equal


def test_table_layout_rejections():
    d = P.GridDims(8, 8, 8)
    with pytest.raises(P.ConfigError):
        P.GpuEngine(d, P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=0))
    with pytest.raises(P.ConfigError):
        P.GpuEngine(d, P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6,
                                    engine=P.ENGINE_SPLIT))
    with P.GpuEngine(d, P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6)) as eng:
        with pytest.raises(P.ConfigError):
            eng.generate(P.GEN_RANDOM, 1)  # random media are not piecewise constant


def test_config3_generator_at_256_cubed_vs_oracle():
    """SURVEY s8d parity procedure: a 256^3 instance of the config-3 layered
    generator against the CPU oracle -- reference layout (TBLOCK) and table
    layout (TBLOCK-table), 4 iterations."""
    d = P.GridDims(256, 256, 256)
    host = P.generate_problem(d, P.GEN_LAYERED, seed=1)
    want = oracle_run(host, 4)
    for opts in (P.GpuOptions(), P.GpuOptions(coeff_layout=P.COEFF_TABLE, n_materials=6)):
        with P.GpuEngine(d, opts) as eng:
            eng.generate(P.GEN_LAYERED, seed=1)
            eng.step(4)
            diff = eng.compare_fields(want)
        assert diff.bitwise_equal, (opts.coeff_layout, diff)
