"""GPU: the exactly-once coverage sanitizer (the
reference's UpdateLog check, tools/main.cpp:20-41).  With the sanitizer on,
every output store of the default kernels is counted and each pass must store
every (component, interior cell) exactly once and no ghost -- over all
engines, z-chunkings, odd step counts, the table layout and multi-slab
contexts (deep TBLOCK halos included).  Results stay bitwise equal to the
oracle, and an uninstrumented schedule is reported as violating."""
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _passes(engine, steps):
    return steps // 2 + steps % 2 if engine == P.ENGINE_TBLOCK else steps


@pytest.mark.parametrize("engine", [P.ENGINE_SPLIT, P.ENGINE_FUSED, P.ENGINE_TBLOCK])
# nx mod 28 = 9, 8, 6 (TBLOCK folds the remainder into 16-lane segments),
# 4, 3 (8-lane segments)
@pytest.mark.parametrize("shape,steps,zc", [((37, 29, 23), 5, 0), ((64, 40, 48), 4, 7),
                                           ((90, 61, 18), 3, 5), ((60, 47, 20), 4, 0),
                                           ((31, 70, 16), 2, 3)])
def test_exactly_once_single_slab(engine, shape, steps, zc):
    d = P.GridDims(*shape)
    with P.GpuEngine(d, P.GpuOptions(engine=engine, z_chunk=zc)) as e:
        e.generate(P.GEN_RANDOM, 3)
        e.set_sanitize(True)
        e.step(steps)
        assert e.coverage() == (_passes(engine, steps), 0)
        got = P.allocate_state(d)
        e.download_fields(got)
    want = P.generate_problem(d, P.GEN_RANDOM, 3)
    O.c_step(shape, want.arrays, steps, threads=8)
    assert P.compare_states(got, want).bitwise_equal


@pytest.mark.parametrize("engine", [P.ENGINE_FUSED, P.ENGINE_TBLOCK])
def test_exactly_once_table_layout(engine):
    d = P.GridDims(45, 33, 40)
    with P.GpuEngine(d, P.GpuOptions(engine=engine, coeff_layout=P.COEFF_TABLE,
                                     n_materials=6)) as e:
        e.generate(P.GEN_LAYERED, 4)
        e.set_sanitize(True)
        e.step(5)
        assert e.coverage() == (_passes(engine, 5), 0)


@pytest.mark.parametrize("engine", [P.ENGINE_SPLIT, P.ENGINE_FUSED, P.ENGINE_TBLOCK])
def test_exactly_once_multi_slab(engine):
    d = P.GridDims(40, 30, 36)
    with P.GpuEngine(d, P.GpuOptions(engine=engine, n_gpus=3, same_device=1)) as e:
        e.generate(P.GEN_RANDOM, 5)
        e.set_sanitize(True)
        e.step(5)
        assert e.coverage() == (_passes(engine, 5), 0)


def test_uninstrumented_schedule_is_reported(monkeypatch):
    """Negative control: the uninstrumented TBLOCK instances store without
    counting, so every interior (component, cell) of every pass must show up
    as a violation."""
    monkeypatch.setenv("THIIM_SANITIZE_UNCOUNTED", "1")
    d = P.GridDims(30, 20, 16)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK)) as e:
        e.generate(P.GEN_RANDOM, 1)
        e.set_sanitize(True)
        e.step(4)
        passes, bad = e.coverage()
    assert passes == 2 and bad == 2 * 12 * d.interior_cells()


def test_sanitizer_needs_enabling():
    with P.GpuEngine(P.GridDims(8, 8, 8)) as e:
        e.generate(P.GEN_RANDOM, 1)
        with pytest.raises(P.GpuError):
            e.coverage()
