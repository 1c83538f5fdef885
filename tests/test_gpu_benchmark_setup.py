"""GPU: the reference's benchmark problem built on the device
(thiim_gpu_init_benchmark) equals build_benchmark_problem
(coefficients.cpp:94-111) bitwise in all 40 arrays -- through the oracle's
restatement, itself pinned to the compiled reference in test_oracle.py -- for
the default and non-default schemes, z-slab contexts and the table layout, and
steps like the oracle from there."""
import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _host(d, **sp):
    return P.ProblemState(d, O.c_benchmark_problem((d.nx, d.ny, d.nz), **sp))


@pytest.mark.parametrize("shape", [(20, 17, 12), (33, 8, 41)])
@pytest.mark.parametrize("sp", [{}, {"omega": 1.1, "tau": 0.7, "delta": 0.5},
                                {"omega": 3.14159265358979323846, "tau": 1.0, "delta": 2.0}])
def test_init_benchmark_equals_reference_setup(shape, sp):
    d = P.GridDims(*shape)
    want = _host(d, **sp)
    with P.GpuEngine(d) as e:
        e.init_benchmark(**sp)
        got = e.download_state()
    for k in range(40):
        assert np.array_equal(got.arrays[k].view(np.uint64), want.arrays[k].view(np.uint64)), k


def test_init_benchmark_slabs_and_stepping():
    d = P.GridDims(24, 20, 28)
    want = _host(d)
    O.c_step((24, 20, 28), want.arrays, 7, threads=8)
    for n in (1, 3):
        with P.GpuEngine(d, P.GpuOptions(n_gpus=n, same_device=1)) as e:
            e.init_benchmark()
            e.step(7)
            got = P.allocate_state(d)
            e.download_fields(got)
        assert P.compare_states(got, want).bitwise_equal, n


@pytest.mark.parametrize("engine", [P.ENGINE_FUSED, P.ENGINE_TBLOCK])
def test_init_benchmark_table_layout(engine):
    d = P.GridDims(30, 22, 36)
    want = _host(d)
    with P.GpuEngine(d, P.GpuOptions(engine=engine, coeff_layout=P.COEFF_TABLE,
                                     n_materials=3)) as e:
        e.init_benchmark()
        mid, tab = e.download_table(3)
        full = P.expand_coefficients(d, mid, tab)
        for k in range(12, 40):
            assert np.array_equal(full.interior(k).view(np.uint64), want.interior(k).view(np.uint64))
        e.step(6)
        got = P.allocate_state(d)
        e.download_fields(got)
    O.c_step((30, 22, 36), want.arrays, 6, threads=8)
    assert P.compare_states(got, want).bitwise_equal


def test_init_benchmark_validation():
    with P.GpuEngine(P.GridDims(8, 8, 8)) as e:
        with pytest.raises(P.ConfigError):
            e.init_benchmark(tau=0.0)
        with pytest.raises(P.ConfigError):
            e.init_benchmark(omega=4.0, tau=1.0)
    with P.GpuEngine(P.GridDims(8, 8, 8), P.GpuOptions(coeff_layout=P.COEFF_TABLE,
                                                       n_materials=2)) as e:
        with pytest.raises(P.ConfigError):
            e.init_benchmark()
