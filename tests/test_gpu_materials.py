"""GPU: per-cell coefficient setup from a material map on the device
(thiim_gpu_init_materials) -- the reference's
build_problem_from_voxels (coefficients.cpp:112-141) with derive_coefficients
(:25-55) evaluated per cell on the GPU.  Its complex division restates libgcc's
__divdc3; both are checked bitwise: the division against the host's own
(C99 complex, the code std::complex<double> calls), the whole setup against the
compiled reference reading the same voxel file."""
import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nan = np.isnan(a) & np.isnan(b)
    return np.all(nan | (a.view(np.uint64) == b.view(np.uint64)))


def test_device_complex_division_is_libgcc():
    rng = np.random.default_rng(5)
    n = 1 << 18
    mant = rng.uniform(-1, 1, (n, 4))
    expo = rng.integers(-320, 310, (n, 4)).astype(np.float64)
    with np.errstate(over="ignore"):
        ops = mant * np.power(10.0, expo)  # includes infinities by design
    # structured edge cases: zero / signed-zero / subnormal / huge / inf / nan parts
    vals = [0.0, -0.0, 1.0, -2.5, 5e-324, 1e-310, 2.2e-308, 1e-300, 1e300, 1.7e308,
            np.inf, -np.inf, np.nan, 3.0e-16, 0.75]
    grid = np.array(np.meshgrid(vals, vals, vals, vals)).reshape(4, -1).T
    typical = rng.uniform(-3, 3, (n, 4))
    for chunk in (ops, grid, typical):
        with np.errstate(all="ignore"):
            want = O.c_cdiv(chunk)
            got = P.selftest_cdiv(chunk)
        assert _same(got, want), np.argwhere(~((np.isnan(got) & np.isnan(want)) |
                                                (got.view(np.uint64) == want.view(np.uint64))))[:5]


def _materials(d, seed, back=True):
    rng = np.random.default_rng(seed)
    m = np.empty((d.nz, d.ny, d.nx, 5))
    m[..., 0] = rng.uniform(-2.0 if back else 0.5, 4.0, m.shape[:3])  # eps re (< 0: back mode)
    m[..., 1] = rng.uniform(0.0, 1.0, m.shape[:3])                    # eps im
    m[..., 2] = rng.uniform(0.5, 2.0, m.shape[:3])                    # mu
    m[..., 3] = rng.uniform(0.0, 1.0, m.shape[:3])                    # sigma
    m[..., 4] = rng.uniform(0.0, 1.0, m.shape[:3])                    # sigma*
    return m


@needs_ref
@pytest.mark.parametrize("shape,sp", [((13, 9, 11), {}), ((24, 17, 20), {"omega": 1.3, "tau": 0.8,
                                                                           "delta": 0.5})])
def test_init_materials_equals_reference_voxels(tmp_path, shape, sp):
    d = P.GridDims(*shape)
    m = _materials(d, 7)
    path = tmp_path / "voxels.bin"
    m.astype("<f8").tofile(path)
    want = O.ref_problem_from_voxels(shape, path, **sp)
    with P.GpuEngine(d) as e:
        e.init_materials(m, **sp)
        got = e.download_state()
    for k in range(40):
        assert np.array_equal(got.arrays[k].view(np.uint64), want[k].view(np.uint64)), k


@needs_ref
@pytest.mark.parametrize("n_gpus", [1, 3])
def test_init_materials_then_steps(tmp_path, n_gpus):
    d = P.GridDims(30, 22, 26)
    m = _materials(d, 9)
    path = tmp_path / "voxels.bin"
    m.astype("<f8").tofile(path)
    want = P.ProblemState(d, O.ref_problem_from_voxels((30, 22, 26), path))
    O.c_step((30, 22, 26), want.arrays, 5, threads=8)
    with P.GpuEngine(d, P.GpuOptions(n_gpus=n_gpus, same_device=1)) as e:
        e.init_materials(m)
        e.step(5)
        got = P.allocate_state(d)
        e.download_fields(got)
    assert P.compare_states(got, want).bitwise_equal


@needs_ref
def test_init_materials_errors_match_reference(tmp_path):
    d = P.GridDims(6, 5, 4)
    m = _materials(d, 3, back=False)
    m[..., 2] = 1.0
    m[2, 3, 1, 4] = -1.0  # sigma*/mu = -1/tau with omega = 0: vanishing H denominator
    m[3, 0, 4, 4] = -1.0
    path = tmp_path / "v.bin"
    m.astype("<f8").tofile(path)
    with pytest.raises(RuntimeError) as ref_err:
        O.ref_problem_from_voxels((6, 5, 4), path, omega=0.0)
    with P.GpuEngine(d) as e:
        with pytest.raises(P.SetupError) as err:
            e.init_materials(m, omega=0.0)
    assert str(ref_err.value).endswith(str(err.value))  # the reference's text, same cell
    assert "(H, forward)" in str(err.value) and "at cell (1,3,2) component Hxy" in str(err.value)
    m[..., 4] = 0.0
    m[1, 1, 1, 2] = 0.0  # mu = 0
    with P.GpuEngine(d) as e:
        with pytest.raises(P.SetupError, match="mu must be nonzero"):
            e.init_materials(m)
        with pytest.raises(P.ConfigError):
            e.init_materials(m[:1])
