"""CPU tests: pin the C oracle (oracle/thiim_oracle.c) before trusting it.

1. golden fixtures produced by the UNMODIFIED reference (tests/golden/);
2. bitwise agreement with the reference library itself (oracle/_ref);
3. the reference's own known-answer tests (tests/test_kernels.cpp,
   test_grid.cpp, test_coefficients.cpp) re-expressed on the oracle.
"""
import glob
import hashlib
import json
import os
import random

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def bits(a):
    return a.view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


# ---------------------------------------------------------------- golden fixtures
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))))
def test_oracle_matches_golden(path):
    z = np.load(path)
    meta = json.loads(str(z["meta"]))
    dims = tuple(meta["dims"])
    if meta["kind"] == "random":
        arrays = O.c_generate(dims, meta["seed"])
    elif meta["kind"] == "layered":
        arrays = O.c_generate(dims, meta["seed"], layered=True)
    else:
        arrays = O.c_benchmark_problem(dims)
    got = [hashlib.sha256(a.tobytes()).hexdigest() for a in arrays]
    assert got == meta["input_sha256"], "inputs differ from the fixture's"
    O.c_step(dims, arrays, meta["steps"])
    for k in range(12):
        assert same(arrays[k], z["fields"][k]), (meta["name"], k)


def test_golden_index_complete():
    idx = json.load(open(os.path.join(GOLDEN, "index.json")))
    assert {m["name"] for m in idx} == {os.path.basename(p)[:-4]
                                        for p in glob.glob(os.path.join(GOLDEN, "*.npz"))}


# ---------------------------------------------------------------- vs the reference library
@need_ref
@pytest.mark.parametrize("dims,steps,threads", [((4, 4, 4), 2, 1), ((9, 7, 6), 5, 1),
                                                ((12, 16, 20), 6, 3), ((17, 5, 11), 3, 4)])
def test_oracle_matches_reference_run_naive(dims, steps, threads):
    a = O.c_generate(dims, 17)
    b = [x.copy() for x in a]
    O.c_step(dims, a, steps, threads=threads)
    O.ref_run_naive(dims, b, steps, threads)
    r = O.ref_compare(dims, a, b)
    assert r["bitwise_equal"], r


@need_ref
def test_oracle_matches_reference_layered():
    dims = (10, 8, 24)
    a = O.c_generate(dims, 2, layered=True)
    b = [x.copy() for x in a]
    O.c_step(dims, a, 3)
    O.ref_run_naive(dims, b, 3, 1)
    assert O.ref_compare(dims, a, b)["bitwise_equal"]


@need_ref
def test_benchmark_problem_builder_matches_reference():
    """build_benchmark_problem (coefficients.cpp:94-111) restated in C."""
    for dims in [(8, 8, 8), (5, 9, 13)]:
        a, b = O.c_benchmark_problem(dims), O.ref_benchmark_problem(dims)
        assert all(same(x, y) for x, y in zip(a, b))


@need_ref
def test_derive_coefficients_matches_reference():
    """derive_coefficients closed forms (coefficients.cpp:25-55), bitwise, over
    random draws in the spirit of test_coefficients.cpp:52-94."""
    rng = random.Random(12345)
    for _ in range(300):
        m = (rng.uniform(-3, 3), rng.uniform(-1, 1), rng.uniform(0.1, 2), rng.uniform(0, 1.5),
             rng.uniform(0, 1.5))
        tau = rng.uniform(0.1, 2.0)
        omega, delta = rng.uniform(0.1, 2.0) / tau, rng.uniform(0.1, 2.0)
        for fam in (0, 1):
            for back in (0, 1):
                x = O.c_derive(m, omega, tau, delta, fam, back)
                y = O.ref_derive(m, omega, tau, delta, fam, back)
                assert same(np.array(x), np.array(y))


@need_ref
def test_spatial_and_mwd_engines_agree_with_oracle():
    """The reference's own blocked engines (CPU baselines) are bitwise equal to
    naive (test_reference_engines.cpp:44-55, test_mwd.cpp:14-26), hence to the oracle."""
    dims = (16, 16, 16)
    a = O.c_generate(dims, 4)
    b = [x.copy() for x in a]
    c = [x.copy() for x in a]
    O.c_step(dims, a, 4)
    O.ref_run_spatial(dims, b, 4, 4, 0, 2)
    _, ex = O.ref_run_mwd(dims, c, 4, 8, 1, 1, 1, 1, 1)
    assert ex == 4
    assert O.ref_compare(dims, a, b)["bitwise_equal"]
    assert O.ref_compare(dims, a, c)["bitwise_equal"]


# ---------------------------------------------------------------- reference KATs on the oracle
def test_grid_layout_kats():
    """test_grid.cpp:9-15 and :26-31."""
    d = P.GridDims(4, 4, 4)
    assert d.px() == 6
    assert d.linear_index(0, 0, 0) == 43
    assert d.linear_index(3, 0, 0) == 46
    assert d.linear_index(3, 3, 3) == 172
    assert P.GridDims(8, 8, 8).padded_cells() * 40 * 16 == 40 * 16 * 10 * 10 * 10
    assert O.c_lib().orc_linear_index(4, 4, 3, 3, 3) == 172


def test_single_cell_kat():
    """test_kernels.cpp:27-43: Hyz, t=0.5, F=2, c=1, shifted sum 0.25, src=0.1 -> 1.35."""
    dims = (4, 4, 4)
    d = P.GridDims(*dims)
    a = O.new_arrays(dims)
    c = int(P.Component.Hyz)
    i, j = d.linear_index(1, 1, 1), d.linear_index(1, 1, 2)
    a[c][i] = 2.0
    a[12 + c][i] = 0.5
    a[24 + c][i] = 1.0
    a[36 + P.source_index(c)][i] = 0.1
    a[int(P.Component.Exy)][j] = 0.25
    O.c_update_region(dims, a, c, 1, 2, 1, 2, 1, 2)
    assert abs(a[c][i].real - 1.35) <= 1e-15 * 1.35 and a[c][i].imag == 0.0


def test_identity_and_zero_kats():
    """test_kernels.cpp:45-61 (identity) and :131-153 (zero fixed point, ghosts)."""
    dims = (8, 8, 8)
    s = P.allocate_state(P.GridDims(*dims))
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")
    for ci in range(12):
        s.interior(12 + ci)[...] = 1.0
        s.interior(ci)[...] = (0.1 * x - 0.2 * y) + 1j * (0.3 * z + 0.01 * x)
    before = P.clone_state(s)
    O.c_step(dims, s.arrays, 1)
    assert P.compare_states(s, before).bitwise_equal
    b = O.c_benchmark_problem((8, 12, 8))
    O.c_step((8, 12, 8), b, 3)
    st = P.ProblemState(P.GridDims(8, 12, 8), b)
    for ci in range(12):
        v = st.view3d(ci).copy()
        v[1:-1, 1:-1, 1:-1] = 0
        assert not np.any(v)


def test_power_of_two_linearity_kat():
    """test_kernels.cpp:155-177 / acceptance criterion 9."""
    a = O.c_benchmark_problem((8, 8, 8))
    b = [x.copy() for x in a]
    for k in range(36, 40):
        b[k] *= 2.0
    O.c_step((8, 8, 8), a, 8)
    O.c_step((8, 8, 8), b, 8)
    for k in range(12):
        assert same(2.0 * a[k], b[k])


# ---------------------------------------------------------------- synthetic inputs
@pytest.mark.parametrize("seed", [1, 2, 0xDEADBEEF])
def test_product_generator_matches_oracle_generator(seed):
    dims = P.GridDims(11, 7, 9)
    s = P.generate_problem(dims, P.GEN_RANDOM, seed)
    o = O.c_generate((11, 7, 9), seed)
    assert all(same(x, y) for x, y in zip(s.arrays, o))
    sl = P.generate_problem(dims, P.GEN_LAYERED, seed)
    ol = O.c_generate((11, 7, 9), seed, layered=True)
    assert all(same(x, y) for x, y in zip(sl.arrays, ol))


def test_generator_distributions():
    d = P.GridDims(20, 20, 20)
    s = P.generate_problem(d, P.GEN_RANDOM, 1)
    for k in range(12):
        v = s.interior(k)
        assert v.real.min() >= -1 and v.real.max() < 1 and v.imag.min() >= -1
        assert abs(v.real.mean()) < 0.05
    for k in range(12, 40):
        assert np.abs(s.interior(k)).max() <= 0.45
    for k in range(40):
        g = s.view3d(k).copy()
        g[1:-1, 1:-1, 1:-1] = 0
        assert not np.any(g), "ghosts must be zero"
    lay = P.generate_problem(P.GridDims(8, 8, 60), P.GEN_LAYERED, 3)
    col = lay.interior(12)[:, 2, 3]
    assert 2 <= len(np.unique(col)) <= 6  # piecewise constant along z


@need_ref
@pytest.mark.parametrize("dims,layered,threads", [((9, 7, 6), False, 1), ((13, 5, 11), False, 4),
                                                  ((16, 12, 30), True, 3), ((6, 9, 14), True, 1)])
def test_reference_shim_generator_matches_oracle(dims, layered, threads):
    """The generator restated inside oracle/_ref (used by bench.py's CPU arms and
    the full-size parity tests) is bitwise the oracle's, and a held reference
    state steps exactly like the reference's run_naive on copied arrays."""
    a = O.c_generate(dims, 11, layered=layered)
    with O.RefState(dims) as r:
        r.generate(11, layered, threads)
        for k in range(40):
            assert same(r.get(k), a[k]), k
        O.ref_run_naive(dims, a, 3, 1)
        r.run_naive(3, threads)
        d = r.compare_fields(a[:12])
        assert d["differing_values"] == 0 and d["first_component"] == -1
        i = dims[0] + 2 + 1 + (dims[0] + 2) * (dims[1] + 2) * 2  # interior (0, 0, 1)
        a[5][i] += 1.0
        d = r.compare_fields(a[:12])
        assert (d["differing_values"], d["first_component"], d["x"], d["y"], d["z"]) == \
            (1, 5, 0, 0, 1)
