"""BASELINE workloads at their full sizes (one B200).

* configs[1] (256^3 x 100 iterations, the bench workload) against the
  reference's own run_naive (oracle/_ref, compiled unmodified) on all host
  threads: bitwise.
* configs[2] (512^3) and configs[4] (1024^2 x 128) on their full grids against
  the reference's run_naive for a bounded number of iterations (5: two TBLOCK
  passes plus the odd remainder step), the problem generated on the device
  (k_generate at full size) and, for the reference, inside oracle/_ref (its
  shim's restated generator) -- 87 GB of reference state + 26 GB of downloaded
  fields in host RAM, compared there with compare_states' field loop.
* configs[2] over all 200 iterations (and configs[4] over all 100) through a
  size-independent property: two schedules that share nothing but the
  arithmetic -- TBLOCK (two steps per pass, TMEM hand-off) and fused (one step
  per pass) -- agree bitwise.
* configs[3] in the reference layout (174 GB: TBLOCK in place, sub-ranges with
  spare planes) against the table layout (TBLOCK-table, material ids) over all
  200 iterations: bitwise (the two contexts run one after the other).
"""
import os

import numpy as np
import pytest

import paper_1510_05218_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def threads():
    return os.cpu_count() or 1


need_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def host_ram_gb():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1e6
    return 0.0


def _full_grid_vs_reference(grid, steps):
    d = P.GridDims(*grid)
    need = 52 * d.padded_cells() * 16 / 1e9 + 8
    if host_ram_gb() < need:
        pytest.skip("needs %.0f GB of host RAM" % need)
    n = d.padded_cells()
    got = [np.empty(n, np.complex128) for _ in range(12)]
    with P.GpuEngine(d, P.GpuOptions()) as e:  # AUTO: TBLOCK (+ fused for the odd step)
        e.generate(P.GEN_RANDOM, 1)
        st = e.step(steps)
        assert st.engine == P.ENGINE_TBLOCK, st.engine
        e.download_fields(got)
    with O.RefState(grid) as r:
        r.generate(1, False, threads())
        r.run_naive(steps, threads())
        diff = r.compare_fields(got)
    assert diff["differing_values"] == 0, diff
    # the fields moved (not a trivial agreement of untouched arrays)
    assert np.isfinite(got[0][n // 2: n // 2 + 4096].view(np.float64)).all()


@need_ref
def test_config2_full_grid_vs_reference():
    _full_grid_vs_reference((512, 512, 512), 5)


@need_ref
def test_config4_full_grid_vs_reference():
    _full_grid_vs_reference((1024, 1024, 128), 5)


full_length = pytest.mark.skipif(
    os.environ.get("THIIM_FULL_LENGTH") != "1",
    reason="THIIM_FULL_LENGTH=1 runs the reference for the whole workload (minutes of CPU time)")


@need_ref
@full_length
def test_config2_full_length_vs_reference():
    """configs[2] over all 200 iterations against the reference's run_naive
    (~4 min on 16 host threads; the round's run is kept under profiles/)."""
    _full_grid_vs_reference((512, 512, 512), 200)


@need_ref
@full_length
def test_config4_full_length_vs_reference():
    """configs[4]'s per-GPU slab over all 100 iterations against run_naive."""
    _full_grid_vs_reference((1024, 1024, 128), 100)


def test_config1_full_workload_vs_reference():
    d = P.GridDims(256, 256, 256)
    s = P.generate_problem(d, P.GEN_RANDOM, seed=1)  # bench.py's problem
    want = P.clone_state(s)
    if O.ref_available():
        O.ref_run_naive((256, 256, 256), want.arrays, 100, threads())
    else:  # GPU box without the prebuilt reference: the pinned C restatement
        O.c_step((256, 256, 256), want.arrays, 100, threads=threads())
    r = P.run_gpu(s, 100)  # default engine (TBLOCK), the bench path
    assert r.engine == "gpu-tblock"
    diff = P.compare_states(s, want)
    assert diff.bitwise_equal, diff


def test_config2_full_workload_tblock_vs_fused():
    d = P.GridDims(512, 512, 512)
    n = d.padded_cells()
    ref = [np.empty(n, np.complex128) for _ in range(12)]  # 26 GB host
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_FUSED)) as a:
        a.generate(P.GEN_RANDOM, 1)
        a.step(200)
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK)) as b:
        b.generate(P.GEN_RANDOM, 1)
        st = b.step(200)
        # 100 passes, each one launch per round of <= one CTA per SM
        assert st.engine == P.ENGINE_TBLOCK and st.kernel_launches % 100 == 0
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff
    # not a trivial agreement: the fields moved and stayed finite
    assert all(np.isfinite(f[n // 2: n // 2 + 4096].view(np.float64)).all() for f in ref)


def test_config4_full_workload_tblock_vs_fused():
    """configs[4] (1024^2 x 128, 100 iterations -- the per-GPU slab of the
    weak-scaling runs) over the whole workload: TBLOCK (24 rounds per pass) and
    the fused one-step sweep agree bitwise."""
    d = P.GridDims(1024, 1024, 128)
    n = d.padded_cells()
    ref = [np.empty(n, np.complex128) for _ in range(12)]
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_FUSED)) as a:
        a.generate(P.GEN_RANDOM, 1)
        a.step(100)
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK)) as b:
        b.generate(P.GEN_RANDOM, 1)
        st = b.step(100)
        assert st.engine == P.ENGINE_TBLOCK
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff
    assert all(np.isfinite(f[n // 2: n // 2 + 4096].view(np.float64)).all() for f in ref)


def test_config3_full_workload_inplace_vs_table():
    """configs[3] (layered 1024^2 x 256, 200 iterations): the reference layout
    (174 GB; AUTO picks TBLOCK in place: it fits once, not twice) against the
    material-id table layout (TBLOCK-table), bitwise."""
    d = P.GridDims(1024, 1024, 256)
    n = d.padded_cells()
    if host_ram_gb() < 12 * n * 16 / 1e9 + 8:
        pytest.skip("needs 52 GB of host RAM")
    ref = [np.empty(n, np.complex128) for _ in range(12)]
    with P.GpuEngine(d, P.GpuOptions()) as a:
        a.generate(P.GEN_LAYERED, 1)
        st = a.step(200)
        assert st.engine == P.ENGINE_TBLOCK_INPLACE, st.engine
        a.download_fields(ref)
    with P.GpuEngine(d, P.GpuOptions(engine=P.ENGINE_TBLOCK, coeff_layout=P.COEFF_TABLE,
                                     n_materials=6)) as b:
        b.generate(P.GEN_LAYERED, 1)
        st = b.step(200)
        assert st.engine == P.ENGINE_TBLOCK
        diff = b.compare_fields(ref)
    assert diff.bitwise_equal, diff
    assert all(np.isfinite(f[n // 2: n // 2 + 4096].view(np.float64)).all() for f in ref)


def test_config2_stream_inplace_vs_device_generated():
    """The e2e stream at configs[2] (bench.py's e2e leg): run_gpu_batch under
    AUTO holds two TBLOCK-in-place contexts (ping-pong state fits once) and
    takes its inputs from host memory (the host generator, 87 GB, pinned);
    its results equal a device-generated (k_generate at full size) ping-pong
    TBLOCK run bitwise -- which also pins the device generator to the host one
    on the full grid."""
    d = P.GridDims(512, 512, 512)
    n = d.padded_cells()
    steps = 6  # three passes per problem: ends on an odd pass (array moved back)
    if host_ram_gb() < 66 * n * 16 / 1e9 + 8:
        pytest.skip("needs %.0f GB of host RAM" % (66 * n * 16 / 1e9 + 8))
    ref = [np.empty(n, np.complex128) for _ in range(12)]
    with P.GpuEngine(d, P.GpuOptions()) as e:
        e.generate(P.GEN_RANDOM, 1)
        st = e.step(steps)
        assert st.engine == P.ENGINE_TBLOCK
        e.download_fields(ref)
    P.release_cached(0)
    host = P.generate_problem(d, P.GEN_RANDOM, 1)
    out = [np.zeros(n, np.complex128) for _ in range(12)]
    L = P.lib()
    bufs = host.arrays + out
    for a in bufs:
        assert L.thiim_gpu_pin_host(a.ctypes.data, a.nbytes) == 0
    try:
        rep = P.run_gpu_batch([host, host], steps, outputs=[out, out])
    finally:
        for a in bufs:
            L.thiim_gpu_unpin_host(a.ctypes.data)
    assert rep.engine == "gpu-tblock-inplace" and rep.depth == 2, rep
    for k in range(12):
        assert np.array_equal(out[k].view(np.uint64), ref[k].view(np.uint64)), k
    assert all(np.isfinite(f[n // 2: n // 2 + 4096].view(np.float64)).all() for f in ref)
