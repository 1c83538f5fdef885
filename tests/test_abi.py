"""CPU tests of the C-ABI boundary (include/thiim_gpu.h): the library loads,
exports every declared entry point, and validates arguments like the
reference (ConfigError / SetupError) before touching a device."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1510_05218_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "thiim_gpu.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(thiim_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ["thiim_gpu_create", "thiim_gpu_upload", "thiim_gpu_init_generated",
              "thiim_gpu_step", "thiim_gpu_download_fields", "thiim_gpu_destroy",
              "thiim_gpu_last_error"]:
        assert f in fns
    assert set(fns) == set(P.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    L = P.lib()
    for f in declared_functions():
        assert hasattr(L, f), f
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True,
                         text=True).stdout
    for f in declared_functions():
        assert re.search(r"\bT %s\b" % f, out), f


def test_library_is_sm100a_cubin():
    out = subprocess.run(["cuobjdump", "-lelf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass, "TMA tensor loads expected in the fused sweep"
    # the TBLOCK level-1 -> level-2 hand-off lives in TMEM: tcgen05.st / .ld
    # (SASS STTM / LDTM) in every k_tblock_tm instance
    tm = [blk for blk in sass.split("Function :")[1:] if blk.split()[0].startswith("_ZN9thiim_gpu11k_tblock_tm")]
    assert tm, "no k_tblock_tm instances"
    for blk in tm:
        assert "UTMALDG" in blk and "LDTM" in blk and "STTM" in blk, blk.split()[0]
    # -fmad=false: no contracted FP64 multiply-add in any stencil / setup kernel.  Only
    # the kernels that divide (IEEE division is an FMA-refined sequence, still correctly
    # rounded -- test_gpu_materials.py pins them bitwise against libgcc) contain DFMA.
    fn, with_fma = None, set()
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
        elif "DFMA" in line:
            with_fma.add(fn)
    divides = ("k_init_materials", "k_selftest_cdiv")
    assert with_fma and all(any(d in f for d in divides) for f in with_fma), sorted(with_fma)


def test_abi_version_and_models():
    assert P.lib().thiim_gpu_abi_version() == 2
    # thiim_gpu_opts: 7 ints of geometry/engine, schedule, band, same_device,
    # 4 reserved, coeff_layout, n_materials
    assert ctypes.sizeof(P._Opts) == 16 * 4
    assert P.balance_model(P.ENGINE_SPLIT) == 1024.0
    assert P.balance_model(P.ENGINE_FUSED) == 832.0
    assert P.balance_model(P.ENGINE_TBLOCK, 2) == 416.0


def test_argument_validation_without_device():
    L = P.lib()
    ctx = ctypes.c_void_p()
    bad = P._Dims(3, 8, 8, 1)
    assert L.thiim_gpu_create(ctypes.byref(bad), None, ctypes.byref(ctx)) == 3  # SetupError
    ghost2 = P._Dims(8, 8, 8, 2)
    assert L.thiim_gpu_create(ctypes.byref(ghost2), None, ctypes.byref(ctx)) == 3
    assert b"invalid grid dims" in L.thiim_gpu_last_error()
    good = P._Dims(8, 8, 8, 1)
    o = P.GpuOptions(n_gpus=9)._c()
    assert L.thiim_gpu_create(ctypes.byref(good), ctypes.byref(o), ctypes.byref(ctx)) == 2
    assert L.thiim_gpu_step(None, 1, None) == 2
    with pytest.raises(P.SetupError):
        P.GpuEngine(P.GridDims(8, 8, 3))
    with pytest.raises(P.ConfigError):
        P.run_gpu(P.allocate_state(P.GridDims(4, 4, 4)), -1)


def test_host_generator_rejects_bad_input():
    L = P.lib()
    arrs = (ctypes.c_void_p * 40)()
    d = P._Dims(8, 8, 8, 1)
    assert L.thiim_generate_host(ctypes.byref(d), 7, 1, arrs) == 2


def test_compare_states_semantics():
    """compare_states (verifier.cpp:13-44): interior only, first mismatch in
    component-major, z, y, x order, bitwise (so -0.0 != +0.0)."""
    d = P.GridDims(5, 4, 6)
    a = P.generate_problem(d, P.GEN_RANDOM, 1)
    b = P.clone_state(a)
    assert P.compare_states(a, b).bitwise_equal
    b.view3d(3)[0, 0, 0] = 99.0  # ghost: ignored
    assert P.compare_states(a, b).bitwise_equal
    b.interior(4)[2, 1, 3] += 1e-12
    b.interior(7)[0, 0, 0] += 1.0
    diff = P.compare_states(a, b)
    assert not diff.bitwise_equal and diff.differing_values == 2
    assert (diff.first_component, diff.x, diff.y, diff.z) == (4, 3, 1, 2)
    c = P.allocate_state(d)
    e = P.allocate_state(d)
    e.interior(0)[0, 0, 0] = -0.0
    assert not P.compare_states(c, e).bitwise_equal


def test_compress_expand_roundtrip():
    d = P.GridDims(10, 9, 30)
    s = P.generate_problem(d, P.GEN_LAYERED, 4)
    mid, tab = P.compress_coefficients(s)
    assert len(tab) == 7  # 6 layers + the all-zero ghost row
    full = P.expand_coefficients(d, mid, tab)
    for k in range(12, 40):
        assert np.array_equal(full.arrays[k].view(np.uint64), s.arrays[k].view(np.uint64))
    with pytest.raises(P.ConfigError):
        P.compress_coefficients(P.generate_problem(d, P.GEN_RANDOM, 1))


def test_tuner_model_ranks_candidates_without_a_device():
    """thiim_gpu_enumerate_candidates: the GPU re-parameterisation of the
    reference's Eq. 11/12 models (autotuner.cpp:15-50) runs on the host."""
    c = P.enumerate_candidates(P.GridDims(512, 512, 512))
    assert len(c) > 20
    assert {x["time_block"] for x in c} == {2, 3}
    m = [x["model_mlups"] for x in c]
    assert all(a >= b * 0.995 for a, b in zip(m, m[1:]))  # best first (0.5% tie window)
    for x in c:
        assert x["balance_model"] == pytest.approx(832.0 / x["time_block"])
        # overlap re-fetch and chunk starts only add bytes
        assert x["model_bytes_per_lup"] >= x["balance_model"]
        assert 0 < x["quantization"] <= 1 and x["l2_set_bytes"] > 0
    # one launch (y-neighbours desynchronised) models more DRAM bytes than rounds
    one = [x for x in c if x["schedule"] == 1 and x["time_block"] == 2 and x["tile_y"] == 15]
    rnd = [x for x in c if x["schedule"] == 0 and x["band"] == 0 and x["time_block"] == 2
           and x["tile_y"] == 15 and x["z_chunk"] == one[0]["z_chunk"]]
    assert one and rnd and one[0]["model_bytes_per_lup"] > rnd[0]["model_bytes_per_lup"]
    # depth 3 is SM-bound in the model (calibrated): it must not rank first
    assert c[0]["time_block"] == 2
    # slabs and the table layout have no depth 3
    c2 = P.enumerate_candidates(P.GridDims(256, 256, 256), P.GpuOptions(n_gpus=2))
    assert {x["time_block"] for x in c2} == {2}
