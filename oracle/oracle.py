"""TEST INFRASTRUCTURE ONLY -- ctypes bindings of the parity oracles.

* ``C``   : oracle/_lib/libthiim_oracle.so, the plain-C restatement
            (thiim_oracle.c) of the reference sweep.
* ``REF`` : oracle/_ref/libthiim_ref.so, the UNMODIFIED reference library
            compiled from /root/reference/proj/src (oracle/Makefile) behind
            ref_shim.cpp.  Built in the dev container; travels prebuilt.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the CPU baseline -- never as the product path.

All functions take ``arrays``: a list of 40 C-contiguous complex128 numpy
vectors in ProblemState order ([0..11] fields, [12..23] t, [24..35] c,
[36..39] src), reference padded layout.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
C_LIB = os.path.join(HERE, "_lib", "libthiim_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libthiim_ref.so")

_c = None
_ref = None


def build(quiet: bool = True) -> None:
    """make -C oracle: the C restatement always, the reference when present."""
    r = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + r.stdout + r.stderr)
    if not quiet:
        print(r.stdout)


def _ptrs(arrays):
    return (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def c_lib() -> ctypes.CDLL:
    global _c
    if _c is None:
        if not os.path.exists(C_LIB):
            build()
        L = ctypes.CDLL(C_LIB)
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_uniform.restype = ctypes.c_double
        L.orc_uniform.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.orc_compare_fields.restype = ctypes.c_uint64
        _c = L
    return _c


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> ctypes.CDLL:
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(
                "oracle/_ref/libthiim_ref.so missing (build with `make -C oracle` where "
                "/root/reference exists)")
        L = ctypes.CDLL(REF_LIB)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_code_balance_naive.restype = ctypes.c_double
        _ref = L
    return _ref


class _OrcState(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("a", ctypes.c_void_p * 40)]


def _st(dims, arrays) -> _OrcState:
    s = _OrcState()
    s.nx, s.ny, s.nz = dims
    for k in range(40):
        assert arrays[k].flags.c_contiguous and arrays[k].dtype == np.complex128
        s.a[k] = arrays[k].ctypes.data
    return s


def new_arrays(dims):
    nx, ny, nz = dims
    n = (nx + 2) * (ny + 2) * (nz + 2)
    return [np.zeros(n, dtype=np.complex128) for _ in range(40)]


# ---------------------------------------------------------------- C restatement
def c_step(dims, arrays, steps: int = 1, threads: int = 1) -> None:
    """steps x step_reference (kernels.cpp:105-113), in place."""
    s = _st(dims, arrays)
    if threads > 1:
        c_lib().orc_run_naive_threads(ctypes.byref(s), steps, threads)
    else:
        c_lib().orc_run_naive(ctypes.byref(s), steps)


def c_step_slab(dims, arrays, halo_lo: bool) -> None:
    """One step of a z-slab (local dims) whose plane below is a halo copy."""
    s = _st(dims, arrays)
    c_lib().orc_step_slab(ctypes.byref(s), 1 if halo_lo else 0)


def c_update_region(dims, arrays, comp, x0, x1, y0, y1, z0, z1) -> None:
    s = _st(dims, arrays)
    c_lib().orc_update_component_region(ctypes.byref(s), comp, x0, x1, y0, y1, z0, z1)


def c_generate(dims, seed: int, layered: bool = False):
    arrays = new_arrays(dims)
    s = _st(dims, arrays)
    if layered:
        c_lib().orc_generate_layered(ctypes.byref(s), ctypes.c_uint64(seed))
    else:
        c_lib().orc_generate_random(ctypes.byref(s), ctypes.c_uint64(seed))
    return arrays


class _Scheme(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in
                ("omega", "tau", "delta", "src_e_re", "src_e_im", "src_h_re", "src_h_im")]


class _Material(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("eps_re", "eps_im", "mu", "sigma", "sigma_star")]


def c_benchmark_problem(dims, omega=0.4, tau=1.0, delta=1.0):
    arrays = new_arrays(dims)
    s = _st(dims, arrays)
    sp = _Scheme(omega, tau, delta, 1.0, 0.0, 1.0, 0.0)
    if c_lib().orc_build_benchmark_problem(ctypes.byref(s), ctypes.byref(sp)) != 0:
        raise RuntimeError("setup error")
    return arrays


def c_fill_uniform(dims, arrays, material=(1.0, 0.0, 1.0, 0.0, 0.0), omega=0.4, tau=1.0,
                   delta=1.0) -> None:
    s = _st(dims, arrays)
    sp = _Scheme(omega, tau, delta, 1.0, 0.0, 1.0, 0.0)
    m = _Material(*material)
    if c_lib().orc_fill_coefficients_uniform(ctypes.byref(s), ctypes.byref(sp), ctypes.byref(m)):
        raise RuntimeError("setup error")


def c_derive(material, omega, tau, delta, family, back):
    out = (ctypes.c_double * 6)()
    sp = _Scheme(omega, tau, delta, 1.0, 0.0, 1.0, 0.0)
    m = _Material(*material)
    t = (ctypes.c_double * 2)()
    c = (ctypes.c_double * 2)()
    s = (ctypes.c_double * 2)()
    rc = c_lib().orc_derive_coefficients(ctypes.byref(m), ctypes.byref(sp), family, back, t, c, s)
    if rc:
        raise RuntimeError("vanishing denominator")
    out[:] = [t[0], t[1], c[0], c[1], s[0], s[1]]
    return list(out)


def c_compare(dims, a, b):
    fc, fx, fy, fz = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    mx = ctypes.c_double()
    sa, sb = _st(dims, a), _st(dims, b)
    n = c_lib().orc_compare_fields(ctypes.byref(sa), ctypes.byref(sb), ctypes.byref(fc),
                                   ctypes.byref(fx), ctypes.byref(fy), ctypes.byref(fz),
                                   ctypes.byref(mx))
    return int(n), mx.value


# ---------------------------------------------------------------- the reference itself
def _ref_check(rc):
    if rc != 0:
        raise RuntimeError("reference error %d: %s" % (rc, ref_lib().ref_last_error().decode()))


def ref_run_naive(dims, arrays, steps: int, threads: int = 1) -> float:
    """reference run_naive (reference_engines.cpp:34-67); fields updated in place.
    Returns the reference's own RunReport.seconds."""
    sec = ctypes.c_double()
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_run_naive(nx, ny, nz, _ptrs(arrays), steps, threads,
                                       ctypes.byref(sec)))
    return sec.value


def ref_run_spatial(dims, arrays, steps: int, block_y: int = 8, block_x: int = 0,
                    threads: int = 1) -> float:
    sec = ctypes.c_double()
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_run_spatial(nx, ny, nz, _ptrs(arrays), steps, block_y, block_x,
                                         threads, ctypes.byref(sec)))
    return sec.value


def ref_run_mwd(dims, arrays, steps, dw, bz, tgz, tgx, tgc, threads):
    sec = ctypes.c_double()
    ex = ctypes.c_int()
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_run_mwd(nx, ny, nz, _ptrs(arrays), steps, dw, bz, tgz, tgx, tgc,
                                     threads, ctypes.byref(sec), ctypes.byref(ex)))
    return sec.value, ex.value


def ref_measure_bandwidth(threads: int, cache_bytes: int = 45 << 20) -> float:
    """reference measure_bandwidth (bandwidth.cpp:12-44): host triad GB/s, best of
    five; cache_bytes defaults to the reference's profile (perf_models.hpp:10)."""
    gbs = ctypes.c_double()
    _ref_check(ref_lib().ref_measure_bandwidth(threads, ctypes.c_ulonglong(cache_bytes),
                                               ctypes.byref(gbs)))
    return gbs.value


def ref_benchmark_problem(dims, omega=0.4, tau=1.0, delta=1.0):
    arrays = new_arrays(dims)
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_build_benchmark_problem(nx, ny, nz, ctypes.c_double(omega),
                                                     ctypes.c_double(tau), ctypes.c_double(delta),
                                                     _ptrs(arrays)))
    return arrays


def ref_problem_from_voxels(dims, path, omega=0.4, tau=1.0, delta=1.0):
    """reference build_problem_from_voxels (coefficients.cpp:112-141) of a voxel file."""
    arrays = new_arrays(dims)
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_build_problem_from_voxels(
        nx, ny, nz, ctypes.c_double(omega), ctypes.c_double(tau), ctypes.c_double(delta),
        str(path).encode(), _ptrs(arrays)))
    return arrays


def c_cdiv(operands):
    """host C99 complex division (libgcc __divdc3) of (n, 4) operands -> (n, 2)."""
    import numpy as np
    a = np.ascontiguousarray(operands, dtype=np.float64).reshape(-1, 4)
    out = np.zeros((a.shape[0], 2), dtype=np.float64)
    c_lib().orc_cdiv_batch(a.shape[0], ctypes.c_void_p(a.ctypes.data), ctypes.c_void_p(out.ctypes.data))
    return out


def ref_derive(material, omega, tau, delta, family, back):
    out = (ctypes.c_double * 6)()
    d = [ctypes.c_double(v) for v in material]
    _ref_check(ref_lib().ref_derive_coefficients(*d, ctypes.c_double(omega), ctypes.c_double(tau),
                                                 ctypes.c_double(delta), family, back, out))
    return list(out)


def ref_update_region(dims, arrays, comp, x0, x1, y0, y1, z0, z1) -> None:
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_update_component_region(nx, ny, nz, _ptrs(arrays), comp, x0, x1, y0,
                                                     y1, z0, z1))


def ref_compare(dims, a, b):
    out = (ctypes.c_longlong * 6)()
    mx = ctypes.c_double()
    nx, ny, nz = dims
    _ref_check(ref_lib().ref_compare_states(nx, ny, nz, _ptrs(a), _ptrs(b), out, ctypes.byref(mx)))
    return {"bitwise_equal": bool(out[0]), "differing_values": int(out[1]),
            "first_component": int(out[2]), "x": int(out[3]), "y": int(out[4]), "z": int(out[5]),
            "max_abs_diff": mx.value}


class RefState:
    """A reference ProblemState held inside oracle/_ref (ref_shim.cpp): generated
    there (the seeded synthetic problem, bitwise c_generate's), stepped with the
    reference's engines in place, compared there -- no host copies of 87-174 GB
    states.  Only libthiim_ref.so is loaded."""

    def __init__(self, dims):
        L = ref_lib()
        L.ref_state_new.restype = ctypes.c_void_p
        L.ref_state_new.argtypes = [ctypes.c_int] * 3
        for f in ("ref_state_generate", "ref_state_run_naive", "ref_state_run_spatial",
                  "ref_state_run_mwd", "ref_state_get", "ref_state_set",
                  "ref_state_compare_fields"):
            getattr(L, f).restype = ctypes.c_int
        L.ref_state_free.argtypes = [ctypes.c_void_p]
        self.dims = tuple(dims)
        self.h = L.ref_state_new(*self.dims)
        if not self.h:
            raise RuntimeError("ref_state_new: " + L.ref_last_error().decode())

    def close(self):
        if self.h:
            ref_lib().ref_state_free(ctypes.c_void_p(self.h))
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def generate(self, seed: int, layered: bool = False, threads: int = 1):
        _ref_check(ref_lib().ref_state_generate(ctypes.c_void_p(self.h), ctypes.c_ulonglong(seed),
                                                int(layered), threads))

    def run_naive(self, steps: int, threads: int = 1) -> float:
        sec = ctypes.c_double()
        _ref_check(ref_lib().ref_state_run_naive(ctypes.c_void_p(self.h), steps, threads,
                                                 ctypes.byref(sec)))
        return sec.value

    def run_spatial(self, steps, block_y=8, block_x=0, threads=1) -> float:
        sec = ctypes.c_double()
        _ref_check(ref_lib().ref_state_run_spatial(ctypes.c_void_p(self.h), steps, block_y,
                                                   block_x, threads, ctypes.byref(sec)))
        return sec.value

    def run_mwd(self, steps, dw, bz, tgz, tgx, tgc, threads):
        sec = ctypes.c_double()
        ex = ctypes.c_int()
        _ref_check(ref_lib().ref_state_run_mwd(ctypes.c_void_p(self.h), steps, dw, bz, tgz, tgx,
                                               tgc, threads, ctypes.byref(sec), ctypes.byref(ex)))
        return sec.value, ex.value

    def get(self, a: int):
        import numpy as np
        nx, ny, nz = self.dims
        out = np.empty((nx + 2) * (ny + 2) * (nz + 2), dtype=np.complex128)
        _ref_check(ref_lib().ref_state_get(ctypes.c_void_p(self.h), a,
                                           ctypes.c_void_p(out.ctypes.data)))
        return out

    def set(self, a: int, arr):
        _ref_check(ref_lib().ref_state_set(ctypes.c_void_p(self.h), a,
                                           ctypes.c_void_p(arr.ctypes.data)))

    def compare_fields(self, fields):
        """compare_states' field loop vs 12 host arrays (padded layout)."""
        out = (ctypes.c_longlong * 5)()
        mx = ctypes.c_double()
        _ref_check(ref_lib().ref_state_compare_fields(ctypes.c_void_p(self.h), _ptrs(fields), out,
                                                      ctypes.byref(mx)))
        return {"differing_values": int(out[0]), "first_component": int(out[1]),
                "x": int(out[2]), "y": int(out[3]), "z": int(out[4]), "max_abs_diff": mx.value}
