"""paper_1510_05218_b200 -- B200-native THIIM split-field sweep engine.

Host-side mirror of the reference C++ driver API for the hot path
(/root/reference/proj/include/thiim, read-only upstream), bound over the
C-ABI of ``libthiim_gpu.so`` (include/thiim_gpu.h).  Names, argument meaning
and error behaviour follow the reference:

==========================  ===========================================  =======================================
here                        reference                                    file:line
==========================  ===========================================  =======================================
``GridDims``                ``thiim::GridDims``                          include/thiim/grid.hpp:12-48
``ProblemState``            ``thiim::ProblemState`` (40 arrays)          include/thiim/state.hpp:49-66
``allocate_state``          ``allocate_state``                           src/state.cpp:5-16
``clone_state``             ``clone_state``                              src/state.cpp:18-29
``Component``               ``thiim::Component``                         include/thiim/components.hpp:17-30
``COMPONENT_TABLE``         ``kComponentTable``                          include/thiim/components.hpp:54-67
``run_gpu``                 ``run_naive`` (the time loop it replaces)    src/reference_engines.cpp:34-67
``RunReport``               ``thiim::RunReport``                         include/thiim/report.hpp:37-52
``compare_states``          ``compare_states``                           src/verifier.cpp:13-44
``ConfigError`` ...         ``ConfigError`` / ``SetupError``             include/thiim/grid.hpp:50-60
==========================  ===========================================  =======================================

The compute path is the CUDA library only: there is no CPU fallback.  If the
library cannot be loaded, importing the engine raises.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import replace, dataclass, field
from typing import Tuple, List, Optional

import numpy as np

__all__ = [
    "ConfigError", "SetupError", "PlanError", "GpuError",
    "GridDims", "ProblemState", "allocate_state", "clone_state", "Component",
    "COMPONENT_TABLE", "GEN_RANDOM", "GEN_LAYERED", "ENGINE_AUTO", "ENGINE_SPLIT",
    "ENGINE_FUSED", "ENGINE_TBLOCK", "ENGINE_TBLOCK_INPLACE", "GpuOptions", "RunReport", "StateDiff", "GpuEngine",
    "run_gpu", "generate_problem", "compare_states", "balance_model", "lib",
    "compress_coefficients", "expand_coefficients", "coeff_compress", "COEFF_FULL", "COEFF_TABLE",
    "COEFF_AUTO",
    "run_gpu_batch", "BatchReport", "release_cached",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# THIIM_LIB: load an alternative build (A/B experiments, tools/build_variant.sh)
LIB_PATH = os.environ.get("THIIM_LIB") or os.path.join(HERE, "libthiim_gpu.so")


# ---------------------------------------------------------------- errors
class ConfigError(RuntimeError):
    """thiim::ConfigError (grid.hpp:50-52)."""


class SetupError(RuntimeError):
    """thiim::SetupError (grid.hpp:58-60)."""


class PlanError(RuntimeError):
    """thiim::PlanError (grid.hpp:54-56)."""


class GpuError(RuntimeError):
    """CUDA / communication / call-order failures of the GPU engine."""


# ---------------------------------------------------------------- layout
@dataclass(frozen=True)
class GridDims:
    """thiim::GridDims (grid.hpp:12-48): interior extents + 1-cell ghost."""

    nx: int
    ny: int
    nz: int
    ghost: int = 1

    def valid(self) -> bool:
        return self.nx >= 4 and self.ny >= 4 and self.nz >= 4 and self.ghost == 1

    def px(self) -> int:
        return self.nx + 2 * self.ghost

    def py(self) -> int:
        return self.ny + 2 * self.ghost

    def pz(self) -> int:
        return self.nz + 2 * self.ghost

    def padded_cells(self) -> int:
        return self.px() * self.py() * self.pz()

    def interior_cells(self) -> int:
        return self.nx * self.ny * self.nz

    def stride_y(self) -> int:
        return self.px()

    def stride_z(self) -> int:
        return self.px() * self.py()

    def linear_index(self, x: int, y: int, z: int) -> int:
        return (z + self.ghost) * self.stride_z() + (y + self.ghost) * self.stride_y() + x + self.ghost


class Component(enum.IntEnum):
    """thiim::Component (components.hpp:17-30)."""

    Exy = 0
    Exz = 1
    Eyx = 2
    Eyz = 3
    Ezx = 4
    Ezy = 5
    Hxy = 6
    Hxz = 7
    Hyx = 8
    Hyz = 9
    Hzx = 10
    Hzy = 11


# kComponentTable (components.hpp:54-67):
# id -> (family 'E'/'H', shift axis 0/1/2, shift sign, operand_a, operand_b, curl_sign, has_source)
C = Component
COMPONENT_TABLE = {
    C.Exy: ("E", 1, -1, C.Hzx, C.Hzy, +1, False),
    C.Exz: ("E", 2, -1, C.Hyx, C.Hyz, -1, True),
    C.Eyx: ("E", 0, -1, C.Hzx, C.Hzy, -1, False),
    C.Eyz: ("E", 2, -1, C.Hxy, C.Hxz, +1, True),
    C.Ezx: ("E", 0, -1, C.Hyx, C.Hyz, +1, False),
    C.Ezy: ("E", 1, -1, C.Hxy, C.Hxz, -1, False),
    C.Hxy: ("H", 1, +1, C.Ezx, C.Ezy, -1, False),
    C.Hxz: ("H", 2, +1, C.Eyx, C.Eyz, +1, True),
    C.Hyx: ("H", 0, +1, C.Ezx, C.Ezy, +1, False),
    C.Hyz: ("H", 2, +1, C.Exy, C.Exz, -1, True),
    C.Hzx: ("H", 0, +1, C.Eyx, C.Eyz, -1, False),
    C.Hzy: ("H", 1, +1, C.Exy, C.Exz, +1, False),
}
del C


def source_index(c: int) -> int:
    """source_index (components.hpp:89-97)."""
    return {1: 0, 3: 1, 7: 2, 9: 3}.get(int(c), -1)


class ProblemState:
    """thiim::ProblemState (state.hpp:49-66): 12 fields, 12 t, 12 c, 4 src.

    Every array is a C-contiguous complex128 numpy vector of padded_cells()
    elements (== interleaved {re, im} doubles, ComplexScalar).  ``arrays``
    lists them in C-ABI order [fields, t, c, src].
    """

    def __init__(self, dims: GridDims, arrays: Optional[List[np.ndarray]] = None):
        if not dims.valid():
            raise SetupError("invalid grid dims (need nx,ny,nz >= 4, ghost = 1)")
        self.dims = dims
        n = dims.padded_cells()
        if arrays is None:
            arrays = [np.zeros(n, dtype=np.complex128) for _ in range(40)]
        if len(arrays) != 40 or any(a.shape != (n,) or a.dtype != np.complex128 for a in arrays):
            raise ConfigError("ProblemState needs 40 complex128 arrays of padded_cells()")
        self.arrays = [np.ascontiguousarray(a) for a in arrays]

    @property
    def fields(self) -> List[np.ndarray]:
        return self.arrays[0:12]

    @property
    def coeff_t(self) -> List[np.ndarray]:
        return self.arrays[12:24]

    @property
    def coeff_c(self) -> List[np.ndarray]:
        return self.arrays[24:36]

    @property
    def coeff_src(self) -> List[np.ndarray]:
        return self.arrays[36:40]

    def field(self, c: int) -> np.ndarray:
        return self.arrays[int(c)]

    def t_of(self, c: int) -> np.ndarray:
        return self.arrays[12 + int(c)]

    def c_of(self, c: int) -> np.ndarray:
        return self.arrays[24 + int(c)]

    def view3d(self, a: int) -> np.ndarray:
        """(pz, py, px) view of array ``a`` (z slowest, x unit stride)."""
        d = self.dims
        return self.arrays[a].reshape(d.pz(), d.py(), d.px())

    def interior(self, a: int) -> np.ndarray:
        return self.view3d(a)[1:-1, 1:-1, 1:-1]

    def zero_fields(self) -> None:
        for f in self.fields:
            f[:] = 0


def allocate_state(dims: GridDims) -> ProblemState:
    """allocate_state (state.cpp:5-16): all 40 arrays zeroed."""
    return ProblemState(dims)


def clone_state(s: ProblemState) -> ProblemState:
    """clone_state (state.cpp:18-29): deep copy of all 40 arrays."""
    return ProblemState(s.dims, [a.copy() for a in s.arrays])


@dataclass
class StateDiff:
    """thiim::StateDiff (verifier.hpp:11-18) plus per-component relative L2."""

    max_abs_diff: float = 0.0
    bitwise_equal: bool = True
    differing_values: int = 0
    first_component: int = 0
    x: int = -1
    y: int = -1
    z: int = -1
    rel_l2: List[float] = field(default_factory=lambda: [0.0] * 12)

    @property
    def max_rel_l2(self) -> float:
        return max(self.rel_l2)


def compare_states(a: ProblemState, b: ProblemState) -> StateDiff:
    """compare_states (verifier.cpp:13-44): exact interior scan of the 12 fields.

    ``rel_l2[k] = ||a_k - b_k|| / ||b_k||`` over the interior is the
    north-star 1e-12 criterion; ``bitwise_equal`` the -fmad=false contract.
    """
    if a.dims != b.dims:
        raise ConfigError("compare_states: dimension mismatch")
    d = StateDiff()
    for ci in range(12):
        va, vb = a.interior(ci), b.interior(ci)
        ba = va.view(np.uint64).reshape(va.shape + (2,))
        bb = vb.view(np.uint64).reshape(vb.shape + (2,))
        neq = np.any(ba != bb, axis=-1)
        n = int(neq.sum())
        if n:
            if d.bitwise_equal:
                z, y, x = np.argwhere(neq)[0]
                d.first_component, d.x, d.y, d.z = ci, int(x), int(y), int(z)
            d.bitwise_equal = False
            d.differing_values += n
            diff = np.maximum(np.abs(va.real - vb.real), np.abs(va.imag - vb.imag))
            d.max_abs_diff = max(d.max_abs_diff, float(diff.max()))
        den = float(np.sqrt(np.sum(np.abs(vb) ** 2)))
        num = float(np.sqrt(np.sum(np.abs(va - vb) ** 2)))
        d.rel_l2[ci] = num / den if den > 0 else num
    return d


# ---------------------------------------------------------------- C-ABI binding
class _Scheme(ctypes.Structure):
    """thiim_scheme (include/thiim_gpu.h) == SchemeParams (coefficients.hpp:21-34)."""
    _fields_ = [("omega", ctypes.c_double), ("tau", ctypes.c_double), ("delta", ctypes.c_double),
                ("se_re", ctypes.c_double), ("se_im", ctypes.c_double),
                ("sh_re", ctypes.c_double), ("sh_im", ctypes.c_double)]


class _Dims(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int), ("ny", ctypes.c_int), ("nz", ctypes.c_int),
                ("ghost", ctypes.c_int)]


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("n_gpus", ctypes.c_int), ("engine", ctypes.c_int),
                ("tile_x", ctypes.c_int), ("tile_y", ctypes.c_int), ("z_chunk", ctypes.c_int),
                ("time_block", ctypes.c_int), ("schedule", ctypes.c_int), ("band", ctypes.c_int),
                ("same_device", ctypes.c_int), ("reserved", ctypes.c_int * 4),
                ("coeff_layout", ctypes.c_int), ("n_materials", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("seconds", ctypes.c_double), ("mlups", ctypes.c_double),
                ("balance_model", ctypes.c_double), ("kernel_seconds", ctypes.c_double),
                ("kernel_launches", ctypes.c_longlong), ("steps", ctypes.c_int),
                ("engine", ctypes.c_int), ("n_gpus", ctypes.c_int),
                ("reserved", ctypes.c_int * 5)]


class _BatchStats(ctypes.Structure):
    _fields_ = [("seconds", ctypes.c_double), ("device_seconds", ctypes.c_double),
                ("upload_seconds", ctypes.c_double), ("kernel_seconds", ctypes.c_double),
                ("download_seconds", ctypes.c_double), ("mlups", ctypes.c_double),
                ("kernel_launches", ctypes.c_longlong), ("h2d_bytes", ctypes.c_longlong),
                ("d2h_bytes", ctypes.c_longlong), ("n_problems", ctypes.c_int),
                ("depth", ctypes.c_int), ("engine", ctypes.c_int), ("reserved", ctypes.c_int * 5)]


class _Diff(ctypes.Structure):
    _fields_ = [("differing_values", ctypes.c_ulonglong), ("max_rel_l2", ctypes.c_double),
                ("rel_l2", ctypes.c_double * 12)]


class _Cand(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("time_block", "tile_y", "z_chunk", "band", "schedule",
                                            "tiles", "rounds")] + \
               [(n, ctypes.c_double) for n in ("balance_model", "model_bytes_per_lup",
                                               "quantization", "model_mlups", "l2_set_bytes")]


class _Trial(ctypes.Structure):
    _fields_ = [("cand", _Cand), ("steps", ctypes.c_int), ("ok", ctypes.c_int),
                ("seconds", ctypes.c_double), ("mlups", ctypes.c_double),
                ("note", ctypes.c_char * 96)]


EXPORTED_SYMBOLS = [
    "thiim_gpu_abi_version", "thiim_gpu_last_error", "thiim_gpu_default_opts",
    "thiim_gpu_balance_model", "thiim_gpu_create", "thiim_gpu_destroy", "thiim_gpu_upload",
    "thiim_gpu_upload_fields", "thiim_gpu_init_generated", "thiim_gpu_step",
    "thiim_gpu_download_fields", "thiim_gpu_download_array", "thiim_gpu_compare_fields",
    "thiim_generate_host", "thiim_gpu_pin_host", "thiim_gpu_unpin_host",
    "thiim_gpu_create_slab", "thiim_gpu_halo_view", "thiim_gpu_slab_info", "thiim_gpu_sync",
    "thiim_gpu_upload_planes", "thiim_gpu_download_fields_planes", "thiim_generate_host_planes",
    "thiim_gpu_upload_table", "thiim_gpu_download_table", "thiim_gpu_set_sanitize",
    "thiim_gpu_coverage", "thiim_scheme_default", "thiim_gpu_init_benchmark",
    "thiim_gpu_init_materials", "thiim_gpu_selftest_cdiv", "thiim_gpu_slab_export",
    "thiim_gpu_slab_import", "thiim_gpu_slab_detach", "thiim_gpu_run_batch",
    "thiim_gpu_release_cached", "thiim_gpu_enumerate_candidates", "thiim_gpu_tune",
    "thiim_coeff_compress",
]

_LIB = None


def lib() -> ctypes.CDLL:
    """Load libthiim_gpu.so (built in-tree by __graft_entry__.build()).  Raises
    if it is missing: there is no fallback compute path."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise GpuError("libthiim_gpu.so not built (%s); run __graft_entry__.build()" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    PP = ctypes.POINTER(ctypes.c_void_p)
    L.thiim_gpu_abi_version.restype = ctypes.c_int
    L.thiim_gpu_last_error.restype = ctypes.c_char_p
    L.thiim_gpu_default_opts.argtypes = [ctypes.POINTER(_Opts)]
    L.thiim_gpu_balance_model.restype = ctypes.c_double
    L.thiim_gpu_balance_model.argtypes = [ctypes.c_int, ctypes.c_int]
    L.thiim_gpu_create.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(_Opts), ctypes.POINTER(P)]
    L.thiim_gpu_destroy.argtypes = [P]
    L.thiim_gpu_upload.argtypes = [P, PP, PP, PP, PP]
    L.thiim_gpu_upload_fields.argtypes = [P, PP]
    L.thiim_gpu_init_generated.argtypes = [P, ctypes.c_int, ctypes.c_uint64]
    L.thiim_gpu_step.argtypes = [P, ctypes.c_int, ctypes.POINTER(_Stats)]
    L.thiim_gpu_download_fields.argtypes = [P, PP]
    L.thiim_gpu_download_array.argtypes = [P, ctypes.c_int, P]
    L.thiim_gpu_compare_fields.argtypes = [P, PP, ctypes.POINTER(_Diff)]
    L.thiim_generate_host.argtypes = [ctypes.POINTER(_Dims), ctypes.c_int, ctypes.c_uint64, PP]
    L.thiim_gpu_upload_table.argtypes = [P, PP, P, P]
    L.thiim_coeff_compress.argtypes = [ctypes.POINTER(_Dims), PP, ctypes.c_int, P, P,
                                       ctypes.POINTER(ctypes.c_int)]
    L.thiim_gpu_download_table.argtypes = [P, P, P]
    L.thiim_gpu_pin_host.argtypes = [P, ctypes.c_size_t]
    L.thiim_gpu_unpin_host.argtypes = [P]
    L.thiim_gpu_set_sanitize.argtypes = [P, ctypes.c_int]
    L.thiim_scheme_default.argtypes = [ctypes.POINTER(_Scheme)]
    L.thiim_gpu_init_benchmark.argtypes = [P, ctypes.POINTER(_Scheme)]
    L.thiim_gpu_init_materials.argtypes = [P, ctypes.POINTER(_Scheme), P]
    L.thiim_gpu_selftest_cdiv.argtypes = [ctypes.c_int, P, P]
    L.thiim_gpu_coverage.argtypes = [P, ctypes.POINTER(ctypes.c_ulonglong),
                                     ctypes.POINTER(ctypes.c_ulonglong)]
    L.thiim_gpu_release_cached.argtypes = [ctypes.c_int]
    L.thiim_gpu_run_batch.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(_Opts), ctypes.c_int,
                                      PP, PP, ctypes.c_int, ctypes.c_int,
                                      ctypes.POINTER(_BatchStats)]
    L.thiim_gpu_enumerate_candidates.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(_Opts),
                                                 ctypes.c_double, ctypes.POINTER(_Cand),
                                                 ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    L.thiim_gpu_tune.argtypes = [ctypes.POINTER(_Dims), ctypes.POINTER(_Opts), ctypes.c_int,
                                 ctypes.c_double, ctypes.c_int, ctypes.POINTER(_Trial),
                                 ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                 ctypes.POINTER(_Opts), ctypes.POINTER(ctypes.c_int)]
    if L.thiim_gpu_abi_version() != 2:
        raise GpuError("libthiim_gpu.so ABI mismatch")
    _LIB = L
    return L


def _ptrs(arrays) -> "ctypes.Array":
    return (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib().thiim_gpu_last_error() or b"").decode()
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise SetupError(msg)
    raise GpuError("thiim_gpu error %d: %s" % (rc, msg))


GEN_RANDOM = 0
GEN_LAYERED = 1
COEFF_FULL = 0
COEFF_TABLE = 1
COEFF_AUTO = 2  # run_gpu only (THIIM_COEFF_AUTO_HOST): TABLE for <= 16 coefficient rows, else FULL
ENGINE_AUTO, ENGINE_SPLIT, ENGINE_FUSED, ENGINE_TBLOCK, ENGINE_TBLOCK_INPLACE = 0, 1, 2, 3, 4
ENGINE_NAMES = {ENGINE_SPLIT: "gpu-split", ENGINE_FUSED: "gpu-fused", ENGINE_TBLOCK: "gpu-tblock",
                ENGINE_TBLOCK_INPLACE: "gpu-tblock-inplace"}


def selftest_cdiv(operands: np.ndarray) -> np.ndarray:
    """Device complex division (libgcc __divdc3 restated) of operands (n, 4) =
    a, b, c, d -> (n, 2) = (a+ib)/(c+id); verification entry."""
    a = np.ascontiguousarray(operands, dtype=np.float64).reshape(-1, 4)
    out = np.zeros((a.shape[0], 2), dtype=np.float64)
    _check(lib().thiim_gpu_selftest_cdiv(a.shape[0], a.ctypes.data, out.ctypes.data))
    return out


def balance_model(engine: int, time_block: int = 0) -> float:
    """Modelled HBM bytes per LUP of an engine (TBLOCK: 832 / time_block, default 2)."""
    return float(lib().thiim_gpu_balance_model(engine, time_block))


@dataclass
class GpuOptions:
    """Mirror of thiim_gpu_opts (include/thiim_gpu.h)."""

    device: int = 0
    n_gpus: int = 1
    engine: int = ENGINE_AUTO
    tile_x: int = 0
    tile_y: int = 0
    z_chunk: int = 0
    time_block: int = 0
    schedule: int = 0  # TBLOCK CTA schedule: 0 auto (rounds, tiles in bands), 1 one launch
    band: int = 0      # TBLOCK rounds: tile columns per band, 0 = auto
    same_device: int = 0  # test knob: all slabs of a multi-slab context on `device`
    coeff_layout: int = 0  # COEFF_FULL (reference layout) or COEFF_TABLE (material ids)
    n_materials: int = 0

    def _c(self) -> _Opts:
        o = _Opts()
        lib().thiim_gpu_default_opts(ctypes.byref(o))
        o.device, o.n_gpus, o.engine = self.device, self.n_gpus, self.engine
        o.tile_x, o.tile_y, o.z_chunk, o.time_block = self.tile_x, self.tile_y, self.z_chunk, self.time_block
        o.schedule, o.band, o.same_device = self.schedule, self.band, self.same_device
        o.coeff_layout, o.n_materials = self.coeff_layout, self.n_materials
        return o


@dataclass
class RunReport:
    """thiim::RunReport (report.hpp:37-52), filled like run_naive does
    (reference_engines.cpp:37-44, 19-23): threads = #GPUs, balance_model = the
    engine's algorithmic bytes/LUP, seconds = device time (CUDA events)."""

    engine: str = ""
    dims: Optional[GridDims] = None
    steps: int = 0
    steps_executed: int = 0
    threads: int = 1
    dw: int = 0
    bz: int = 0
    seconds: float = 0.0
    mlups: Optional[float] = None
    balance_model: float = 0.0
    cache_model_bytes: int = 0
    predicted_mlups: Optional[float] = None
    verification: str = "skipped"
    kernel_launches: int = 0


class GpuEngine:
    """A device-resident problem (one thiim_gpu_ctx)."""

    def __init__(self, dims: GridDims, opts: Optional[GpuOptions] = None):
        self.dims = dims
        self.opts = opts or GpuOptions()
        L = lib()
        self._ctx = ctypes.c_void_p()
        d = _Dims(dims.nx, dims.ny, dims.nz, dims.ghost)
        o = self.opts._c()
        _check(L.thiim_gpu_create(ctypes.byref(d), ctypes.byref(o), ctypes.byref(self._ctx)))

    def close(self) -> None:
        if self._ctx:
            lib().thiim_gpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def upload(self, s: ProblemState) -> None:
        if s.dims != self.dims:
            raise ConfigError("state dims do not match the engine")
        a = s.arrays
        _check(lib().thiim_gpu_upload(self._ctx, _ptrs(a[0:12]), _ptrs(a[12:24]), _ptrs(a[24:36]),
                                      _ptrs(a[36:40])))

    def upload_fields(self, s: ProblemState) -> None:
        _check(lib().thiim_gpu_upload_fields(self._ctx, _ptrs(s.arrays[0:12])))

    def generate(self, kind: int = GEN_RANDOM, seed: int = 1) -> None:
        _check(lib().thiim_gpu_init_generated(self._ctx, kind, seed))

    def init_benchmark(self, omega: float = 0.4, tau: float = 1.0, delta: float = 1.0,
                       source_e: complex = 1.0 + 0j, source_h: complex = 1.0 + 0j) -> None:
        """build_benchmark_problem (coefficients.cpp:94-111) on the device."""
        sp = _Scheme(omega, tau, delta, source_e.real, source_e.imag, source_h.real,
                     source_h.imag)
        _check(lib().thiim_gpu_init_benchmark(self._ctx, ctypes.byref(sp)))

    def init_materials(self, materials: np.ndarray, omega: float = 0.4, tau: float = 1.0,
                       delta: float = 1.0, source_e: complex = 1.0 + 0j,
                       source_h: complex = 1.0 + 0j) -> None:
        """build_problem_from_voxels (coefficients.cpp:112-141) on the device;
        `materials`: (nz, ny, nx, 5) float64 = eps re/im, mu, sigma, sigma*."""
        m = np.ascontiguousarray(materials, dtype=np.float64)
        if m.size != self.dims.interior_cells() * 5:
            raise ConfigError("material map must hold nx*ny*nz records of 5 doubles")
        sp = _Scheme(omega, tau, delta, source_e.real, source_e.imag, source_h.real,
                     source_h.imag)
        _check(lib().thiim_gpu_init_materials(self._ctx, ctypes.byref(sp), m.ctypes.data))

    def step(self, steps: int) -> _Stats:
        st = _Stats()
        _check(lib().thiim_gpu_step(self._ctx, steps, ctypes.byref(st)))
        return st

    def download_fields(self, s) -> None:
        """Into a ProblemState's fields, or into a list of 12 padded arrays."""
        fs = s.arrays[0:12] if isinstance(s, ProblemState) else list(s)
        if len(fs) != 12:
            raise ConfigError("download_fields needs 12 arrays")
        _check(lib().thiim_gpu_download_fields(self._ctx, _ptrs(fs)))

    def set_sanitize(self, on: bool = True) -> None:
        """Exactly-once store coverage check after every pass (debug mode)."""
        _check(lib().thiim_gpu_set_sanitize(self._ctx, int(bool(on))))

    def coverage(self) -> Tuple[int, int]:
        """(passes checked, (component, cell) violations) since set_sanitize."""
        p, v = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        _check(lib().thiim_gpu_coverage(self._ctx, ctypes.byref(p), ctypes.byref(v)))
        return p.value, v.value

    def upload_table(self, fields: List[np.ndarray], material_id: np.ndarray,
                     table: np.ndarray) -> None:
        """THIIM_COEFF_TABLE contexts: 12 field arrays, uint8 material id per
        padded cell, table [n_materials][28] complex128 (t, c, src order)."""
        mid = np.ascontiguousarray(material_id, dtype=np.uint8)
        tab = np.ascontiguousarray(table, dtype=np.complex128)
        _check(lib().thiim_gpu_upload_table(self._ctx, _ptrs(fields[0:12]), mid.ctypes.data,
                                            tab.ctypes.data))

    def download_table(self, n_materials: int):
        n = self.dims.padded_cells()
        mid = np.zeros(n, dtype=np.uint8)
        tab = np.zeros((n_materials, 28), dtype=np.complex128)
        _check(lib().thiim_gpu_download_table(self._ctx, mid.ctypes.data, tab.ctypes.data))
        return mid, tab

    def download_array(self, a: int, out: np.ndarray) -> None:
        _check(lib().thiim_gpu_download_array(self._ctx, a, out.ctypes.data))

    def download_state(self) -> ProblemState:
        s = allocate_state(self.dims)
        for a in range(40):
            self.download_array(a, s.arrays[a])
        return s

    def compare_fields(self, ref) -> StateDiff:
        """On-device comparison with a ProblemState's fields or 12 padded arrays."""
        fs = ref.arrays[0:12] if isinstance(ref, ProblemState) else list(ref)
        if len(fs) != 12:
            raise ConfigError("compare_fields needs 12 arrays")
        out = _Diff()
        _check(lib().thiim_gpu_compare_fields(self._ctx, _ptrs(fs), ctypes.byref(out)))
        d = StateDiff()
        d.differing_values = int(out.differing_values)
        d.bitwise_equal = d.differing_values == 0
        d.rel_l2 = list(out.rel_l2)
        return d


def generate_problem(dims: GridDims, kind: int = GEN_RANDOM, seed: int = 1) -> ProblemState:
    """Host copy of the seeded synthetic problem (bitwise equal to the device
    generator)."""
    s = allocate_state(dims)
    d = _Dims(dims.nx, dims.ny, dims.nz, dims.ghost)
    _check(lib().thiim_generate_host(ctypes.byref(d), kind, seed, _ptrs(s.arrays)))
    return s


def compress_coefficients(state: ProblemState, max_materials: int = 16):
    """Material ids + coefficient table of a piecewise-constant problem (the
    THIIM_COEFF_TABLE layout).  Raises ConfigError if the medium has more than
    `max_materials` distinct coefficient rows."""
    coef = np.stack(state.arrays[12:40], axis=1)  # (cells, 28)
    rows, ids = np.unique(coef.view(np.uint64).reshape(len(coef), 56), axis=0, return_inverse=True)
    if len(rows) > max_materials:
        raise ConfigError("medium has %d distinct coefficient rows (> %d)" % (len(rows), max_materials))
    table = rows.view(np.complex128).reshape(len(rows), 28)
    return ids.astype(np.uint8).reshape(-1), np.ascontiguousarray(table)


def coeff_compress(state: ProblemState, max_materials: int = 16):
    """Native compression (thiim_coeff_compress) of the interior coefficient
    rows: (material_id, table) of the THIIM_COEFF_TABLE layout when the medium
    has at most `max_materials` distinct rows, else None.  Ghost cells' ids are
    0 (no engine reads their coefficients)."""
    d = _Dims(state.dims.nx, state.dims.ny, state.dims.nz, state.dims.ghost)
    mid = np.empty(state.dims.padded_cells(), np.uint8)
    tab = np.empty((max(1, max_materials), 28), np.complex128)
    n = ctypes.c_int()
    _check(lib().thiim_coeff_compress(ctypes.byref(d), _ptrs(state.arrays[12:40]), max_materials,
                                      mid.ctypes.data, tab.ctypes.data, ctypes.byref(n)))
    if n.value == 0:
        return None
    return mid, np.ascontiguousarray(tab[:n.value])


def expand_coefficients(dims: GridDims, material_id: np.ndarray, table: np.ndarray) -> ProblemState:
    """Inverse of compress_coefficients (fields left zero)."""
    s = allocate_state(dims)
    full = table[material_id]  # (cells, 28)
    for k in range(28):
        s.arrays[12 + k][:] = full[:, k]
    return s


def run_gpu(state: ProblemState, steps: int, opts: Optional[GpuOptions] = None) -> RunReport:
    """Drop-in for run_naive(state, steps) (reference_engines.cpp:34-67): uploads
    ``state``, runs ``steps`` THIIM iterations on the GPU(s), downloads the 12
    fields back into ``state`` in place, returns a RunReport."""
    if steps < 0:
        raise ConfigError("steps must be >= 0")
    opts = opts or GpuOptions()
    packed = None
    if opts.coeff_layout == COEFF_AUTO:
        # piecewise-constant media run in the compressed layout (192.5 instead
        # of 416 B/LUP with TBLOCK), bitwise the same results
        packed = coeff_compress(state)
        opts = replace(opts, coeff_layout=COEFF_TABLE if packed else COEFF_FULL,
                       n_materials=len(packed[1]) if packed else opts.n_materials)
    with GpuEngine(state.dims, opts) as eng:
        if packed:
            eng.upload_table(state.fields, packed[0], packed[1])
        else:
            eng.upload(state)
        st = eng.step(steps)
        eng.download_fields(state)
    r = RunReport(engine=ENGINE_NAMES.get(st.engine, "gpu") + ("-table" if packed else ""),
                  dims=state.dims, steps=steps,
                  steps_executed=steps, threads=st.n_gpus, seconds=st.seconds,
                  balance_model=st.balance_model, kernel_launches=st.kernel_launches)
    if steps > 0 and st.seconds > 0:
        r.mlups = state.dims.interior_cells() * steps / st.seconds / 1e6
    return r


@dataclass
class BatchReport:
    """Result of run_gpu_batch: host wall clock of the whole call plus the
    device time of each phase summed over the problems."""

    engine: str = ""
    n_problems: int = 0
    depth: int = 0
    steps: int = 0
    seconds: float = 0.0
    device_seconds: float = 0.0
    upload_seconds: float = 0.0
    kernel_seconds: float = 0.0
    download_seconds: float = 0.0
    mlups: float = 0.0
    kernel_launches: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0


def release_cached(device: int = 0) -> None:
    """Return the device pool's cached, unused pages to the driver."""
    _check(lib().thiim_gpu_release_cached(device))


def run_gpu_batch(states: List[ProblemState], steps: int, opts: Optional[GpuOptions] = None,
                  outputs: Optional[List[List[np.ndarray]]] = None, depth: int = 0) -> BatchReport:
    """run_naive (reference_engines.cpp:34-67) over a stream of independent
    problems on one GPU, pipelined (thiim_gpu_run_batch): problem i uploads
    while i-1 computes and i-2 downloads.  ``outputs[i]`` (12 complex128
    arrays of padded_cells()) receives problem i's fields; without it each
    state is updated in place, and then the states must not share arrays.
    Pin the host arrays (lib().thiim_gpu_pin_host) for the copies to overlap."""
    if steps < 0:
        raise ConfigError("steps must be >= 0")
    opts = opts or GpuOptions()
    if not states:
        return BatchReport(n_problems=0, steps=steps)
    dims = states[0].dims
    n = dims.padded_cells()
    for s in states:
        if s.dims != dims:
            raise ConfigError("all problems of a batch need the same grid dims")
    if outputs is not None:
        if len(outputs) != len(states):
            raise ConfigError("outputs needs one 12-array field set per problem")
        for fs in outputs:
            if len(fs) != 12 or any(a.shape != (n,) or a.dtype != np.complex128
                                    or not a.flags.c_contiguous for a in fs):
                raise ConfigError("outputs: 12 C-contiguous complex128 arrays of padded_cells()")
    ins = _ptrs([a for s in states for a in s.arrays])
    outs = _ptrs([a for fs in outputs for a in fs]) if outputs is not None else None
    d = _Dims(dims.nx, dims.ny, dims.nz, dims.ghost)
    o = opts._c()
    st = _BatchStats()
    _check(lib().thiim_gpu_run_batch(ctypes.byref(d), ctypes.byref(o), len(states), ins, outs,
                                     steps, depth, ctypes.byref(st)))
    return BatchReport(engine=ENGINE_NAMES.get(st.engine, "gpu"), n_problems=st.n_problems,
                       depth=st.depth, steps=steps, seconds=st.seconds,
                       device_seconds=st.device_seconds, upload_seconds=st.upload_seconds,
                       kernel_seconds=st.kernel_seconds, download_seconds=st.download_seconds,
                       mlups=st.mlups, kernel_launches=st.kernel_launches,
                       h2d_bytes=st.h2d_bytes, d2h_bytes=st.d2h_bytes)


# ---------------------------------------------------------------- auto-tuner
_CAND_KEYS = ("time_block", "tile_y", "z_chunk", "band", "schedule", "tiles", "rounds",
              "balance_model", "model_bytes_per_lup", "quantization", "model_mlups",
              "l2_set_bytes")


def _cand_dict(c: _Cand) -> dict:
    return {k: getattr(c, k) for k in _CAND_KEYS}


def enumerate_candidates(dims: GridDims, opts: Optional[GpuOptions] = None,
                         hbm_gbs: float = 0.0) -> List[dict]:
    """TBLOCK candidates ranked by the GPU re-parameterisation of the
    reference's models (enumerate_candidates, autotuner.cpp:15-50): modelled
    DRAM bytes/LUP (Eq. 12 analogue) x wave quantisation, L2 fit of the
    deeper levels' coefficient planes (Eq. 11 analogue).  No device needed."""
    d = _Dims(dims.nx, dims.ny, dims.nz, dims.ghost)
    o = (opts or GpuOptions())._c()
    n = ctypes.c_int()
    _check(lib().thiim_gpu_enumerate_candidates(ctypes.byref(d), ctypes.byref(o), hbm_gbs, None, 0,
                                                ctypes.byref(n)))
    arr = (_Cand * max(1, n.value))()
    _check(lib().thiim_gpu_enumerate_candidates(ctypes.byref(d), ctypes.byref(o), hbm_gbs, arr,
                                                n.value, ctypes.byref(n)))
    return [_cand_dict(arr[i]) for i in range(n.value)]


@dataclass
class TuneResult:
    """tune's result (autotuner.hpp TuneResult): the trial table, the winner
    as GpuOptions and its bitwise verification."""
    table: List[dict] = field(default_factory=list)
    best: Optional[GpuOptions] = None
    winner_verification: str = "skipped"


def tune(dims: GridDims, steps: int = 8, opts: Optional[GpuOptions] = None,
         min_seconds: float = 0.5, max_trials: int = 8) -> TuneResult:
    """tune (autotuner.cpp:62-142) for the GPU knobs: times the model's best
    candidates, picks the deepest time block within 2% of the fastest and
    verifies it bitwise against the fused engine."""
    d = _Dims(dims.nx, dims.ny, dims.nz, dims.ghost)
    o = (opts or GpuOptions())._c()
    cap = max_trials + 2
    tab = (_Trial * cap)()
    n = ctypes.c_int()
    w = _Opts()
    ver = ctypes.c_int()
    _check(lib().thiim_gpu_tune(ctypes.byref(d), ctypes.byref(o), steps, min_seconds, max_trials,
                                tab, cap, ctypes.byref(n), ctypes.byref(w), ctypes.byref(ver)))
    rows = []
    for i in range(n.value):
        t = tab[i]
        r = _cand_dict(t.cand)
        r.update(steps=t.steps, ok=bool(t.ok), seconds=t.seconds, mlups=t.mlups,
                 note=t.note.decode(errors="replace"))
        rows.append(r)
    best = GpuOptions(device=w.device, n_gpus=w.n_gpus, engine=w.engine, tile_x=w.tile_x,
                      tile_y=w.tile_y, z_chunk=w.z_chunk, time_block=w.time_block,
                      schedule=w.schedule, band=w.band, same_device=w.same_device,
                      coeff_layout=w.coeff_layout, n_materials=w.n_materials)
    return TuneResult(table=rows, best=best,
                      winner_verification="bitwise-equal vs gpu-fused" if ver.value else "failed")
