"""Multi-GPU z-slab decomposition, one process per GPU.

The grid's interior planes are split into contiguous z-slabs exactly like the
reference's threaded engines split them among workers (z_slab,
reference_engines.cpp:26-30).  Each rank owns one slab context
(thiim_gpu_create_slab) whose boundary planes are either global ghosts or
halo copies of the neighbour's boundary planes.  Before every THIIM step the
ranks exchange, per interface:

    lower rank  SEND_UP   : E x6 + Hxy,Hxz,Hyx,Hyz of its last plane  -> upper RECV_DOWN
    upper rank  SEND_DOWN : E x6 of its first plane                   -> lower RECV_UP

The upper rank recomputes H_new on the received plane inside its sweep, so a
step needs no mid-step exchange.  With the TBLOCK engine (two steps per HBM
pass) slabs are "deep": two-plane halos of all 12 fields, exchanged after
every 2-step pass (include/thiim_gpu.h).  Either way the driver loop is
step(k <= exchange_period), then exchange -- the uploaded halos are valid for
the first pass.  The exchange is torch.distributed
point-to-point (batch_isend_irecv: NCCL over NVLink on GPUs, gloo on CPU for
the tests); the engine object supplies the plane buffers, so the same logic
drives the CUDA engine and the CPU test double.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import numpy as np

from . import (GEN_RANDOM, GridDims, GpuOptions, ProblemState, _check, _Dims, _ptrs, _Stats, lib)

SEND_DOWN, RECV_DOWN, SEND_UP, RECV_UP = 0, 1, 2, 3
N_ARRAYS = {SEND_DOWN: 6, RECV_DOWN: 10, SEND_UP: 10, RECV_UP: 6}


def slab_bounds(nz: int, world: int, rank: int) -> Tuple[int, int]:
    """Static z partition of reference_engines.cpp:26-30."""
    base, rem = divmod(nz, world)
    z0 = rank * base + min(rank, rem)
    return z0, z0 + base + (1 if rank < rem else 0)


class _HaloView(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p), ("array_stride_bytes", ctypes.c_longlong),
                ("plane_bytes", ctypes.c_longlong), ("n_arrays", ctypes.c_int),
                ("device", ctypes.c_int)]


class _CudaPlane:
    """__cuda_array_interface__ over one device array-plane (float64 view)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes // 8,), "typestr": "<f8",
                                         "data": (ptr, False), "version": 3, "strides": None}


class _SlabInfo(ctypes.Structure):
    _fields_ = [("own_z0", ctypes.c_int), ("own_z1", ctypes.c_int), ("local_z0", ctypes.c_int),
                ("local_z1", ctypes.c_int), ("exchange_period", ctypes.c_int),
                ("engine", ctypes.c_int), ("device_ordered", ctypes.c_int)]


class _SlabExport(ctypes.Structure):
    """thiim_slab_export (include/thiim_gpu.h)."""
    _fields_ = [("ipc", ctypes.c_ubyte * 64), ("stride", ctypes.c_longlong),
                ("nz_local", ctypes.c_int), ("ext_lo", ctypes.c_int), ("ext_hi", ctypes.c_int),
                ("nfield_sets", ctypes.c_int), ("device", ctypes.c_int), ("px", ctypes.c_int),
                ("pxy", ctypes.c_longlong), ("counter_offset", ctypes.c_longlong)]


class SlabGpuEngine:
    """One rank's slab of the global grid on its GPU (AUTO: TBLOCK deep-halo slab)."""

    def __init__(self, global_dims: GridDims, z0: int, z1: int, opts: Optional[GpuOptions] = None):
        self.dims, self.z0, self.z1 = global_dims, z0, z1
        self.opts = opts or GpuOptions()
        L = lib()
        L.thiim_gpu_create_slab.argtypes = [ctypes.POINTER(_Dims), ctypes.c_int, ctypes.c_int,
                                            ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]
        L.thiim_gpu_halo_view.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(_HaloView)]
        L.thiim_gpu_sync.argtypes = [ctypes.c_void_p]
        self._ctx = ctypes.c_void_p()
        d = _Dims(global_dims.nx, global_dims.ny, global_dims.nz, global_dims.ghost)
        o = self.opts._c()
        _check(L.thiim_gpu_create_slab(ctypes.byref(d), z0, z1, ctypes.byref(o),
                                       ctypes.byref(self._ctx)))
        L.thiim_gpu_slab_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(_SlabInfo)]
        info = _SlabInfo()
        _check(L.thiim_gpu_slab_info(self._ctx, ctypes.byref(info)))
        # padded planes this rank's host buffers hold: [local_z0, local_z1 + 2)
        self.local_z0, self.local_z1 = info.local_z0, info.local_z1
        self.exchange_period = info.exchange_period
        self.engine = info.engine
        self.peer_stores = False
        self.device_ordered = False

    def close(self):
        if self._ctx:
            lib().thiim_gpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def generate(self, kind: int = GEN_RANDOM, seed: int = 1):
        _check(lib().thiim_gpu_init_generated(self._ctx, kind, seed))

    def upload(self, s: ProblemState):
        a = s.arrays
        _check(lib().thiim_gpu_upload(self._ctx, _ptrs(a[0:12]), _ptrs(a[12:24]), _ptrs(a[24:36]),
                                      _ptrs(a[36:40])))

    def download_fields(self, s: ProblemState):
        _check(lib().thiim_gpu_download_fields(self._ctx, _ptrs(s.arrays[0:12])))

    # rank-local host buffers: global padded planes [local_z0, local_z1 + 2)
    def local_host_problem(self, kind: int = GEN_RANDOM, seed: int = 1) -> List[np.ndarray]:
        pxy = (self.dims.nx + 2) * (self.dims.ny + 2)
        n = self.local_z1 - self.local_z0 + 2
        arrays = [np.zeros(n * pxy, dtype=np.complex128) for _ in range(40)]
        d = _Dims(self.dims.nx, self.dims.ny, self.dims.nz, self.dims.ghost)
        _check(lib().thiim_generate_host_planes(ctypes.byref(d), kind, seed, self.local_z0,
                                                self.local_z1 + 2, _ptrs(arrays)))
        return arrays

    def owned_planes(self, arrays: List[np.ndarray], k: int) -> np.ndarray:
        """Interior planes [z0, z1) of host array k of local_host_problem()."""
        pxy = (self.dims.nx + 2) * (self.dims.ny + 2)
        a = self.z0 - self.local_z0 + 1
        return arrays[k][a * pxy:(a + self.z1 - self.z0) * pxy]

    def upload_local(self, arrays: List[np.ndarray]):
        _check(lib().thiim_gpu_upload_planes(self._ctx, _ptrs(arrays), self.local_z0))

    def download_local(self, arrays: List[np.ndarray]):
        _check(lib().thiim_gpu_download_fields_planes(self._ctx, _ptrs(arrays[0:12]),
                                                      self.local_z0))

    def step(self, steps: int = 1):
        st = _Stats()
        _check(lib().thiim_gpu_step(self._ctx, steps, ctypes.byref(st)))
        return st

    def halo(self, which: int):
        """The halo array-planes as torch CUDA tensors aliasing engine memory."""
        import torch
        v = _HaloView()
        _check(lib().thiim_gpu_halo_view(self._ctx, which, ctypes.byref(v)))
        dev = torch.device("cuda", v.device)
        return [torch.as_tensor(_CudaPlane(v.base + k * v.array_stride_bytes, v.plane_bytes),
                                device=dev) for k in range(v.n_arrays)]

    def sync(self):
        _check(lib().thiim_gpu_sync(self._ctx))

    def enable_peer_stores(self, rank: int, world: int, group=None) -> bool:
        """Map the neighbour ranks' slabs (CUDA IPC) so that every TBLOCK pass
        writes their halo planes itself -- no exchange after 2-step passes, a
        barrier instead (run_distributed).  Collective: all ranks call it; all
        end up enabled or all stay on the exchange."""
        import torch
        import torch.distributed as dist
        L = lib()
        L.thiim_gpu_slab_export.argtypes = [ctypes.c_void_p, ctypes.POINTER(_SlabExport)]
        L.thiim_gpu_slab_import.argtypes = [ctypes.c_void_p, ctypes.c_int,
                                            ctypes.POINTER(_SlabExport)]
        L.thiim_gpu_slab_detach.argtypes = [ctypes.c_void_p]
        mine = _SlabExport()
        ok = self.exchange_period == 2 and L.thiim_gpu_slab_export(self._ctx, ctypes.byref(mine)) == 0
        parts = [None] * world
        dist.all_gather_object(parts, bytes(mine) if ok else None, group=group)
        ok = all(p is not None for p in parts)
        if ok:
            for which, nb in ((0, rank - 1), (1, rank + 1)):
                if 0 <= nb < world:
                    ex = _SlabExport.from_buffer_copy(parts[nb])
                    ok = ok and L.thiim_gpu_slab_import(self._ctx, which, ctypes.byref(ex)) == 0
        flag = torch.tensor([1 if ok else 0], dtype=torch.int32,
                            device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.peer_stores = bool(flag.item())
        if not self.peer_stores:
            L.thiim_gpu_slab_detach(self._ctx)
        # passes ordered on the devices (pass counters) on every rank, or a
        # host barrier after every pass on all of them
        info = _SlabInfo()
        _check(L.thiim_gpu_slab_info(self._ctx, ctypes.byref(info)))
        flag = torch.tensor([info.device_ordered if self.peer_stores else 0], dtype=torch.int32,
                            device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.device_ordered = bool(flag.item())
        return self.peer_stores


class HaloExchanger:
    """Between-step halo exchange of one rank with its z-neighbours."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def barrier(self) -> None:
        import torch.distributed as dist
        dist.barrier(group=self.group)

    def exchange(self, engine) -> int:
        """Returns the number of bytes this rank sent."""
        import torch
        import torch.distributed as dist
        ops: List = []
        sent = 0
        if self.rank + 1 < self.world:
            up = self.rank + 1
            for t in engine.halo(SEND_UP):
                ops.append(dist.P2POp(dist.isend, t, up, self.group))
                sent += t.numel() * 8
            for t in engine.halo(RECV_UP):
                ops.append(dist.P2POp(dist.irecv, t, up, self.group))
        if self.rank > 0:
            down = self.rank - 1
            for t in engine.halo(SEND_DOWN):
                ops.append(dist.P2POp(dist.isend, t, down, self.group))
                sent += t.numel() * 8
            for t in engine.halo(RECV_DOWN):
                ops.append(dist.P2POp(dist.irecv, t, down, self.group))
        if ops:
            staged = ops[0].tensor.is_cuda and dist.get_backend(self.group) == "gloo"
            if staged:
                # gloo moves host tensors only: stage device planes through host memory
                host_ops, backs = [], []
                for op in ops:
                    h = op.tensor.detach().cpu() if op.op is dist.isend else torch.empty(
                        op.tensor.shape, dtype=op.tensor.dtype)
                    host_ops.append(dist.P2POp(op.op, h, op.peer, self.group))
                    if op.op is dist.irecv:
                        backs.append((op.tensor, h))
                for req in dist.batch_isend_irecv(host_ops):
                    req.wait()
                for dev, h in backs:
                    dev.copy_(h)
                torch.cuda.synchronize()
            else:
                for req in dist.batch_isend_irecv(ops):
                    req.wait()
                if torch.cuda.is_available() and ops[0].tensor.is_cuda:
                    torch.cuda.synchronize()
        return sent


def run_distributed(engine, steps: int, exchanger: HaloExchanger) -> dict:
    """`steps` THIIM iterations of the decomposed grid: passes of up to
    engine.exchange_period steps, each followed by the halo exchange."""
    period = max(1, int(getattr(engine, "exchange_period", 1)))
    sent = 0
    launches = 0
    done = 0
    if getattr(engine, "peer_stores", False) and steps > 0:
        # upload / generate write both field sets of this slab, halos included:
        # no neighbour's pass may store into them before every rank is done
        exchanger.barrier()
    if getattr(engine, "device_ordered", False) and steps >= 2:
        # every pass waits on the devices for the neighbours' previous pass
        # (pass counters): all 2-step passes in one call, no host sync between
        k = steps - steps % 2
        st = engine.step(k)
        launches += getattr(st, "kernel_launches", 0)
        done = k
    while done < steps:
        k = min(period, steps - done)
        st = engine.step(k)
        launches += getattr(st, "kernel_launches", 0)
        if getattr(engine, "peer_stores", False) and k == 2:
            exchanger.barrier()  # the pass wrote the neighbours' halos itself
        else:
            sent += exchanger.exchange(engine)
        done += k
    if getattr(engine, "device_ordered", False) and steps > 0:
        # every rank's step has returned, i.e. its stream has seen the neighbours'
        # final counters: from here a rank may destroy its slab (the mapped
        # counters and halos the neighbours' streams were polling / storing into)
        exchanger.barrier()
    return {"halo_bytes_sent": sent, "kernel_launches": launches}
