"""Multi-rank z-slab decomposition on CPU (gloo, world_size 2 and 3).

The halo-exchange logic of paper_1510_05218_b200/distributed.py (which
planes, which arrays, which direction, before every step) drives a CPU test
double of the slab engine whose step is the C oracle's slab step; the
gathered result must be BITWISE equal to the undecomposed oracle run.  The
GPU path uses the same HaloExchanger over NCCL with the CUDA slab engine.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1510_05218_b200 as P
from paper_1510_05218_b200 import distributed as D
from oracle import oracle as O


class SlabCpuEngine:
    """Test double of SlabGpuEngine: local planes [z0-1, z1] of every array."""

    def __init__(self, global_arrays, dims, z0, z1):
        self.dims, self.z0, self.z1 = dims, z0, z1
        pxy = (dims.nx + 2) * (dims.ny + 2)
        self.pxy = pxy
        self.local = [np.ascontiguousarray(a[z0 * pxy:(z1 + 2) * pxy]) for a in global_arrays]
        self.ldims = (dims.nx, dims.ny, z1 - z0)

    def plane(self, k, p):
        return torch.from_numpy(self.local[k][p * self.pxy:(p + 1) * self.pxy].view(np.float64))

    def halo(self, which):
        nz = self.z1 - self.z0
        plane = {D.SEND_DOWN: 1, D.RECV_DOWN: 0, D.SEND_UP: nz, D.RECV_UP: nz + 1}[which]
        return [self.plane(k, plane) for k in range(D.N_ARRAYS[which])]

    def step(self, n=1):
        for _ in range(n):
            O.c_step_slab(self.ldims, self.local, self.z0 > 0)


class SlabCpuDeepEngine:
    """Test double of a TBLOCK (deep-halo) slab: local interior planes
    [z0-e_lo, z1+e_hi) -- one extended plane per internal interface -- plus a
    ghost each side; a pass of k <= 2 steps is k oracle slab steps on that
    extended domain, and every view is two planes of all 12 fields
    (include/thiim_gpu.h, deep-halo protocol)."""

    exchange_period = 2

    def __init__(self, global_arrays, dims, z0, z1):
        self.dims, self.z0, self.z1 = dims, z0, z1
        self.elo, self.ehi = int(z0 > 0), int(z1 < dims.nz)
        self.lz0, self.lz1 = z0 - self.elo, z1 + self.ehi
        self.pxy = pxy = (dims.nx + 2) * (dims.ny + 2)
        self.local = [np.ascontiguousarray(a[self.lz0 * pxy:(self.lz1 + 2) * pxy])
                      for a in global_arrays]
        self.ldims = (dims.nx, dims.ny, self.lz1 - self.lz0)

    def halo(self, which):
        nzl = self.lz1 - self.lz0
        first = {D.SEND_DOWN: 1 + self.elo, D.RECV_DOWN: 0, D.SEND_UP: nzl - 1 - self.ehi,
                 D.RECV_UP: nzl}[which]
        p = self.pxy
        return [torch.from_numpy(self.local[k][first * p:(first + 2) * p].view(np.float64))
                for k in range(12)]

    def step(self, n=1):
        assert n <= 2, "deep slabs exchange after at most two steps"
        for _ in range(n):
            O.c_step_slab(self.ldims, self.local, self.lz0 > 0)

    def owned(self, k):
        a = self.z0 - self.lz0 + 1
        return self.local[k][a * self.pxy:(a + self.z1 - self.z0) * self.pxy]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, shape, steps, seed, out_dir, deep=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dims = P.GridDims(*shape)
    arrays = O.c_generate(shape, seed)
    z0, z1 = D.slab_bounds(dims.nz, world, rank)
    eng = (SlabCpuDeepEngine if deep else SlabCpuEngine)(arrays, dims, z0, z1)
    stats = D.run_distributed(eng, steps, D.HaloExchanger(rank, world))
    pxy = eng.pxy
    owned = [eng.owned(k) for k in range(12)] if deep else \
        [a[pxy:(z1 - z0 + 1) * pxy] for a in eng.local[:12]]
    np.save(os.path.join(out_dir, "r%d.npy" % rank), np.stack(owned))
    np.save(os.path.join(out_dir, "s%d.npy" % rank), np.array([stats["halo_bytes_sent"]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,steps", [(2, (9, 7, 12), 5), (3, (6, 5, 14), 4),
                                               (2, (8, 8, 8), 1)])
def test_slab_decomposition_matches_single_domain(tmp_path, world, shape, steps):
    mp.spawn(_worker, args=(world, _free_port(), shape, steps, 21, str(tmp_path)), nprocs=world,
             join=True)
    ref = O.c_generate(shape, 21)
    O.c_step(shape, ref, steps)
    dims = P.GridDims(*shape)
    pxy = (dims.nx + 2) * (dims.ny + 2)
    sent = 0
    for r in range(world):
        z0, z1 = D.slab_bounds(dims.nz, world, r)
        got = np.load(tmp_path / ("r%d.npy" % r))
        for k in range(12):
            want = ref[k][(z0 + 1) * pxy:(z1 + 1) * pxy]
            assert np.array_equal(got[k].view(np.uint64), want.view(np.uint64)), (r, k)
        sent += int(np.load(tmp_path / ("s%d.npy" % r))[0])
    # 16 array-planes cross each interface per step (10 up, 6 down)
    assert sent == steps * (world - 1) * 16 * pxy * 16


@pytest.mark.parametrize("world,shape,steps", [(2, (9, 7, 12), 5), (3, (6, 5, 14), 4),
                                               (2, (8, 8, 8), 2), (3, (7, 6, 15), 7)])
def test_deep_halo_decomposition_matches_single_domain(tmp_path, world, shape, steps):
    """The TBLOCK slab protocol: two-plane halos of all 12 fields exchanged
    after every pass of <= 2 steps; bitwise equal to the undecomposed run."""
    mp.spawn(_worker, args=(world, _free_port(), shape, steps, 23, str(tmp_path), True),
             nprocs=world, join=True)
    ref = O.c_generate(shape, 23)
    O.c_step(shape, ref, steps)
    dims = P.GridDims(*shape)
    pxy = (dims.nx + 2) * (dims.ny + 2)
    sent = 0
    for r in range(world):
        z0, z1 = D.slab_bounds(dims.nz, world, r)
        got = np.load(tmp_path / ("r%d.npy" % r))
        for k in range(12):
            want = ref[k][(z0 + 1) * pxy:(z1 + 1) * pxy]
            assert np.array_equal(got[k].view(np.uint64), want.view(np.uint64)), (r, k)
        sent += int(np.load(tmp_path / ("s%d.npy" % r))[0])
    # per pass and interface: 2 planes x 12 fields each way
    passes = (steps + 1) // 2
    assert sent == passes * (world - 1) * 48 * pxy * 16


def test_slab_bounds_match_reference_z_slab():
    assert [D.slab_bounds(10, 3, r) for r in range(3)] == [(0, 4), (4, 7), (7, 10)]
    assert [D.slab_bounds(256, 8, r)[1] - D.slab_bounds(256, 8, r)[0] for r in range(8)] == [32] * 8


def test_missing_halo_exchange_is_detected(tmp_path):
    """Fault injection: skipping the exchange must break bitwise equality."""
    dims = P.GridDims(6, 6, 10)
    arrays = O.c_generate((6, 6, 10), 4)
    lo, hi = SlabCpuEngine(arrays, dims, 0, 5), SlabCpuEngine(arrays, dims, 5, 10)
    for _ in range(3):
        lo.step()
        hi.step()
    ref = O.c_generate((6, 6, 10), 4)
    O.c_step((6, 6, 10), ref, 3)
    pxy = 64
    got = np.concatenate([lo.local[0][pxy:6 * pxy], hi.local[0][pxy:6 * pxy]])
    assert not np.array_equal(got, ref[0][pxy:11 * pxy])


def test_peer_store_protocol_orders_upload_before_first_pass():
    """Host logic only: with IPC peer stores, run_distributed barriers once on
    entry (an upload / generate rewrites the halos a neighbour's first pass
    stores into -- the race the 2-rank GPU test caught) and after every 2-step
    pass; the odd remainder step still exchanges."""
    calls = []

    class Eng:
        exchange_period = 2
        peer_stores = True

        def step(self, k):
            calls.append(("step", k))
            return type("S", (), {"kernel_launches": 1})()

    class Ex:
        def barrier(self):
            calls.append(("barrier",))

        def exchange(self, eng):
            calls.append(("exchange",))
            return 8

    st = D.run_distributed(Eng(), 5, Ex())
    assert calls == [("barrier",), ("step", 2), ("barrier",), ("step", 2), ("barrier",),
                     ("step", 1), ("exchange",)]
    assert st == {"halo_bytes_sent": 8, "kernel_launches": 3}
    calls.clear()
    D.run_distributed(Eng(), 0, Ex())
    assert calls == []


def test_device_ordered_peer_stores_enqueue_all_passes_at_once():
    """Host logic only: with device-side pass counters (device_ordered), the
    2-step passes of a call go to the library in ONE step call -- no host
    barrier between passes; one barrier on entry and one on exit (after it a
    rank may destroy the slab its neighbours' streams were polling), the odd
    remainder step still exchanges."""
    calls = []

    class Eng:
        exchange_period = 2
        peer_stores = True
        device_ordered = True

        def step(self, k):
            calls.append(("step", k))
            return type("S", (), {"kernel_launches": k // 2 or 1})()

    class Ex:
        def barrier(self):
            calls.append(("barrier",))

        def exchange(self, eng):
            calls.append(("exchange",))
            return 8

    st = D.run_distributed(Eng(), 9, Ex())
    assert calls == [("barrier",), ("step", 8), ("step", 1), ("exchange",), ("barrier",)]
    assert st == {"halo_bytes_sent": 8, "kernel_launches": 5}
    calls.clear()
    D.run_distributed(Eng(), 4, Ex())
    assert calls == [("barrier",), ("step", 4), ("barrier",)]
