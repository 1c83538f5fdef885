// thiim_fused_tma.cuh -- engine FUSED: one z-streamed H->E sweep per
// THIIM step, operands staged by TMA.
//
// Each CTA owns a 30 x (BY-2) x-y tile and streams z over a chunk.  At plane z
// it computes H_new(z) then E_new(z) (reference step_reference order,
// kernels.cpp:105-113): E_new(z) needs H_new at x-1, y-1 (shared memory) and
// z-1 (registers, carried); H_new(z) needs E_old at x+1, y+1 (shared memory) and
// z+1 (the plane fetched one iteration ahead).  Fields are ping-ponged: a
// neighbouring CTA may already have written its edge (the reference's in-place
// update is only safe one family at a time).  The thread block is the tile
// plus a one-cell ring; the -x/-y ring recomputes the four H components the
// tile needs there, bitwise like the owner; at a global boundary the ring sits
// on ghost cells whose stored values are used unchanged.
//
// One producer warp streams the 40 array-planes a z-plane needs (E_old(z+1) x6;
// per H component F, t, c (, src); per E component t, c (, src)) as 4-D TMA
// boxes (cp.async.bulk.tensor, SASS UTMALDG) in 12 groups through a grouped
// mbarrier ring (thiim_ring.cuh); BY consumer warps read them from shared
// memory.  Algorithmic traffic: 40 reads + 12 writes x 16 B = 832 B/LUP.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_producer.cuh"
#include "thiim_ring.cuh"

namespace thiim_gpu {

template <int BY, int NG>
struct FusedSmem {
  Ring<BY, NG> ring;
  double2 sE[3][BY][32];  // E_old sums (x, y, z physical components) at plane z
  double2 sH[3][BY][32];  // H_new sums at plane z
};

template <int BY, int NG, bool COUNT = false>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_fused_tma(Grid g, Arrays A, const __grid_constant__ TmaMaps maps, int zc, int tiles_x,
                int fb, int cb) {
  constexpr int BX = 32, TX = BX - 2, TY = BY - 2, NCOMP = 32 * BY;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  FusedSmem<BY, NG>& sm = *reinterpret_cast<FusedSmem<BY, NG>*>(smem_raw);
  // x-tiles enumerate fastest: x-neighbours share the DRAM blocks at their
  // (unaligned) box edges, so running them together lets the second fetch hit
  // in L2 (measured: 5.7% excess DRAM reads vs 19% y-fastest)
  const int bty = blockIdx.x / tiles_x, btx = blockIdx.x % tiles_x;
  const int xb = btx * TX - 1, yb = bty * TY - 1;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const long long pxy = g.pxy;

  if (tx == 0 && ty == 0) {
    ring_init(sm.ring, BY);
    fence_mbar_init();
  }
  __syncthreads();

  if (ty == BY) {  // ---------------- producer warp (one elected lane)
    if (tx == 0) {
#pragma unroll
      for (int b = 0; b < NBOX; ++b) tma_prefetch_desc(&maps.m[b]);
      // straight-line sequence (thiim_producer.cuh): 40 boxes in 12 groups
      RingProducer<BY, NG> P(sm.ring, maps, xb, yb);
      for (int z = z0; z < z1; ++z) produce_plane_ct<false>(P, fb, cb, z);
    }
    return;
  }

  // ---------------- consumer warps: thread (tx, ty) owns cell (xb+tx, yb+ty)
  const int x = xb + tx, y = yb + ty;
  const bool inpad = (x <= g.nx) && (y <= g.ny);
  const bool interior = (x >= 0) && (x < g.nx) && (y >= 0) && (y < g.ny);
  const bool ring_x = (tx == 0) && (ty >= 1) && (ty <= BY - 2) && (y < g.ny);
  const bool ring_y = (ty == 0) && (tx >= 1) && (tx <= BX - 2) && (x < g.nx);
  const bool own = interior && tx >= 1 && tx <= BX - 2 && ty >= 1 && ty <= BY - 2;
  // which H components this thread updates (ring cells on ghosts keep H_old)
  const bool upd_x = own || (ring_y && y >= 0);                         // Hxy, Hxz
  const bool upd_y = own || (ring_x && x >= 0);                         // Hyx, Hyz
  const bool upd_z = own || (ring_x && x >= 0) || (ring_y && y >= 0);  // Hzx, Hzy
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  long long i = g.idx(xs, ys, z0);

  // prologue: E_old(z0) splits; H_new sums at z0-1 for own cells (direct loads)
  double2 e[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) e[k] = inpad ? __ldg(A.f[k] + i) : make_double2(0.0, 0.0);
  double2 pHx = make_double2(0.0, 0.0), pHy = make_double2(0.0, 0.0);
  {
    const long long im = i - pxy;
    if (z0 == 0 && !g.halo_lo) {
      if (own) {
        pHx = csum(__ldg(A.f[HXY] + im), __ldg(A.f[HXZ] + im));
        pHy = csum(__ldg(A.f[HYX] + im), __ldg(A.f[HYZ] + im));
      }
    } else {
      if (inpad) {
        double2 m[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) m[k] = __ldg(A.f[k] + im);
        sm.sE[0][ty][tx] = csum(m[EXY], m[EXZ]);
        sm.sE[1][ty][tx] = csum(m[EYX], m[EYZ]);
        sm.sE[2][ty][tx] = csum(m[EZX], m[EZY]);
      }
      named_sync(1, NCOMP);
      if (own) {
        const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
        const double2 nEx = csum(e[EXY], e[EXZ]), nEy = csum(e[EYX], e[EYZ]);
        const double2 hxy = upd(__ldg(A.f[HXY] + im), __ldg(A.t[HXY] + im), __ldg(A.c[HXY] + im),
                                sm.sE[2][ty + 1][tx], sEz);
        const double2 hxz = upd_src(__ldg(A.f[HXZ] + im), __ldg(A.t[HXZ] + im),
                                    __ldg(A.c[HXZ] + im), nEy, sEy, __ldg(A.src[SRC_HXZ] + im));
        const double2 hyx = upd(__ldg(A.f[HYX] + im), __ldg(A.t[HYX] + im), __ldg(A.c[HYX] + im),
                                sm.sE[2][ty][tx + 1], sEz);
        const double2 hyz = upd_src(__ldg(A.f[HYZ] + im), __ldg(A.t[HYZ] + im),
                                    __ldg(A.c[HYZ] + im), nEx, sEx, __ldg(A.src[SRC_HYZ] + im));
        pHx = csum(hxy, hxz);
        pHy = csum(hyx, hyz);
      }
      named_sync(1, NCOMP);
    }
  }

  auto& R = sm.ring;
  RingCursor rc = ring_cursor(R);
#define RD(k, b) ring_read(R, rc, k, b, tx, ty)
  for (int z = z0; z < z1; ++z, i += pxy) {
    // (a) E_old(z+1) splits (carried to the next plane); E sums at z to smem
    double2 en[6];
    ring_wait(R, rc);
#pragma unroll
    for (int k = 0; k < 4; ++k) en[k] = RD(k, BOX_A);
    ring_release(R, rc, tx, ring_dep(en[0], en[1], en[2], en[3]));
    ring_wait(R, rc);
    en[4] = RD(0, BOX_A);
    en[5] = RD(1, BOX_A);
    ring_release(R, rc, tx, ring_dep(en[4], en[5]));
    // own sums from registers; neighbours read them from shared memory
    const double2 sEx = csum(e[EXY], e[EXZ]), sEy = csum(e[EYX], e[EYZ]), sEz = csum(e[EZX], e[EZY]);
    if (inpad) {
      sm.sE[0][ty][tx] = sEx;
      sm.sE[1][ty][tx] = sEy;
      sm.sE[2][ty][tx] = sEz;
    }
    named_sync(1, NCOMP);

    // (b) H half-step at plane z (own cells: all six; ring: the four needed)
    const double2 nEx = csum(en[EXY], en[EXZ]), nEy = csum(en[EYX], en[EYZ]);
    double2 h[6];
    {  // Hxy
      ring_wait(R, rc);
      h[0] = RD(0, BOX_BY);
      const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY);
      ring_release(R, rc, tx, ring_dep(h[0], c, t));
      if (upd_x) h[0] = upd(h[0], t, c, sm.sE[2][ty + 1][tx], sEz);
    }
    {  // Hxz
      ring_wait(R, rc);
      h[1] = RD(0, BOX_BY);
      const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY), s = RD(3, BOX_BY);
      ring_release(R, rc, tx, ring_dep(h[1], s, c, t));
      if (upd_x) h[1] = upd_src(h[1], t, c, nEy, sEy, s);
    }
    {  // Hyx
      ring_wait(R, rc);
      h[2] = RD(0, BOX_BX);
      const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX);
      ring_release(R, rc, tx, ring_dep(h[2], c, t));
      if (upd_y) h[2] = upd(h[2], t, c, sm.sE[2][ty][tx + 1], sEz);
    }
    {  // Hyz
      ring_wait(R, rc);
      h[3] = RD(0, BOX_BX);
      const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX), s = RD(3, BOX_BX);
      ring_release(R, rc, tx, ring_dep(h[3], s, c, t));
      if (upd_y) h[3] = upd_src(h[3], t, c, nEx, sEx, s);
    }
    {  // Hzx
      ring_wait(R, rc);
      h[4] = RD(0, BOX_B);
      const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
      ring_release(R, rc, tx, ring_dep(h[4], c, t));
      if (upd_z) h[4] = upd(h[4], t, c, sm.sE[1][ty][tx + 1], sEy);
    }
    {  // Hzy
      ring_wait(R, rc);
      h[5] = RD(0, BOX_B);
      const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
      ring_release(R, rc, tx, ring_dep(h[5], c, t));
      if (upd_z) h[5] = upd(h[5], t, c, sm.sE[0][ty + 1][tx], sEx);
    }
    if (own) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        A.fo[HXY + k][i] = h[k];
        mark<COUNT>(A, HXY + k, i);
      }
    }
    const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
    if (own || ring_x || ring_y) {
      sm.sH[0][ty][tx] = sHx;
      sm.sH[1][ty][tx] = sHy;
      sm.sH[2][ty][tx] = sHz;
    }
    named_sync(1, NCOMP);

    // (c) E half-step at plane z for own cells
    {  // Exy, Eyx
      ring_wait(R, rc);
      const double2 t0 = RD(0, BOX_C), c0 = RD(1, BOX_C), t1 = RD(2, BOX_C), c1 = RD(3, BOX_C);
      ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
      if (own) {
        A.fo[EXY][i] = upd(e[EXY], t0, c0, sm.sH[2][ty - 1][tx], sHz);
        A.fo[EYX][i] = upd(e[EYX], t1, c1, sm.sH[2][ty][tx - 1], sHz);
        mark<COUNT>(A, EXY, i);
        mark<COUNT>(A, EYX, i);
      }
    }
    {  // Exz
      ring_wait(R, rc);
      const double2 t = RD(0, BOX_C), c = RD(1, BOX_C), s = RD(2, BOX_C);
      ring_release(R, rc, tx, ring_dep(s, c, t));
      if (own) {
        A.fo[EXZ][i] = upd_src(e[EXZ], t, c, pHy, sHy, s);
        mark<COUNT>(A, EXZ, i);
      }
    }
    {  // Eyz
      ring_wait(R, rc);
      const double2 t = RD(0, BOX_C), c = RD(1, BOX_C), s = RD(2, BOX_C);
      ring_release(R, rc, tx, ring_dep(s, c, t));
      if (own) {
        A.fo[EYZ][i] = upd_src(e[EYZ], t, c, pHx, sHx, s);
        mark<COUNT>(A, EYZ, i);
      }
    }
    {  // Ezx, Ezy
      ring_wait(R, rc);
      const double2 t0 = RD(0, BOX_C), c0 = RD(1, BOX_C), t1 = RD(2, BOX_C), c1 = RD(3, BOX_C);
      ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
      if (own) {
        A.fo[EZX][i] = upd(e[EZX], t0, c0, sm.sH[1][ty][tx - 1], sHy);
        A.fo[EZY][i] = upd(e[EZY], t1, c1, sm.sH[0][ty - 1][tx], sHx);
        mark<COUNT>(A, EZX, i);
        mark<COUNT>(A, EZY, i);
      }
    }
    pHx = sHx;
    pHy = sHy;
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = en[k];
  }
#undef RD
}

}  // namespace thiim_gpu
