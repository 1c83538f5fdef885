// thiim_fused_tma.cuh -- engine FUSED, bulk-async staged variant (default).
//
// Same numerics and tiling as k_fused (thiim_fused.cuh): one z-streamed H->E
// sweep per step, ping-pong fields, a 32 x BY thread tile = the (32-2) x (BY-2)
// own cells plus a one-cell ring whose -x/-y side recomputes the H sums the
// tile needs.  What changes is how operands reach the SM:
//
//   * one PRODUCER warp streams every array-plane the tile needs -- 40 per
//     z-plane: E_old(z+1) x6, then per H component F,t,c(,src), then per E
//     component t,c(,src) -- as 1-D bulk copies (cp.async.bulk, the TMA
//     engine; SASS UBLKCP), one 512-B row segment per lane, into a ring of
//     NBUF shared-memory slots of 32 x BY x 16 B, each guarded by a
//     full/empty mbarrier pair;
//   * BY CONSUMER warps take the slots in the same order, each thread reading
//     its own cell's element (LDS.128, conflict-free), and release them.
//
// Up to NBUF x 8 KB of loads are in flight per SM independent of register
// pressure, so the sweep is no longer latency-bound on the per-plane
// barriers.  Algorithmic traffic: 40 reads + 12 writes x 16 B = 832 B/LUP.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"

namespace thiim_gpu {

// Array-plane order the producer streams and the consumers take, per z-plane,
// as array slots of the slab allocation (the 4th coordinate of its tensor
// map).  Entries 0..5 are read at plane z+1, the rest at plane z.
struct SeqSlots {
  int s[40];
};

// field_slot(k): slot of input field k; coeff_slot(a): slot of array a (12..39)
template <class FS, class CS>
inline SeqSlots make_seq(FS field_slot, CS coeff_slot) {
  SeqSlots S;
  int k = 0;
  for (int c = EXY; c <= EZY; ++c) S.s[k++] = field_slot(c);
  const int hsrc[6] = {-1, SRC_HXZ, -1, SRC_HYZ, -1, -1};
  for (int c = HXY; c <= HZY; ++c) {
    S.s[k++] = field_slot(c);
    S.s[k++] = coeff_slot(12 + c);
    S.s[k++] = coeff_slot(24 + c);
    if (hsrc[c - HXY] >= 0) S.s[k++] = coeff_slot(36 + hsrc[c - HXY]);
  }
  const int esrc[6] = {-1, SRC_EXZ, -1, SRC_EYZ, -1, -1};
  for (int c = EXY; c <= EZY; ++c) {
    S.s[k++] = coeff_slot(12 + c);
    S.s[k++] = coeff_slot(24 + c);
    if (esrc[c] >= 0) S.s[k++] = coeff_slot(36 + esrc[c]);
  }
  return S;
}

template <int BY, int NBUF>
struct TmaSmem {
  double2 buf[NBUF][BY][32];
  double2 sE[3][BY][32];
  double2 sH[3][BY][32];
  uint64_t full[NBUF];
  uint64_t empty[NBUF];
};

template <int BY, int NBUF>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_fused_tma(Grid g, Arrays A, const __grid_constant__ CUtensorMap tmap, SeqSlots S, int zc) {
  constexpr int BX = 32, TX = BX - 2, TY = BY - 2, NCOMP = 32 * BY;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TmaSmem<BY, NBUF>& sm = *reinterpret_cast<TmaSmem<BY, NBUF>*>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int xb = blockIdx.x * TX - 1, yb = blockIdx.y * TY - 1;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const long long px = g.px, pxy = g.pxy;

  if (tx == 0 && ty == 0) {
    for (int k = 0; k < NBUF; ++k) {
      mbar_init(&sm.full[k], 1);
      mbar_init(&sm.empty[k], BY);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (ty == BY) {
    // ---------------- producer warp: one elected lane issues one TMA box
    // (32 cells x BY rows = BY*512 B) per array-plane
    if (tx == 0) {
      tma_prefetch_desc(&tmap);
      int slot = 0;
      uint32_t phase = 0;
      const int c0 = 2 * (xb + 1), c1 = yb + 1;  // x in doubles, padded y
      for (int z = z0; z < z1; ++z) {
#pragma unroll 1
        for (int s = 0; s < 40; ++s) {
          mbar_wait(&sm.empty[slot], phase ^ 1);
          mbar_arrive_expect_tx(&sm.full[slot], BY * BX * 16);
          tma_load_4d(&sm.buf[slot][0][0], &tmap, c0, c1, z + 1 + (s < 6 ? 1 : 0), S.s[s],
                      &sm.full[slot]);
          if (++slot == NBUF) {
            slot = 0;
            phase ^= 1;
          }
        }
      }
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
  const bool upd_x = own || (ring_y && y >= 0);               // Hxy, Hxz
  const bool upd_y = own || (ring_x && x >= 0);               // Hyx, Hyz
  const bool upd_z = own || (ring_x && x >= 0) || (ring_y && y >= 0);  // Hzx, Hzy
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  long long i = g.idx(xs, ys, z0);

  // prologue: E_old(z0) splits; H_new sums at z0-1 for own cells (direct loads)
  double2 e[6];
  if (inpad) {
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = __ldg(A.f[k] + i);
  }
  double2 pHx = make_double2(0.0, 0.0), pHy = make_double2(0.0, 0.0);
  {
    const long long im = i - pxy;
    if (z0 == 0) {
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

  int slot = 0;
  uint32_t phase = 0;
  auto take = [&]() -> double2 {
    mbar_wait(&sm.full[slot], phase);
    const double2 v = sm.buf[slot][ty][tx];
    __syncwarp();
    if (tx == 0) mbar_arrive(&sm.empty[slot]);
    if (++slot == NBUF) {
      slot = 0;
      phase ^= 1;
    }
    return v;
  };

  for (int z = z0; z < z1; ++z, i += pxy) {
    // (a) E_old(z+1) splits (carried to the next plane); E sums at z to smem
    double2 en[6];
#pragma unroll
    for (int k = 0; k < 6; ++k) en[k] = take();
    if (inpad) {
      sm.sE[0][ty][tx] = csum(e[EXY], e[EXZ]);
      sm.sE[1][ty][tx] = csum(e[EYX], e[EYZ]);
      sm.sE[2][ty][tx] = csum(e[EZX], e[EZY]);
    }
    named_sync(1, NCOMP);

    // (b) H half-step at plane z (own cells: all six; ring: the four needed)
    const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
    const double2 nEx = csum(en[EXY], en[EXZ]), nEy = csum(en[EYX], en[EYZ]);
    double2 hxy = take();
    {
      const double2 t = take(), c = take();
      if (upd_x) hxy = upd(hxy, t, c, sm.sE[2][ty + 1][tx], sEz);
    }
    double2 hxz = take();
    {
      const double2 t = take(), c = take(), s = take();
      if (upd_x) hxz = upd_src(hxz, t, c, nEy, sEy, s);
    }
    double2 hyx = take();
    {
      const double2 t = take(), c = take();
      if (upd_y) hyx = upd(hyx, t, c, sm.sE[2][ty][tx + 1], sEz);
    }
    double2 hyz = take();
    {
      const double2 t = take(), c = take(), s = take();
      if (upd_y) hyz = upd_src(hyz, t, c, nEx, sEx, s);
    }
    double2 hzx = take();
    {
      const double2 t = take(), c = take();
      if (upd_z) hzx = upd(hzx, t, c, sm.sE[1][ty][tx + 1], sEy);
    }
    double2 hzy = take();
    {
      const double2 t = take(), c = take();
      if (upd_z) hzy = upd(hzy, t, c, sm.sE[0][ty + 1][tx], sEx);
    }
    if (own) {
      A.fo[HXY][i] = hxy;
      A.fo[HXZ][i] = hxz;
      A.fo[HYX][i] = hyx;
      A.fo[HYZ][i] = hyz;
      A.fo[HZX][i] = hzx;
      A.fo[HZY][i] = hzy;
    }
    if (own || ring_x || ring_y) {
      sm.sH[0][ty][tx] = csum(hxy, hxz);
      sm.sH[1][ty][tx] = csum(hyx, hyz);
      sm.sH[2][ty][tx] = csum(hzx, hzy);
    }
    named_sync(1, NCOMP);

    // (c) E half-step at plane z (own cells)
    const double2 sHx = sm.sH[0][ty][tx], sHy = sm.sH[1][ty][tx], sHz = sm.sH[2][ty][tx];
    {
      const double2 t = take(), c = take();
      if (own) A.fo[EXY][i] = upd(e[EXY], t, c, sm.sH[2][ty - 1][tx], sHz);
    }
    {
      const double2 t = take(), c = take(), s = take();
      if (own) A.fo[EXZ][i] = upd_src(e[EXZ], t, c, pHy, sHy, s);
    }
    {
      const double2 t = take(), c = take();
      if (own) A.fo[EYX][i] = upd(e[EYX], t, c, sm.sH[2][ty][tx - 1], sHz);
    }
    {
      const double2 t = take(), c = take(), s = take();
      if (own) A.fo[EYZ][i] = upd_src(e[EYZ], t, c, pHx, sHx, s);
    }
    {
      const double2 t = take(), c = take();
      if (own) A.fo[EZX][i] = upd(e[EZX], t, c, sm.sH[1][ty][tx - 1], sHy);
    }
    {
      const double2 t = take(), c = take();
      if (own) A.fo[EZY][i] = upd(e[EZY], t, c, sm.sH[0][ty - 1][tx], sHx);
    }
    pHx = sHx;
    pHy = sHy;
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = en[k];
  }
}

}  // namespace thiim_gpu
