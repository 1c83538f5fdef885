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

// Array-plane order the producer streams and the consumers take, per z-plane:
// the array slot of the slab allocation (4th tensor-map coordinate) and the
// box shape.  Entries 0..5 are read at plane z+1, the rest at plane z.
//
// Box shapes (thread tile = 32 x BY cells, own cells = [1,30] x [1,BY-2]):
//   BOX_A  32 x BY     everything (E_old: own, both rings, +x/+y neighbours)
//   BOX_B  31 x (BY-1) own + ring_x + ring_y        (Hzx, Hzy operands)
//   BOX_BX 31 x (BY-2) own + ring_x (x0-1 column)   (Hyx, Hyz operands)
//   BOX_BY 30 x (BY-1) own + ring_y (y0-1 row)      (Hxy, Hxz operands)
//   BOX_C  30 x (BY-2) own only                     (E-phase coefficients)
// Fetching only what each group needs keeps the tile overlap (re-read by the
// neighbouring CTA) at ~7% instead of ~22%.
enum : int { BOX_A = 0, BOX_B = 1, BOX_BX = 2, BOX_BY = 3, BOX_C = 4, NBOX = 5 };

struct SeqSlots {
  int s[40];
  int box[40];
};

struct TmaMaps {
  CUtensorMap m[NBOX];
};

// geometry of a box kind: first thread column/row it covers, width, height
template <int BY>
struct BoxGeom {
  __host__ __device__ static constexpr int x0(int b) { return b >= BOX_BY ? 1 : 0; }
  __host__ __device__ static constexpr int y0(int b) { return (b == BOX_BX || b == BOX_C) ? 1 : 0; }
  __host__ __device__ static constexpr int w(int b) { return b == BOX_A ? 32 : b <= BOX_BX ? 31 : 30; }
  __host__ __device__ static constexpr int h(int b) {
    return b == BOX_A ? BY : (b == BOX_B || b == BOX_BY) ? BY - 1 : BY - 2;
  }
};

// field_slot(k): slot of input field k; coeff_slot(a): slot of array a (12..39)
template <class FS, class CS>
inline SeqSlots make_seq(FS field_slot, CS coeff_slot) {
  SeqSlots S;
  int k = 0;
  for (int c = EXY; c <= EZY; ++c) {
    S.box[k] = BOX_A;
    S.s[k++] = field_slot(c);
  }
  const int hsrc[6] = {-1, SRC_HXZ, -1, SRC_HYZ, -1, -1};
  const int hbox[6] = {BOX_BY, BOX_BY, BOX_BX, BOX_BX, BOX_B, BOX_B};
  for (int c = HXY; c <= HZY; ++c) {
    const int b = hbox[c - HXY];
    S.box[k] = b; S.s[k++] = field_slot(c);
    S.box[k] = b; S.s[k++] = coeff_slot(12 + c);
    S.box[k] = b; S.s[k++] = coeff_slot(24 + c);
    if (hsrc[c - HXY] >= 0) { S.box[k] = b; S.s[k++] = coeff_slot(36 + hsrc[c - HXY]); }
  }
  const int esrc[6] = {-1, SRC_EXZ, -1, SRC_EYZ, -1, -1};
  for (int c = EXY; c <= EZY; ++c) {
    S.box[k] = BOX_C; S.s[k++] = coeff_slot(12 + c);
    S.box[k] = BOX_C; S.s[k++] = coeff_slot(24 + c);
    if (esrc[c] >= 0) { S.box[k] = BOX_C; S.s[k++] = coeff_slot(36 + esrc[c]); }
  }
  return S;
}

template <int BY, int NBUF>
struct TmaSmem {
  double2 buf[NBUF][BY * 32];  // one box per slot, packed with the box's own pitch
  double2 sE[3][BY][32];
  double2 sH[3][BY][32];
  uint64_t full[NBUF];
  uint64_t empty[NBUF];
};

template <int BY, int NBUF>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_fused_tma(Grid g, Arrays A, const __grid_constant__ TmaMaps maps, SeqSlots S, int zc,
                int tiles_y, int tiles_x, int x_fastest) {
  constexpr int BX = 32, TX = BX - 2, TY = BY - 2, NCOMP = 32 * BY;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TmaSmem<BY, NBUF>& sm = *reinterpret_cast<TmaSmem<BY, NBUF>*>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  // x-tiles enumerate fastest by default: x-neighbours share the DRAM blocks
  // at their (unaligned) box edges, so running them together lets the second
  // fetch hit in L2 (measured: 5.7% excess DRAM reads vs 19% y-fastest)
  const int bty = x_fastest ? blockIdx.x / tiles_x : blockIdx.x % tiles_y;
  const int btx = x_fastest ? blockIdx.x % tiles_x : blockIdx.x / tiles_y;
  const int xb = btx * TX - 1, yb = bty * TY - 1;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const long long pxy = g.pxy;

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
#pragma unroll
      for (int b = 0; b < NBOX; ++b) tma_prefetch_desc(&maps.m[b]);
      int slot = 0;
      uint32_t phase = 0;
      using G = BoxGeom<BY>;
      for (int z = z0; z < z1; ++z) {
#pragma unroll 1
        for (int s = 0; s < 40; ++s) {
          const int b = S.box[s];
          mbar_wait(&sm.empty[slot], phase ^ 1);
          mbar_arrive_expect_tx(&sm.full[slot], (uint32_t)(G::w(b) * G::h(b) * 16));
          // x in doubles, padded y / plane coordinates
          tma_load_4d(&sm.buf[slot][0], &maps.m[b], 2 * (xb + 1 + G::x0(b)), yb + 1 + G::y0(b),
                      z + 1 + (s < 6 ? 1 : 0), S.s[s], &sm.full[slot]);
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

  int slot = 0;
  uint32_t phase = 0;
  // wait for the next slot, read this thread's element if the slot's box
  // covers it, release the slot
  auto take = [&](const int b) -> double2 {
    using G = BoxGeom<BY>;
    mbar_wait(&sm.full[slot], phase);
    const int cx = tx - G::x0(b), cy = ty - G::y0(b);
    double2 v = make_double2(0.0, 0.0);
    if (cx >= 0 && cx < G::w(b) && cy >= 0 && cy < G::h(b)) v = sm.buf[slot][cy * G::w(b) + cx];
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
    for (int k = 0; k < 6; ++k) en[k] = take(BOX_A);
    if (inpad) {
      sm.sE[0][ty][tx] = csum(e[EXY], e[EXZ]);
      sm.sE[1][ty][tx] = csum(e[EYX], e[EYZ]);
      sm.sE[2][ty][tx] = csum(e[EZX], e[EZY]);
    }
    named_sync(1, NCOMP);

    // (b) H half-step at plane z (own cells: all six; ring: the four needed)
    const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
    const double2 nEx = csum(en[EXY], en[EXZ]), nEy = csum(en[EYX], en[EYZ]);
    double2 hxy = take(BOX_BY);
    {
      const double2 t = take(BOX_BY), c = take(BOX_BY);
      if (upd_x) hxy = upd(hxy, t, c, sm.sE[2][ty + 1][tx], sEz);
    }
    double2 hxz = take(BOX_BY);
    {
      const double2 t = take(BOX_BY), c = take(BOX_BY), s = take(BOX_BY);
      if (upd_x) hxz = upd_src(hxz, t, c, nEy, sEy, s);
    }
    double2 hyx = take(BOX_BX);
    {
      const double2 t = take(BOX_BX), c = take(BOX_BX);
      if (upd_y) hyx = upd(hyx, t, c, sm.sE[2][ty][tx + 1], sEz);
    }
    double2 hyz = take(BOX_BX);
    {
      const double2 t = take(BOX_BX), c = take(BOX_BX), s = take(BOX_BX);
      if (upd_y) hyz = upd_src(hyz, t, c, nEx, sEx, s);
    }
    double2 hzx = take(BOX_B);
    {
      const double2 t = take(BOX_B), c = take(BOX_B);
      if (upd_z) hzx = upd(hzx, t, c, sm.sE[1][ty][tx + 1], sEy);
    }
    double2 hzy = take(BOX_B);
    {
      const double2 t = take(BOX_B), c = take(BOX_B);
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
      const double2 t = take(BOX_C), c = take(BOX_C);
      if (own) A.fo[EXY][i] = upd(e[EXY], t, c, sm.sH[2][ty - 1][tx], sHz);
    }
    {
      const double2 t = take(BOX_C), c = take(BOX_C), s = take(BOX_C);
      if (own) A.fo[EXZ][i] = upd_src(e[EXZ], t, c, pHy, sHy, s);
    }
    {
      const double2 t = take(BOX_C), c = take(BOX_C);
      if (own) A.fo[EYX][i] = upd(e[EYX], t, c, sm.sH[2][ty][tx - 1], sHz);
    }
    {
      const double2 t = take(BOX_C), c = take(BOX_C), s = take(BOX_C);
      if (own) A.fo[EYZ][i] = upd_src(e[EYZ], t, c, pHx, sHx, s);
    }
    {
      const double2 t = take(BOX_C), c = take(BOX_C);
      if (own) A.fo[EZX][i] = upd(e[EZX], t, c, sm.sH[1][ty][tx - 1], sHy);
    }
    {
      const double2 t = take(BOX_C), c = take(BOX_C);
      if (own) A.fo[EZY][i] = upd(e[EZY], t, c, sm.sH[0][ty - 1][tx], sHx);
    }
    pHx = sHx;
    pHy = sHy;
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = en[k];
  }
}

}  // namespace thiim_gpu
