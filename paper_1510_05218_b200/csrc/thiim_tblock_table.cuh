// thiim_tblock_table.cuh -- engine TBLOCK with compressed coefficients
// (THIIM_COEFF_TABLE): two THIIM steps per HBM pass over a piecewise-constant
// medium (BASELINE config 3's layered stack).
//
// k_tblock_tm's two-level wavefront (level 1 at plane q on the tile grown by
// one ring, level 2 at plane q-1 on the 28 x (BY-4) output tile, the level-1 ->
// level-2 hand-off of E^1 / H^1 in each thread's TMEM lane) combined with
// k_fused_table's coefficient source: a uint8 material id per cell and the
// [n_mat][28] table in shared memory.  Level 2 therefore streams nothing from
// HBM at all -- its coefficients are table rows selected by the material id
// level 1 loaded one iteration earlier -- and the only TMA traffic is level
// 1's 12 field boxes per plane: (12 x 16 read + 12 x 16 written + 1) / 2
// = 192.5 B/LUP.  Arithmetic is operation for operation that of the other
// engines on the same coefficient values, so results are bitwise equal.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_fused_table.cuh"
#include "thiim_producer.cuh"
#include "thiim_ring.cuh"
#include "thiim_tblock.cuh"
#include "thiim_tmem.cuh"

namespace thiim_gpu {

template <int BY, int NG>
struct TbTableSmem {
  Ring<BY, NG> ring;
  double2 sE[3][BY][32];
  double2 sH[3][BY][32];
  double2 tab[kMaxMaterials][28];
  uint32_t tmem_base;
};

template <int BY, int NG, bool COUNT = false, bool DEEP = false>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_tblock_table(Grid g, Arrays A, TableGrid T, const __grid_constant__ TmaMaps maps,
                   const __grid_constant__ PeerOut po, int fb, int zc, int tiles_x, TileOrder ord) {
  constexpr int NCOMP = 32 * BY;
  constexpr int TX2 = 28, TY2 = BY - 4;
  constexpr int LAG = 1;
  static_assert(BY <= 16, "TMEM carry layout: at most 4 consumer warps per lane quadrant");
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TbTableSmem<BY, NG>& sm = *reinterpret_cast<TbTableSmem<BY, NG>*>(smem_raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  // (tile, z-chunk) of this CTA: rounds of <= one CTA per SM, tiles in
  // vertical bands (TileOrder, thiim_tblock.cuh); the chunk by repeated
  // subtraction keeps z0 on the uniform datapath
  int chunk = 0, it = ord.item0 + (int)blockIdx.x;
  while (it >= ord.nbt) {
    it -= ord.nbt;
    ++chunk;
  }
  const int b = band_tile(it, tiles_x, ord);
  const int xb = (b % tiles_x) * TX2 - 2, yb = (b / tiles_x) * TY2 - 2;
  const int z0 = chunk * zc;
  const int z1 = min(DEEP ? po.st1 : g.nz, z0 + zc);  // deep slabs: level 2 stops at st1 - 1
  const long long pxy = g.pxy;
  const int qs = max(z0 - 1, 0);
  const int q1 = min(z1, g.nz - 1);
  const int qe = z1 + LAG - 1;

  for (int k = ty * 32 + tx; k < T.n_mat * 28; k += 32 * (BY + 1))
    sm.tab[k / 28][k % 28] = T.table[k];
  if (ty == 0) tm_alloc<512>(&sm.tmem_base);
  if (tx == 0 && ty == 0) {
    ring_init(sm.ring, BY);
    fence_mbar_init();
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();

  if (ty == BY) {  // ---------------- producer warp (one elected lane)
    if (tx == 0) {
#pragma unroll
      for (int b = 0; b < NBOX; ++b) tma_prefetch_desc(&maps.m[b]);
      const uint64_t drop = policy_evict_first();
      RingProducer<BY, NG> P(sm.ring, maps, xb, yb);
      for (int q = qs; q <= q1; ++q) produce_table_plane_ct(P, fb, q, drop);
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const uint32_t tcar = tm_warp_addr(sm.tmem_base, ty, 128 * (ty >> 2));
  const uint32_t tnext = tcar + 96;
  const int x = xb + tx, y = yb + ty;
  const bool inpad = (x >= -1) && (x <= g.nx) && (y >= -1) && (y <= g.ny);
  const bool interior = (x >= 0) && (x < g.nx) && (y >= 0) && (y < g.ny);
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  const bool own1 = tx >= 1 && tx <= 30 && ty >= 1 && ty <= BY - 2;
  const bool rx1 = (tx == 0) && (ty >= 1) && (ty <= BY - 2);
  const bool ry1 = (ty == 0) && (tx >= 1) && (tx <= 30);
  const bool own2 = tx >= 2 && tx <= 29 && ty >= 2 && ty <= BY - 3;
  const bool rx2 = (tx == 1) && (ty >= 2) && (ty <= BY - 3);
  const bool ry2 = (ty == 1) && (tx >= 2) && (tx <= 29);
  const bool upd1_x = (own1 || ry1) && interior;
  const bool upd1_y = (own1 || rx1) && interior;
  const bool upd1_z = (own1 || rx1 || ry1) && interior;
  const bool upd2_x = (own2 || ry2) && interior;
  const bool upd2_y = (own2 || rx2) && interior;
  const bool upd2_z = (own2 || rx2 || ry2) && interior;
  // material id of this thread's cell at interior plane z (padded plane z+1)
  // (raw byte loaded one plane ahead, range-checked where it is used, so no
  // compare right after the load exposes its latency)
  auto mat_raw = [&](int z) -> int {
    if (!inpad) return 0;
    return __ldg(T.mat + (long long)(z + 1) * T.mplane + (long long)(ys + 1) * T.mp + (xs + 1));
  };
  auto mat_ok = [&](int m) -> int { return m < T.n_mat ? m : 0; };
  auto mat_at = [&](int z) -> int { return mat_ok(mat_raw(z)); };

  auto& R = sm.ring;
  RingCursor rc = ring_cursor(R);
#define RD(k, b) ring_read<true>(R, rc, k, b, tx, ty)

  // ---- level-1 prologue: E_old splits at qs (to TMEM), H^1 sums at qs-1
  double2 pH1x = make_double2(0.0, 0.0), pH1y = make_double2(0.0, 0.0);
  {
    double2 e[6];
    const long long i1 = g.idx(xs, ys, qs);
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = inpad ? __ldg(A.f[k] + i1) : make_double2(0.0, 0.0);
    tm_st6(tnext, e);
    const long long im = i1 - pxy;
    if (qs == 0 && !g.halo_lo) {
      if (own1 && inpad) {  // ghost plane below the grid: H never updated
        pH1x = csum(__ldg(A.f[HXY] + im), __ldg(A.f[HXZ] + im));
        pH1y = csum(__ldg(A.f[HYX] + im), __ldg(A.f[HYZ] + im));
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
      if (own1 && inpad) {
        if (interior) {
          const double2* C = sm.tab[mat_at(qs - 1)];
          const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
          const double2 nEx = csum(e[EXY], e[EXZ]), nEy = csum(e[EYX], e[EYZ]);
          const double2 hxy = upd(__ldg(A.f[HXY] + im), C[HXY], C[12 + HXY], sm.sE[2][ty + 1][tx], sEz);
          const double2 hxz =
              upd_src(__ldg(A.f[HXZ] + im), C[HXZ], C[12 + HXZ], nEy, sEy, C[24 + SRC_HXZ]);
          const double2 hyx = upd(__ldg(A.f[HYX] + im), C[HYX], C[12 + HYX], sm.sE[2][ty][tx + 1], sEz);
          const double2 hyz =
              upd_src(__ldg(A.f[HYZ] + im), C[HYZ], C[12 + HYZ], nEx, sEx, C[24 + SRC_HYZ]);
          pH1x = csum(hxy, hxz);
          pH1y = csum(hyx, hyz);
        } else {
          pH1x = csum(__ldg(A.f[HXY] + im), __ldg(A.f[HXZ] + im));
          pH1y = csum(__ldg(A.f[HYX] + im), __ldg(A.f[HYZ] + im));
        }
      }
      named_sync(1, NCOMP);
    }
  }
  double2 pH2x = make_double2(0.0, 0.0), pH2y = make_double2(0.0, 0.0);
  double2 nE2x = make_double2(0.0, 0.0), nE2y = make_double2(0.0, 0.0);
  const uint64_t first = policy_evict_first();
  int mid1_next = mat_raw(qs);  // level-1 material id (raw), one plane ahead
  int mid_last = 0;            // material id of the last level-1 plane

  for (int q = qs; q <= qe; ++q) {
    // level 2 sweeps plane q-1: the plane level 1 swept in the previous iteration
    const int mid2 = mid_last;
    // ================= level 1 at plane q (step n) -> TMEM slot q&1
    if (q <= q1) {
      const int mid1 = mat_ok(mid1_next);
      mid_last = mid1;
      if (q + 1 <= q1) mid1_next = mat_raw(q + 1);
      const double2* C = sm.tab[mid1];
      const uint32_t tslot = tcar + 48 * (q & 1);
      double2 e[6];
      tm_ld6(tnext, e);  // E_old(q)
      double2 nEx, nEy;
      double2 h45[2];
      {
        double2 en[6];
        ring_wait(R, rc);
#pragma unroll
        for (int k = 0; k < 4; ++k) en[k] = RD(k, BOX_A);
        ring_release(R, rc, tx, ring_dep(en[0], en[1], en[2], en[3]));
        ring_wait(R, rc);
        en[4] = RD(0, BOX_A);
        en[5] = RD(1, BOX_A);
        h45[0] = RD(2, BOX_B);
        h45[1] = RD(3, BOX_B);
        ring_release(R, rc, tx, ring_dep(en[4], en[5], h45[0], h45[1]));
        tm_st6(tnext, en);  // E_old(q+1) for the next plane
        nEx = csum(en[EXY], en[EXZ]);
        nEy = csum(en[EYX], en[EYZ]);
      }
      // own sums from registers; neighbours read them from shared memory
      const double2 sEx = csum(e[EXY], e[EXZ]), sEy = csum(e[EYX], e[EYZ]),
                    sEz = csum(e[EZX], e[EZY]);
      if (inpad) {
        sm.sE[0][ty][tx] = sEx;
        sm.sE[1][ty][tx] = sEy;
        sm.sE[2][ty][tx] = sEz;
      }
      named_sync(1, NCOMP);
      double2 h[6];
      ring_wait(R, rc);
      h[0] = RD(0, BOX_BY);
      h[1] = RD(1, BOX_BY);
      h[2] = RD(2, BOX_BX);
      h[3] = RD(3, BOX_BX);
      ring_release(R, rc, tx, ring_dep(h[0], h[1], h[2], h[3]));
      h[4] = h45[0];
      h[5] = h45[1];
      if (upd1_x) {
        h[0] = upd(h[0], C[HXY], C[12 + HXY], sm.sE[2][ty + 1][tx], sEz);
        h[1] = upd_src(h[1], C[HXZ], C[12 + HXZ], nEy, sEy, C[24 + SRC_HXZ]);
      }
      if (upd1_y) {
        h[2] = upd(h[2], C[HYX], C[12 + HYX], sm.sE[2][ty][tx + 1], sEz);
        h[3] = upd_src(h[3], C[HYZ], C[12 + HYZ], nEx, sEx, C[24 + SRC_HYZ]);
      }
      if (upd1_z) {
        h[4] = upd(h[4], C[HZX], C[12 + HZX], sm.sE[1][ty][tx + 1], sEy);
        h[5] = upd(h[5], C[HZY], C[12 + HZY], sm.sE[0][ty + 1][tx], sEx);
      }
      const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
      if (own1 || rx1 || ry1) {
        sm.sH[0][ty][tx] = sHx;
        sm.sH[1][ty][tx] = sHy;
        sm.sH[2][ty][tx] = sHz;
      }
      tm_st6(tslot + 24, h);  // H^1(q)
      named_sync(1, NCOMP);
      if (own1 && interior) {
        e[EXY] = upd(e[EXY], C[EXY], C[12 + EXY], sm.sH[2][ty - 1][tx], sHz);
        e[EXZ] = upd_src(e[EXZ], C[EXZ], C[12 + EXZ], pH1y, sHy, C[24 + SRC_EXZ]);
        e[EYX] = upd(e[EYX], C[EYX], C[12 + EYX], sm.sH[2][ty][tx - 1], sHz);
        e[EYZ] = upd_src(e[EYZ], C[EYZ], C[12 + EYZ], pH1x, sHx, C[24 + SRC_EYZ]);
        e[EZX] = upd(e[EZX], C[EZX], C[12 + EZX], sm.sH[1][ty][tx - 1], sHy);
        e[EZY] = upd(e[EZY], C[EZY], C[12 + EZY], sm.sH[0][ty - 1][tx], sHx);
      }
      tm_st6(tslot, e);  // E^1(q) (ghost cells pass through unchanged)
      nE2x = csum(e[EXY], e[EXZ]);
      nE2y = csum(e[EYX], e[EYZ]);
      pH1x = sHx;
      pH1y = sHy;
    }

    // ================= level 2 at plane r = q-1 (step n+1) -> output set
    const int r = q - LAG;
    if (r >= z0 - 1 && r < z1) {
      const long long i = g.idx(xs, ys, r);
      // level-2 outputs: owned planes locally, boundary planes also into the
      // neighbours' halos (multi-GPU contexts, peer memory)
      const bool st_ok = r >= po.st0 && r < po.st1;
      const bool lo_ok = po.lo[0] != nullptr && r >= po.lo_r0 && r < po.lo_r1;
      const bool hi_ok = po.hi[0] != nullptr && r >= po.hi_r0 && r < po.hi_r1;
      auto put = [&](int comp, const double2 v) {
        if constexpr (!DEEP) {  // whole-z context: every plane, locally
          st_hint(A.fo[comp] + i, v, first);
          mark<COUNT>(A, comp, i);
        } else {
          if (st_ok) {
            st_hint(A.fo[comp] + i, v, first);
            mark<COUNT>(A, comp, i);
          }
          if (lo_ok) st_hint(po.lo[comp] + i + po.lo_shift, v, first);
          if (hi_ok) st_hint(po.hi[comp] + i + po.hi_shift, v, first);
        }
      };
      const bool plane_ok = r >= 0;
      const double2* C = sm.tab[mid2];
      double2 nEx = nE2x, nEy = nE2y;
      if (q > q1) {  // plane r+1 is the top ghost plane: level 1 did not run
        double2 e[6];
        tm_ld6(tnext, e);
        nEx = csum(e[EXY], e[EXZ]);
        nEy = csum(e[EYX], e[EYZ]);
      }
      double2 e1[6], h[6];
      if (plane_ok) {
        const uint32_t tslot = tcar + 48 * (r & 1);
        tm_ld6(tslot, e1);
        tm_ld6(tslot + 24, h);
      } else {  // ghost plane -1: never updated, read the input set
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          e1[k] = inpad ? __ldg(A.f[k] + i) : make_double2(0.0, 0.0);
          h[k] = inpad ? __ldg(A.f[HXY + k] + i) : make_double2(0.0, 0.0);
        }
      }
      // own sums from registers; neighbours read them from shared memory
      const double2 sEx = csum(e1[EXY], e1[EXZ]), sEy = csum(e1[EYX], e1[EYZ]),
                    sEz = csum(e1[EZX], e1[EZY]);
      if (inpad) {
        sm.sE[0][ty][tx] = sEx;
        sm.sE[1][ty][tx] = sEy;
        sm.sE[2][ty][tx] = sEz;
      }
      named_sync(1, NCOMP);
      if (upd2_x && plane_ok) {
        h[0] = upd(h[0], C[HXY], C[12 + HXY], sm.sE[2][ty + 1][tx], sEz);
        h[1] = upd_src(h[1], C[HXZ], C[12 + HXZ], nEy, sEy, C[24 + SRC_HXZ]);
      }
      if (upd2_y && plane_ok) {
        h[2] = upd(h[2], C[HYX], C[12 + HYX], sm.sE[2][ty][tx + 1], sEz);
        h[3] = upd_src(h[3], C[HYZ], C[12 + HYZ], nEx, sEx, C[24 + SRC_HYZ]);
      }
      if (upd2_z && plane_ok) {
        h[4] = upd(h[4], C[HZX], C[12 + HZX], sm.sE[1][ty][tx + 1], sEy);
        h[5] = upd(h[5], C[HZY], C[12 + HZY], sm.sE[0][ty + 1][tx], sEx);
      }
      if (r == z0 - 1) {
        // chunk prologue: only the H_new sums of the plane below the chunk
        if (own2) {
          pH2x = csum(h[0], h[1]);
          pH2y = csum(h[2], h[3]);
        }
        named_sync(1, NCOMP);  // sE reads done before the next level-1 writes
        continue;
      }
      if (own2 && interior) {
#pragma unroll
        for (int k = 0; k < 6; ++k) put(HXY + k, h[k]);
      }
      const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
      if (own2 || rx2 || ry2) {
        sm.sH[0][ty][tx] = sHx;
        sm.sH[1][ty][tx] = sHy;
        sm.sH[2][ty][tx] = sHz;
      }
      named_sync(1, NCOMP);
      if (own2 && interior) {
        put(EXY, upd(e1[EXY], C[EXY], C[12 + EXY], sm.sH[2][ty - 1][tx], sHz));
        put(EXZ, upd_src(e1[EXZ], C[EXZ], C[12 + EXZ], pH2y, sHy, C[24 + SRC_EXZ]));
        put(EYX, upd(e1[EYX], C[EYX], C[12 + EYX], sm.sH[2][ty][tx - 1], sHz));
        put(EYZ, upd_src(e1[EYZ], C[EYZ], C[12 + EYZ], pH2x, sHx, C[24 + SRC_EYZ]));
        put(EZX, upd(e1[EZX], C[EZX], C[12 + EZX], sm.sH[1][ty][tx - 1], sHy));
        put(EZY, upd(e1[EZY], C[EZY], C[12 + EZY], sm.sH[0][ty - 1][tx], sHx));
      }
      pH2x = sHx;
      pH2y = sHy;
    }
  }
#undef RD
  tm_fence_before();
  named_sync(1, NCOMP);
  tm_fence_after();
  if (ty == 0) tm_dealloc<512>(sm.tmem_base);
}

}  // namespace thiim_gpu
