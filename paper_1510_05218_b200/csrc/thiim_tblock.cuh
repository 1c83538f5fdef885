// thiim_tblock.cuh -- engine TBLOCK: two THIIM steps per HBM pass.
//
// The paper's idea (wavefront temporal blocking, arXiv 1510.05218 s II)
// re-derived for B200.  One CTA owns an x-y tile and streams z.  Per iteration
// q it runs
//   level 1 at plane q   (step n):   the fused plane sweep over the tile grown by
//                                    one cell per side (28 x (BY-4) output tile
//                                    + two rings in the 32 x BY thread tile);
//   level 2 at plane q-1 (step n+1): the same sweep on the output tile, which
//                                    writes the ping-pong field set.
// Halo cells are recomputed redundantly by neighbouring CTAs (bitwise
// identical); chunk starts recompute one level-1 plane and one level-2 H plane
// below.  DRAM traffic: 832 / 2 = 416 B/LUP plus tile-overlap re-fetch.
//
// k_tblock_tm: the level-1 -> level-2 hand-off (E^1 / H^1 of plane q-1,
// computed by the same thread) lives in the thread's TMEM lane; a remainder
// tile column of <= 12 grid columns runs as folded CTAs of 8- or 16-lane
// segments; deep-halo slabs of multi-GPU contexts write their neighbours' halo
// planes directly (peer stores).  See the comments at k_tblock_tm and
// DESIGN.md "Temporal blocking".  (Its predecessor -- the hand-off through an
// L2-resident scratch ring, 5.4 vs 11.0 GLUP/s at 256^3 -- and the
// pattern-only ceiling builds are recorded in DESIGN.md, not shipped.)
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_fused_tma.cuh"
#include "thiim_ring.cuh"
#include "thiim_producer.cuh"
#include "thiim_tmem.cuh"

namespace thiim_gpu {

// ---------------------------------------------------------------------------
// k_tblock_tm: the same two-level wavefront with the level-1 -> level-2
// hand-off kept on chip.  Every value level 2 reads at its own cell from level 1
// (E^1 and H^1 of plane r, 12 double2) was computed by the SAME thread one
// iteration earlier, so it never needs to leave the thread: it is parked in the
// thread's TMEM lane (double-buffered by plane parity), together with the
// E_old splits level 1 carries to the next plane.  That removes the L2 scratch
// ring (12 array-planes written and re-fetched per iteration), its ready
// barriers and the register spills of the register-carried variant; level 2's
// producer sequence shrinks to the 8 coefficient groups.
//
// TMEM columns per warp (warp w: lanes 32*(w%4).., columns 128*(w/4)..):
//   [0,48)   slot 0: E^1 (24 cols), H^1 (24 cols)   -- planes with r even
//   [48,96)  slot 1: same                            -- r odd
//   [96,120) E_old splits of the next level-1 plane
template <int BY, int NG>
struct TmSmem {
  static constexpr int SROWS = BY;
  Ring<BY, NG> ring;
  double2 sE[3][SROWS][32];
  double2 sH[3][SROWS][32];
  uint32_t tmem_base;
};

// One CTA's sweep.  W = 32: the 32 x BY thread tile of one 28 x (BY-4) output
// tile at (xb, yb0).  W < 32 (a folded remainder CTA): the warp rows split into
// 32/W segments of W lanes, each the thread tile of a (W-4) x (BY-4) output
// tile, stacked in y from yb0 -- the same sweep on narrow tiles, so a remainder
// column of <= W-4 grid columns costs 32/W times fewer CTAs than full tiles
// (256 = 9 x 28 + 4: the tenth tile column ran 24 nearly empty CTAs per chunk).
template <int BY, int NG, bool COUNT, int W, int DEEP>
__device__ __forceinline__ void tblock_tm_body(TmSmem<BY, NG>& sm, const Grid& g, const Arrays& A,
                                               const TmaMaps& maps, const TmaMaps& cmaps,
                                               const PeerOut& po, int fb, int cb, int zc, int chunk,
                                               int zlo, int zhi, int xb, int yb0) {
  constexpr int NCOMP = 32 * BY;
  constexpr int TY2 = BY - 4;
  constexpr int LAG = 1;
  static_assert(BY <= 16, "TMEM carry layout: at most 4 consumer warps per lane quadrant");
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int lx = W == 32 ? tx : tx % W, seg = W == 32 ? 0 : tx / W;
  const int yb = yb0 + seg * TY2;
  const int z0 = zlo + chunk * zc;
  const int z1 = min(zhi, z0 + zc);
  const long long pxy = g.pxy;
  const int qs = max(z0 - 1, 0);
  const int q1 = min(z1, g.nz - 1);
  const int qe = z1 + LAG - 1;

  if (ty == 0) tm_alloc<512>(&sm.tmem_base);
  if (tx == 0 && ty == 0) {
    ring_init(sm.ring, BY);
    fence_mbar_init();
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();

  if (ty == BY) {
    // ------------------------------------------------------------ producer
    if (tx == 0) {
#pragma unroll
      for (int b = 0; b < NBOX; ++b) {
        tma_prefetch_desc(&maps.m[b]);
        tma_prefetch_desc(&cmaps.m[b]);
      }
      // L2 policies: level-1 fields evict_first (read once), level-1
      // coefficients evict_last (level 2 re-reads them one plane later, their
      // last use: evict_first) -- the best of the measured policy sets
#ifndef THIIM_TB_FIELD_POL  // A/B builds only (tools/build_variant.sh): 1 = evict_normal fields
#define THIIM_TB_FIELD_POL 0
#endif
      const uint64_t pf1 = THIIM_TB_FIELD_POL ? policy_evict_normal() : policy_evict_first(),
                     pc1 = policy_evict_last(), pc2 = policy_evict_first();
      RingProducer<BY, NG, W> P(sm.ring, maps, cmaps, xb, yb0);
      for (int q = qs; q <= qe; ++q) {
        // level 1 keeps coefficients in L2 for level 2 (their last use)
        if (q <= q1) produce_plane_ct<true>(P, fb, cb, q, pf1, pc1);
        const int r = q - LAG;
        if (r >= z0 - 1 && r < z1) {
          produce_level2_coef_ct(P, cb, r, pc2);
        }
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const uint32_t tcar = tm_warp_addr(sm.tmem_base, ty, 128 * (ty >> 2));
  const uint32_t tnext = tcar + 96;
  const int x = xb + lx, y = yb + ty;
  const bool inpad = (x >= -1) && (x <= g.nx) && (y >= -1) && (y <= g.ny);
  const bool interior = (x >= 0) && (x < g.nx) && (y >= 0) && (y < g.ny);
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  // segment-relative roles (x +-1 neighbours of every thread that reads one lie
  // in its own segment)
  const bool own1 = lx >= 1 && lx <= W - 2 && ty >= 1 && ty <= BY - 2;
  const bool rx1 = (lx == 0) && (ty >= 1) && (ty <= BY - 2);
  const bool ry1 = (ty == 0) && (lx >= 1) && (lx <= W - 2);
  const bool own2 = lx >= 2 && lx <= W - 3 && ty >= 2 && ty <= BY - 3;
  const bool rx2 = (lx == 1) && (ty >= 2) && (ty <= BY - 3);
  const bool ry2 = (ty == 1) && (lx >= 2) && (lx <= W - 3);
  const bool upd1_x = (own1 || ry1) && interior;
  const bool upd1_y = (own1 || rx1) && interior;
  const bool upd1_z = (own1 || rx1 || ry1) && interior;
  const bool upd2_x = (own2 || ry2) && interior;
  const bool upd2_y = (own2 || rx2) && interior;
  const bool upd2_z = (own2 || rx2 || ry2) && interior;

  auto& R = sm.ring;
  RingCursor rc = ring_cursor(R);
#define RD(k, b) ring_read_seg<BY, W>(R, rc, k, b, lx, ty, seg)

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
          const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
          const double2 nEx = csum(e[EXY], e[EXZ]), nEy = csum(e[EYX], e[EYZ]);
          const double2 hxy = upd(__ldg(A.f[HXY] + im), __ldg(A.t[HXY] + im),
                                  __ldg(A.c[HXY] + im), sm.sE[2][ty + 1][tx], sEz);
          const double2 hxz = upd_src(__ldg(A.f[HXZ] + im), __ldg(A.t[HXZ] + im),
                                      __ldg(A.c[HXZ] + im), nEy, sEy, __ldg(A.src[SRC_HXZ] + im));
          const double2 hyx = upd(__ldg(A.f[HYX] + im), __ldg(A.t[HYX] + im),
                                  __ldg(A.c[HYX] + im), sm.sE[2][ty][tx + 1], sEz);
          const double2 hyz = upd_src(__ldg(A.f[HYZ] + im), __ldg(A.t[HYZ] + im),
                                      __ldg(A.c[HYZ] + im), nEx, sEx, __ldg(A.src[SRC_HYZ] + im));
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

  for (int q = qs; q <= qe; ++q) {
    // ================= level 1 at plane q (step n) -> TMEM slot q&1
    if (q <= q1) {
      const uint32_t tslot = tcar + 48 * (q & 1);
      double2 e[6];
      tm_ld6(tnext, e);  // E_old(q)
      double2 nEx, nEy;
      {
        double2 en[6];
        ring_wait(R, rc);
#pragma unroll
        for (int k = 0; k < 4; ++k) en[k] = RD(k, BOX_A);
        ring_release(R, rc, tx, ring_dep(en[0], en[1], en[2], en[3]));
        ring_wait(R, rc);
        en[4] = RD(0, BOX_A);
        en[5] = RD(1, BOX_A);
        ring_release(R, rc, tx, ring_dep(en[4], en[5]));
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
      {
        ring_wait(R, rc);
        h[0] = RD(0, BOX_BY);
        const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY);
        ring_release(R, rc, tx, ring_dep(h[0], c, t));
        if (upd1_x) h[0] = upd(h[0], t, c, sm.sE[2][ty + 1][tx], sEz);
      }
      {
        ring_wait(R, rc);
        h[1] = RD(0, BOX_BY);
        const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY), s = RD(3, BOX_BY);
        ring_release(R, rc, tx, ring_dep(h[1], s, c, t));
        if (upd1_x) h[1] = upd_src(h[1], t, c, nEy, sEy, s);
      }
      {
        ring_wait(R, rc);
        h[2] = RD(0, BOX_BX);
        const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX);
        ring_release(R, rc, tx, ring_dep(h[2], c, t));
        if (upd1_y) h[2] = upd(h[2], t, c, sm.sE[2][ty][tx + 1], sEz);
      }
      {
        ring_wait(R, rc);
        h[3] = RD(0, BOX_BX);
        const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX), s = RD(3, BOX_BX);
        ring_release(R, rc, tx, ring_dep(h[3], s, c, t));
        if (upd1_y) h[3] = upd_src(h[3], t, c, nEx, sEx, s);
      }
      {
        ring_wait(R, rc);
        h[4] = RD(0, BOX_B);
        const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
        ring_release(R, rc, tx, ring_dep(h[4], c, t));
        if (upd1_z) h[4] = upd(h[4], t, c, sm.sE[1][ty][tx + 1], sEy);
      }
      {
        ring_wait(R, rc);
        h[5] = RD(0, BOX_B);
        const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
        ring_release(R, rc, tx, ring_dep(h[5], c, t));
        if (upd1_z) h[5] = upd(h[5], t, c, sm.sE[0][ty + 1][tx], sEx);
      }
      const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
      if (own1 || rx1 || ry1) {
        sm.sH[0][ty][tx] = sHx;
        sm.sH[1][ty][tx] = sHy;
        sm.sH[2][ty][tx] = sHz;
      }
      tm_st6(tslot + 24, h);  // H^1(q)
      named_sync(1, NCOMP);
      const bool ue = own1 && interior;
      {
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_C), c0 = RD(1, BOX_C), t1 = RD(2, BOX_C), c1 = RD(3, BOX_C);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (ue) {
          e[EXY] = upd(e[EXY], t0, c0, sm.sH[2][ty - 1][tx], sHz);
          e[EYX] = upd(e[EYX], t1, c1, sm.sH[2][ty][tx - 1], sHz);
        }
      }
      {
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_C), c = RD(1, BOX_C), s = RD(2, BOX_C);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (ue) e[EXZ] = upd_src(e[EXZ], t, c, pH1y, sHy, s);
      }
      {
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_C), c = RD(1, BOX_C), s = RD(2, BOX_C);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (ue) e[EYZ] = upd_src(e[EYZ], t, c, pH1x, sHx, s);
      }
      {
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_C), c0 = RD(1, BOX_C), t1 = RD(2, BOX_C), c1 = RD(3, BOX_C);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (ue) {
          e[EZX] = upd(e[EZX], t0, c0, sm.sH[1][ty][tx - 1], sHy);
          e[EZY] = upd(e[EZY], t1, c1, sm.sH[0][ty - 1][tx], sHx);
        }
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
      auto put = [&](int comp, const double2 v) {
        if constexpr (DEEP == 0) {  // whole-z context: every plane, locally
          st_hint(A.fo[comp] + i, v, first);
          mark<COUNT>(A, comp, i);
        } else if constexpr (DEEP == 2) {  // view: chunks cover only [st0, st1)
          st_hint(A.fo[comp] + i, v, first);
        } else {
          if (st_ok) {
            st_hint(A.fo[comp] + i, v, first);
            mark<COUNT>(A, comp, i);
          }
          if constexpr (DEEP == 1) {  // multi-GPU slab: boundary planes into the neighbours
            const bool lo_ok = po.lo[0] != nullptr && r >= po.lo_r0 && r < po.lo_r1;
            const bool hi_ok = po.hi[0] != nullptr && r >= po.hi_r0 && r < po.hi_r1;
            if (lo_ok) st_hint(po.lo[comp] + i + po.lo_shift, v, first);
            if (hi_ok) st_hint(po.hi[comp] + i + po.hi_shift, v, first);
          }
        }
      };
      const bool plane_ok = r >= 0;
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
      const bool u2x = upd2_x && plane_ok, u2y = upd2_y && plane_ok, u2z = upd2_z && plane_ok;
      {  // Hxy, Hyx
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_H2), c0 = RD(1, BOX_H2), t1 = RD(2, BOX_H2), c1 = RD(3, BOX_H2);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (u2x) h[0] = upd(h[0], t0, c0, sm.sE[2][ty + 1][tx], sEz);
        if (u2y) h[2] = upd(h[2], t1, c1, sm.sE[2][ty][tx + 1], sEz);
      }
      {  // Hxz
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_H2), c = RD(1, BOX_H2), s = RD(2, BOX_H2);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (u2x) h[1] = upd_src(h[1], t, c, nEy, sEy, s);
      }
      {  // Hyz
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_H2), c = RD(1, BOX_H2), s = RD(2, BOX_H2);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (u2y) h[3] = upd_src(h[3], t, c, nEx, sEx, s);
      }
      {  // Hzx, Hzy
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_H2), c0 = RD(1, BOX_H2), t1 = RD(2, BOX_H2), c1 = RD(3, BOX_H2);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (u2z) h[4] = upd(h[4], t0, c0, sm.sE[1][ty][tx + 1], sEy);
        if (u2z) h[5] = upd(h[5], t1, c1, sm.sE[0][ty + 1][tx], sEx);
      }
      if (r == z0 - 1) {
        // chunk prologue: only the H_new sums of the plane below the chunk
        if (own2) {
          pH2x = csum(h[0], h[1]);
          pH2y = csum(h[2], h[3]);
        }
        for (int k = 0; k < 4; ++k) {  // E-coefficient groups, unused here
          ring_wait(R, rc);
          ring_release(R, rc, tx, ring_dep());
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
      const bool ue = own2 && interior;
      {  // Exy, Eyx
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_E2), c0 = RD(1, BOX_E2), t1 = RD(2, BOX_E2), c1 = RD(3, BOX_E2);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (ue) {
          put(EXY, upd(e1[EXY], t0, c0, sm.sH[2][ty - 1][tx], sHz));
          put(EYX, upd(e1[EYX], t1, c1, sm.sH[2][ty][tx - 1], sHz));
        }
      }
      {  // Exz
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_E2), c = RD(1, BOX_E2), s = RD(2, BOX_E2);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (ue) {
          put(EXZ, upd_src(e1[EXZ], t, c, pH2y, sHy, s));
        }
      }
      {  // Eyz
        ring_wait(R, rc);
        const double2 t = RD(0, BOX_E2), c = RD(1, BOX_E2), s = RD(2, BOX_E2);
        ring_release(R, rc, tx, ring_dep(s, c, t));
        if (ue) {
          put(EYZ, upd_src(e1[EYZ], t, c, pH2x, sHx, s));
        }
      }
      {  // Ezx, Ezy
        ring_wait(R, rc);
        const double2 t0 = RD(0, BOX_E2), c0 = RD(1, BOX_E2), t1 = RD(2, BOX_E2), c1 = RD(3, BOX_E2);
        ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
        if (ue) {
          put(EZX, upd(e1[EZX], t0, c0, sm.sH[1][ty][tx - 1], sHy));
          put(EZY, upd(e1[EZY], t1, c1, sm.sH[0][ty - 1][tx], sHx));
        }
      }
      pH2x = sHx;
      pH2y = sHy;
    }
  }
#undef RD
  // release TMEM once every consumer warp is done with it
  tm_fence_before();
  named_sync(1, NCOMP);
  tm_fence_after();
  if (ty == 0) tm_dealloc<512>(sm.tmem_base);
}


// Which (tile, z-chunk) a CTA sweeps.  Items are numbered chunk-major; within
// a chunk the n_main full tiles come in vertical BANDS of `band` tile columns
// (row by row inside a band), then the folded remainder CTAs.  A launch covers
// items [item0, item0 + gridDim.x).  The host launches a pass as ROUNDS of at
// most one CTA per SM, so every CTA of a round starts at once and a round's
// tiles form a compact band x rows block whose y- and x-neighbours stream the
// same z-planes at the same time: their overlapping box rows are fetched from
// DRAM once and hit in L2 for the neighbour.  (One launch of all items lets
// the hardware start CTAs as SMs free up: y-neighbours then run tiles_x/148 of
// a CTA lifetime apart -- tens of planes -- and re-fetch every overlap row.)
// band = tiles_x with one launch is the plain x-fastest order.
struct TileOrder {
  int item0;    // first item of this launch
  int nbt;      // items per z-chunk (n_main + folded CTAs)
  int band;     // tile columns per band (1..tiles_x)
  int tiles_y;  // tile rows
};

__device__ __forceinline__ int band_tile(int t, int tiles_x, const TileOrder& o) {
  const int full = tiles_x / o.band, per = o.band * o.tiles_y;
  int row, col;
  if (t < full * per) {
    const int bi = t / per, r = t - bi * per;
    row = r / o.band;
    col = bi * o.band + (r - row * o.band);
  } else {
    const int w = tiles_x - full * o.band, r = t - full * per;
    row = r / w;
    col = full * o.band + (r - row * w);
  }
  return row * tiles_x + col;
}

// DEEP: 0 whole-z context; 1 deep-halo slab of a multi-GPU context (owned
// planes [st0, st1) stored locally, boundary planes also into the neighbours'
// halos); 2 sub-range view of TBLOCK in place (owned planes only, no peers)
template <int BY, int NG, bool COUNT = false, int WF = 0, int DEEP = 0>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_tblock_tm(Grid g, Arrays A, const __grid_constant__ TmaMaps maps,
                const __grid_constant__ TmaMaps maps_f, const __grid_constant__ TmaMaps cmaps,
                const __grid_constant__ TmaMaps cmaps_f, const __grid_constant__ PeerOut po, int fb,
                int cb, int zc, int tiles_x, int n_main, TileOrder ord) {
  constexpr int TX2 = 28, TY2 = BY - 4;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TmSmem<BY, NG>& sm = *reinterpret_cast<TmSmem<BY, NG>*>(smem_raw);
  // chunk = item / nbt by repeated subtraction: every operand is CTA-uniform and
  // so stays on the uniform datapath (an integer division goes through MUFU on
  // the vector side, which made z0 and the loop bounds per-thread registers:
  // +1 spill and 5% slower, measured)
  int chunk = 0, it = ord.item0 + (int)blockIdx.x;
  while (it >= ord.nbt) {
    it -= ord.nbt;
    ++chunk;
  }
  const int t = it;
  // in-place views and deep-halo slabs (the latter without folded tiles) end
  // their chunks at the last owned plane st1 - 1: the plane above is
  // recomputed by level 1 as halo, but its level-2 outputs are never stored.
  // (In the folded deep-slab instances the extra bound cost registers -- 12 ->
  // 40 B of spills, -1% -- so those sweep to the top as before;
  // launch_tblock2_t matches.)
  const int zhi = DEEP == 2 || (DEEP == 1 && WF == 0) ? po.st1 : g.nz;
  const int zlo = DEEP == 2 ? po.st0 : 0;
  if (t < n_main) {  // full tiles
    const int b = band_tile(t, tiles_x, ord);
    tblock_tm_body<BY, NG, COUNT, 32, DEEP>(sm, g, A, maps, cmaps, po, fb, cb, zc, chunk, zlo, zhi,
                                            (b % tiles_x) * TX2 - 2, (b / tiles_x) * TY2 - 2);
  } else if constexpr (WF > 0) {  // folded remainder column: 32/WF y-tiles per CTA
    tblock_tm_body<BY, NG, COUNT, WF, DEEP>(sm, g, A, maps_f, cmaps_f, po, fb, cb, zc, chunk, zlo, zhi,
                                            tiles_x * TX2 - 2, (t - n_main) * (32 / WF) * TY2 - 2);
  }
}

}  // namespace thiim_gpu
