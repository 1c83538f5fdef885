// thiim_tblock3.cuh -- engine TBLOCK at time-block depth 3: three THIIM steps
// per HBM pass (832 / 3 = 277 B/LUP algorithmic).
//
// The same wavefront as k_tblock_tm (thiim_tblock.cuh) one level deeper.  A
// CTA owns a 32 x BY thread tile and streams z; per iteration q it runs
//   level 1 at plane q   : the fused plane sweep (all 40 arrays from the ring),
//   level 2 at plane q-1 : coefficients from the ring (L2 hits of level 1's
//                          evict_last boxes), fields from level 1,
//   level 3 at plane q-2 : likewise from level 2; stores the output tile
//                          (32-6) x (BY-6) into the other field set.
// Level j updates E on its own cells [j, 31-j] x [j, BY-1-j] and H there plus
// on the -x/-y ring at j-1 (the dependency cone of one step grows one cell per
// side), so the output tile is 26 x (BY-6); halo cells are recomputed
// redundantly and bitwise like their owners.
//
// Hand-offs.  Everything a level reads at its own cell from the level below
// (E^{j-1}, H^{j-1} of its plane: 12 double2) was computed by the same thread
// one iteration earlier, so it lives in the thread's TMEM lane.  Depth 2 keeps
// two slots per hand-off (plane parity); depth 3 needs two hand-offs, and 2 x 2
// slots + the E_old carry (216 columns) exceed the 128 columns a warp owns when
// four consumer warps share a lane quadrant.  So each hand-off is ONE slot,
// swapped: level j reads its plane's values out of the slot and parks the
// values level j-1 just computed in the same columns (tm_swap6, two values at a
// time), before level j overwrites the registers.  TMEM per warp: stash 1
// [0,48), stash 2 [48,96), E_old carry [96,120), level 3's H sums [120,128).
//
// Chunk z-range [z0, z1): level j's full planes are [z0-(3-j), z1+(3-j)-1]
// (clamped to the grid) and one plane below them is its prologue (H sums only,
// for the E update of the first full plane); below z = 0 the prologue is the
// ghost plane, whose H values never change.  The top ghost plane's E values
// (plane nz, never updated) stand in for a level's missing z+1 plane.
//
// Whole-z contexts only (a deep-halo slab would need three halo planes): the
// multi-GPU and in-place paths run depth 2.  W = 32 (no folded remainder CTAs).
// Coefficient boxes: level 1 evict_last, level 2 evict_last (level 3 re-reads
// them one plane later), level 3 evict_first.  Memory-system ceiling of this
// access pattern (tools/depth_ceiling.cu): 13.6 / 12.9 GLUP/s at 512^2 x 256 /
// 1024^2 x 128 vs 11.1 / 11.9 for depth 2.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_producer.cuh"
#include "thiim_ring.cuh"
#include "thiim_tblock.cuh"
#include "thiim_tmem.cuh"

namespace thiim_gpu {

// Cells level J touches (thread coordinates, W = 32), evaluated where used
// (compares against constants) rather than held in registers.
template <int BY, int J>
struct LevelMask {
  int tx, ty;
  bool interior;
  __device__ bool own() const { return tx >= J && tx <= 31 - J && ty >= J && ty <= BY - 1 - J; }
  __device__ bool rx() const { return tx == J - 1 && ty >= J && ty <= BY - 1 - J; }
  __device__ bool ry() const { return ty == J - 1 && tx >= J && tx <= 31 - J; }
  __device__ bool upd_x() const { return (own() || ry()) && interior; }  // Hxy, Hxz
  __device__ bool upd_y() const { return (own() || rx()) && interior; }  // Hyx, Hyz
  __device__ bool upd_z() const { return (own() || rx() || ry()) && interior; }  // Hzx, Hzy
  __device__ bool hsum() const { return own() || rx() || ry(); }  // H sums for the E phase
  __device__ bool ue() const { return own() && interior; }         // E components
};

// One coefficient-only level (j >= 2) at plane r.  In: e/h = E^{j-1}(r),
// H^{j-1}(r) at the thread's cell; nEx/nEy = E^{j-1}(r+1) sums; pHx/pHy =
// H^j(r-1) sums.  Reads its 8 coefficient groups (boxes BH / BE) from the ring.
// mode 0 (ghost plane) / 1 (prologue): H^j only (no update on the ghost plane),
// pH <- its sums, the E groups are consumed unread.  mode 2: H^j and E^j; out:
// e/h = E^j(r), H^j(r) (cells a level does not update pass their input
// through), pH <- H^j(r) sums.
template <int BY, int NG, int J, int BH, int BE>
__device__ __forceinline__ void coef_level(TmSmem<BY, NG>& sm, RingCursor& rc, int tx, int ty,
                                           const LevelMask<BY, J>& m, bool inpad, int mode, double2* e,
                                           double2* h, double2 nEx, double2 nEy, double2& pHx,
                                           double2& pHy) {
  constexpr int NCOMP = 32 * BY;
  auto& R = sm.ring;
  if (ty < J - 1 || ty > BY - J) {
    // a warp row outside the level's region (H rows [J-1, BY-1-J], their +y
    // neighbours' E sums up to BY-J): nothing to compute or exchange -- keep
    // the ring and barrier protocol only (its values pass through unchanged
    // and are never read at this level or the next)
    named_sync(1, NCOMP);
    for (int k = 0; k < 4; ++k) {
      ring_wait(R, rc);
      ring_release(R, rc, tx, ring_dep());
    }
    if (mode == 2) named_sync(1, NCOMP);
    for (int k = 0; k < 4; ++k) {
      ring_wait(R, rc);
      ring_release(R, rc, tx, ring_dep());
    }
    if (mode != 2) named_sync(1, NCOMP);
    return;
  }
#define RD(k, b) ring_read<false>(R, rc, k, b, tx, ty)
  const double2 sEx = csum(e[EXY], e[EXZ]), sEy = csum(e[EYX], e[EYZ]), sEz = csum(e[EZX], e[EZY]);
  if (inpad) {
    sm.sE[0][ty][tx] = sEx;
    sm.sE[1][ty][tx] = sEy;
    sm.sE[2][ty][tx] = sEz;
  }
  named_sync(1, NCOMP);
  const bool ok = mode != 0;
  const bool ux = m.upd_x() && ok, uy = m.upd_y() && ok, uz = m.upd_z() && ok;
  {  // Hxy, Hyx
    ring_wait(R, rc);
    const double2 t0 = RD(0, BH), c0 = RD(1, BH), t1 = RD(2, BH), c1 = RD(3, BH);
    ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
    if (ux) h[0] = upd(h[0], t0, c0, sm.sE[2][ty + 1][tx], sEz);
    if (uy) h[2] = upd(h[2], t1, c1, sm.sE[2][ty][tx + 1], sEz);
  }
  {  // Hxz
    ring_wait(R, rc);
    const double2 t = RD(0, BH), c = RD(1, BH), s = RD(2, BH);
    ring_release(R, rc, tx, ring_dep(s, c, t));
    if (ux) h[1] = upd_src(h[1], t, c, nEy, sEy, s);
  }
  {  // Hyz
    ring_wait(R, rc);
    const double2 t = RD(0, BH), c = RD(1, BH), s = RD(2, BH);
    ring_release(R, rc, tx, ring_dep(s, c, t));
    if (uy) h[3] = upd_src(h[3], t, c, nEx, sEx, s);
  }
  {  // Hzx, Hzy
    ring_wait(R, rc);
    const double2 t0 = RD(0, BH), c0 = RD(1, BH), t1 = RD(2, BH), c1 = RD(3, BH);
    ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
    if (uz) h[4] = upd(h[4], t0, c0, sm.sE[1][ty][tx + 1], sEy);
    if (uz) h[5] = upd(h[5], t1, c1, sm.sE[0][ty + 1][tx], sEx);
  }
  const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]);
  if (mode != 2) {
    // prologue / ghost plane: only the H sums the next plane's E update needs
    pHx = sHx;
    pHy = sHy;
    for (int k = 0; k < 4; ++k) {  // E-coefficient groups, unused here
      ring_wait(R, rc);
      ring_release(R, rc, tx, ring_dep());
    }
    named_sync(1, NCOMP);  // sE reads done before the next level's writes
    return;
  }
  const double2 sHz = csum(h[4], h[5]);
  if (m.hsum()) {
    sm.sH[0][ty][tx] = sHx;
    sm.sH[1][ty][tx] = sHy;
    sm.sH[2][ty][tx] = sHz;
  }
  named_sync(1, NCOMP);
  const bool ue = m.ue();
  {  // Exy, Eyx
    ring_wait(R, rc);
    const double2 t0 = RD(0, BE), c0 = RD(1, BE), t1 = RD(2, BE), c1 = RD(3, BE);
    ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
    if (ue) {
      e[EXY] = upd(e[EXY], t0, c0, sm.sH[2][ty - 1][tx], sHz);
      e[EYX] = upd(e[EYX], t1, c1, sm.sH[2][ty][tx - 1], sHz);
    }
  }
  {  // Exz
    ring_wait(R, rc);
    const double2 t = RD(0, BE), c = RD(1, BE), s = RD(2, BE);
    ring_release(R, rc, tx, ring_dep(s, c, t));
    if (ue) e[EXZ] = upd_src(e[EXZ], t, c, pHy, sHy, s);
  }
  {  // Eyz
    ring_wait(R, rc);
    const double2 t = RD(0, BE), c = RD(1, BE), s = RD(2, BE);
    ring_release(R, rc, tx, ring_dep(s, c, t));
    if (ue) e[EYZ] = upd_src(e[EYZ], t, c, pHx, sHx, s);
  }
  {  // Ezx, Ezy
    ring_wait(R, rc);
    const double2 t0 = RD(0, BE), c0 = RD(1, BE), t1 = RD(2, BE), c1 = RD(3, BE);
    ring_release(R, rc, tx, ring_dep(c1, t1, c0, t0));
    if (ue) {
      e[EZX] = upd(e[EZX], t0, c0, sm.sH[1][ty][tx - 1], sHy);
      e[EZY] = upd(e[EZY], t1, c1, sm.sH[0][ty - 1][tx], sHx);
    }
  }
  pHx = sHx;
  pHy = sHy;
#undef RD
}

// Ex, Ey sums of the top ghost plane's E values (never updated), parked by
// level 1 as the E_old carry of its last plane (EXY, EXZ, EYX, EYZ: columns 0-15)
__device__ __forceinline__ void top_ghost_sums(uint32_t tnext, double2& nEx, double2& nEy) {
  double2 t[2];
  tm_ld2(tnext, t);
  nEx = csum(t[0], t[1]);
  tm_ld2(tnext + 8, t);
  nEy = csum(t[0], t[1]);
}

template <int BY, int NG, bool COUNT>
__device__ __forceinline__ void tblock3_body(TmSmem<BY, NG>& sm, const Grid& g, const Arrays& A,
                                             const TmaMaps& maps, int fb, int cb, int zc, int chunk,
                                             int xb, int yb) {
  constexpr int NCOMP = 32 * BY;
  static_assert(BY <= 16, "TMEM carry layout: at most 4 consumer warps per lane quadrant");
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int z0 = chunk * zc;
  const int z1 = min(g.nz, z0 + zc);
  const long long pxy = g.pxy;
  // level ranges (see the header): full planes [lo_j, hi_j], prologue p_j = lo_j - 1
  const int lo1 = max(z0 - 2, 0), hi1 = min(z1 + 1, g.nz - 1);
  const int p2 = max(z0 - 2, -1), hi2 = min(z1, g.nz - 1);
  const int p3 = max(z0 - 1, -1), hi3 = z1 - 1;
  const int qs = lo1, qe = hi3 + 2;

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
      for (int b = 0; b < NBOX; ++b) tma_prefetch_desc(&maps.m[b]);
      // fields are read once (evict_first); coefficients stay in L2 (evict_last)
      // until level 3 re-reads them two planes later (evict_first)
      const uint64_t first = policy_evict_first(), last = policy_evict_last();
      RingProducer<BY, NG> P(sm.ring, maps, xb, yb);
      for (int q = qs; q <= qe; ++q) {
        if (q <= hi1) produce_plane_ct<true>(P, fb, cb, q, first, last);
        const int r2 = q - 1, r3 = q - 2;
        if (r2 >= p2 && r2 <= hi2) produce_levelj_coef_ct<BOX_H2, BOX_E2>(P, cb, r2, last);
        if (r3 >= p3 && r3 <= hi3) produce_levelj_coef_ct<BOX_H3, BOX_E3>(P, cb, r3, first);
      }
    }
    return;
  }

  // -------------------------------------------------------------- consumers
  const uint32_t tcar = tm_warp_addr(sm.tmem_base, ty, 128 * (ty >> 2));
  const uint32_t ts1 = tcar, ts2 = tcar + 48, tnext = tcar + 96, tph3 = tcar + 120;
  const int x = xb + tx, y = yb + ty;
  const bool inpad = (x >= -1) && (x <= g.nx) && (y >= -1) && (y <= g.ny);
  const bool interior = (x >= 0) && (x < g.nx) && (y >= 0) && (y < g.ny);
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  const LevelMask<BY, 1> m1{tx, ty, interior};
  const LevelMask<BY, 2> m2{tx, ty, interior};
  const LevelMask<BY, 3> m3{tx, ty, interior};

  auto& R = sm.ring;
  RingCursor rc = ring_cursor(R);
#define RD(k, b) ring_read<false>(R, rc, k, b, tx, ty)

  // ---- level-1 prologue: E_old splits at qs (to TMEM), H^1 sums at qs-1
  double2 pH1x = make_double2(0.0, 0.0), pH1y = make_double2(0.0, 0.0);
  {
    double2 e[6];
    const long long i1 = g.idx(xs, ys, qs);
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = inpad ? __ldg(A.f[k] + i1) : make_double2(0.0, 0.0);
    tm_st6(tnext, e);
    const long long im = i1 - pxy;
    if (qs == 0) {
      if (m1.own() && inpad) {  // ghost plane below the grid: H never updated
        pH1x = csum(__ldg(A.f[HXY] + im), __ldg(A.f[HXZ] + im));
        pH1y = csum(__ldg(A.f[HYX] + im), __ldg(A.f[HYZ] + im));
      }
    } else {
      if (inpad) {
        double2 mm[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) mm[k] = __ldg(A.f[k] + im);
        sm.sE[0][ty][tx] = csum(mm[EXY], mm[EXZ]);
        sm.sE[1][ty][tx] = csum(mm[EYX], mm[EYZ]);
        sm.sE[2][ty][tx] = csum(mm[EZX], mm[EZY]);
      }
      named_sync(1, NCOMP);
      if (m1.own() && inpad) {
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
  double2 pH2x = make_double2(0.0, 0.0), pH2y = pH2x;
  {  // level 3's carried H sums live in TMEM [120,128) between its planes
    const double2 z2[2] = {pH2x, pH2x};
    tm_st2(tph3, z2);
  }
  double2 nE2x = pH2x, nE2y = pH2x, nE3x = pH2x, nE3y = pH2x;
  const uint64_t first = policy_evict_first();

  for (int q = qs; q <= qe; ++q) {
    const int r2 = q - 1, r3 = q - 2;
    const bool run1 = q <= hi1;
    const bool run2 = r2 >= p2 && r2 <= hi2;
    const bool run3 = r3 >= p3 && r3 <= hi3;
    double2 e[6], h[6];  // the values the level just run produced at its cell
    // ================= level 1 at plane q -> e, h = E^1(q), H^1(q)
    if (run1) {
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
      const double2 sEx = csum(e[EXY], e[EXZ]), sEy = csum(e[EYX], e[EYZ]),
                    sEz = csum(e[EZX], e[EZY]);
      if (inpad) {
        sm.sE[0][ty][tx] = sEx;
        sm.sE[1][ty][tx] = sEy;
        sm.sE[2][ty][tx] = sEz;
      }
      named_sync(1, NCOMP);
      {
        ring_wait(R, rc);
        h[0] = RD(0, BOX_BY);
        const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY);
        ring_release(R, rc, tx, ring_dep(h[0], c, t));
        if (m1.upd_x()) h[0] = upd(h[0], t, c, sm.sE[2][ty + 1][tx], sEz);
      }
      {
        ring_wait(R, rc);
        h[1] = RD(0, BOX_BY);
        const double2 t = RD(1, BOX_BY), c = RD(2, BOX_BY), s = RD(3, BOX_BY);
        ring_release(R, rc, tx, ring_dep(h[1], s, c, t));
        if (m1.upd_x()) h[1] = upd_src(h[1], t, c, nEy, sEy, s);
      }
      {
        ring_wait(R, rc);
        h[2] = RD(0, BOX_BX);
        const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX);
        ring_release(R, rc, tx, ring_dep(h[2], c, t));
        if (m1.upd_y()) h[2] = upd(h[2], t, c, sm.sE[2][ty][tx + 1], sEz);
      }
      {
        ring_wait(R, rc);
        h[3] = RD(0, BOX_BX);
        const double2 t = RD(1, BOX_BX), c = RD(2, BOX_BX), s = RD(3, BOX_BX);
        ring_release(R, rc, tx, ring_dep(h[3], s, c, t));
        if (m1.upd_y()) h[3] = upd_src(h[3], t, c, nEx, sEx, s);
      }
      {
        ring_wait(R, rc);
        h[4] = RD(0, BOX_B);
        const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
        ring_release(R, rc, tx, ring_dep(h[4], c, t));
        if (m1.upd_z()) h[4] = upd(h[4], t, c, sm.sE[1][ty][tx + 1], sEy);
      }
      {
        ring_wait(R, rc);
        h[5] = RD(0, BOX_B);
        const double2 t = RD(1, BOX_B), c = RD(2, BOX_B);
        ring_release(R, rc, tx, ring_dep(h[5], c, t));
        if (m1.upd_z()) h[5] = upd(h[5], t, c, sm.sE[0][ty + 1][tx], sEx);
      }
      const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
      if (m1.hsum()) {
        sm.sH[0][ty][tx] = sHx;
        sm.sH[1][ty][tx] = sHy;
        sm.sH[2][ty][tx] = sHz;
      }
      named_sync(1, NCOMP);
      const bool ue = m1.ue();
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
      nE2x = csum(e[EXY], e[EXZ]);
      nE2y = csum(e[EYX], e[EYZ]);
      pH1x = sHx;
      pH1y = sHy;
    }

    // ================= level 2 at plane r2 = q-1 -> e, h = E^2(r2), H^2(r2)
    const bool full2 = run2 && r2 > p2;
    if (run2) {
      if (r2 < 0) {  // ghost plane below the grid: never updated, the input set
        if (run1) {
          tm_st6(ts1, e);
          tm_st6(ts1 + 24, h);
        }
        const long long i = g.idx(xs, ys, r2);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          e[k] = inpad ? __ldg(A.f[k] + i) : make_double2(0.0, 0.0);
          h[k] = inpad ? __ldg(A.f[HXY + k] + i) : make_double2(0.0, 0.0);
        }
      } else if (run1) {  // E^1/H^1(r2) out of stash 1, E^1/H^1(q) in
        tm_xchg6(ts1, e);
        tm_xchg6(ts1 + 24, h);
      } else {
        tm_ld6(ts1, e);
        tm_ld6(ts1 + 24, h);
      }
      double2 nEx = nE2x, nEy = nE2y;
      if (!run1) top_ghost_sums(tnext, nEx, nEy);  // plane r2+1 is the top ghost plane
      coef_level<BY, NG, 2, BOX_H2, BOX_E2>(sm, rc, tx, ty, m2, inpad, r2 < 0 ? 0 : full2 ? 2 : 1, e,
                                            h, nEx, nEy, pH2x, pH2y);
      if (full2) {
        nE3x = csum(e[EXY], e[EXZ]);
        nE3y = csum(e[EYX], e[EYZ]);
      }
    } else if (run1) {
      tm_st6(ts1, e);  // level 2 has not started yet: park E^1/H^1(q)
      tm_st6(ts1 + 24, h);
    }

    // ================= level 3 at plane r3 = q-2 -> output set
    if (run3) {
      if (r3 < 0) {  // ghost plane below the grid
        if (full2) {
          tm_st6(ts2, e);
          tm_st6(ts2 + 24, h);
        }
        const long long i = g.idx(xs, ys, r3);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          e[k] = inpad ? __ldg(A.f[k] + i) : make_double2(0.0, 0.0);
          h[k] = inpad ? __ldg(A.f[HXY + k] + i) : make_double2(0.0, 0.0);
        }
      } else if (full2) {  // E^2/H^2(r3) out of stash 2, E^2/H^2(r2) in
        tm_xchg6(ts2, e);
        tm_xchg6(ts2 + 24, h);
      } else {
        tm_ld6(ts2, e);
        tm_ld6(ts2 + 24, h);
      }
      double2 nEx = nE3x, nEy = nE3y;
      if (!full2) top_ghost_sums(tnext, nEx, nEy);  // plane r3+1 is the top ghost plane
      const bool full3 = r3 > p3;
      double2 pH3[2];
      tm_ld2(tph3, pH3);
      coef_level<BY, NG, 3, BOX_H3, BOX_E3>(sm, rc, tx, ty, m3, inpad, r3 < 0 ? 0 : full3 ? 2 : 1, e,
                                            h, nEx, nEy, pH3[0], pH3[1]);
      tm_st2(tph3, pH3);
      if (full3 && m3.ue()) {
        const long long i = g.idx(xs, ys, r3);
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          st_hint(A.fo[HXY + k] + i, h[k], first);
          mark<COUNT>(A, HXY + k, i);
        }
#pragma unroll
        for (int k = 0; k < 6; ++k) {
          st_hint(A.fo[k] + i, e[k], first);
          mark<COUNT>(A, k, i);
        }
      }
    } else if (full2) {
      tm_st6(ts2, e);  // level 3 has not started yet: park E^2/H^2(r2)
      tm_st6(ts2 + 24, h);
    }
  }
#undef RD
  // release TMEM once every consumer warp is done with it
  tm_fence_before();
  named_sync(1, NCOMP);
  tm_fence_after();
  if (ty == 0) tm_dealloc<512>(sm.tmem_base);
}

template <int BY, int NG, bool COUNT = false>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_tblock3_tm(Grid g, Arrays A, const __grid_constant__ TmaMaps maps, int fb, int cb, int zc,
                 int tiles_x, TileOrder ord) {
  constexpr int TX3 = 26, TY3 = BY - 6;
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
  const int b = band_tile(it, tiles_x, ord);
  tblock3_body<BY, NG, COUNT>(sm, g, A, maps, fb, cb, zc, chunk, (b % tiles_x) * TX3 - 3,
                              (b / tiles_x) * TY3 - 3);
}

}  // namespace thiim_gpu
