// thiim_producer.cuh -- compile-time producer sequences for the TMA ring.
//
// The producer is a single lane issuing ~40 (fused) or ~68 (TBLOCK) TMA boxes
// per plane.  Interpreting a runtime sequence (GroupSeq in param space: one
// LDC per element, box geometry by branch, R2UR of every operand) costs ~100+
// dependent cycles per box, which starved the TBLOCK consumers (ncu: 51% of
// warp samples on full-barrier waits while the producer almost never waited
// for an empty slot).  Here the sequence is straight-line code: box shapes,
// byte counts and L2 policies are template constants, only the slot bases
// (which field set is current) and the tile / plane coordinates are runtime.
//
// The group order and contents equal seq_plane / seq_level2_coef, which the
// consumer code reads in the same order.
#pragma once

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_ring.cuh"

namespace thiim_gpu {

// W < 32: a folded CTA -- its boxes (BoxGeom<BY, W>, `maps` built for W) span
// all 32/W segments' rows, one TMA per array as for a full tile.
template <int BY, int NG, int W = 32>
struct RingProducer {
  using Gm = BoxGeom<BY, W>;
  static_assert(32 % W == 0, "segment width must divide 32");
  Ring<BY, NG>& R;
  const TmaMaps& maps;   // field arrays
  const TmaMaps& cmaps;  // coefficient arrays (the same maps unless the field
                         // arrays have their own plane stride: TBLOCK in place)
  int xb, yb;  // interior coordinates of thread (0,0) (of segment 0)
  int gi = 0;
  uint32_t ph = 0;

  __device__ RingProducer(Ring<BY, NG>& r, const TmaMaps& m, int xb_, int yb_)
      : R(r), maps(m), cmaps(m), xb(xb_), yb(yb_) {}
  __device__ RingProducer(Ring<BY, NG>& r, const TmaMaps& m, const TmaMaps& cm, int xb_, int yb_)
      : R(r), maps(m), cmaps(cm), xb(xb_), yb(yb_) {}

  template <int BYTES>
  __device__ __forceinline__ void begin() {
    mbar_wait(&R.empty[gi], ph ^ 1);
    mbar_arrive_expect_tx(&R.full[gi], (uint32_t)BYTES);
  }
  // a group of N boxes of kind B
  template <int B, int N>
  __device__ __forceinline__ void begin_group() {
    static_assert(Gm::w(B) * Gm::h(B) <= 32 * BY, "box exceeds a ring box slot");
    begin<N * Gm::bytes(B)>();
  }
  __device__ __forceinline__ void end() {
    if (++gi == NG) {
      gi = 0;
      ph ^= 1;
    }
  }
  // box k of the current group: array `slot` at padded plane `pz`
  template <int B>
  __device__ __forceinline__ void box(int k, int slot, int pz) {
    tma_load_4d(&R.buf[gi][k][0], &maps.m[B], 2 * (xb + 1 + Gm::x0(B)), yb + 1 + Gm::y0(B), pz, slot,
                &R.full[gi]);
  }
  template <int B>
  __device__ __forceinline__ void box(int k, int slot, int pz, uint64_t pol) {
    tma_load_4d_hint(&R.buf[gi][k][0], &maps.m[B], 2 * (xb + 1 + Gm::x0(B)), yb + 1 + Gm::y0(B), pz,
                     slot, &R.full[gi], pol);
  }
  // a coefficient array's box (cmaps)
  template <int B>
  __device__ __forceinline__ void cbox(int k, int slot, int pz) {
    tma_load_4d(&R.buf[gi][k][0], &cmaps.m[B], 2 * (xb + 1 + Gm::x0(B)), yb + 1 + Gm::y0(B), pz, slot,
                &R.full[gi]);
  }
  template <int B>
  __device__ __forceinline__ void cbox(int k, int slot, int pz, uint64_t pol) {
    tma_load_4d_hint(&R.buf[gi][k][0], &cmaps.m[B], 2 * (xb + 1 + Gm::x0(B)), yb + 1 + Gm::y0(B), pz,
                     slot, &R.full[gi], pol);
  }
};

// Slot bases: field component c of the current set = fb + c; coefficient
// array a (12..39 in the reference's 40-array order) = cb + (a - 12).
//
// One fused / level-1 plane z (seq_plane): E_old(z+1) x6, then per H component
// F, t, c (, src), then the E coefficients.  HINT: per-class L2 policies
// (fields, coefficients) or none.
template <bool HINT, class PR>
__device__ __forceinline__ void produce_plane_ct(PR& P, int fb, int cb, int z, uint64_t pf = 0,
                                                 uint64_t pc = 0) {
  const int p0 = z + 1, p1 = z + 2;
#define BOXF(B, k, slot, pz) \
  do {                        \
    if (HINT)                 \
      P.template box<B>(k, slot, pz, pf); \
    else                      \
      P.template box<B>(k, slot, pz);     \
  } while (0)
#define BOXC(B, k, slot, pz) \
  do {                        \
    if (HINT)                 \
      P.template cbox<B>(k, slot, pz, pc); \
    else                      \
      P.template cbox<B>(k, slot, pz);     \
  } while (0)
  P.template begin_group<BOX_A, 4>();
  BOXF(BOX_A, 0, fb + EXY, p1);
  BOXF(BOX_A, 1, fb + EXZ, p1);
  BOXF(BOX_A, 2, fb + EYX, p1);
  BOXF(BOX_A, 3, fb + EYZ, p1);
  P.end();
  P.template begin_group<BOX_A, 2>();
  BOXF(BOX_A, 0, fb + EZX, p1);
  BOXF(BOX_A, 1, fb + EZY, p1);
  P.end();
  P.template begin_group<BOX_BY, 3>();  // Hxy
  BOXF(BOX_BY, 0, fb + HXY, p0);
  BOXC(BOX_BY, 1, cb + HXY, p0);
  BOXC(BOX_BY, 2, cb + 12 + HXY, p0);
  P.end();
  P.template begin_group<BOX_BY, 4>();  // Hxz
  BOXF(BOX_BY, 0, fb + HXZ, p0);
  BOXC(BOX_BY, 1, cb + HXZ, p0);
  BOXC(BOX_BY, 2, cb + 12 + HXZ, p0);
  BOXC(BOX_BY, 3, cb + 24 + SRC_HXZ, p0);
  P.end();
  P.template begin_group<BOX_BX, 3>();  // Hyx
  BOXF(BOX_BX, 0, fb + HYX, p0);
  BOXC(BOX_BX, 1, cb + HYX, p0);
  BOXC(BOX_BX, 2, cb + 12 + HYX, p0);
  P.end();
  P.template begin_group<BOX_BX, 4>();  // Hyz
  BOXF(BOX_BX, 0, fb + HYZ, p0);
  BOXC(BOX_BX, 1, cb + HYZ, p0);
  BOXC(BOX_BX, 2, cb + 12 + HYZ, p0);
  BOXC(BOX_BX, 3, cb + 24 + SRC_HYZ, p0);
  P.end();
  P.template begin_group<BOX_B, 3>();  // Hzx
  BOXF(BOX_B, 0, fb + HZX, p0);
  BOXC(BOX_B, 1, cb + HZX, p0);
  BOXC(BOX_B, 2, cb + 12 + HZX, p0);
  P.end();
  P.template begin_group<BOX_B, 3>();  // Hzy
  BOXF(BOX_B, 0, fb + HZY, p0);
  BOXC(BOX_B, 1, cb + HZY, p0);
  BOXC(BOX_B, 2, cb + 12 + HZY, p0);
  P.end();
  P.template begin_group<BOX_C, 4>();  // Exy, Eyx
  BOXC(BOX_C, 0, cb + EXY, p0);
  BOXC(BOX_C, 1, cb + 12 + EXY, p0);
  BOXC(BOX_C, 2, cb + EYX, p0);
  BOXC(BOX_C, 3, cb + 12 + EYX, p0);
  P.end();
  P.template begin_group<BOX_C, 3>();  // Exz
  BOXC(BOX_C, 0, cb + EXZ, p0);
  BOXC(BOX_C, 1, cb + 12 + EXZ, p0);
  BOXC(BOX_C, 2, cb + 24 + SRC_EXZ, p0);
  P.end();
  P.template begin_group<BOX_C, 3>();  // Eyz
  BOXC(BOX_C, 0, cb + EYZ, p0);
  BOXC(BOX_C, 1, cb + 12 + EYZ, p0);
  BOXC(BOX_C, 2, cb + 24 + SRC_EYZ, p0);
  P.end();
  P.template begin_group<BOX_C, 4>();  // Ezx, Ezy
  BOXC(BOX_C, 0, cb + EZX, p0);
  BOXC(BOX_C, 1, cb + 12 + EZX, p0);
  BOXC(BOX_C, 2, cb + EZY, p0);
  BOXC(BOX_C, 3, cb + 12 + EZY, p0);
  P.end();
#undef BOXF
#undef BOXC
}

// The 28 coefficient planes of a deeper level at plane r, policy `pol`, in 8
// groups (the consumer's read order), boxed to that level's regions: BH / BE =
// BOX_H2 / BOX_E2 (level 2) or BOX_H3 / BOX_E3 (level 3).
template <int BH, int BE, class PR>
__device__ __forceinline__ void produce_levelj_coef_ct(PR& P, int cb, int r, uint64_t pol) {
  const int p0 = r + 1;
  P.template begin_group<BH, 4>();  // Hxy t c, Hyx t c
  P.template cbox<BH>(0, cb + HXY, p0, pol);
  P.template cbox<BH>(1, cb + 12 + HXY, p0, pol);
  P.template cbox<BH>(2, cb + HYX, p0, pol);
  P.template cbox<BH>(3, cb + 12 + HYX, p0, pol);
  P.end();
  P.template begin_group<BH, 3>();  // Hxz t c src
  P.template cbox<BH>(0, cb + HXZ, p0, pol);
  P.template cbox<BH>(1, cb + 12 + HXZ, p0, pol);
  P.template cbox<BH>(2, cb + 24 + SRC_HXZ, p0, pol);
  P.end();
  P.template begin_group<BH, 3>();  // Hyz t c src
  P.template cbox<BH>(0, cb + HYZ, p0, pol);
  P.template cbox<BH>(1, cb + 12 + HYZ, p0, pol);
  P.template cbox<BH>(2, cb + 24 + SRC_HYZ, p0, pol);
  P.end();
  P.template begin_group<BH, 4>();  // Hzx t c, Hzy t c
  P.template cbox<BH>(0, cb + HZX, p0, pol);
  P.template cbox<BH>(1, cb + 12 + HZX, p0, pol);
  P.template cbox<BH>(2, cb + HZY, p0, pol);
  P.template cbox<BH>(3, cb + 12 + HZY, p0, pol);
  P.end();
  P.template begin_group<BE, 4>();  // Exy t c, Eyx t c
  P.template cbox<BE>(0, cb + EXY, p0, pol);
  P.template cbox<BE>(1, cb + 12 + EXY, p0, pol);
  P.template cbox<BE>(2, cb + EYX, p0, pol);
  P.template cbox<BE>(3, cb + 12 + EYX, p0, pol);
  P.end();
  P.template begin_group<BE, 3>();  // Exz t c src
  P.template cbox<BE>(0, cb + EXZ, p0, pol);
  P.template cbox<BE>(1, cb + 12 + EXZ, p0, pol);
  P.template cbox<BE>(2, cb + 24 + SRC_EXZ, p0, pol);
  P.end();
  P.template begin_group<BE, 3>();  // Eyz t c src
  P.template cbox<BE>(0, cb + EYZ, p0, pol);
  P.template cbox<BE>(1, cb + 12 + EYZ, p0, pol);
  P.template cbox<BE>(2, cb + 24 + SRC_EYZ, p0, pol);
  P.end();
  P.template begin_group<BE, 4>();  // Ezx t c, Ezy t c
  P.template cbox<BE>(0, cb + EZX, p0, pol);
  P.template cbox<BE>(1, cb + 12 + EZX, p0, pol);
  P.template cbox<BE>(2, cb + EZY, p0, pol);
  P.template cbox<BE>(3, cb + 12 + EZY, p0, pol);
  P.end();
}

template <class PR>
__device__ __forceinline__ void produce_level2_coef_ct(PR& P, int cb, int r, uint64_t pol) {
  produce_levelj_coef_ct<BOX_H2, BOX_E2>(P, cb, r, pol);
}

// Table-layout plane z (seq_table's 12 arrays, in three full groups instead of
// its four): E_old(z+1) x6, H_old(z) x6 -- the only HBM-streamed arrays when
// coefficients come from the material table.
template <int BY, int NG>
__device__ __forceinline__ void produce_table_plane_ct(RingProducer<BY, NG>& P, int fb, int z,
                                                       uint64_t pol) {
  using Gm = BoxGeom<BY>;
  constexpr int SA = Gm::bytes(BOX_A), SB = Gm::bytes(BOX_B), SBX = Gm::bytes(BOX_BX),
                SBY = Gm::bytes(BOX_BY);
  const int p0 = z + 1, p1 = z + 2;
  P.template begin<4 * SA>();
  P.template box<BOX_A>(0, fb + EXY, p1, pol);
  P.template box<BOX_A>(1, fb + EXZ, p1, pol);
  P.template box<BOX_A>(2, fb + EYX, p1, pol);
  P.template box<BOX_A>(3, fb + EYZ, p1, pol);
  P.end();
  // three full groups per plane: the z-components of E_old ride with Hzx/Hzy
  P.template begin<2 * SA + 2 * SB>();
  P.template box<BOX_A>(0, fb + EZX, p1, pol);
  P.template box<BOX_A>(1, fb + EZY, p1, pol);
  P.template box<BOX_B>(2, fb + HZX, p0, pol);
  P.template box<BOX_B>(3, fb + HZY, p0, pol);
  P.end();
  P.template begin<2 * SBY + 2 * SBX>();
  P.template box<BOX_BY>(0, fb + HXY, p0, pol);
  P.template box<BOX_BY>(1, fb + HXZ, p0, pol);
  P.template box<BOX_BX>(2, fb + HYX, p0, pol);
  P.template box<BOX_BX>(3, fb + HYZ, p0, pol);
  P.end();
}

}  // namespace thiim_gpu
