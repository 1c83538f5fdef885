// thiim_ring.cuh -- grouped TMA ring shared by the fused and temporally
// blocked sweeps.
//
// The ring holds NG group slots of G boxes each (a box = one array-plane of the
// 32 x BY thread tile, up to BY*32 double2).  One producer lane fills a group
// with up to G TMA loads that all complete on the group's `full` mbarrier
// (expect_tx = the group's total bytes); every consumer warp waits on it once,
// reads its elements of all boxes, and releases the group once (one proxy
// fence + one arrive on `empty`).  Grouping the array-planes a component needs
// (F, t, c, src) cuts the per-box wait/fence/arrive latency chain that
// otherwise bounds the sweep (measured: 80 sequential takes per plane pair).
//
// Cross-proxy WAR: consumers read slots with generic-proxy LDS and the
// producer overwrites them with async-proxy TMA writes, so a slot may only be
// released once the warp's reads of it have LANDED -- an mbarrier arrive
// issued right after the LDS overtakes them (measured: reads of a slot raced
// its refill whenever the ring ran full).  Two ways to order them:
//   * fence.proxy.async.shared::cta before the arrive (THIIM_RING_FENCE=1):
//     lowers to MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC, which also drains every
//     other outstanding access of the thread (~15% of TBLOCK's warp samples);
//   * (default) a data dependency: the arrive's address is offset by a token
//     = AND of the loaded registers AND a zero the compiler cannot see (read
//     from shared memory at run time -- a literal 0 is folded away by ptxas,
//     which reintroduced the race), so the warp cannot issue the arrive before
//     those LDS have written back: the read is complete before the producer
//     can observe the phase and refill the slot.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"

namespace thiim_gpu {

// Box shapes within the 32 x BY thread tile (own cells = [1,30] x [1,BY-2] for a
// one-level sweep):
//   BOX_A  32 x BY     everything (E_old: own, both rings, +x/+y neighbours)
//   BOX_B  31 x (BY-1) own + ring_x + ring_y        (Hzx, Hzy operands)
//   BOX_BX 31 x (BY-2) own + ring_x (x0-1 column)   (Hyx, Hyz operands)
//   BOX_BY 30 x (BY-1) own + ring_y (y0-1 row)      (Hxy, Hxz operands)
//   BOX_C  30 x (BY-2) own only                     (E-phase coefficients)
// and for the deeper levels of the temporally blocked sweep, whose regions
// shrink by one ring per level (level j: own cells [j, 31-j] x [j, BY-1-j],
// H updated also on the -x/-y ring at j-1):
//   BOX_H2 29 x (BY-3) level-2 own + its -x/-y ring  (level-2 H coefficients)
//   BOX_E2 28 x (BY-4) level-2 own                   (level-2 E coefficients)
//   BOX_H3 27 x (BY-5), BOX_E3 26 x (BY-6)           (level 3, depth-3 sweep)
// Fetching only what each group needs keeps the tile overlap (re-read by the
// neighbouring CTA) at ~7% instead of ~22%.
enum : int {
  BOX_A = 0, BOX_B = 1, BOX_BX = 2, BOX_BY = 3, BOX_C = 4, BOX_H2 = 5, BOX_E2 = 6,
  BOX_H3 = 7, BOX_E3 = 8, NBOX = 9
};

// W: width of the thread tile the boxes belong to -- 32 (one warp row), or a
// narrower segment of a folded CTA (k_tblock_tm's remainder tiles).  A folded
// CTA's 32/W segments are consecutive y-tiles (BY - 4 rows apart), so one box
// serves all of them: 32 - W columns narrower and (32/W - 1)(BY - 4) rows taller;
// segment s reads rows s(BY - 4) + [0, h_seg).
template <int BY, int W = 32>
struct BoxGeom {
  __host__ __device__ static constexpr int x0(int b) {
    return b == BOX_E3 ? 3
           : (b == BOX_E2 || b == BOX_H3) ? 2
           : (b == BOX_BY || b == BOX_C || b == BOX_H2) ? 1
                                                        : 0;
  }
  __host__ __device__ static constexpr int y0(int b) {
    return b == BOX_E3 ? 3
           : (b == BOX_E2 || b == BOX_H3) ? 2
           : (b == BOX_BX || b == BOX_C || b == BOX_H2) ? 1
                                                        : 0;
  }
  __host__ __device__ static constexpr int w(int b) {
    return (b == BOX_A ? 32 : b <= BOX_BX ? 31 : b <= BOX_C ? 30 : 34 - b) - (32 - W);
  }
  __host__ __device__ static constexpr int h_seg(int b) {  // rows one segment reads
    return b == BOX_A                      ? BY
           : (b == BOX_B || b == BOX_BY)   ? BY - 1
           : (b == BOX_BX || b == BOX_C)   ? BY - 2
                                           : BY + 2 - b;
  }
  __host__ __device__ static constexpr int h(int b) {  // box rows
    return h_seg(b) + (32 / W - 1) * (BY - 4);
  }
  __host__ __device__ static constexpr int bytes(int b) { return w(b) * h(b) * 16; }
};

struct TmaMaps {
  CUtensorMap m[NBOX];
};

// One element of a producer sequence.
struct SeqElem {
  short slot;   // array slot of the allocation (4th map coordinate), or scratch component
  char box;     // BOX_* (main) -- scratch boxes are always the full tile
  char src;     // 0 main at plane z, 1 main at plane z+1, 2 level-1 field of plane r
  char coef;    // 1 if a coefficient array (L2 policy)
  char pad[3];
};

// A producer sequence: groups of up to 4 elements.
struct GroupSeq {
  int ngroups;
  int nelem;
  unsigned char gsize[24];
  SeqElem e[96];
};

template <int BY, int NG>
struct alignas(128) Ring {
  static constexpr int G = 4;
  double2 buf[NG][G][BY * 32];
  uint64_t full[NG];
  uint64_t empty[NG];
  uint32_t zero;  // 0, written at init: the opaque operand of the release token
};

// consumer-side cursor
struct RingCursor {
  int g = 0;
  uint32_t ph = 0;
  uint32_t zero = 0;  // loaded from Ring::zero by ring_cursor()
};

template <int BY, int NG>
__device__ __forceinline__ void ring_init(Ring<BY, NG>& r, int consumer_warps) {
  for (int k = 0; k < NG; ++k) {
    mbar_init(&r.full[k], 1);
    mbar_init(&r.empty[k], consumer_warps);
  }
  r.zero = 0;
}

// consumer cursor (after the barrier that publishes ring_init)
template <int BY, int NG>
__device__ __forceinline__ RingCursor ring_cursor(Ring<BY, NG>& r) {
  RingCursor c;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(c.zero) : "r"(smem_u32(&r.zero)));
  return c;
}

template <int BY, int NG>
__device__ __forceinline__ void ring_wait(Ring<BY, NG>& r, const RingCursor& c) {
  mbar_wait(&r.full[c.g], c.ph);
}

// element k (box kind b) of the current group, for thread (tx, ty).
// UNBOUNDED = false: threads outside box b get 0.  UNBOUNDED = true: the load
// is unconditional -- a thread outside the box reads some other element of the
// same (completed) slot, which is fine because every thread that USES a value
// of box b lies inside it by construction of the box shapes.  That drops the
// per-read register clears and predicates (CS2R zero-fills were 12.7% of the
// TBLOCK kernel's instructions) but adds shared-memory wavefronts for the
// out-of-box lanes: measured, the table kernels gain 6% (17.8 vs 16.8 GLUP/s)
// and the shared-memory-heavy TBLOCK kernel loses 7%, so it stays bounded.
// Unbounded indices stay inside the slot: the largest is 31*BY < 32*BY
// (BOX_B, bottom row) and negative ones (top row / left column of an offset
// box) are clamped to 0.
template <int BY>
__device__ __forceinline__ int ring_index(int b, int tx, int ty) {
  using Gm = BoxGeom<BY>;
  return max(0, (ty - Gm::y0(b)) * Gm::w(b) + (tx - Gm::x0(b)));
}
template <bool UNBOUNDED = false, int BY, int NG>
__device__ __forceinline__ double2 ring_read(Ring<BY, NG>& r, const RingCursor& c, int k, int b,
                                             int tx, int ty) {
  if constexpr (UNBOUNDED) {
    return r.buf[c.g][k][ring_index<BY>(b, tx, ty)];
  } else {
    using Gm = BoxGeom<BY>;
    const int cx = tx - Gm::x0(b), cy = ty - Gm::y0(b);
    if (cx >= 0 && cx < Gm::w(b) && cy >= 0 && cy < Gm::h(b)) return r.buf[c.g][k][cy * Gm::w(b) + cx];
    return make_double2(0.0, 0.0);
  }
}

#ifndef THIIM_RING_FENCE
#define THIIM_RING_FENCE 0
#endif

// AND of the low words of both halves of every value read from a group
// (ring_release masks it with the opaque zero)
template <class... T>
__device__ __forceinline__ uint32_t ring_dep(const T&... v) {
  uint32_t acc = 0xffffffffu;
  ((acc &= (uint32_t)__double2loint(v.x) & (uint32_t)__double2loint(v.y)), ...);
  return acc;
}

// release the current group; `dep` = ring_dep(every value read from it)
// bounded read for thread (lx, ty) of segment `seg` of a folded CTA (W < 32):
// the segment's window starts seg * (BY - 4) rows into the shared box
template <int BY, int W, int NG>
__device__ __forceinline__ double2 ring_read_seg(Ring<BY, NG>& r, const RingCursor& c, int k, int b,
                                                 int lx, int ty, int seg) {
  if constexpr (W == 32) {
    return ring_read(r, c, k, b, lx, ty);
  } else {
    using Gm = BoxGeom<BY, W>;
    const int cx = lx - Gm::x0(b), cy = ty - Gm::y0(b);
    if (cx >= 0 && cx < Gm::w(b) && cy >= 0 && cy < Gm::h_seg(b))
      return r.buf[c.g][k][(seg * (BY - 4) + cy) * Gm::w(b) + cx];
    return make_double2(0.0, 0.0);
  }
}

template <int BY, int NG>
__device__ __forceinline__ void ring_release(Ring<BY, NG>& r, RingCursor& c, int tx, uint32_t dep) {
#if THIIM_RING_FENCE == 1
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  dep = 0;
#elif THIIM_RING_FENCE == 2
  dep = 0;  // NO ordering: test builds only (tools/stress_ring.py must then fail)
#endif
  __syncwarp();
  if (tx == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&r.empty[c.g]) +
                                                                  (dep & c.zero))
                 : "memory");
  if (++c.g == NG) {
    c.g = 0;
    c.ph ^= 1;
  }
}

}  // namespace thiim_gpu
