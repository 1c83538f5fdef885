// thiim_tmem.cuh -- tensor memory (TMEM) as thread-private carry storage.
//
// The sweeps keep no MMA accumulators, but TMEM (512 columns x 128 lanes x
// 32 bit per SM) is also the largest per-thread storage on the SM: warp w may
// address lanes 32*(w%4) .. 32*(w%4)+31, thread t of the warp owns lane
// 32*(w%4)+t, and 32x32b loads / stores move N consecutive 32-bit columns of
// that lane to / from N registers.  The temporally blocked sweep parks the
// values it carries between its two time levels there instead of in
// registers (which spilled) or an L2 scratch ring (which cost L2->SM bandwidth).
//
// Every access is warp-collective (.sync.aligned): call from converged,
// warp-uniform code only.  Loads and stores complete inside the same asm
// statement (wait::ld / wait::st), so the compiler never sees a register
// before its TMEM load has landed and stores may be followed by loads of the
// same columns at any later point.
#pragma once

#include <cstdint>

#include "thiim_async.cuh"

namespace thiim_gpu {

// One warp allocates `ncols` (power of two, 32..512) columns; the base address
// lands in *dst (shared memory).  Callers fence + barrier before reading it.
template <int NCOLS>
__device__ __forceinline__ void tm_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "n"(NCOLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <int NCOLS>
__device__ __forceinline__ void tm_dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(NCOLS)
               : "memory");
}

__device__ __forceinline__ void tm_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tm_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// lane base of warp w in a TMEM address (lane in bits 31:16, column in 15:0)
__device__ __forceinline__ uint32_t tm_warp_addr(uint32_t base, int warp, int col) {
  return base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)col;
}

#define THIIM_LO(v) __double2loint(v)
#define THIIM_HI(v) __double2hiint(v)

// six double2 = 24 columns of the thread's lane, starting at `a`
__device__ __forceinline__ void tm_st6(uint32_t a, const double2* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15, %16};\n\t"
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%17], {%18, %19, %20, %21, %22, %23, %24, %25};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(a),
      "r"(THIIM_LO(v[0].x)), "r"(THIIM_HI(v[0].x)), "r"(THIIM_LO(v[0].y)), "r"(THIIM_HI(v[0].y)),
      "r"(THIIM_LO(v[1].x)), "r"(THIIM_HI(v[1].x)), "r"(THIIM_LO(v[1].y)), "r"(THIIM_HI(v[1].y)),
      "r"(THIIM_LO(v[2].x)), "r"(THIIM_HI(v[2].x)), "r"(THIIM_LO(v[2].y)), "r"(THIIM_HI(v[2].y)),
      "r"(THIIM_LO(v[3].x)), "r"(THIIM_HI(v[3].x)), "r"(THIIM_LO(v[3].y)), "r"(THIIM_HI(v[3].y)),
      "r"(a + 16), "r"(THIIM_LO(v[4].x)), "r"(THIIM_HI(v[4].x)), "r"(THIIM_LO(v[4].y)),
      "r"(THIIM_HI(v[4].y)), "r"(THIIM_LO(v[5].x)), "r"(THIIM_HI(v[5].x)), "r"(THIIM_LO(v[5].y)),
      "r"(THIIM_HI(v[5].y))
      : "memory");
}

__device__ __forceinline__ void tm_ld6(uint32_t a, double2* v) {
  uint32_t r[24];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, "
      "%12, %13, %14, %15}, [%24];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%16, %17, %18, %19, %20, %21, %22, %23}, [%25];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23])
      : "r"(a), "r"(a + 16)
      : "memory");
#pragma unroll
  for (int k = 0; k < 6; ++k)
    v[k] = make_double2(__hiloint2double((int)r[4 * k + 1], (int)r[4 * k]),
                        __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]));
}

// two double2 = 8 columns
__device__ __forceinline__ void tm_st2(uint32_t a, const double2* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n\t"
      "tcgen05.wait::st.sync.aligned;" ::"r"(a),
      "r"(THIIM_LO(v[0].x)), "r"(THIIM_HI(v[0].x)), "r"(THIIM_LO(v[0].y)), "r"(THIIM_HI(v[0].y)),
      "r"(THIIM_LO(v[1].x)), "r"(THIIM_HI(v[1].x)), "r"(THIIM_LO(v[1].y)), "r"(THIIM_HI(v[1].y))
      : "memory");
}

__device__ __forceinline__ void tm_ld2(uint32_t a, double2* v) {
  uint32_t r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(a)
      : "memory");
#pragma unroll
  for (int k = 0; k < 2; ++k)
    v[k] = make_double2(__hiloint2double((int)r[4 * k + 1], (int)r[4 * k]),
                        __hiloint2double((int)r[4 * k + 3], (int)r[4 * k + 2]));
}

// Single-buffered hand-off: exchange the six values in `v` with the six
// parked at `a`, two at a time (the register peak is the six values plus one
// pair).
__device__ __forceinline__ void tm_xchg6(uint32_t a, double2* v) {
#pragma unroll
  for (int p = 0; p < 3; ++p) {
    double2 t[2];
    tm_ld2(a + 8 * p, t);
    tm_st2(a + 8 * p, v + 2 * p);
    v[2 * p] = t[0];
    v[2 * p + 1] = t[1];
  }
}

#undef THIIM_LO
#undef THIIM_HI

}  // namespace thiim_gpu
