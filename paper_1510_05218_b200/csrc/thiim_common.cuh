// thiim_common.cuh -- primitives shared by every THIIM sweep kernel.
//
// * The per-cell update (reference kernels.cpp:43-51) with explicit
//   round-to-nearest intrinsics on the device, so no multiply-add can ever be
//   contracted whatever the compiler flags: bitwise identical to the reference
//   built without FMA (its default x86-64 build).
// * The padded grid layout (reference grid.hpp:12-48).
// * The counter-based synthetic problem generator, host and device.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#if defined(__CUDA_ARCH__)
#define THIIM_HD __host__ __device__ __forceinline__
#else
#define THIIM_HD inline
#endif

namespace thiim_gpu {

// ---- exact FP helpers: device uses _rn intrinsics (never fused); the host
// side is compiled with -ffp-contract=off.
THIIM_HD double fmul(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
THIIM_HD double fadd(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
THIIM_HD double fsub(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}

// Physical-component sum A+B of the two splits one component differentiates
// (components.hpp:55-66).  IEEE addition is commutative, so forming the sum
// once per cell and sharing it between its two consumers is bitwise safe.
THIIM_HD double2 csum(double2 a, double2 b) {
  return make_double2(fadd(a.x, b.x), fadd(a.y, b.y));
}

// F_new = t*F + c*(S[j] - S[i]) (+ src), exact order of kernels.cpp:43-51:
//   dr=(a_j+b_j)-(a_i+b_i); tr=t.re*f.re-t.im*f.im; ti=t.re*f.im+t.im*f.re;
//   cr=c.re*dr-c.im*di;     ci=c.re*di+c.im*dr;     f=(tr+cr)(+src)
THIIM_HD double2 upd(double2 f, double2 t, double2 c, double2 sj, double2 si) {
  const double dr = fsub(sj.x, si.x);
  const double di = fsub(sj.y, si.y);
  const double tr = fsub(fmul(t.x, f.x), fmul(t.y, f.y));
  const double ti = fadd(fmul(t.x, f.y), fmul(t.y, f.x));
  const double cr = fsub(fmul(c.x, dr), fmul(c.y, di));
  const double ci = fadd(fmul(c.x, di), fmul(c.y, dr));
  return make_double2(fadd(tr, cr), fadd(ti, ci));
}
THIIM_HD double2 upd_src(double2 f, double2 t, double2 c, double2 sj, double2 si, double2 s) {
  const double2 r = upd(f, t, c, sj, si);
  return make_double2(fadd(r.x, s.x), fadd(r.y, s.y));
}

// ---- component ids (components.hpp:17-30) and array slots
enum : int { EXY = 0, EXZ, EYX, EYZ, EZX, EZY, HXY, HXZ, HYX, HYZ, HZX, HZY };
// source_index (components.hpp:89-97)
enum : int { SRC_EXZ = 0, SRC_EYZ = 1, SRC_HXZ = 2, SRC_HYZ = 3 };

// Padded layout of one slab (grid.hpp:34-43): index (z+1)*pxy + (y+1)*px + (x+1).
struct Grid {
  int nx, ny, nz;  // interior extents of this slab
  long long px, pxy;
  // 1 when the plane below local z = 0 holds a neighbour slab's interior
  // plane (a halo copy) rather than the global ghost plane: the fused sweep
  // then recomputes H_new there instead of reading the never-updated ghost.
  int halo_lo;
  THIIM_HD long long idx(int x, int y, int z) const {
    return (long long)(z + 1) * pxy + (long long)(y + 1) * px + (long long)(x + 1);
  }
};

// Device pointers of one slab.  f: fields read this sweep; fo: fields written
// (== f for the in-place split engine; the other ping-pong set for fused).
struct Arrays {
  double2* f[12];
  double2* fo[12];
  const double2* t[12];
  const double2* c[12];
  const double2* src[4];
  unsigned* cnt = nullptr;  // sanitizer: per (component, padded cell) store counts
  long long cstride = 0;
};

// Where a TBLOCK pass stores its level-2 outputs (the interior local plane r of
// a slab): locally for r in [st0, st1) -- a deep slab's owned planes -- and, in a
// multi-GPU context, also straight into the neighbour slabs' halo planes over
// NVLink / NVSwitch peer memory (lo / hi: the neighbour's output field set,
// element shift my index -> its index), which replaces the halo exchange step.
struct PeerOut {
  double2* lo[12];  // lower neighbour (null: none)
  double2* hi[12];  // upper neighbour
  long long lo_shift, hi_shift;
  int lo_r0, lo_r1, hi_r0, hi_r1;  // my interior planes sent down / up
  int st0, st1;                    // my interior planes stored locally
};

// Sanitizer hook at every output store of the default kernels (their COUNT
// instances only): counts how often (component, cell) is written in a pass;
// k_coverage then demands exactly once per interior cell, never on a ghost.
template <bool COUNT>
__device__ __forceinline__ void mark(const Arrays& A, int comp, long long i) {
  if constexpr (COUNT) atomicAdd(A.cnt + (long long)comp * A.cstride + i, 1u);
}

// ---- synthetic problem generator
THIIM_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
THIIM_HD uint64_t gen_key(uint64_t seed, int array_id) {
  return splitmix64(splitmix64(seed) ^ ((uint64_t)(array_id + 1) * 0x9E3779B97F4A7C15ull));
}
THIIM_HD uint64_t gen_bits(uint64_t key, uint64_t counter, int draw) {
  return splitmix64(key + (counter << 8) + (uint64_t)draw);
}
THIIM_HD double gen_u(uint64_t key, uint64_t counter, int draw) {
  return fmul((double)(gen_bits(key, counter, draw) >> 11), 0x1.0p-53);
}
// field value: re, im ~ U[-1, 1)
THIIM_HD double2 gen_field(uint64_t key, uint64_t counter) {
  return make_double2(fsub(fmul(2.0, gen_u(key, counter, 0)), 1.0),
                      fsub(fmul(2.0, gen_u(key, counter, 1)), 1.0));
}
// coefficient value: uniform in the disk |z| <= 0.45 by rejection
THIIM_HD double2 gen_disk(uint64_t key, uint64_t counter) {
  const double r = 0.45;
  const double r2 = fmul(r, r);
  for (int k = 0; k < 64; ++k) {
    const double re = fmul(r, fsub(fmul(2.0, gen_u(key, counter, 2 * k)), 1.0));
    const double im = fmul(r, fsub(fmul(2.0, gen_u(key, counter, 2 * k + 1)), 1.0));
    if (fadd(fmul(re, re), fmul(im, im)) <= r2) return make_double2(re, im);
  }
  return make_double2(0.0, 0.0);
}
// config 3 layer id of interior cell (x,y,z) of a grid with nz interior planes
THIIM_HD int gen_layer(uint64_t seed, int nx, int nz, int x, int y, int z) {
  int layer = 0;
  for (int k = 1; k <= 5; ++k) {
    const uint64_t key = gen_key(seed, 64 + k);
    const int h = (int)((gen_bits(key, (uint64_t)y * (uint64_t)nx + (uint64_t)x, 0) >> 11) % 17ull) - 8;
    if (z >= k * nz / 6 + h) ++layer;
  }
  return layer;
}

}  // namespace thiim_gpu
