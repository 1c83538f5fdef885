// thiim_split.cuh -- engine SPLIT: one H sweep then one E sweep per step,
// in place (H reads only E, E reads only H: components.hpp:55-66, so the
// in-place update of one family is race-free), z-streamed per thread.
//
// Algorithmic traffic per LUP: each sweep reads 6 own fields + 6 operand
// fields + 6 t + 6 c + 2 src and writes 6 fields: 2 x 32 x 16 B = 1024 B.
//
// Thread (x, y) of a CTA walks z over one chunk; warp = 32 consecutive x, so
// every array access is a coalesced 512-B row segment of 16-B (LDG.128)
// elements.  The x-neighbour sum comes from the next/previous lane by
// shuffle, the z-neighbour sum is carried in registers from the previous
// plane, the y-neighbour sum is re-read (L1/L2 hit).
#pragma once

#include "thiim_common.cuh"

namespace thiim_gpu {

constexpr int kSplitBX = 32;  // warp along x

__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

// H half-step on planes [z0, z1) of the chunk (reference kHOrder,
// components.hpp:80-86; shift +1, E operands).
template <int BY, bool COUNT = false>
__global__ void __launch_bounds__(kSplitBX* BY)
    k_split_h(Grid g, Arrays A, int zc) {
  const int lane = threadIdx.x;
  const int x = blockIdx.x * kSplitBX + lane;
  const int y = blockIdx.y * BY + threadIdx.y;
  if (y >= g.ny) return;  // whole warp (one row) leaves together
  const bool act = x < g.nx;
  const int xs = act ? x : g.nx - 1;  // clamp for address generation
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const bool fetch_x = (lane == kSplitBX - 1) || (x + 1 == g.nx);
  const long long px = g.px, pxy = g.pxy;

  // E sums at plane z0 (own cell)
  long long i = g.idx(xs, y, z0);
  double2 sEx = csum(ldg2(A.f[EXY] + i), ldg2(A.f[EXZ] + i));
  double2 sEy = csum(ldg2(A.f[EYX] + i), ldg2(A.f[EYZ] + i));
  double2 sEz = csum(ldg2(A.f[EZX] + i), ldg2(A.f[EZY] + i));

  for (int z = z0; z < z1; ++z, i += pxy) {
    const long long ip = i + pxy;
    // E sums at z+1 (plane nz is the ghost plane)
    const double2 nEx = csum(ldg2(A.f[EXY] + ip), ldg2(A.f[EXZ] + ip));
    const double2 nEy = csum(ldg2(A.f[EYX] + ip), ldg2(A.f[EYZ] + ip));
    const double2 nEz = csum(ldg2(A.f[EZX] + ip), ldg2(A.f[EZY] + ip));
    // E sums at y+1 (row ny is the ghost row)
    const long long iy = i + px;
    const double2 yEx = csum(ldg2(A.f[EXY] + iy), ldg2(A.f[EXZ] + iy));
    const double2 yEz = csum(ldg2(A.f[EZX] + iy), ldg2(A.f[EZY] + iy));
    // E sums at x+1: neighbour lane, or memory at the warp edge / ghost column
    double2 xEy, xEz;
    xEy.x = __shfl_down_sync(0xffffffffu, sEy.x, 1);
    xEy.y = __shfl_down_sync(0xffffffffu, sEy.y, 1);
    xEz.x = __shfl_down_sync(0xffffffffu, sEz.x, 1);
    xEz.y = __shfl_down_sync(0xffffffffu, sEz.y, 1);
    if (fetch_x) {
      xEy = csum(ldg2(A.f[EYX] + i + 1), ldg2(A.f[EYZ] + i + 1));
      xEz = csum(ldg2(A.f[EZX] + i + 1), ldg2(A.f[EZY] + i + 1));
    }
    if (act) {
      double2* F;
      F = A.f[HXY] + i; *F = upd(*F, ldg2(A.t[HXY] + i), ldg2(A.c[HXY] + i), yEz, sEz);
      F = A.f[HXZ] + i; *F = upd_src(*F, ldg2(A.t[HXZ] + i), ldg2(A.c[HXZ] + i), nEy, sEy, ldg2(A.src[SRC_HXZ] + i));
      F = A.f[HYX] + i; *F = upd(*F, ldg2(A.t[HYX] + i), ldg2(A.c[HYX] + i), xEz, sEz);
      F = A.f[HYZ] + i; *F = upd_src(*F, ldg2(A.t[HYZ] + i), ldg2(A.c[HYZ] + i), nEx, sEx, ldg2(A.src[SRC_HYZ] + i));
      F = A.f[HZX] + i; *F = upd(*F, ldg2(A.t[HZX] + i), ldg2(A.c[HZX] + i), xEy, sEy);
      F = A.f[HZY] + i; *F = upd(*F, ldg2(A.t[HZY] + i), ldg2(A.c[HZY] + i), yEx, sEx);
#pragma unroll
      for (int k = HXY; k <= HZY; ++k) mark<COUNT>(A, k, i);
    }
    sEx = nEx;
    sEy = nEy;
    sEz = nEz;
  }
}

// E half-step (reference kEOrder, components.hpp:73-79; shift -1, H operands).
template <int BY, bool COUNT = false>
__global__ void __launch_bounds__(kSplitBX* BY)
    k_split_e(Grid g, Arrays A, int zc) {
  const int lane = threadIdx.x;
  const int x = blockIdx.x * kSplitBX + lane;
  const int y = blockIdx.y * BY + threadIdx.y;
  if (y >= g.ny) return;
  const bool act = x < g.nx;
  const int xs = act ? x : g.nx - 1;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const bool fetch_x = (lane == 0);  // x-1 of lane 0 (ghost column when x == 0)
  const long long px = g.px, pxy = g.pxy;

  // H sums at plane z0-1 (ghost plane when z0 == 0); H is already new there.
  long long i = g.idx(xs, y, z0);
  const long long im = i - pxy;
  double2 pHx = csum(ldg2(A.f[HXY] + im), ldg2(A.f[HXZ] + im));
  double2 pHy = csum(ldg2(A.f[HYX] + im), ldg2(A.f[HYZ] + im));

  for (int z = z0; z < z1; ++z, i += pxy) {
    const double2 sHx = csum(ldg2(A.f[HXY] + i), ldg2(A.f[HXZ] + i));
    const double2 sHy = csum(ldg2(A.f[HYX] + i), ldg2(A.f[HYZ] + i));
    const double2 sHz = csum(ldg2(A.f[HZX] + i), ldg2(A.f[HZY] + i));
    const long long iy = i - px;
    const double2 yHx = csum(ldg2(A.f[HXY] + iy), ldg2(A.f[HXZ] + iy));
    const double2 yHz = csum(ldg2(A.f[HZX] + iy), ldg2(A.f[HZY] + iy));
    double2 xHy, xHz;
    xHy.x = __shfl_up_sync(0xffffffffu, sHy.x, 1);
    xHy.y = __shfl_up_sync(0xffffffffu, sHy.y, 1);
    xHz.x = __shfl_up_sync(0xffffffffu, sHz.x, 1);
    xHz.y = __shfl_up_sync(0xffffffffu, sHz.y, 1);
    if (fetch_x) {
      xHy = csum(ldg2(A.f[HYX] + i - 1), ldg2(A.f[HYZ] + i - 1));
      xHz = csum(ldg2(A.f[HZX] + i - 1), ldg2(A.f[HZY] + i - 1));
    }
    if (act) {
      double2* F;
      F = A.f[EXY] + i; *F = upd(*F, ldg2(A.t[EXY] + i), ldg2(A.c[EXY] + i), yHz, sHz);
      F = A.f[EXZ] + i; *F = upd_src(*F, ldg2(A.t[EXZ] + i), ldg2(A.c[EXZ] + i), pHy, sHy, ldg2(A.src[SRC_EXZ] + i));
      F = A.f[EYX] + i; *F = upd(*F, ldg2(A.t[EYX] + i), ldg2(A.c[EYX] + i), xHz, sHz);
      F = A.f[EYZ] + i; *F = upd_src(*F, ldg2(A.t[EYZ] + i), ldg2(A.c[EYZ] + i), pHx, sHx, ldg2(A.src[SRC_EYZ] + i));
      F = A.f[EZX] + i; *F = upd(*F, ldg2(A.t[EZX] + i), ldg2(A.c[EZX] + i), xHy, sHy);
      F = A.f[EZY] + i; *F = upd(*F, ldg2(A.t[EZY] + i), ldg2(A.c[EZY] + i), yHx, sHx);
#pragma unroll
      for (int k = EXY; k <= EZY; ++k) mark<COUNT>(A, k, i);
    }
    pHx = sHx;
    pHy = sHy;
  }
}

}  // namespace thiim_gpu
