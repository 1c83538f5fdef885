// thiim_fused.cuh -- engine FUSED: one kernel per THIIM step.
//
// Each CTA owns an x-y tile of TX x TY cells and streams z over a chunk of
// planes.  At plane z it computes H_new(z) and then E_new(z) (reference
// step_reference order, kernels.cpp:105-113): E_new(z) needs H_new at
// x-1, y-1 (same plane, from shared memory) and at z-1 (carried in registers
// from the previous plane); H_new(z) needs E_old at x+1, y+1 (shared memory)
// and z+1 (the plane loaded one iteration ahead).
//
// Fields are ping-ponged (read set f, write set fo): a neighbouring CTA may
// already have written its E_new/H_new at the shared tile edge, so the in-place
// update of the reference (safe there because one family is swept at a time)
// would race here.  Ghost cells are never written, in either set.
//
// The thread block covers the tile plus a one-cell ring: BX = TX+2,
// BY = TY+2.  Ring threads at -x / -y recompute the four H components the tile
// needs there (Hzx,Hzy,Hyx,Hyz at x0-1; Hzx,Hzy,Hxy,Hxz at y0-1) from the
// same inputs as the owning CTA -- bitwise identical.  Ring threads at +x / +y
// only load E.  At a global boundary the ring sits on ghost cells, whose
// stored values are used unchanged (exactly what the reference reads).
//
// Algorithmic traffic per LUP: 40 arrays read + 12 written = 832 B.
#pragma once

#include "thiim_common.cuh"

namespace thiim_gpu {

template <int BX, int BY>
struct RegFusedSmem {
  double2 sE[3][BY][BX];  // E_old sums (x, y, z physical components) at plane z
  double2 sH[3][BY][BX];  // H_new sums at plane z
};

template <int BX, int BY, int MINB>
__global__ void __launch_bounds__(BX* BY, MINB)
    k_fused(Grid g, Arrays A, int zc) {
  constexpr int TX = BX - 2, TY = BY - 2;
  __shared__ RegFusedSmem<BX, BY> sm;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int x = blockIdx.x * TX - 1 + tx;
  const int y = blockIdx.y * TY - 1 + ty;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);

  const bool inpad = (x <= g.nx) && (y <= g.ny);
  const bool interior = (x >= 0) && (x < g.nx) && (y >= 0) && (y < g.ny);
  const bool ring_x = (tx == 0) && (ty >= 1) && (ty <= BY - 2) && (y < g.ny);
  const bool ring_y = (ty == 0) && (tx >= 1) && (tx <= BX - 2) && (x < g.nx);
  const bool own = interior && tx >= 1 && tx <= BX - 2 && ty >= 1 && ty <= BY - 2;
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;  // safe address for idle threads
  const long long pxy = g.pxy;
  long long i = g.idx(xs, ys, z0);

  // ---- prologue: E_old at plane z0 (carried), H_new sums at z0-1 for own cells.
  double2 e[6];
  if (inpad) {
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = __ldg(A.f[k] + i);
  }
  double2 pHx = make_double2(0.0, 0.0), pHy = make_double2(0.0, 0.0);
  {
    const long long im = i - pxy;
    if (z0 == 0 && !g.halo_lo) {
      // ghost plane below the grid: H never updated there
      if (own) {
        pHx = csum(__ldg(A.f[HXY] + im), __ldg(A.f[HXZ] + im));
        pHy = csum(__ldg(A.f[HYX] + im), __ldg(A.f[HYZ] + im));
      }
    } else {
      double2 m[6];
      if (inpad) {
#pragma unroll
        for (int k = 0; k < 6; ++k) m[k] = __ldg(A.f[k] + im);
        sm.sE[0][ty][tx] = csum(m[EXY], m[EXZ]);
        sm.sE[1][ty][tx] = csum(m[EYX], m[EYZ]);
        sm.sE[2][ty][tx] = csum(m[EZX], m[EZY]);
      }
      __syncthreads();
      if (own) {
        const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
        const double2 nEx = csum(e[EXY], e[EXZ]), nEy = csum(e[EYX], e[EYZ]);
        const double2 hxy = upd(__ldg(A.f[HXY] + im), __ldg(A.t[HXY] + im), __ldg(A.c[HXY] + im),
                                sm.sE[2][ty + 1][tx], sEz);
        const double2 hxz = upd_src(__ldg(A.f[HXZ] + im), __ldg(A.t[HXZ] + im), __ldg(A.c[HXZ] + im),
                                    nEy, sEy, __ldg(A.src[SRC_HXZ] + im));
        const double2 hyx = upd(__ldg(A.f[HYX] + im), __ldg(A.t[HYX] + im), __ldg(A.c[HYX] + im),
                                sm.sE[2][ty][tx + 1], sEz);
        const double2 hyz = upd_src(__ldg(A.f[HYZ] + im), __ldg(A.t[HYZ] + im), __ldg(A.c[HYZ] + im),
                                    nEx, sEx, __ldg(A.src[SRC_HYZ] + im));
        pHx = csum(hxy, hxz);
        pHy = csum(hyx, hyz);
      }
      __syncthreads();
    }
  }

  for (int z = z0; z < z1; ++z, i += pxy) {
    // (a) E_old at z+1 (plane nz is the ghost plane); E sums at z to smem.
    double2 en[6];
    const long long ip = i + pxy;
    if (inpad) {
#pragma unroll
      for (int k = 0; k < 6; ++k) en[k] = __ldg(A.f[k] + ip);
      sm.sE[0][ty][tx] = csum(e[EXY], e[EXZ]);
      sm.sE[1][ty][tx] = csum(e[EYX], e[EYZ]);
      sm.sE[2][ty][tx] = csum(e[EZX], e[EZY]);
    }
    __syncthreads();

    // (b) H half-step at plane z: own cells (all six) and the -x / -y ring.
    if (own) {
      const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
      const double2 nEx = csum(en[EXY], en[EXZ]), nEy = csum(en[EYX], en[EYZ]);
      const double2 hxy = upd(__ldg(A.f[HXY] + i), __ldg(A.t[HXY] + i), __ldg(A.c[HXY] + i),
                              sm.sE[2][ty + 1][tx], sEz);
      const double2 hxz = upd_src(__ldg(A.f[HXZ] + i), __ldg(A.t[HXZ] + i), __ldg(A.c[HXZ] + i),
                                  nEy, sEy, __ldg(A.src[SRC_HXZ] + i));
      const double2 hyx = upd(__ldg(A.f[HYX] + i), __ldg(A.t[HYX] + i), __ldg(A.c[HYX] + i),
                              sm.sE[2][ty][tx + 1], sEz);
      const double2 hyz = upd_src(__ldg(A.f[HYZ] + i), __ldg(A.t[HYZ] + i), __ldg(A.c[HYZ] + i),
                                  nEx, sEx, __ldg(A.src[SRC_HYZ] + i));
      const double2 hzx = upd(__ldg(A.f[HZX] + i), __ldg(A.t[HZX] + i), __ldg(A.c[HZX] + i),
                              sm.sE[1][ty][tx + 1], sEy);
      const double2 hzy = upd(__ldg(A.f[HZY] + i), __ldg(A.t[HZY] + i), __ldg(A.c[HZY] + i),
                              sm.sE[0][ty + 1][tx], sEx);
      A.fo[HXY][i] = hxy;
      A.fo[HXZ][i] = hxz;
      A.fo[HYX][i] = hyx;
      A.fo[HYZ][i] = hyz;
      A.fo[HZX][i] = hzx;
      A.fo[HZY][i] = hzy;
      sm.sH[0][ty][tx] = csum(hxy, hxz);
      sm.sH[1][ty][tx] = csum(hyx, hyz);
      sm.sH[2][ty][tx] = csum(hzx, hzy);
    } else if (ring_x) {  // cell (x0-1, y): Hy and Hz sums
      double2 hzx = __ldg(A.f[HZX] + i), hzy = __ldg(A.f[HZY] + i);
      double2 hyx = __ldg(A.f[HYX] + i), hyz = __ldg(A.f[HYZ] + i);
      if (x >= 0) {
        const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
        const double2 nEx = csum(en[EXY], en[EXZ]);
        hzx = upd(hzx, __ldg(A.t[HZX] + i), __ldg(A.c[HZX] + i), sm.sE[1][ty][tx + 1], sEy);
        hzy = upd(hzy, __ldg(A.t[HZY] + i), __ldg(A.c[HZY] + i), sm.sE[0][ty + 1][tx], sEx);
        hyx = upd(hyx, __ldg(A.t[HYX] + i), __ldg(A.c[HYX] + i), sm.sE[2][ty][tx + 1], sEz);
        hyz = upd_src(hyz, __ldg(A.t[HYZ] + i), __ldg(A.c[HYZ] + i), nEx, sEx,
                      __ldg(A.src[SRC_HYZ] + i));
      }
      sm.sH[1][ty][tx] = csum(hyx, hyz);
      sm.sH[2][ty][tx] = csum(hzx, hzy);
    } else if (ring_y) {  // cell (x, y0-1): Hx and Hz sums
      double2 hzx = __ldg(A.f[HZX] + i), hzy = __ldg(A.f[HZY] + i);
      double2 hxy = __ldg(A.f[HXY] + i), hxz = __ldg(A.f[HXZ] + i);
      if (y >= 0) {
        const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
        const double2 nEy = csum(en[EYX], en[EYZ]);
        hzx = upd(hzx, __ldg(A.t[HZX] + i), __ldg(A.c[HZX] + i), sm.sE[1][ty][tx + 1], sEy);
        hzy = upd(hzy, __ldg(A.t[HZY] + i), __ldg(A.c[HZY] + i), sm.sE[0][ty + 1][tx], sEx);
        hxy = upd(hxy, __ldg(A.t[HXY] + i), __ldg(A.c[HXY] + i), sm.sE[2][ty + 1][tx], sEz);
        hxz = upd_src(hxz, __ldg(A.t[HXZ] + i), __ldg(A.c[HXZ] + i), nEy, sEy,
                      __ldg(A.src[SRC_HXZ] + i));
      }
      sm.sH[0][ty][tx] = csum(hxy, hxz);
      sm.sH[2][ty][tx] = csum(hzx, hzy);
    }
    __syncthreads();

    // (c) E half-step at plane z for own cells.
    if (own) {
      const double2 sHx = sm.sH[0][ty][tx], sHy = sm.sH[1][ty][tx], sHz = sm.sH[2][ty][tx];
      A.fo[EXY][i] = upd(e[EXY], __ldg(A.t[EXY] + i), __ldg(A.c[EXY] + i), sm.sH[2][ty - 1][tx], sHz);
      A.fo[EXZ][i] = upd_src(e[EXZ], __ldg(A.t[EXZ] + i), __ldg(A.c[EXZ] + i), pHy, sHy,
                             __ldg(A.src[SRC_EXZ] + i));
      A.fo[EYX][i] = upd(e[EYX], __ldg(A.t[EYX] + i), __ldg(A.c[EYX] + i), sm.sH[2][ty][tx - 1], sHz);
      A.fo[EYZ][i] = upd_src(e[EYZ], __ldg(A.t[EYZ] + i), __ldg(A.c[EYZ] + i), pHx, sHx,
                             __ldg(A.src[SRC_EYZ] + i));
      A.fo[EZX][i] = upd(e[EZX], __ldg(A.t[EZX] + i), __ldg(A.c[EZX] + i), sm.sH[1][ty][tx - 1], sHy);
      A.fo[EZY][i] = upd(e[EZY], __ldg(A.t[EZY] + i), __ldg(A.c[EZY] + i), sm.sH[0][ty - 1][tx], sHx);
      pHx = sHx;
      pHy = sHy;
    }
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = en[k];
  }
}

}  // namespace thiim_gpu
