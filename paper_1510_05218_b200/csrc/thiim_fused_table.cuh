// thiim_fused_table.cuh -- engine FUSED with compressed coefficients
// (THIIM_COEFF_TABLE) for piecewise-constant media such as BASELINE config 3's
// layered thin-film stack.
//
// The reference stores 28 coefficient arrays per cell (state.hpp:49-66, 448 of
// its 640 B/cell) even when the medium has a handful of materials.  Here a
// cell stores a uint8 material id; the [n_materials][28] table lives in
// shared memory.  Per plane the producer streams 12 TMA boxes -- E_old(z+1)
// x6, H_old x6 -- instead of 40, each consumer thread loads its cell's
// material id one plane ahead (1 B), so the sweep moves
// 12 x 16 read + 12 x 16 written + 1 = 385 B/LUP instead of 832.  The
// arithmetic is k_fused_tma's, operation for operation, on the same
// coefficient values, so results are bitwise those of the FULL layout.
// Material ids use a pitched layout (row pitch rounded to 16 B); host uploads
// and downloads convert.
#pragma once

#include <cuda.h>

#include "thiim_async.cuh"
#include "thiim_common.cuh"
#include "thiim_fused_tma.cuh"
#include "thiim_ring.cuh"

namespace thiim_gpu {

constexpr int kMaxMaterials = 16;

struct TableMaps {
  TmaMaps f;  // field boxes (same shapes as the FULL layout)
};

struct TableGrid {
  const uint8_t* mat;  // pitched material ids
  long long mp, mplane;  // row pitch and plane stride in bytes
  const double2* table;  // [n_mat][28] in global memory
  int n_mat;
};

// Table-layout plane sequence (4 groups, 12 boxes).
template <class FS>
inline void seq_table(GroupSeq& S, FS fslot) {
  S.ngroups = 0;
  S.nelem = 0;
  auto add = [&](int slot, int box, int src) {
    SeqElem& e = S.e[S.nelem++];
    e.slot = (short)slot;
    e.box = (char)box;
    e.src = (char)src;
    e.coef = 0;
    S.gsize[S.ngroups - 1]++;
  };
  auto group = [&]() { S.gsize[S.ngroups++] = 0; };
  group();  // G0: E_old(z+1) Exy Exz Eyx Eyz
  for (int c : {EXY, EXZ, EYX, EYZ}) add(fslot(c), BOX_A, 1);
  group();  // G1: E_old(z+1) Ezx Ezy
  for (int c : {EZX, EZY}) add(fslot(c), BOX_A, 1);
  group();  // G2: H_old Hxy Hxz Hyx Hyz
  add(fslot(HXY), BOX_BY, 0);
  add(fslot(HXZ), BOX_BY, 0);
  add(fslot(HYX), BOX_BX, 0);
  add(fslot(HYZ), BOX_BX, 0);
  group();  // G3: H_old Hzx Hzy
  add(fslot(HZX), BOX_B, 0);
  add(fslot(HZY), BOX_B, 0);
}

template <int BY, int NG>
struct TableSmem {
  Ring<BY, NG> ring;
  double2 sE[3][BY][32];
  double2 sH[3][BY][32];
  double2 tab[kMaxMaterials][28];  // t x12, c x12, src x4 per material
};

template <int BY, int NG, bool COUNT = false>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_fused_table(Grid g, Arrays A, TableGrid T, const __grid_constant__ TableMaps maps,
                  const __grid_constant__ GroupSeq S, int zc, int tiles_x) {
  constexpr int BX = 32, TX = BX - 2, TY = BY - 2, NCOMP = 32 * BY;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  TableSmem<BY, NG>& sm = *reinterpret_cast<TableSmem<BY, NG>*>(smem_raw);
  const int bty = blockIdx.x / tiles_x, btx = blockIdx.x % tiles_x;
  const int xb = btx * TX - 1, yb = bty * TY - 1;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int z0 = blockIdx.z * zc;
  const int z1 = min(g.nz, z0 + zc);
  const long long pxy = g.pxy;

  for (int k = ty * 32 + tx; k < T.n_mat * 28; k += 32 * (BY + 1))
    sm.tab[k / 28][k % 28] = T.table[k];
  if (tx == 0 && ty == 0) {
    ring_init(sm.ring, BY);
    fence_mbar_init();
  }
  __syncthreads();

  if (ty == BY) {  // ---------------- producer warp (one elected lane)
    if (tx == 0) {
      using Gm = BoxGeom<BY>;
#pragma unroll
      for (int b = 0; b < NBOX; ++b) tma_prefetch_desc(&maps.f.m[b]);
      auto& R = sm.ring;
      int gi = 0;
      uint32_t ph = 0;
      for (int z = z0; z < z1; ++z) {
        int e = 0;
        for (int gr = 0; gr < S.ngroups; ++gr) {
          const int n = S.gsize[gr];
          int bytes = 0;
          for (int k = 0; k < n; ++k) bytes += Gm::bytes(S.e[e + k].box);
          mbar_wait(&R.empty[gi], ph ^ 1);
          mbar_arrive_expect_tx(&R.full[gi], (uint32_t)bytes);
          for (int k = 0; k < n; ++k, ++e) {
            const SeqElem el = S.e[e];
            const int b = el.box;
            tma_load_4d(&R.buf[gi][k][0], &maps.f.m[b], 2 * (xb + 1 + Gm::x0(b)),
                        yb + 1 + Gm::y0(b), z + 1 + el.src, el.slot, &R.full[gi]);
          }
          if (++gi == NG) {
            gi = 0;
            ph ^= 1;
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
  const bool upd_x = own || (ring_y && y >= 0);
  const bool upd_y = own || (ring_x && x >= 0);
  const bool upd_z = own || (ring_x && x >= 0) || (ring_y && y >= 0);
  const int xs = inpad ? x : 0, ys = inpad ? y : 0;
  long long i = g.idx(xs, ys, z0);
  // material id of this thread's cell at local padded plane zp: the raw byte
  // (loaded one plane ahead) and its range check at the point of use, so the
  // load's latency is not exposed by a compare right after it
  auto mat_raw = [&](int zp) -> int {
    return __ldg(T.mat + (long long)zp * T.mplane + (long long)(ys + 1) * T.mp + (xs + 1));
  };
  auto mat_ok = [&](int m) -> int { return m < T.n_mat ? m : 0; };
  auto mat_at = [&](int zp) -> int { return mat_ok(mat_raw(zp)); };

  double2 e[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) e[k] = inpad ? __ldg(A.f[k] + i) : make_double2(0.0, 0.0);
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
        const double2* C = sm.tab[mat_at(z0)];  // local padded plane of z0-1
        const double2 sEx = sm.sE[0][ty][tx], sEy = sm.sE[1][ty][tx], sEz = sm.sE[2][ty][tx];
        const double2 nEx = csum(e[EXY], e[EXZ]), nEy = csum(e[EYX], e[EYZ]);
        const double2 hxy = upd(__ldg(A.f[HXY] + im), C[HXY], C[12 + HXY], sm.sE[2][ty + 1][tx], sEz);
        const double2 hxz = upd_src(__ldg(A.f[HXZ] + im), C[HXZ], C[12 + HXZ], nEy, sEy, C[24 + SRC_HXZ]);
        const double2 hyx = upd(__ldg(A.f[HYX] + im), C[HYX], C[12 + HYX], sm.sE[2][ty][tx + 1], sEz);
        const double2 hyz = upd_src(__ldg(A.f[HYZ] + im), C[HYZ], C[12 + HYZ], nEx, sEx, C[24 + SRC_HYZ]);
        pHx = csum(hxy, hxz);
        pHy = csum(hyx, hyz);
      }
      named_sync(1, NCOMP);
    }
  }

  auto& R = sm.ring;
  RingCursor rc = ring_cursor(R);
#define RD(k, b) ring_read<true>(R, rc, k, b, tx, ty)
  int mid_next = inpad ? mat_raw(z0 + 1) : 0;  // material id, one plane ahead
  for (int z = z0; z < z1; ++z, i += pxy) {
    const int mid = mat_ok(mid_next);
    if (inpad && z + 1 < z1) mid_next = mat_raw(z + 2);
    double2 en[6];
    ring_wait(R, rc);
#pragma unroll
    for (int k = 0; k < 4; ++k) en[k] = RD(k, BOX_A);
    ring_release(R, rc, tx, ring_dep(en[0], en[1], en[2], en[3]));
    ring_wait(R, rc);
    en[4] = RD(0, BOX_A);
    en[5] = RD(1, BOX_A);
    ring_release(R, rc, tx, ring_dep(en[4], en[5]));
    const double2* C = sm.tab[mid];
    // own sums from registers; neighbours read them from shared memory
    const double2 sEx = csum(e[EXY], e[EXZ]), sEy = csum(e[EYX], e[EYZ]),
                  sEz = csum(e[EZX], e[EZY]);
    if (inpad) {
      sm.sE[0][ty][tx] = sEx;
      sm.sE[1][ty][tx] = sEy;
      sm.sE[2][ty][tx] = sEz;
    }
    named_sync(1, NCOMP);
    const double2 nEx = csum(en[EXY], en[EXZ]), nEy = csum(en[EYX], en[EYZ]);
    double2 h[6];
    ring_wait(R, rc);
    h[0] = RD(0, BOX_BY);
    h[1] = RD(1, BOX_BY);
    h[2] = RD(2, BOX_BX);
    h[3] = RD(3, BOX_BX);
    ring_release(R, rc, tx, ring_dep(h[0], h[1], h[2], h[3]));
    ring_wait(R, rc);
    h[4] = RD(0, BOX_B);
    h[5] = RD(1, BOX_B);
    ring_release(R, rc, tx, ring_dep(h[4], h[5]));
    if (upd_x) {
      h[0] = upd(h[0], C[HXY], C[12 + HXY], sm.sE[2][ty + 1][tx], sEz);
      h[1] = upd_src(h[1], C[HXZ], C[12 + HXZ], nEy, sEy, C[24 + SRC_HXZ]);
    }
    if (upd_y) {
      h[2] = upd(h[2], C[HYX], C[12 + HYX], sm.sE[2][ty][tx + 1], sEz);
      h[3] = upd_src(h[3], C[HYZ], C[12 + HYZ], nEx, sEx, C[24 + SRC_HYZ]);
    }
    if (upd_z) {
      h[4] = upd(h[4], C[HZX], C[12 + HZX], sm.sE[1][ty][tx + 1], sEy);
      h[5] = upd(h[5], C[HZY], C[12 + HZY], sm.sE[0][ty + 1][tx], sEx);
    }
    if (own) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        A.fo[HXY + k][i] = h[k];
        mark<COUNT>(A, HXY + k, i);
      }
    }
    const double2 sHx = csum(h[0], h[1]), sHy = csum(h[2], h[3]), sHz = csum(h[4], h[5]);
    if (own || ring_x || ring_y) {
      sm.sH[0][ty][tx] = sHx;
      sm.sH[1][ty][tx] = sHy;
      sm.sH[2][ty][tx] = sHz;
    }
    named_sync(1, NCOMP);

    if (own) {
      A.fo[EXY][i] = upd(e[EXY], C[EXY], C[12 + EXY], sm.sH[2][ty - 1][tx], sHz);
      A.fo[EXZ][i] = upd_src(e[EXZ], C[EXZ], C[12 + EXZ], pHy, sHy, C[24 + SRC_EXZ]);
      A.fo[EYX][i] = upd(e[EYX], C[EYX], C[12 + EYX], sm.sH[2][ty][tx - 1], sHz);
      A.fo[EYZ][i] = upd_src(e[EYZ], C[EYZ], C[12 + EYZ], pHx, sHx, C[24 + SRC_EYZ]);
      A.fo[EZX][i] = upd(e[EZX], C[EZX], C[12 + EZX], sm.sH[1][ty][tx - 1], sHy);
      A.fo[EZY][i] = upd(e[EZY], C[EZY], C[12 + EZY], sm.sH[0][ty - 1][tx], sHx);
#pragma unroll
      for (int k = EXY; k <= EZY; ++k) mark<COUNT>(A, k, i);
    }
    pHx = sHx;
    pHy = sHy;
#pragma unroll
    for (int k = 0; k < 6; ++k) e[k] = en[k];
  }
#undef RD
}

// Generator for the table layout: fields as THIIM_GEN_* and the layer id of
// THIIM_GEN_LAYERED as the material id (pitched), one thread per padded cell.
__global__ void k_generate_table(Grid g, int z_global0, int nz_global, Arrays A, uint64_t seed,
                                 uint8_t* mat, long long mp, long long mplane) {
  const long long n = (long long)(g.nz + 2) * g.pxy;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long r = p - (long long)zp * g.pxy;
    const int yp = (int)(r / g.px);
    const int xp = (int)(r - (long long)yp * g.px);
    const int x = xp - 1, y = yp - 1, z = z_global0 + zp - 1;
    const bool interior = x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < nz_global;
    const uint64_t gidx = (uint64_t)(z + 1) * (uint64_t)g.pxy + (uint64_t)r;
    for (int a = 0; a < 12; ++a)
      A.f[a][p] = interior ? gen_field(gen_key(seed, a), gidx) : make_double2(0.0, 0.0);
    mat[(long long)zp * mplane + (long long)yp * mp + xp] =
        interior ? (uint8_t)gen_layer(seed, g.nx, nz_global, x, y, z) : (uint8_t)0;
  }
}

}  // namespace thiim_gpu
