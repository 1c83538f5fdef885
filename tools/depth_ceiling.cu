// depth_ceiling.cu -- memory-system ceiling of a depth-k temporally blocked
// THIIM sweep (not product code).
//
// A pattern-only stand-in for a k-level TBLOCK kernel: the producer lane of a
// 32 x BY thread tile streams exactly the TMA boxes a k-level wavefront would
// need -- level 1 at plane q: the 40 array-planes of the fused sweep (E_old of
// plane q+1, F/t/c/src of the six H components, t/c/src of the six E
// components; the product's 12 groups and box shapes), and for every level
// j = 2..k at plane q-j+1 the 28 coefficient planes boxed to that level's
// region (H: (33-2j) x (BY+1-2j) at (j-1, j-1), E: (32-2j) x (BY-2j) at (j, j))
// -- through the product's 6-slot group ring; consumers wait for and release
// every group and the last level stores 12 fields of its (32-2k) x (BY-2k)
// output tile.  No arithmetic: the time is what the access pattern costs the
// memory system (DRAM, L2 -> SM, TMA issue), i.e. an upper bound on a real
// depth-k kernel built this way.  Tiles run in rounds of <= one CTA per SM in
// bands, like the product's TBLOCK schedule.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -o tools/depth_ceiling tools/depth_ceiling.cu
//   tools/depth_ceiling NX NY NZ [reps]      (prints one JSON line per depth)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_1510_05218_b200/csrc/thiim_async.cuh"

using namespace thiim_gpu;

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__,       \
                  __LINE__);                                                         \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

constexpr int NG = 6;      // ring group slots
constexpr int GMAX = 4;    // boxes per group
constexpr int NARR = 52;   // 12 + 12 fields, 28 coefficients
constexpr int FIN = 0, FOUT = 12, COEF = 24;
constexpr int MAXK = 4;

// box kinds: 5 level-1 shapes, then (H, E) per level 2..MAXK
constexpr int NB = 5 + 2 * (MAXK - 1);
struct Maps {
  CUtensorMap m[NB];
};

__host__ __device__ constexpr int bx0(int b) {
  return b < 5 ? (b == 0 ? 0 : b == 1 ? 1 : b == 2 ? 0 : b == 3 ? 0 : 1)
               : ((b - 5) / 2 + 2) - ((b - 5) % 2 == 0 ? 1 : 0);
}
__host__ __device__ constexpr int by0(int b) {
  return b < 5 ? (b == 0 ? 0 : b == 1 ? 0 : b == 2 ? 1 : b == 3 ? 0 : 1) : bx0(b);
}
__host__ __device__ constexpr int bw(int b) {
  return b < 5 ? (b == 0 ? 32 : b == 1 ? 30 : b == 2 ? 31 : b == 3 ? 31 : 30)
               : ((b - 5) % 2 == 0 ? 33 : 32) - 2 * ((b - 5) / 2 + 2);
}
template <int BY>
__host__ __device__ constexpr int bh(int b) {
  return b < 5 ? (b == 0 ? BY : b == 1 ? BY - 1 : b == 2 ? BY - 2 : b == 3 ? BY - 1 : BY - 2)
               : ((b - 5) % 2 == 0 ? BY + 1 : BY) - 2 * ((b - 5) / 2 + 2);
}
// level-1 kinds: 0 E_old (A), 1 Hx* (BY), 2 Hy* (BX), 3 Hz* (B), 4 E coefs (C)
__host__ __device__ constexpr int hbox(int j) { return 5 + 2 * (j - 2); }
__host__ __device__ constexpr int ebox(int j) { return 6 + 2 * (j - 2); }

template <int BY>
struct Smem {
  double2 buf[NG][GMAX][BY * 32];
  uint64_t full[NG], empty[NG];
};

template <int BY>
struct Prod {
  Smem<BY>& S;
  const Maps& M;
  int xb, yb;
  int g = 0;
  uint32_t ph = 0;
  int k = 0;
  __device__ Prod(Smem<BY>& s, const Maps& m, int x, int y) : S(s), M(m), xb(x), yb(y) {}
  __device__ void begin(uint32_t bytes) {
    mbar_wait(&S.empty[g], ph ^ 1);
    mbar_arrive_expect_tx(&S.full[g], bytes);
    k = 0;
  }
  __device__ void box(int b, int arr, int pz, uint64_t pol) {
    tma_load_4d_hint(&S.buf[g][k++][0], &M.m[b], 2 * (xb + 1 + bx0(b)), yb + 1 + by0(b), pz, arr,
                     &S.full[g], pol);
  }
  __device__ void end() {
    if (++g == NG) {
      g = 0;
      ph ^= 1;
    }
  }
  template <int B>
  __device__ static constexpr uint32_t bytes() {
    return (uint32_t)(bw(B) * bh<BY>(B) * 16);
  }
  // the product's level-1 plane (thiim_producer.cuh produce_plane_ct)
  __device__ void level1(int z, uint64_t pf, uint64_t pc) {
    const int p0 = z + 1, p1 = z + 2;
    begin(4 * bytes<0>());
    for (int c = 0; c < 4; ++c) box(0, FIN + c, p1, pf);
    end();
    begin(2 * bytes<0>());
    for (int c = 4; c < 6; ++c) box(0, FIN + c, p1, pf);
    end();
    const int hb[6] = {1, 1, 2, 2, 3, 3};
    const int nsrc[6] = {0, 1, 0, 1, 0, 0};
    for (int h = 0; h < 6; ++h) {
      const int b = hb[h];
      const uint32_t by = b == 1 ? bytes<1>() : b == 2 ? bytes<2>() : bytes<3>();
      begin((3 + nsrc[h]) * by);
      box(b, FIN + 6 + h, p0, pf);
      box(b, COEF + 6 + h, p0, pc);
      box(b, COEF + 18 + h, p0, pc);
      if (nsrc[h]) box(b, COEF + 24 + (h == 1 ? 2 : 3), p0, pc);
      end();
    }
    // E coefficients: t/c of the six E components + two src (the 14 arrays
    // the H groups above do not read)
    const int ne[4] = {4, 3, 3, 4};
    const int ea[14] = {0, 12, 1, 13, 2, 14, 24, 3, 15, 25, 4, 16, 5, 17};
    for (int e = 0, a = 0; e < 4; ++e) {
      begin(ne[e] * bytes<4>());
      for (int k2 = 0; k2 < ne[e]; ++k2) box(4, COEF + ea[a++], p0, pc);
      end();
    }
  }
  // the 28 coefficient planes of level j (8 groups), boxed to its region
  template <int J>
  __device__ void levelj(int r, uint64_t pol) {
    const int p0 = r + 1;
    const int n[8] = {4, 3, 3, 4, 4, 3, 3, 4};
    int a = 0;
    for (int gi = 0; gi < 8; ++gi) {
      const int b = gi < 4 ? hbox(J) : ebox(J);
      begin(n[gi] * (gi < 4 ? bytes<hbox(J)>() : bytes<ebox(J)>()));
      for (int k2 = 0; k2 < n[gi]; ++k2) box(b, COEF + (a++ % 28), p0, pol);
      end();
    }
  }
};

struct Order {
  int item0, tiles_x, tiles_y, band;
};

template <int BY, int K>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_pattern(const __grid_constant__ Maps M, double2* out, long long stride, int nx, int ny, int nz,
              Order o) {
  constexpr int TXO = 32 - 2 * K, TYO = BY - 2 * K;
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem<BY>& S = *reinterpret_cast<Smem<BY>*>(raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  // band order (thiim_tblock.cuh band_tile)
  const int t = o.item0 + (int)blockIdx.x;
  const int full = o.tiles_x / o.band, per = o.band * o.tiles_y;
  int row, col;
  if (t < full * per) {
    const int bi = t / per, r = t - bi * per;
    row = r / o.band;
    col = bi * o.band + r % o.band;
  } else {
    const int w = o.tiles_x - full * o.band, r = t - full * per;
    row = r / w;
    col = full * o.band + r % w;
  }
  const int xb = col * TXO - K, yb = row * TYO - K;
  if (tx == 0 && ty == 0) {
    for (int g = 0; g < NG; ++g) {
      mbar_init(&S.full[g], 1);
      mbar_init(&S.empty[g], BY);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int qe = nz - 1 + K - 1;
  if (ty == BY) {
    if (tx == 0) {
      const uint64_t first = policy_evict_first(), last = policy_evict_last();
      Prod<BY> P(S, M, xb, yb);
      for (int q = 0; q <= qe; ++q) {
        if (q < nz) P.level1(q, first, last);
        if (K >= 2 && q - 1 >= 0 && q - 1 < nz) P.template levelj<2>(q - 1, K == 2 ? first : last);
        if (K >= 3 && q - 2 >= 0 && q - 2 < nz) P.template levelj<3>(q - 2, K == 3 ? first : last);
        if (K >= 4 && q - 3 >= 0 && q - 3 < nz) P.template levelj<4>(q - 3, first);
      }
    }
    return;
  }
  int g = 0;
  uint32_t ph = 0;
  auto take = [&](int n) {
    for (int i = 0; i < n; ++i) {
      mbar_wait(&S.full[g], ph);
      __syncwarp();
      if (tx == 0) mbar_arrive(&S.empty[g]);
      if (++g == NG) {
        g = 0;
        ph ^= 1;
      }
    }
  };
  const uint64_t first = policy_evict_first();
  const int x = xb + tx, y = yb + ty;
  const bool own = tx >= K && tx < 32 - K && ty >= K && ty < BY - K && x < nx && y < ny && x >= 0 &&
                   y >= 0;
  const long long px = nx + 2, pxy = px * (ny + 2);
  for (int q = 0; q <= qe; ++q) {
    if (q < nz) take(12);
    for (int j = 2; j <= K; ++j)
      if (q - (j - 1) >= 0 && q - (j - 1) < nz) take(8);
    const int r = q - (K - 1);
    if (r >= 0 && r < nz && own) {
      const long long i = (long long)(r + 1) * pxy + (long long)(y + 1) * px + (x + 1);
      for (int c = 0; c < 12; ++c) st_hint(out + c * stride + i, make_double2(0.0, 0.0), first);
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int BY, int K>
void run(double2* buf, long long stride, int nx, int ny, int nz, int reps, int sms) {
  Maps M;
  auto fn = encode_fn();
  const long long px = nx + 2, py = ny + 2;
  const cuuint64_t dims[4] = {(cuuint64_t)(2 * px), (cuuint64_t)py, (cuuint64_t)(nz + 2), NARR};
  const cuuint64_t strides[3] = {(cuuint64_t)px * 16, (cuuint64_t)(px * py * 16),
                                 (cuuint64_t)stride * 16};
  for (int b = 0; b < NB; ++b) {
    const int w = std::max(1, bw(b)), h = std::max(1, bh<BY>(b));
    const cuuint32_t box[4] = {(cuuint32_t)(2 * w), (cuuint32_t)h, 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (fn(&M.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, buf, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      std::printf("tensor map %d failed\n", b);
      std::exit(1);
    }
  }
  constexpr int TXO = 32 - 2 * K, TYO = BY - 2 * K;
  Order o;
  o.tiles_x = (nx + TXO - 1) / TXO;
  o.tiles_y = (ny + TYO - 1) / TYO;
  const long long items = (long long)o.tiles_x * o.tiles_y;
  const long long rounds = (items + sms - 1) / sms, per_round = (items + rounds - 1) / rounds;
  const double bb = std::sqrt((double)std::min<long long>(per_round, sms) * 23.0 / 50.0);
  const int nb = std::max(1, (int)std::ceil(o.tiles_x / bb));
  o.band = (o.tiles_x + nb - 1) / nb;
  const size_t smem = sizeof(Smem<BY>);
  CK(cudaFuncSetAttribute(k_pattern<BY, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  auto pass = [&]() {
    for (long long i0 = 0; i0 < items; i0 += per_round) {
      o.item0 = (int)i0;
      const unsigned n = (unsigned)std::min<long long>(per_round, items - i0);
      k_pattern<BY, K><<<n, dim3(32, BY + 1), smem>>>(M, buf + FOUT * stride, stride, nx, ny, nz, o);
    }
  };
  pass();
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) pass();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double per_pass = ms * 1e-3 / reps;
  const double cells = (double)nx * ny * nz;
  const double glups = cells * K / per_pass / 1e9;
  std::printf("{\"depth\": %d, \"tile_y\": %d, \"grid\": [%d, %d, %d], \"output_tile\": [%d, %d], "
              "\"tiles\": %lld, \"rounds\": %lld, \"band\": %d, \"ms_per_pass\": %.3f, "
              "\"pattern_glups\": %.3f, \"algorithmic_bytes_per_lup\": %.1f, "
              "\"algorithmic_gbs\": %.1f}\n",
              K, BY, nx, ny, nz, TXO, TYO, items, rounds, o.band, per_pass * 1e3, glups, 832.0 / K,
              cells * 832.0 / per_pass / 1e9);
  std::fflush(stdout);
}

int main(int argc, char** argv) {
  const int nx = argc > 1 ? std::atoi(argv[1]) : 512;
  const int ny = argc > 2 ? std::atoi(argv[2]) : 512;
  const int nz = argc > 3 ? std::atoi(argv[3]) : 256;
  const int reps = argc > 4 ? std::atoi(argv[4]) : 3;
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long stride = ((long long)(nx + 2) * (ny + 2) * (nz + 2) + 15) / 16 * 16;
  double2* buf = nullptr;
  CK(cudaMalloc(&buf, (size_t)stride * NARR * sizeof(double2)));
  CK(cudaMemset(buf, 0, (size_t)stride * NARR * sizeof(double2)));
  run<15, 2>(buf, stride, nx, ny, nz, reps, sms);
  run<15, 3>(buf, stride, nx, ny, nz, reps, sms);
  run<15, 4>(buf, stride, nx, ny, nz, reps, sms);
  run<16, 2>(buf, stride, nx, ny, nz, reps, sms);
  run<16, 3>(buf, stride, nx, ny, nz, reps, sms);
  CK(cudaFree(buf));
  return 0;
}
