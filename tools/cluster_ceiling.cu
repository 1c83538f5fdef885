// cluster_ceiling.cu -- memory-system ceiling of depth-2 TBLOCK with CTA
// pairs sharing their y-halo through distributed shared memory (not product
// code; DESIGN.md "Round scheduling" / "Next").
//
// Pattern-only, like tools/depth_ceiling.cu: the product's producer stream of
// level-1 (40 array-planes in 12 groups) and level-2 (28 coefficient planes in
// 8 groups) TMA boxes through a 6-slot group ring, consumers that wait for and
// release every group, four consumer barriers per iteration at the product's
// exchange points, and the level-2 output stores -- no arithmetic.
//   MODE 0  the product's overlapped tiles: a 32 x 15 thread tile per CTA,
//           28 x 11 output tile (2 halo rows/columns per side recomputed).
//   MODE 1  CTA pairs (cluster 2 x 1 x 1) stacked in y: the pair's 32 x 30
//           thread rows cover a 28 x 26 output tile; the rows at the pair's
//           internal edge are not recomputed, their neighbour sums cross to the
//           partner CTA (st.shared::cluster + a remote mbarrier arrive, E sums
//           down and H sums up, twice per iteration), so the pair's boxes do not
//           overlap in y and level 2's boxes grow to 14 / 13 rows.
//   MODE 2  MODE 1's tiling and cluster launch without the exchange (its cost)
//   MODE 3  MODE 0's overlapped tiles launched as y-adjacent cluster pairs
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//        -o tools/cluster_ceiling tools/cluster_ceiling.cu
//   tools/cluster_ceiling NX NY NZ [reps]   (one JSON line per mode)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

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

constexpr int BY = 15;
constexpr int NG = 6;
constexpr int GMAX = 4;
constexpr int NARR = 52;
constexpr int FIN = 0, FOUT = 12, COEF = 24;

// box kinds 0..4: level 1 (A, BY, BX, B, C of thiim_producer.cuh);
// 5/6: level-2 H / E boxes of MODE 0 (29 x 12 at (1,1), 28 x 11 at (2,2));
// 7/8: level-2 H / E boxes of MODE 1 (29 x 14, 28 x 13; y offset by rank)
constexpr int NB = 9;
struct Maps {
  CUtensorMap m[NB];
};
__host__ __device__ constexpr int bx0(int b) {
  return b == 0 ? 0 : b == 1 ? 1 : b == 2 ? 0 : b == 3 ? 0 : b == 4 ? 1 : (b == 5 || b == 7) ? 1 : 2;
}
__host__ __device__ constexpr int by0(int b) {
  return b == 0 ? 0 : b == 1 ? 0 : b == 2 ? 1 : b == 3 ? 0 : b == 4 ? 1 : b == 5 ? 1 : b == 6 ? 2 : 0;
}
__host__ __device__ constexpr int bw(int b) {
  return b == 0 ? 32 : b == 1 ? 30 : b == 2 ? 31 : b == 3 ? 31 : b == 4 ? 30 : (b == 5 || b == 7) ? 29 : 28;
}
__host__ __device__ constexpr int bh(int b) {
  return b == 0 ? BY : b == 1 ? BY - 1 : b == 2 ? BY - 2 : b == 3 ? BY - 1 : b == 4 ? BY - 2
       : b == 5 ? 12 : b == 6 ? 11 : b == 7 ? 14 : 13;
}

struct Smem {
  double2 buf[NG][GMAX][BY * 32];
  uint64_t full[NG], empty[NG];
  double2 sx[3][BY + 2][32];  // exchange sums (+ the partner's row)
  uint64_t xbar;              // partner's boundary row landed
};

struct Prod {
  Smem& S;
  const Maps& M;
  int xb, yb;
  int g = 0;
  uint32_t ph = 0;
  int k = 0;
  __device__ Prod(Smem& s, const Maps& m, int x, int y) : S(s), M(m), xb(x), yb(y) {}
  __device__ void begin(uint32_t bytes) {
    mbar_wait(&S.empty[g], ph ^ 1);
    mbar_arrive_expect_tx(&S.full[g], bytes);
    k = 0;
  }
  __device__ void box(int b, int arr, int pz, uint64_t pol, int dy = 0) {
    tma_load_4d_hint(&S.buf[g][k++][0], &M.m[b], 2 * (xb + 1 + bx0(b)), yb + 1 + by0(b) + dy, pz,
                     arr, &S.full[g], pol);
  }
  __device__ void end() {
    if (++g == NG) {
      g = 0;
      ph ^= 1;
    }
  }
  __device__ void level1(int z, uint64_t pf, uint64_t pc) {
    const int p0 = z + 1, p1 = z + 2;
    begin(4 * bw(0) * bh(0) * 16);
    for (int c = 0; c < 4; ++c) box(0, FIN + c, p1, pf);
    end();
    begin(2 * bw(0) * bh(0) * 16);
    for (int c = 4; c < 6; ++c) box(0, FIN + c, p1, pf);
    end();
    const int hb[6] = {1, 1, 2, 2, 3, 3};
    const int nsrc[6] = {0, 1, 0, 1, 0, 0};
    for (int h = 0; h < 6; ++h) {
      const int b = hb[h];
      begin((3 + nsrc[h]) * bw(b) * bh(b) * 16);
      box(b, FIN + 6 + h, p0, pf);
      box(b, COEF + 6 + h, p0, pc);
      box(b, COEF + 18 + h, p0, pc);
      if (nsrc[h]) box(b, COEF + 24 + (h == 1 ? 2 : 3), p0, pc);
      end();
    }
    const int ne[4] = {4, 3, 3, 4};
    const int ea[14] = {0, 12, 1, 13, 2, 14, 24, 3, 15, 25, 4, 16, 5, 17};
    for (int e = 0, a = 0; e < 4; ++e) {
      begin(ne[e] * bw(4) * bh(4) * 16);
      for (int k2 = 0; k2 < ne[e]; ++k2) box(4, COEF + ea[a++], p0, pc);
      end();
    }
  }
  __device__ void level2(int r, uint64_t pol, int hb, int eb, int dyh, int dye) {
    const int p0 = r + 1;
    const int n[8] = {4, 3, 3, 4, 4, 3, 3, 4};
    int a = 0;
    for (int gi = 0; gi < 8; ++gi) {
      const int b = gi < 4 ? hb : eb;
      begin(n[gi] * bw(b) * bh(b) * 16);
      for (int k2 = 0; k2 < n[gi]; ++k2) box(b, COEF + (a++ % 28), p0, pol, gi < 4 ? dyh : dye);
      end();
    }
  }
};

struct Order {
  int item0, tiles_x, tiles_y, band;
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster(uint32_t a, double2 v) {
  asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void arrive_remote(uint32_t a) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void wait_acq_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "W_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

template <int MODE>
__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_pattern(const __grid_constant__ Maps M, double2* out, long long stride, int nx, int ny, int nz,
              Order o) {
  constexpr int TXO = 28;
  constexpr int TYO = MODE == 0 ? 11 : MODE == 3 ? 22 : 26;  // output rows per tile / pair
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int rank = MODE >= 1 ? (int)cluster_rank() : 0;
  const int t = o.item0 + (int)(MODE >= 1 ? blockIdx.x / 2 : blockIdx.x);
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
  const int xb = col * TXO - 2;
  const int yb = MODE == 0 ? row * TYO - 2 : MODE == 3 ? row * TYO - 2 + rank * 11
                                            : row * TYO - 2 + rank * BY;
  if (tx == 0 && ty == 0) {
    for (int g = 0; g < NG; ++g) {
      mbar_init(&S.full[g], 1);
      mbar_init(&S.empty[g], BY);
    }
    mbar_init(&S.xbar, 32);
    fence_mbar_init();
  }
  __syncthreads();
  if (MODE >= 1) cluster_sync_all();  // partner's barriers initialised
  const int qe = nz;
  if (ty == BY) {
    if (tx == 0) {
      const uint64_t first = policy_evict_first(), last = policy_evict_last();
      Prod P(S, M, xb, yb);
      for (int q = 0; q <= qe; ++q) {
        if (q < nz) P.level1(q, first, last);
        if (q - 1 >= 0 && q - 1 < nz) {
          if (MODE == 0 || MODE == 3)
            P.level2(q - 1, first, 5, 6, 0, 0);
          else  // rank 0: H rows [1, 15), E rows [2, 15); rank 1: [0, 14), [0, 13)
            P.level2(q - 1, first, 7, 8, rank == 0 ? 1 : 0, rank == 0 ? 2 : 0);
        }
      }
    }
    if (MODE >= 1) cluster_sync_all();
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
  // one exchange point: every consumer publishes 3 sums; MODE 1's boundary
  // warps also send theirs to the partner (E sums down: rank 1 row 0 ->
  // rank 0 row BY; H sums up: rank 0 row BY-1 -> rank 1 row -1) and the
  // receiving boundary warp waits for them
  uint32_t xph = 0;
  double acc = 0.0;
  const uint32_t prow_e = smem_u32(&S.sx[0][BY + 1][tx]), prow_h = smem_u32(&S.sx[0][0][tx]);
  auto exchange = [&](bool down, double v) {
    const double2 s = make_double2(v, v);
    for (int c = 0; c < 3; ++c) S.sx[c][ty + 1][tx] = s;
    if (MODE == 1) {
      const bool send = down ? (rank == 1 && ty == 0) : (rank == 0 && ty == BY - 1);
      const bool recv = down ? (rank == 0 && ty == BY - 1) : (rank == 1 && ty == 0);
      if (send) {
        const uint32_t base = down ? prow_e : prow_h;
        const uint32_t peer = rank ^ 1;
        for (int c = 0; c < 3; ++c)
          st_cluster(mapa(base + c * (BY + 2) * 32 * 16, peer), s);
        arrive_remote(mapa(smem_u32(&S.xbar), peer));
      }
      if (recv) {
        wait_acq_cluster(&S.xbar, xph);
        xph ^= 1;
      }
    }
    named_sync(1, 32 * BY);
    const int yn = down ? ty + 2 : ty;  // y+1 / y-1 neighbour row
    for (int c = 0; c < 3; ++c) acc += S.sx[c][yn][tx].x;
    named_sync(1, 32 * BY);
  };
  const uint64_t first = policy_evict_first();
  const int x = xb + tx, y = yb + ty;
  const bool own = MODE == 0 || MODE == 3 ? (tx >= 2 && tx < 30 && ty >= 2 && ty < BY - 2)
                             : (tx >= 2 && tx < 30 && (rank == 0 ? ty >= 2 : ty < BY - 2));
  const bool in = own && x >= 0 && x < nx && y >= 0 && y < ny;
  const long long px = nx + 2, pxy = px * (ny + 2);
  for (int q = 0; q <= qe; ++q) {
    if (q < nz) {
      take(2);
      exchange(true, acc);
      take(6);
      exchange(false, acc);
      take(4);
    }
    const int r = q - 1;
    if (r >= 0 && r < nz) {
      exchange(true, acc);
      take(4);
      exchange(false, acc);
      take(4);
      if (in) {
        const long long i = (long long)(r + 1) * pxy + (long long)(y + 1) * px + (x + 1);
        for (int c = 0; c < 12; ++c)
          st_hint(out + c * stride + i, make_double2(acc * 0.0, 0.0), first);
      }
    }
  }
  if (MODE >= 1) cluster_sync_all();  // the partner may still send into this CTA
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

template <int MODE>
void run(double2* buf, long long stride, int nx, int ny, int nz, int reps, int sms) {
  Maps M;
  auto fn = encode_fn();
  const long long px = nx + 2, py = ny + 2;
  const cuuint64_t dims[4] = {(cuuint64_t)(2 * px), (cuuint64_t)py, (cuuint64_t)(nz + 2), NARR};
  const cuuint64_t strides[3] = {(cuuint64_t)px * 16, (cuuint64_t)(px * py * 16),
                                 (cuuint64_t)stride * 16};
  for (int b = 0; b < NB; ++b) {
    const cuuint32_t box[4] = {(cuuint32_t)(2 * bw(b)), (cuuint32_t)bh(b), 1, 1};
    const cuuint32_t es[4] = {1, 1, 1, 1};
    if (fn(&M.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, buf, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      std::printf("tensor map %d failed\n", b);
      std::exit(1);
    }
  }
  constexpr int TYO = MODE == 0 ? 11 : MODE == 3 ? 22 : 26;
  const int ctas_per_item = MODE == 0 ? 1 : 2;
  Order o;
  o.tiles_x = (nx + 27) / 28;
  o.tiles_y = (ny + TYO - 1) / TYO;
  const long long items = (long long)o.tiles_x * o.tiles_y;
  const long long slots = sms / ctas_per_item;
  const long long rounds = (items + slots - 1) / slots, per_round = (items + rounds - 1) / rounds;
  // product band rule on the round's CTA block (a pair is 2 tiles tall)
  const double bb = std::sqrt((double)std::min<long long>(per_round, slots) * ctas_per_item * 23.0 / 50.0);
  const int nb = std::max(1, (int)std::ceil(o.tiles_x / bb));
  o.band = (o.tiles_x + nb - 1) / nb;
  const size_t smem = sizeof(Smem);
  CK(cudaFuncSetAttribute(k_pattern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (MODE >= 1)
    CK(cudaFuncSetAttribute(k_pattern<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  auto pass = [&]() {
    for (long long i0 = 0; i0 < items; i0 += per_round) {
      o.item0 = (int)i0;
      const unsigned n = (unsigned)std::min<long long>(per_round, items - i0);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(n * ctas_per_item);
      cfg.blockDim = dim3(32, BY + 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = ctas_per_item;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k_pattern<MODE>, M, buf + FOUT * stride, stride, nx, ny, nz, o));
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
  std::printf("{\"mode\": %d, \"grid\": [%d, %d, %d], \"items\": %lld, \"rounds\": %lld, "
              "\"band\": %d, \"ms_per_pass\": %.3f, \"pattern_glups\": %.3f}\n",
              MODE, nx, ny, nz, items, rounds, o.band, per_pass * 1e3, cells * 2 / per_pass / 1e9);
  std::fflush(stdout);
}

int main(int argc, char** argv) {
  const int nx = argc > 1 ? std::atoi(argv[1]) : 512;
  const int ny = argc > 2 ? std::atoi(argv[2]) : 512;
  const int nz = argc > 3 ? std::atoi(argv[3]) : 256;
  const int reps = argc > 4 ? std::atoi(argv[4]) : 3;
  const int which = argc > 5 ? std::atoi(argv[5]) : -1;
  int sms = 148;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const long long stride = ((long long)(nx + 2) * (ny + 2) * (nz + 2) + 15) / 16 * 16;
  double2* buf = nullptr;
  CK(cudaMalloc(&buf, (size_t)stride * NARR * sizeof(double2)));
  CK(cudaMemset(buf, 0, (size_t)stride * NARR * sizeof(double2)));
  for (int rep = 0; rep < 2; ++rep) {
    if (which <= 0) run<0>(buf, stride, nx, ny, nz, reps, sms);
    if (which < 0 || which == 1) run<1>(buf, stride, nx, ny, nz, reps, sms);
    if (which < 0 || which == 2) run<2>(buf, stride, nx, ny, nz, reps, sms);
    if (which < 0 || which == 3) run<3>(buf, stride, nx, ny, nz, reps, sms);
  }
  CK(cudaFree(buf));
  return 0;
}
