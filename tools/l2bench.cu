// l2bench.cu -- L2 -> SM throughput of TMA boxes vs LDG.128 (not product code).
//
// A `foot`-MB buffer of random doubles (L2-resident when < ~100 MB) is read
// repeatedly by (a) one producer lane per CTA issuing 4-D... here 2-D TMA boxes of
// 32 x BY double2 into a ring of smem slots drained by consumer warps, and
// (b) plain LDG.128 loads (ld.global.cg).  Reports GB/s.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x)                                                                               \
  do {                                                                                      \
    cudaError_t e = (x);                                                                    \
    if (e != cudaSuccess) {                                                                 \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);        \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

__device__ __forceinline__ uint32_t su(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int BY = 16, NBUF = 20, BOXB = BY * 32 * 16;

__global__ void __launch_bounds__(32 * (BY + 1), 1)
    k_tma(const __grid_constant__ CUtensorMap m, int nrows_boxes, int iters, double* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  double2* buf = (double2*)raw;
  uint64_t* full = (uint64_t*)(raw + NBUF * BOXB);
  uint64_t* empty = full + NBUF;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (tx == 0 && ty == 0) {
    for (int k = 0; k < NBUF; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&full[k])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(&empty[k])), "r"(BY));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int slot = 0;
  uint32_t phase = 0;
  if (ty == BY) {
    if (tx == 0) {
      for (int it = 0; it < iters; ++it) {
        const int row = (blockIdx.x * 131 + it * 7) % nrows_boxes;
        asm volatile(
            "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                su(&empty[slot])),
            "r"(phase ^ 1)
            : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&full[slot])),
                     "r"(BOXB)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], "
            "[%1, {%2, %3}], [%4];" ::"r"(su(buf + slot * BY * 32)),
            "l"(&m), "r"(0), "r"(row * BY), "r"(su(&full[slot]))
            : "memory");
        if (++slot == NBUF) { slot = 0; phase ^= 1; }
      }
    }
    return;
  }
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    asm volatile(
        "{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
            su(&full[slot])),
        "r"(phase)
        : "memory");
    const double2 v = buf[slot * BY * 32 + ty * 32 + tx];
    acc += v.x;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (tx == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(&empty[slot])) : "memory");
    if (++slot == NBUF) { slot = 0; phase ^= 1; }
  }
  if (acc == 1.2345) *sink = acc;
}

__global__ void k_ldg(const double2* __restrict__ a, long long n, int reps, double* sink) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(a + (i * 7 + r * 1031) % n);
      s += v.x + v.y;
    }
  if (s == 123.456) *sink = s;
}

__global__ void k_fill(double2* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = make_double2((double)(i * 2654435761ull % 1000003) * 1e-3, (double)(i % 977) + 0.5);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  double* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t smem = NBUF * BOXB + 2 * NBUF * 8;
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int mb : {16, 32, 64, 96, 128, 512, 4096}) {
    const long long n = (long long)mb * (1 << 20) / 16;
    double2* a;
    CK(cudaMalloc(&a, n * 16));
    k_fill<<<sms * 4, 256>>>(a, n);
    CK(cudaDeviceSynchronize());
    // TMA: view as rows of 32 double2 (64 doubles)
    const long long rows = n / 32;
    CUtensorMap m;
    const cuuint64_t dims[2] = {64, (cuuint64_t)rows};
    const cuuint64_t str[1] = {512};
    const cuuint32_t box[2] = {64, BY};
    const cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4000;
    const int nboxes = (int)(rows / BY);
    k_tma<<<sms, dim3(32, BY + 1), smem>>>(m, nboxes, 100, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_tma<<<sms, dim3(32, BY + 1), smem>>>(m, nboxes, iters, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tma = (double)sms * iters * BOXB / (ms * 1e-3) / 1e9;
    const int reps = (int)(4096 / mb) + 2;
    k_ldg<<<sms * 8, 512>>>(a, n, 1, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_ldg<<<sms * 8, 512>>>(a, n, reps, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double ldg = (double)n * 16 * reps / (ms * 1e-3) / 1e9;
    printf("footprint %5d MB: TMA boxes %.0f GB/s   LDG.128 %.0f GB/s\n", mb, tma, ldg);
    cudaFree(a);
  }
  return 0;
}
