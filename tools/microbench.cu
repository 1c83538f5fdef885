// microbench.cu -- B200 ceilings for the THIIM sweep design (not product code).
//
//   stream<NIN,NOUT>  elementwise over NIN input + NOUT output double2 arrays of
//                     n elements (the "ideal" zero-reuse sweep: 40/12 is one
//                     fused LUP = 832 B, 26/6 one split half-sweep = 512 B)
//   l2read            repeated reads of an L2-resident buffer
//   fp64              DMUL/DADD throughput (dependent chains, many warps)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

template <int NIN, int NOUT>
struct Ptrs {
  const double2* in[NIN];
  double2* out[NOUT];
};

template <int NIN, int NOUT>
__global__ void __launch_bounds__(256) k_stream(Ptrs<NIN, NOUT> p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double2 acc[NOUT];
#pragma unroll
    for (int k = 0; k < NOUT; ++k) acc[k] = make_double2(0, 0);
#pragma unroll
    for (int j = 0; j < NIN; ++j) {
      const double2 v = __ldg(p.in[j] + i);
      acc[j % NOUT].x += v.x;
      acc[j % NOUT].y += v.y;
    }
#pragma unroll
    for (int k = 0; k < NOUT; ++k) p.out[k][i] = acc[k];
  }
}

__global__ void k_l2read(const double2* __restrict__ a, long long n, int reps, double* sink) {
  double s = 0;
  for (int r = 0; r < reps; ++r)
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
      const double2 v = __ldcg(a + i);
      s += v.x + v.y;
    }
  if (s == 123.456) *sink = s;
}

__global__ void k_fp64(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.9999999, d = blockIdx.x * 1e-5;
  double e = a + 1, f = d + 2, g = a * 3, h = d * 4;
  for (int i = 0; i < iters; ++i) {
    a = __dmul_rn(a, b); d = __dmul_rn(d, c); e = __dadd_rn(e, b); f = __dadd_rn(f, c);
    g = __dmul_rn(g, c); h = __dadd_rn(h, b); b = __dadd_rn(b, 1e-17); c = __dmul_rn(c, 1.0);
  }
  if (a + d + e + f + g + h == 1.2345) out[0] = a;
}

template <int NIN, int NOUT>
int run_stream(long long n, int sms) {
  std::vector<double2*> bufs(NIN + NOUT);
  for (auto& b : bufs) {
    CK(cudaMalloc(&b, n * sizeof(double2)));
    CK(cudaMemset(b, 0, n * sizeof(double2)));
  }
  Ptrs<NIN, NOUT> p;
  for (int j = 0; j < NIN; ++j) p.in[j] = bufs[j];
  for (int k = 0; k < NOUT; ++k) p.out[k] = bufs[NIN + k];
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {2, 4, 8, 16, 64}) {
    const int grid = bps * sms;
    k_stream<NIN, NOUT><<<grid, 256>>>(p, n);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) k_stream<NIN, NOUT><<<grid, 256>>>(p, n);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)n * 16.0 * (NIN + NOUT) * reps;
    printf("stream<%d,%d> n=%lld grid=%d: %.1f GB/s  (%.1f M elem/s)\n", NIN, NOUT, n, grid,
           bytes / (ms * 1e-3) / 1e9, (double)n * reps / (ms * 1e-3) / 1e6);
  }
  for (auto& b : bufs) cudaFree(b);
  return 0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("SMs %d, L2 %d bytes\n", sms, l2);
  const long long n = 17173512;  // 258^3 padded cells of the 256^3 grid
  if (run_stream<40, 12>(n, sms)) return 1;
  if (run_stream<26, 6>(n, sms)) return 1;
  if (run_stream<1, 1>(n * 16, sms)) return 1;
  // L2 read bandwidth at several footprints
  double* sink;
  CK(cudaMalloc(&sink, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (long long mb : {8, 16, 32, 48, 64, 96, 128, 256}) {
    const long long ne = mb * (1 << 20) / 16;
    double2* a;
    CK(cudaMalloc(&a, ne * 16));
    CK(cudaMemset(a, 0, ne * 16));
    const int reps = (int)(2048 / mb) + 1;
    k_l2read<<<sms * 8, 512>>>(a, ne, 1, sink);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    k_l2read<<<sms * 8, 512>>>(a, ne, reps, sink);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("l2read %4lld MB: %.1f GB/s\n", mb, (double)ne * 16 * reps / (ms * 1e-3) / 1e9);
    cudaFree(a);
  }
  // FP64 pipe: 8 ops per iteration per thread
  double* o;
  CK(cudaMalloc(&o, 8));
  const int iters = 20000;
  k_fp64<<<sms * 16, 256>>>(o, 100);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_fp64<<<sms * 16, 256>>>(o, iters);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)sms * 16 * 256 * iters * 8;
  printf("fp64 dmul/dadd: %.2f Tops/s (%.1f ops/clk/SM at 1.965 GHz)\n", ops / (ms * 1e-3) / 1e12,
         ops / (ms * 1e-3) / sms / 1.965e9);
  return 0;
}
