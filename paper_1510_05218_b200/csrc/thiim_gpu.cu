// thiim_gpu.cu -- libthiim_gpu.so: the C-ABI declared in include/thiim_gpu.h.
//
// One context = one problem split into z-slabs, one slab per GPU.  Each slab
// holds the reference padded layout for its planes [z0-1, z1] (the outer
// planes are global ghosts or halo copies of the neighbour slab's boundary
// planes) in one device allocation:
//   [F0: 12 field arrays][F1: 12 field arrays, fused engines only]
//   [t: 12][c: 12][src: 4]
// each array `stride` elements (padded plane count x (nx+2)(ny+2), rounded up
// to 256 B).  Upload/download are plain plane-range copies: no layout change.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <omp.h>

// ring depth (slots) of the default TBLOCK kernel (experiment builds override)
#ifndef THIIM_TB_NG
#define THIIM_TB_NG 6
#endif

#include "../../include/thiim_gpu.h"
#include "thiim_common.cuh"
#include "thiim_complex.cuh"
#include "thiim_fused_table.cuh"
#include "thiim_fused_tma.cuh"
#include "thiim_split.cuh"
#include "thiim_tblock.cuh"
#include "thiim_tblock3.cuh"
#include "thiim_tblock_table.cuh"

using namespace thiim_gpu;

namespace {

thread_local std::string g_err;

// One-time per-device setup flags (function attributes, pool configuration):
// an atomic bit per device, set only after the setup succeeded.  The setups
// are idempotent, so two host threads racing on one device merely both do it;
// devices >= 32 redo it every time.
bool setup_needed(const std::atomic<unsigned>& mask, int dev) {
  return dev < 0 || dev >= 32 || !(mask.load() >> dev & 1u);
}
void setup_done(std::atomic<unsigned>& mask, int dev) {
  if (dev >= 0 && dev < 32) mask.fetch_or(1u << dev);
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(THIIM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

constexpr int kSplitBY = 4;

struct Slab {
  int device = 0;
  int z0 = 0, z1 = 0;  // global interior planes [z0, z1) held as local interior
  Grid g{};            // local grid: nz = z1 - z0
  // owned planes [own0, own1); a TBLOCK ("deep") slab also holds one extended
  // plane per internal interface (ext_lo / ext_hi) that the exchange refreshes
  int own0 = 0, own1 = 0, ext_lo = 0, ext_hi = 0;
  bool deep = false;
  unsigned* cnt = nullptr;                 // sanitizer store counts [12][stride] (or null)
  bool ipc_buf = false;  // buf from cudaMalloc (exportable by IPC), not the pool
  // neighbour slabs of other processes, imported by IPC (multi-process peer stores)
  struct Peer {
    double2* base = nullptr;
    long long stride = 0;
    int nz = 0, ext_lo = 0, ext_hi = 0;
    unsigned long long* counter = nullptr;  // its pass counter (mapped)
  } peer[2];
  // multi-process peer stores: this slab's pass counter (in buf, exported) and
  // the number of TBLOCK passes enqueued so far
  unsigned long long* counter = nullptr;
  long long counter_offset = 0;
  unsigned long long passes = 0;
  unsigned long long* cov_bad = nullptr;   // sanitizer violations (device)
  double2* buf = nullptr;
  size_t stride = 0;   // elements per array
  int nfield_sets = 1;
  int cur = 0;         // current field set
  bool table = false;  // THIIM_COEFF_TABLE: no coefficient arrays, material ids + table
  uint8_t* mat = nullptr;  // pitched material ids (table layout)
  long long mp = 0, mplane = 0;
  double2* tab = nullptr;  // [kMaxMaterials][28]
  int n_mat = 0;

  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t ev_pass = nullptr;  // last TBLOCK pass (peer-store ordering between slabs)
  // CUDA graph of two TBLOCK passes (4 steps) per starting field set, replayed
  // by thiim_gpu_step on whole-z contexts (launch-bound small grids)
  cudaGraphExec_t pass_graph[2] = {nullptr, nullptr};
  long long pass_graph_launches[2] = {0, 0};  // kernel launches one replay runs
  int pass_graph_depth[2] = {0, 0};           // time-block depth of the captured passes
  // 4-D tensor maps over the allocation {x (doubles), y, plane, array slot},
  // one set of box shapes per tile height (8 / 16 rows), built lazily
  TmaMaps maps[6];  // tile heights 8, 16, 15, 12, 14, 13 (map_index)
  bool maps_ok[6] = {false, false, false, false, false, false};
  TmaMaps maps_seg[6][2];  // the same for 16- / 8-lane segments (folded TBLOCK tiles)
  bool maps_seg_ok[6][2] = {};
  TmaMaps fmaps[6];  // the one-step (fused) sweeps' maps: no L2 promotion (ensure_tmap)
  bool fmaps_ok[6] = {false, false, false, false, false, false};

  // TBLOCK in place (THIIM_ENGINE_TBLOCK_INPLACE, one whole-z slab, no second
  // field set): sub-range length; the field arrays carry a gap of ip_L + 2
  // planes (fstride, see launch_tblock_inplace)
  int ip_L = 0;
  // sub-range views only: where the TBLOCK pass stores its outputs (field k at
  // fo_base + k * fo_stride - fo_shift) instead of the other field set
  double2* fo_base = nullptr;
  long long fo_stride = 0, fo_shift = 0;

  // TBLOCK in place (r02): the field arrays get their own stride (nz + 2 + D
  // planes: the array plus the D-plane gap it oscillates into); views of it
  // address the coefficients through their own base (cbuf) and tensor maps
  size_t fstride = 0;        // elements per field array (0: `stride`)
  double2* cbuf = nullptr;   // views: first coefficient array, plane-shifted like buf
  TmaMaps cmaps[6];          // views: coefficient maps (tile heights as `maps`)
  bool cmaps_ok[6] = {false, false, false, false, false, false};
  TmaMaps cmaps_seg[6][2];
  bool cmaps_seg_ok[6][2] = {};
  int ip_pos = 0;            // field planes start at plane ip_pos of their region (0 / D)
  unsigned* ring_nz = nullptr;  // in place: some field ghost-ring cell is non-zero (device)

  size_t fs() const { return fstride ? fstride : stride; }
  double2* field(int set, int k) const { return buf + (size_t)(set * 12 + k) * fs(); }
  double2* coeff(int a) const {  // a in 12..39 (FULL layout only)
    if (table) return nullptr;
    if (cbuf) return cbuf + (size_t)(a - 12) * stride;
    return buf + (size_t)nfield_sets * 12 * fs() + (size_t)(a - 12) * stride;
  }
  int n_arrays() const { return nfield_sets * 12 + (table ? 0 : 28); }
  double2* array(int a) const { return a < 12 ? field(cur, a) : coeff(a); }
  Arrays arrays(int in_set, int out_set) const {
    Arrays A;
    for (int k = 0; k < 12; ++k) {
      A.f[k] = field(in_set, k);
      A.fo[k] = fo_base ? fo_base + k * fo_stride - fo_shift : field(out_set, k);
      A.t[k] = coeff(12 + k);
      A.c[k] = coeff(24 + k);
    }
    for (int k = 0; k < 4; ++k) A.src[k] = coeff(36 + k);
    A.cnt = cnt;
    A.cstride = (long long)stride;
    return A;
  }
};

}  // namespace

struct thiim_gpu_ctx {
  thiim_dims dims{};
  thiim_gpu_opts opts{};
  int depth = 2;  // TBLOCK time-block depth (3: one whole-z slab, reference layout)
  int engine = THIIM_ENGINE_FUSED;
  std::vector<Slab> slabs;
  bool loaded = false;
  bool sanitize = false;               // exactly-once store coverage per pass
  bool peer_stores = false;  // deep slabs write each other's halos from the kernel
  bool ipc_ordered = false;  // IPC peer stores ordered by device pass counters
  unsigned long long cov_passes = 0;
  long long pxy() const { return (long long)(dims.nx + 2) * (dims.ny + 2); }
};

// ------------------------------------------------------------------ kernels

namespace {

// Device generator: one thread per padded cell of the slab, all 40 arrays.
__global__ void k_generate(Grid g, int z_global0, int nz_global, Arrays A, int kind,
                           uint64_t seed, const double2* __restrict__ layer_table) {
  const long long n = (long long)(g.nz + 2) * g.pxy;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long r = p - (long long)zp * g.pxy;
    const int yp = (int)(r / g.px);
    const int xp = (int)(r - (long long)yp * g.px);
    const int x = xp - 1, y = yp - 1, zl = zp - 1;
    const int z = z_global0 + zl;  // global interior plane
    const bool interior = x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < nz_global;
    // the counter is the GLOBAL padded index, so slabs reproduce the 1-GPU problem
    const uint64_t gidx = (uint64_t)(z + 1) * (uint64_t)g.pxy + (uint64_t)r;
    for (int a = 0; a < 40; ++a) {
      double2 v = make_double2(0.0, 0.0);
      if (interior) {
        if (a < 12) {
          v = gen_field(gen_key(seed, a), gidx);
        } else if (kind == THIIM_GEN_LAYERED) {
          v = layer_table[(a - 12) * 6 + gen_layer(seed, g.nx, nz_global, x, y, z)];
        } else {
          v = gen_disk(gen_key(seed, a), gidx);
        }
      }
      double2* dst = a < 12 ? A.f[a] : a < 24 ? const_cast<double2*>(A.t[a - 12])
                                       : a < 36 ? const_cast<double2*>(A.c[a - 24])
                                                : const_cast<double2*>(A.src[a - 36]);
      dst[p] = v;
    }
  }
}

// Benchmark problem (build_benchmark_problem, coefficients.cpp:94-111): fields
// and ghosts zero, every interior cell the same 24 t / c values, the 4 source
// arrays non-zero on the injection plane only.  One thread per padded cell.
struct BenchValues {
  double2 v[28];  // t x12, c x12, src x4 (reference array order 12..39)
};
__global__ void k_init_benchmark(Grid g, int z_global0, int nz_global, Arrays A, BenchValues bv,
                                 int zsrc) {
  const long long n = (long long)(g.nz + 2) * g.pxy;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long r = p - (long long)zp * g.pxy;
    const int yp = (int)(r / g.px);
    const int xp = (int)(r - (long long)yp * g.px);
    const int z = z_global0 + zp - 1;
    const bool interior = xp >= 1 && xp <= g.nx && yp >= 1 && yp <= g.ny && z >= 0 && z < nz_global;
    const double2 zero = make_double2(0.0, 0.0);
    for (int a = 0; a < 12; ++a) A.f[a][p] = zero;
    for (int k = 0; k < 12; ++k) {
      const_cast<double2*>(A.t[k])[p] = interior ? bv.v[k] : zero;
      const_cast<double2*>(A.c[k])[p] = interior ? bv.v[12 + k] : zero;
    }
    for (int k = 0; k < 4; ++k)
      const_cast<double2*>(A.src[k])[p] = (interior && z == zsrc) ? bv.v[24 + k] : zero;
  }
}

// Same problem in the table layout: material id 0 (ghost), 1 (interior), 2
// (interior, injection plane); fields zero.
__global__ void k_init_benchmark_table(Grid g, int z_global0, int nz_global, Arrays A,
                                       uint8_t* mat, long long mp, long long mplane, int zsrc) {
  const long long n = (long long)(g.nz + 2) * g.pxy;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long r = p - (long long)zp * g.pxy;
    const int yp = (int)(r / g.px);
    const int xp = (int)(r - (long long)yp * g.px);
    const int z = z_global0 + zp - 1;
    const bool interior = xp >= 1 && xp <= g.nx && yp >= 1 && yp <= g.ny && z >= 0 && z < nz_global;
    for (int a = 0; a < 12; ++a) A.f[a][p] = make_double2(0.0, 0.0);
    mat[(long long)zp * mplane + (long long)yp * mp + xp] =
        interior ? (uint8_t)(z == zsrc ? 2 : 1) : (uint8_t)0;
  }
}

// build_problem_from_voxels (coefficients.cpp:112-141) on the device: the 28
// coefficients of every interior cell from its material record (eps re/im, mu,
// sigma, sigma*; x fastest), derive_coefficients (coefficients.cpp:25-55) per
// family and iteration mode with the host build's complex arithmetic
// (thiim_complex.cuh), fill_coefficients' sign folding (:63-66); fields zero,
// ghosts zero, sources on the injection plane only.  The first failing
// (component, z, y, x) in the reference's loop order is kept as
// key = ((comp * ncells + cell) << 3) | code (atomicMin; code 1 mu, 2 eps,
// 3 / 4 vanishing denominator in forward / back mode).
struct SchemeDev {
  double tau, delta;
  dcx ep_h, em_h, em_1, ep_1;  // expi(+wt/2), expi(-wt/2), expi(-wt), expi(+wt)
  dcx src_e, src_h;
  int zsrc;
};
__global__ void k_init_materials(Grid g, int z_global0, int nz_global, Arrays A,
                                 const double* __restrict__ mats, int z_mat0, SchemeDev sp,
                                 unsigned long long* err) {
  static constexpr double kCurl[12] = {+1, -1, -1, +1, +1, -1, -1, +1, +1, -1, -1, +1};
  const long long n = (long long)(g.nz + 2) * g.pxy;
  const unsigned long long ncells = (unsigned long long)g.nx * g.ny * nz_global;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long rr = p - (long long)zp * g.pxy;
    const int yp = (int)(rr / g.px);
    const int xp = (int)(rr - (long long)yp * g.px);
    const int x = xp - 1, y = yp - 1, z = z_global0 + zp - 1;
    const bool interior = x >= 0 && x < g.nx && y >= 0 && y < g.ny && z >= 0 && z < nz_global;
    const double2 zero = make_double2(0.0, 0.0);
    for (int a = 0; a < 12; ++a) A.f[a][p] = zero;
    if (!interior) {
      for (int k = 0; k < 12; ++k) {
        const_cast<double2*>(A.t[k])[p] = zero;
        const_cast<double2*>(A.c[k])[p] = zero;
      }
      for (int k = 0; k < 4; ++k) const_cast<double2*>(A.src[k])[p] = zero;
      continue;
    }
    const double* m = mats + (((long long)(z - z_mat0) * g.ny + y) * g.nx + x) * 5;
    const dcx eps = cx(m[0], m[1]);
    const double mu = m[2], sigma = m[3], sigma_star = m[4];
    const unsigned long long cell = ((unsigned long long)z * g.ny + y) * g.nx + x;
    auto fail_at = [&](int comp, unsigned code) {
      atomicMin(err, (((unsigned long long)comp * ncells + cell) << 3) | code);
    };
    // per-cell checks of fill_coefficients (:70-72), first component first
    if (mu == 0.0) { fail_at(0, 1); continue; }
    if (eps.re == 0.0 && eps.im == 0.0) { fail_at(0, 2); continue; }
    // H family (:29-36)
    const dcx den_h = cadd(sp.ep_h, cx(sp.tau * sigma_star / mu, 0.0));
    const bool bad_h = den_h.re == 0.0 && den_h.im == 0.0;
    const dcx t_h = cdiv(sp.em_h, den_h);
    const dcx c_h = cdiv(cx(sp.tau / (mu * sp.delta), 0.0), den_h);
    const dcx s_h = cdiv(cscale(sp.tau, sp.src_h), den_h);
    // E family: forward (:37-45) or back (:46-53) by select_mode (coefficients.hpp:50-53)
    dcx t_e, c_e, s_e;
    bool bad_e;
    const dcx ed = cscale(sp.delta, eps);  // eps * delta
    if (!(eps.re < 0.0)) {
      const dcx den = cadd(cx(1.0, 0.0), cdiv(cx(sp.tau * sigma, 0.0), eps));
      bad_e = den.re == 0.0 && den.im == 0.0;
      t_e = cdiv(sp.em_1, den);
      c_e = cdiv(cmul(cdiv(cx(sp.tau, 0.0), ed), sp.em_h), den);
      s_e = cdiv(cmul(cscale(sp.tau, sp.em_1), sp.src_e), den);
    } else {
      const dcx den = csub(cx(1.0 / sp.tau, 0.0), cdiv(cx(sigma, 0.0), eps));
      bad_e = den.re == 0.0 && den.im == 0.0;
      t_e = cdiv(sp.ep_1, cscale(sp.tau, den));
      c_e = cdiv(cmul(cneg(cdiv(cx(1.0, 0.0), ed)), sp.ep_h), den);
      s_e = cdiv(cneg(sp.src_e), den);
    }
    if (bad_e) fail_at(EXY, eps.re < 0.0 ? 4 : 3);  // E components come first in the table
    if (bad_h) fail_at(HXY, 3);                     // H: always forward
    for (int k = 0; k < 12; ++k) {
      const bool e = k < HXY;
      const double sign = (e ? -1.0 : 1.0) * kCurl[k];
      const dcx t = e ? t_e : t_h, c = cscale(sign, e ? c_e : c_h);
      const_cast<double2*>(A.t[k])[p] = make_double2(t.re, t.im);
      const_cast<double2*>(A.c[k])[p] = make_double2(c.re, c.im);
    }
    const bool on = z == sp.zsrc;
    const_cast<double2*>(A.src[SRC_EXZ])[p] = on ? make_double2(s_e.re, s_e.im) : zero;
    const_cast<double2*>(A.src[SRC_EYZ])[p] = on ? make_double2(s_e.re, s_e.im) : zero;
    const_cast<double2*>(A.src[SRC_HXZ])[p] = on ? make_double2(s_h.re, s_h.im) : zero;
    const_cast<double2*>(A.src[SRC_HYZ])[p] = on ? make_double2(s_h.re, s_h.im) : zero;
  }
}

__global__ void k_selftest_cdiv(int n, const double* in, double* out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const dcx q = cdiv(cx(in[4 * i], in[4 * i + 1]), cx(in[4 * i + 2], in[4 * i + 3]));
    out[2 * i] = q.re;
    out[2 * i + 1] = q.im;
  }
}

// Sanitizer check of one pass (the reference's exactly-once
// UpdateLog coverage, tools/main.cpp:20-41): every (component, interior cell) of
// the slab's local grid was stored exactly once, no ghost ever; the counts are
// reset for the next pass.
// Interior cells (x/y ghost ring excluded) of `nplanes` consecutive padded
// planes of the 12 fields, src -> dst: TBLOCK-in-place copy-back.  The ring is
// input data the sweep never writes, and the spare planes never hold it.
struct Planes12 {
  double2* p[12];
};
// The x / y ghost ring of `nplanes` consecutive padded planes of the 12 fields,
// src -> dst (TBLOCK in place: the sweep stores interior cells only, and the
// ring -- input data, never updated -- must follow the planes it belongs to).
// grid: x = ring segments (grid-stride), y = plane, z = field
__global__ void k_copy_ring(Planes12 dst, Planes12 src, int nplanes, int nx, int ny, long long px,
                            long long pxy, const unsigned* nonzero) {
  if (*nonzero == 0) return;  // every ring cell of the field region is +0.0: nothing moves
  const int k = blockIdx.z, z = blockIdx.y;
  double2* __restrict__ d = dst.p[k] + (long long)z * pxy;
  const double2* __restrict__ sp = src.p[k] + (long long)z * pxy;
  const long long last = (long long)(ny + 1) * px;
  const int ncell = 2 * (int)px + 2 * ny;  // rows y = -1, ny; columns x = -1, nx
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
    long long i;
    if (c < px) i = c;
    else if (c < 2 * px) i = last + (c - px);
    else {
      const int r = c - 2 * (int)px;  // 0 .. 2 ny - 1
      const int y = 1 + (r >> 1);
      i = (long long)y * px + ((r & 1) ? nx + 1 : 0);
    }
    d[i] = sp[i];
  }
}

// *nonzero |= 1 when any x/y ghost-ring cell of planes [0, nplanes) of the 12
// field arrays is not +0.0 (bitwise).  TBLOCK in place runs it once per call
// over the whole field region (array + gap): when every ring cell is zero --
// the device generators' and the usual uploaded states' Dirichlet halo --
// moving the rings with the array is a no-op and k_copy_ring exits at once.
__global__ void k_ring_nonzero(Planes12 src, int nplanes, int nx, int ny, long long px,
                               long long pxy, unsigned* nonzero) {
  const int k = blockIdx.z;
  const long long last = (long long)(ny + 1) * px;
  const int ncell = 2 * (int)px + 2 * ny;
  bool nz = false;
  for (int z = blockIdx.y; z < nplanes; z += gridDim.y) {
    const double2* __restrict__ sp = src.p[k] + (long long)z * pxy;
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncell; c += gridDim.x * blockDim.x) {
      long long i;
      if (c < px) i = c;
      else if (c < 2 * px) i = last + (c - px);
      else {
        const int r = c - 2 * (int)px;
        i = (long long)(1 + (r >> 1)) * px + ((r & 1) ? nx + 1 : 0);
      }
      const double2 v = sp[i];
      nz |= (__double_as_longlong(v.x) | __double_as_longlong(v.y)) != 0;
    }
  }
  if (__syncthreads_or(nz) && threadIdx.x == 0) atomicOr(nonzero, 1u);
}

__global__ void k_coverage(Grid g, unsigned* cnt, long long cstride, int r0, int r1,
                           unsigned long long* bad) {
  const long long n = (long long)(g.nz + 2) * g.pxy;
  unsigned long long b = 0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
       p += (long long)gridDim.x * blockDim.x) {
    const int zp = (int)(p / g.pxy);
    const long long r = p - (long long)zp * g.pxy;
    const int yp = (int)(r / g.px);
    const int xp = (int)(r - (long long)yp * g.px);
    const bool interior =
        xp >= 1 && xp <= g.nx && yp >= 1 && yp <= g.ny && zp >= 1 + r0 && zp <= r1;  // r: zp - 1
    const unsigned want = interior ? 1u : 0u;
    for (int k = 0; k < 12; ++k) {
      unsigned* c = cnt + (long long)k * cstride + p;
      b += *c != want;
      *c = 0u;
    }
  }
  for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  if ((threadIdx.x & 31) == 0 && b) atomicAdd(bad, b);
}

// Interior comparison of one field array against a reference copy.
// acc[0] += sum |a-b|^2, acc[1] += sum |b|^2; cnt += bit mismatches.
__global__ void k_compare(Grid g, const double2* __restrict__ a, const double2* __restrict__ b,
                          double* acc, unsigned long long* cnt) {
  double num = 0.0, den = 0.0;
  unsigned long long c = 0;
  const long long n = (long long)g.nx * g.ny * g.nz;
  for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(q % g.nx);
    const long long r = q / g.nx;
    const int y = (int)(r % g.ny);
    const int z = (int)(r / g.ny);
    const long long i = g.idx(x, y, z);
    const double2 va = a[i], vb = b[i];
    const double dr = va.x - vb.x, di = va.y - vb.y;
    num += dr * dr + di * di;
    den += vb.x * vb.x + vb.y * vb.y;
    if (__double_as_longlong(va.x) != __double_as_longlong(vb.x) ||
        __double_as_longlong(va.y) != __double_as_longlong(vb.y))
      ++c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], num);
    atomicAdd(&acc[1], den);
    atomicAdd(cnt, c);
  }
}

int sm_count(int dev) {
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int pick_zchunk(const thiim_gpu_ctx* ctx, const Slab& s, long long cols, int user) {
  if (user > 0) return std::min(user, s.g.nz);
  // enough CTAs for >= ~8 per SM, but chunks no shorter than 16 planes
  const long long want = 8LL * sm_count(s.device);
  long long chunks = (want + cols - 1) / cols;
  chunks = std::max(1LL, std::min(chunks, (long long)std::max(1, s.g.nz / 16)));
  (void)ctx;
  return (int)((s.g.nz + chunks - 1) / chunks);
}

// Exchange halo planes between neighbouring slabs (single-process multi-GPU).
// which: 0 = E top halo (slab s's plane z1 <- slab s+1's first interior plane),
//        1 = H bottom halo (slab s's plane z0-1 <- slab s-1's last interior plane).
int exchange(thiim_gpu_ctx* ctx, int which) {
  const int n = (int)ctx->slabs.size();
  if (n < 2) return THIIM_OK;
  const long long pxy = ctx->pxy();
  const size_t bytes = (size_t)pxy * sizeof(double2);
  for (int s = 0; s < n; ++s) {
    Slab& me = ctx->slabs[s];
    if (which == 0 && s + 1 < n) {
      const Slab& nb = ctx->slabs[s + 1];
      for (int k = EXY; k <= EZY; ++k)
        CK(cudaMemcpyPeerAsync(me.field(me.cur, k) + (size_t)(me.g.nz + 1) * pxy, me.device,
                               nb.field(nb.cur, k) + (size_t)1 * pxy, nb.device, bytes,
                               me.stream));
    }
    if (which == 1 && s > 0) {
      const Slab& nb = ctx->slabs[s - 1];
      for (int k = HXY; k <= HZY; ++k)
        CK(cudaMemcpyPeerAsync(me.field(me.cur, k), me.device,
                               nb.field(nb.cur, k) + (size_t)nb.g.nz * pxy, nb.device, bytes,
                               me.stream));
    }
  }
  // the copies are issued on the receiver's stream; the sender must not
  // overwrite before they land: serialize by synchronizing all streams.
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
  }
  return THIIM_OK;
}

// Fused engines (single-process multi-GPU): before a step, each interface gets
// the lower slab's last plane (E + Hxy,Hxz,Hyx,Hyz: the upper slab recomputes
// H_new there) and the upper slab's first plane (E) copied into the halo
// planes, peer to peer over NVLink.  Same data the multi-process path moves
// with NCCL (thiim_gpu_halo_view).
int exchange_fused(thiim_gpu_ctx* ctx) {
  const int n = (int)ctx->slabs.size();
  const size_t pbytes = (size_t)ctx->pxy() * sizeof(double2);
  for (auto& sl : ctx->slabs) {  // previous step finished everywhere
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
  }
  for (int s = 0; s + 1 < n; ++s) {
    Slab& lo = ctx->slabs[s];
    Slab& hi = ctx->slabs[s + 1];
    CK(cudaSetDevice(hi.device));
    for (int k = 0; k < 10; ++k)  // lo's plane nz -> hi's plane 0
      CK(cudaMemcpyPeerAsync(hi.field(hi.cur, k), hi.device,
                             lo.field(lo.cur, k) + (size_t)lo.g.nz * lo.g.pxy, lo.device, pbytes,
                             hi.stream));
    CK(cudaSetDevice(lo.device));
    for (int k = 0; k < 6; ++k)  // hi's plane 1 -> lo's plane nz+1
      CK(cudaMemcpyPeerAsync(lo.field(lo.cur, k) + (size_t)(lo.g.nz + 1) * lo.g.pxy, lo.device,
                             hi.field(hi.cur, k) + (size_t)hi.g.pxy, hi.device, pbytes, lo.stream));
  }
  return THIIM_OK;
}

// Deep-halo exchange (TBLOCK slabs), after a pass: per interface the lower
// slab's two last owned planes -> the upper slab's ghost + extended planes, and
// the upper slab's two first owned planes -> the lower slab's extended + ghost
// planes; all 12 fields of the current set.
int deep_first_plane(const Slab& sl, int which) {  // local padded plane of a 2-plane view
  switch (which) {
    case THIIM_HALO_SEND_DOWN: return 1 + sl.ext_lo;         // owned own0, own0+1
    case THIIM_HALO_RECV_DOWN: return 0;                     // ghost own0-2, extended own0-1
    case THIIM_HALO_SEND_UP: return sl.g.nz - 1 - sl.ext_hi;  // owned own1-2, own1-1
    default: return sl.g.nz;                                 // extended own1, ghost own1+1
  }
}

// Store plan of slab `k` for its next TBLOCK pass (before any slab of the pass
// is launched: launches flip the current field set).  Deep slabs store their
// owned planes; with peer stores they also write their two boundary planes at
// each internal interface straight into the neighbour's halo (SEND_* -> RECV_*
// of the deep-halo protocol, the neighbour's output set).
// Stream memory operations (driver API) for the device-side pass counters of
// multi-process peer stores.
struct StreamMemOps {
  CUresult (*wait64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
  CUresult (*write64)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
};
const StreamMemOps* stream_mem_ops() {
  static StreamMemOps ops{nullptr, nullptr};
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* w = nullptr;
    void* v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue64", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q2 == cudaDriverEntryPointSuccess) {
      ops.wait64 = reinterpret_cast<decltype(ops.wait64)>(w);
      ops.write64 = reinterpret_cast<decltype(ops.write64)>(v);
    }
    cudaGetLastError();
  }
  return ops.wait64 && ops.write64 ? &ops : nullptr;
}
CUresult stream_wait_geq(cudaStream_t s, unsigned long long* addr, unsigned long long v) {
  return stream_mem_ops()->wait64((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ);
}
// default flags: a system-scope memory fence orders the prior work's stores
// (the pass's peer stores) before the counter write
CUresult stream_write(cudaStream_t s, unsigned long long* addr, unsigned long long v) {
  return stream_mem_ops()->write64((CUstream)s, (CUdeviceptr)addr, v, CU_STREAM_WRITE_VALUE_DEFAULT);
}

PeerOut peer_out(const thiim_gpu_ctx* ctx, int k) {
  const Slab& sl = ctx->slabs[k];
  PeerOut po{};
  po.st0 = sl.deep ? sl.ext_lo : 0;
  po.st1 = sl.deep ? sl.g.nz - sl.ext_hi : sl.g.nz;
  if (!ctx->peer_stores) return po;
  const long long pxy = sl.g.pxy;
  if (ctx->slabs.size() == 1) {  // neighbours in other processes (IPC), same cur parity
    const int out = sl.cur ^ 1;
    if (const Slab::Peer& p = sl.peer[0]; p.base) {  // lower: its RECV_UP = its plane nz
      for (int c = 0; c < 12; ++c) po.lo[c] = p.base + (size_t)(out * 12 + c) * p.stride;
      po.lo_r0 = sl.ext_lo;
      po.lo_r1 = sl.ext_lo + 2;
      po.lo_shift = (long long)(p.nz - deep_first_plane(sl, THIIM_HALO_SEND_DOWN)) * pxy;
    }
    if (const Slab::Peer& p = sl.peer[1]; p.base) {  // upper: its RECV_DOWN = its plane 0
      for (int c = 0; c < 12; ++c) po.hi[c] = p.base + (size_t)(out * 12 + c) * p.stride;
      po.hi_r0 = sl.g.nz - 2 - sl.ext_hi;
      po.hi_r1 = sl.g.nz - sl.ext_hi;
      po.hi_shift = (long long)(0 - deep_first_plane(sl, THIIM_HALO_SEND_UP)) * pxy;
    }
    return po;
  }
  if (k > 0) {
    const Slab& lo = ctx->slabs[k - 1];
    for (int c = 0; c < 12; ++c) po.lo[c] = lo.field(lo.cur ^ 1, c);
    po.lo_r0 = sl.ext_lo;
    po.lo_r1 = sl.ext_lo + 2;
    po.lo_shift = (long long)(deep_first_plane(lo, THIIM_HALO_RECV_UP) -
                              deep_first_plane(sl, THIIM_HALO_SEND_DOWN)) * pxy;
  }
  if (k + 1 < (int)ctx->slabs.size()) {
    const Slab& hi = ctx->slabs[k + 1];
    for (int c = 0; c < 12; ++c) po.hi[c] = hi.field(hi.cur ^ 1, c);
    po.hi_r0 = sl.g.nz - 2 - sl.ext_hi;
    po.hi_r1 = sl.g.nz - sl.ext_hi;
    po.hi_shift = (long long)(deep_first_plane(hi, THIIM_HALO_RECV_DOWN) -
                              deep_first_plane(sl, THIIM_HALO_SEND_UP)) * pxy;
  }
  return po;
}

// make slab k's stream wait for its neighbours' last pass (their peer stores
// into k's halos, and their reads of the halos k's next pass overwrites)
int wait_neighbours(thiim_gpu_ctx* ctx, int k) {
  Slab& sl = ctx->slabs[k];
  CK(cudaSetDevice(sl.device));
  if (k > 0) CK(cudaStreamWaitEvent(sl.stream, ctx->slabs[k - 1].ev_pass, 0));
  if (k + 1 < (int)ctx->slabs.size()) CK(cudaStreamWaitEvent(sl.stream, ctx->slabs[k + 1].ev_pass, 0));
  return THIIM_OK;
}

int exchange_deep(thiim_gpu_ctx* ctx) {
  const int n = (int)ctx->slabs.size();
  const size_t bytes2 = 2 * (size_t)ctx->pxy() * sizeof(double2);
  for (auto& sl : ctx->slabs) {  // the pass finished everywhere
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
  }
  for (int s = 0; s + 1 < n; ++s) {
    Slab& lo = ctx->slabs[s];
    Slab& hi = ctx->slabs[s + 1];
    const size_t lo_send = (size_t)deep_first_plane(lo, THIIM_HALO_SEND_UP) * lo.g.pxy;
    const size_t lo_recv = (size_t)deep_first_plane(lo, THIIM_HALO_RECV_UP) * lo.g.pxy;
    const size_t hi_send = (size_t)deep_first_plane(hi, THIIM_HALO_SEND_DOWN) * hi.g.pxy;
    const size_t hi_recv = (size_t)deep_first_plane(hi, THIIM_HALO_RECV_DOWN) * hi.g.pxy;
    CK(cudaSetDevice(hi.device));
    for (int k = 0; k < 12; ++k)
      CK(cudaMemcpyPeerAsync(hi.field(hi.cur, k) + hi_recv, hi.device, lo.field(lo.cur, k) + lo_send,
                             lo.device, bytes2, hi.stream));
    CK(cudaSetDevice(lo.device));
    for (int k = 0; k < 12; ++k)
      CK(cudaMemcpyPeerAsync(lo.field(lo.cur, k) + lo_recv, lo.device, hi.field(hi.cur, k) + hi_send,
                             hi.device, bytes2, lo.stream));
  }
  return THIIM_OK;
}

int launch_split(thiim_gpu_ctx* ctx, Slab& s, int fam, long long* launches) {
  CK(cudaSetDevice(s.device));
  const Arrays A = s.arrays(s.cur, s.cur);
  const dim3 block(kSplitBX, kSplitBY);
  const long long cols = (long long)((s.g.nx + kSplitBX - 1) / kSplitBX) *
                         ((s.g.ny + kSplitBY - 1) / kSplitBY);
  const int zc = pick_zchunk(ctx, s, cols, ctx->opts.z_chunk);
  const dim3 grid((s.g.nx + kSplitBX - 1) / kSplitBX, (s.g.ny + kSplitBY - 1) / kSplitBY,
                  (s.g.nz + zc - 1) / zc);
  if (fam == 0)
    (s.cnt ? k_split_h<kSplitBY, true> : k_split_h<kSplitBY, false>)<<<grid, block, 0, s.stream>>>(
        s.g, A, zc);
  else
    (s.cnt ? k_split_e<kSplitBY, true> : k_split_e<kSplitBY, false>)<<<grid, block, 0, s.stream>>>(
        s.g, A, zc);
  CK(cudaGetLastError());
  ++*launches;
  return THIIM_OK;
}

// z-chunk count for a grid of `cols` column tiles with `per_sm` resident CTAs
// per SM: minimise (waves x planes-per-CTA incl. ~1.5 planes of prologue).
int balanced_zchunk(const Slab& s, long long cols, int per_sm, int user) {
  if (user > 0) return std::min(user, s.g.nz);
  const long long slots = (long long)sm_count(s.device) * per_sm;
  double best = 1e300;
  int best_c = 1;
  for (int c = 1; c <= std::max(1, s.g.nz / 4); ++c) {
    const int planes = (s.g.nz + c - 1) / c;
    const long long ctas = cols * c;
    const long long waves = (ctas + slots - 1) / slots;
    const double t = (double)waves * (planes + 1.5);
    if (t < best - 1e-9) {
      best = t;
      best_c = c;
    }
  }
  return (s.g.nz + best_c - 1) / best_c;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

int map_index(int by) {
  return by == 8 ? 0 : by == 16 ? 1 : by == 15 ? 2 : by == 12 ? 3 : by == 14 ? 4 : by == 13 ? 5 : -1;
}
// (each tile height gets its own set of box shapes)

// tensor maps for tile height `by` and thread-tile width `width` (32, or a
// 16 / 8 lane segment of a folded CTA: every box 32 - width columns narrower)
TmaMaps& tmaps(Slab& s, int by, int width = 32, bool fused = false) {
  const int w = map_index(by);
  if (fused) return s.fmaps[w];
  return width == 32 ? s.maps[w] : s.maps_seg[w][width == 16 ? 0 : 1];
}
// coefficient maps: the same maps unless the slab is a view with its own
// coefficient base (TBLOCK in place)
TmaMaps& ctmaps(Slab& s, int by, int width = 32) {
  if (!s.cbuf) return tmaps(s, by, width);
  const int w = map_index(by);
  return width == 32 ? s.cmaps[w] : s.cmaps_seg[w][width == 16 ? 0 : 1];
}

// L2 promotion (measured, profiles/r02x_l2_promotion.md): the TBLOCK sweeps take
// 64-B promotion -- box rows start 16 B into a 32-B sector, and fetching the
// sector pair brings the x-neighbour's overlap along: 3.4% fewer DRAM read bytes
// per pass at configs[2], +0.2-0.3% on every TBLOCK kernel; 128 B: no change;
// 256 B: -1% and +7% DRAM reads.  The one-step sweeps (`fused`: their own map
// set) stay without promotion (64 B: -1.8%).
int ensure_tmap(Slab& s, int by, int width = 32, bool fused = false) {
  const int w = map_index(by);
  if (w < 0) return fail(THIIM_ERR_CONFIG, "no tensor maps for tile height " + std::to_string(by));
  if (width != 32 && width != 16 && width != 8)
    return fail(THIIM_ERR_CONFIG, "no tensor maps for tile width " + std::to_string(width));
  if (fused && (width != 32 || s.cbuf))
    return fail(THIIM_ERR_CONFIG, "internal: the one-step sweeps run full-width tiles, no views");
  bool& ok = fused ? s.fmaps_ok[w]
                   : width == 32 ? s.maps_ok[w] : s.maps_seg_ok[w][width == 16 ? 0 : 1];
  if (ok) return THIIM_OK;
  auto fn = get_encode_fn();
  if (!fn) return fail(THIIM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  int bw[NBOX] = {32, 31, 31, 30, 30, 29, 28, 27, 26};  // BoxGeom
  for (int b = 0; b < NBOX; ++b) bw[b] = std::max(1, bw[b] - (32 - width));
  int bh[NBOX] = {by, by - 1, by - 2, by - 1, by - 2, by - 3, by - 4, by - 5, by - 6};
  for (int b = 0; b < NBOX; ++b) bh[b] += (32 / width - 1) * (by - 4);  // folded: all segments
  // one map set over `narr` arrays of `astride` elements from `base`
  auto encode = [&](TmaMaps& out, void* base, int narr, size_t astride) -> int {
    const cuuint64_t dims[4] = {(cuuint64_t)(2 * s.g.px), (cuuint64_t)(s.g.pxy / s.g.px),
                                (cuuint64_t)(s.g.nz + 2), (cuuint64_t)narr};
    const cuuint64_t strides[3] = {(cuuint64_t)s.g.px * 16, (cuuint64_t)s.g.pxy * 16,
                                   (cuuint64_t)astride * 16};
    const CUtensorMapL2promotion promo =
        fused ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    for (int b = 0; b < NBOX; ++b) {
      const cuuint32_t box[4] = {(cuuint32_t)(2 * bw[b]), (cuuint32_t)bh[b], 1, 1};
      const cuuint32_t estr[4] = {1, 1, 1, 1};
      CUresult r = fn(&out.m[b], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, base, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS)
        return fail(THIIM_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
    }
    return THIIM_OK;
  };
  int r;
  if (s.cbuf) {  // view with separate field / coefficient strides (TBLOCK in place)
    if ((r = encode(tmaps(s, by, width), s.buf, 12 * s.nfield_sets, s.fs()))) return r;
    if ((r = encode(ctmaps(s, by, width), s.cbuf, 28, s.stride))) return r;
  } else {
    if (s.fs() != s.stride)
      return fail(THIIM_ERR_CONFIG, "internal: field stride differs; the sweep needs a view");
    if ((r = encode(tmaps(s, by, width, fused), s.buf, s.n_arrays(), s.stride))) return r;
  }
  ok = true;
  return THIIM_OK;
}

template <int BY, int NG>
int launch_fused_tma_t(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  const Arrays A = s.arrays(s.cur, s.cur ^ 1);
  const int cur = s.cur, nf = s.nfield_sets;
  int r = ensure_tmap(s, BY, 32, true);
  if (r) return r;
  constexpr int TX = 30, TY = BY - 2;
  const size_t smem = sizeof(FusedSmem<BY, NG>);
  static std::atomic<unsigned> attr_set{0};  // the attribute is per function and device
  if (setup_needed(attr_set, s.device)) {
    CK(cudaFuncSetAttribute(k_fused_tma<BY, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    CK(cudaFuncSetAttribute(k_fused_tma<BY, NG, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    setup_done(attr_set, s.device);
  }
  const long long cols = (long long)((s.g.nx + TX - 1) / TX) * ((s.g.ny + TY - 1) / TY);
  const int zc = balanced_zchunk(s, cols, 1, ctx->opts.z_chunk);
  const int tiles_y = (s.g.ny + TY - 1) / TY;
  const int tiles_x = (s.g.nx + TX - 1) / TX;
  const dim3 grid(tiles_x * tiles_y, 1, (s.g.nz + zc - 1) / zc);
  const dim3 block(32, BY + 1);
  (s.cnt ? k_fused_tma<BY, NG, true> : k_fused_tma<BY, NG, false>)<<<grid, block, smem, s.stream>>>(
      s.g, A, tmaps(s, BY, 32, true), zc, tiles_x, cur * 12, nf * 12);
  CK(cudaGetLastError());
  s.cur ^= 1;
  ++*launches;
  return THIIM_OK;
}

// ---- TBLOCK (two steps per pass)
// z-chunks of a TBLOCK launch: minimise waves x (planes + overhead) over one
// CTA per SM.  A chunk start re-does ~2 planes of level-1/level-2 work, re-reads
// their boxes and fills the ring from empty; measured at configs[4] (r02y: one
// 128-plane chunk in 24 rounds vs two 64-plane chunks in 47, +1.4%) the whole
// costs the depth-2 kernel ~4.7 plane-iterations, hence its 4.5
int tblock_zchunk(const Slab& s, long long cols, double overhead = 2.0, int span = 0) {
  const long long slots = sm_count(s.device);
  const int nz = span > 0 ? span : s.g.nz;  // planes the chunks cover
  double best = 1e300;
  int best_c = 1;
  for (int c = 1; c <= std::max(1, nz / 8); ++c) {
    const int planes = (nz + c - 1) / c;
    const long long waves = (cols * c + slots - 1) / slots;
    const double t = (double)waves * (planes + overhead);
    if (t < best - 1e-9) {
      best = t;
      best_c = c;
    }
  }
  return (nz + best_c - 1) / best_c;
}

// slot bases of the 4-D tensor maps: current field set, first coefficient
int cur_slot(const Slab& s) { return s.cur * 12; }
int nf_slot(const Slab& s) { return s.nfield_sets * 12; }

// Tile columns per band of a round-scheduled TBLOCK pass (TileOrder,
// thiim_tblock.cuh).  A round of G tiles as a band x (G / band) block re-fetches
// the y-overlap of its `band` bottom tiles (~50 KB per tile-plane of level-1
// boxes: 105 array-rows of ~30 cells) and the x-overlap of its G / band side
// tiles (~23 KB: 1445 cells); band ~ sqrt(G * 23 / 50) ~ 8 minimises the sum.
// Bands are made equal-width.
int tblock_band(int tiles_x, int per_round, int user) {
  if (user > 0) return std::min(user, tiles_x);
  const double b = std::sqrt((double)per_round * 23.0 / 50.0);
  const int nb = std::max(1, (int)std::ceil(tiles_x / b));
  return (tiles_x + nb - 1) / nb;
}

template <int BY, int NG>
int launch_tblock2_t(thiim_gpu_ctx* ctx, Slab& s, long long* launches, const PeerOut& po) {
  if (!s.deep && (s.g.halo_lo || s.z1 < ctx->dims.nz))
    return fail(THIIM_ERR_CONFIG, "TBLOCK on a slab needs a deep-halo slab context");
  const Arrays A = s.arrays(s.cur, s.cur ^ 1);
  const int cur = s.cur, nf = s.nfield_sets;
  int r = ensure_tmap(s, BY);
  if (r) return r;
  const size_t smem = sizeof(TmSmem<BY, NG>);
  static std::atomic<unsigned> attr_set{0};
  if (setup_needed(attr_set, s.device)) {
    const int tm_smem = (int)smem;
    CK(cudaFuncSetAttribute(k_tblock_tm<BY, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            tm_smem));
    CK(cudaFuncSetAttribute(k_tblock_tm<BY, NG, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, tm_smem));
    if constexpr (BY == 15) {
      for (auto f : {k_tblock_tm<BY, NG, false, 8>, k_tblock_tm<BY, NG, true, 8>,
                     k_tblock_tm<BY, NG, false, 16>, k_tblock_tm<BY, NG, true, 16>,
                     k_tblock_tm<BY, NG, false, 0, 1>, k_tblock_tm<BY, NG, true, 0, 1>,
                     k_tblock_tm<BY, NG, false, 8, 1>, k_tblock_tm<BY, NG, true, 8, 1>,
                     k_tblock_tm<BY, NG, false, 16, 1>, k_tblock_tm<BY, NG, true, 16, 1>,
                     k_tblock_tm<BY, NG, false, 0, 2>, k_tblock_tm<BY, NG, false, 8, 2>,
                     k_tblock_tm<BY, NG, false, 16, 2>})
        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, tm_smem));
    }
    setup_done(attr_set, s.device);
  }
  constexpr int TX2 = 28, TY2 = BY - 4;
  int tiles_x = (s.g.nx + TX2 - 1) / TX2;
  const int tiles_y = (s.g.ny + TY2 - 1) / TY2;
  // remainder column of <= 12 grid columns: folded CTAs of 16- or 8-lane
  // segments (2 or 4 y-tiles per CTA) instead of a column of full tiles
  int wf = 0, n_fold = 0;
  const int rem = s.g.nx - (s.g.nx / TX2) * TX2;
  static const bool no_fold = std::getenv("THIIM_NO_FOLD") != nullptr;  // A/B knob
  if constexpr (BY == 15) {
    if (!no_fold && s.g.nx >= TX2 && rem > 0 && rem <= 12) {
      wf = rem <= 4 ? 8 : 16;
      tiles_x = s.g.nx / TX2;
      n_fold = (tiles_y + 32 / wf - 1) / (32 / wf);
      if ((r = ensure_tmap(s, BY, wf))) return r;
    }
  }
  const int n_main = tiles_x * tiles_y, nbt = n_main + n_fold;
  // in-place views, and deep slabs without folded tiles: chunks cover planes
  // [0, st1) (level 2 stops below the top halo plane; k_tblock_tm zhi)
  const bool view = s.deep && s.fo_base != nullptr;
  const int span = view ? po.st1 - po.st0 : s.deep && wf == 0 ? po.st1 : s.g.nz;
  int zc = ctx->opts.z_chunk;
  if (zc <= 0) zc = tblock_zchunk(s, (long long)nbt, 4.5, span);
  const int nchunks = (span + zc - 1) / zc;
  const long long items = (long long)nbt * nchunks;
  // CTA schedule: rounds of at most one CTA per SM in band order (default), or
  // (schedule 1) one launch of every item in x-fastest order
  const int sms = sm_count(s.device);
  const bool one_launch = ctx->opts.schedule == 1;
  const long long rounds = one_launch ? 1 : (items + sms - 1) / sms;
  const long long per_round = (items + rounds - 1) / rounds;
  TileOrder ord;
  ord.nbt = nbt;
  ord.tiles_y = tiles_y;
  ord.band = one_launch ? tiles_x : tblock_band(tiles_x, (int)std::min<long long>(per_round, sms),
                                                 ctx->opts.band);
  const dim3 block(32, BY + 1);
  // sanitizer negative control (tests only): THIIM_SANITIZE_UNCOUNTED=1 runs the
  // uninstrumented instances while the sanitizer is on, so every store must be
  // reported missing
  const bool c = s.cnt != nullptr && !std::getenv("THIIM_SANITIZE_UNCOUNTED");
  if (view && c) return fail(THIIM_ERR_CONFIG, "the sanitizer does not count in-place views");
  auto kern = c ? k_tblock_tm<BY, NG, true> : k_tblock_tm<BY, NG, false>;
  if constexpr (BY == 15) {
    if (view) {  // in-place sub-range view: owned-plane stores only
      kern = wf == 8 ? k_tblock_tm<BY, NG, false, 8, 2>
             : wf == 16 ? k_tblock_tm<BY, NG, false, 16, 2> : k_tblock_tm<BY, NG, false, 0, 2>;
    } else if (s.deep) {  // owned-plane stores + peer stores (multi-GPU slabs)
      kern = wf == 8    ? (c ? k_tblock_tm<BY, NG, true, 8, 1> : k_tblock_tm<BY, NG, false, 8, 1>)
             : wf == 16 ? (c ? k_tblock_tm<BY, NG, true, 16, 1>
                             : k_tblock_tm<BY, NG, false, 16, 1>)
                        : (c ? k_tblock_tm<BY, NG, true, 0, 1> : k_tblock_tm<BY, NG, false, 0, 1>);
    } else {
      if (wf == 8) kern = c ? k_tblock_tm<BY, NG, true, 8> : k_tblock_tm<BY, NG, false, 8>;
      if (wf == 16) kern = c ? k_tblock_tm<BY, NG, true, 16> : k_tblock_tm<BY, NG, false, 16>;
    }
  } else if (s.deep) {
    return fail(THIIM_ERR_CONFIG, "deep-halo slabs run TBLOCK at tile height 15");
  }
  for (long long it0 = 0; it0 < items; it0 += per_round) {
    ord.item0 = (int)it0;
    const unsigned n = (unsigned)std::min<long long>(per_round, items - it0);
    kern<<<n, block, smem, s.stream>>>(s.g, A, tmaps(s, BY), tmaps(s, BY, wf ? wf : 32),
                                       ctmaps(s, BY), ctmaps(s, BY, wf ? wf : 32), po, cur * 12,
                                       s.cbuf ? 0 : nf * 12, zc, tiles_x, n_main, ord);
    CK(cudaGetLastError());
    ++*launches;
  }
  s.cur ^= 1;
  return THIIM_OK;
}

template <int BY, int NG>
int launch_tblock_table_t(thiim_gpu_ctx* ctx, Slab& s, long long* launches, const PeerOut& po) {
  if (!s.deep && (s.g.halo_lo || s.z1 < ctx->dims.nz))
    return fail(THIIM_ERR_CONFIG, "TBLOCK on a slab needs a deep-halo slab context");
  const Arrays A = s.arrays(s.cur, s.cur ^ 1);
  int r = ensure_tmap(s, BY);
  if (r) return r;
  TableGrid T;
  T.mat = s.mat;
  T.mp = s.mp;
  T.mplane = s.mplane;
  T.table = s.tab;
  T.n_mat = s.n_mat;
  const size_t smem = sizeof(TbTableSmem<BY, NG>);
  static std::atomic<unsigned> attr_set{0};
  if (setup_needed(attr_set, s.device)) {
    CK(cudaFuncSetAttribute(k_tblock_table<BY, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    CK(cudaFuncSetAttribute(k_tblock_table<BY, NG, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tblock_table<BY, NG, false, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(k_tblock_table<BY, NG, true, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    setup_done(attr_set, s.device);
  }
  constexpr int TX2 = 28, TY2 = BY - 4;
  const int tiles_x = (s.g.nx + TX2 - 1) / TX2, tiles_y = (s.g.ny + TY2 - 1) / TY2;
  int zc = ctx->opts.z_chunk;
  const int nbt = tiles_x * tiles_y;
  const int span = s.deep ? po.st1 : s.g.nz;  // deep slabs: up to the last owned plane
  if (zc <= 0) zc = tblock_zchunk(s, (long long)nbt, 2.0, span);
  const long long items = (long long)nbt * ((span + zc - 1) / zc);
  // rounds of <= one CTA per SM with the tiles in bands, like k_tblock_tm: the
  // y-neighbours of a round stream the same planes together and share their
  // overlapping field rows in L2 (schedule 1: one launch, x-fastest)
  const int sms = sm_count(s.device);
  const bool one_launch = ctx->opts.schedule == 1;
  const long long rounds = one_launch ? 1 : (items + sms - 1) / sms;
  const long long per_round = (items + rounds - 1) / rounds;
  TileOrder ord;
  ord.nbt = nbt;
  ord.tiles_y = tiles_y;
  ord.band = one_launch ? tiles_x : tblock_band(tiles_x, (int)std::min<long long>(per_round, sms),
                                                 ctx->opts.band);
  auto kern = s.deep ? (s.cnt ? k_tblock_table<BY, NG, true, true> : k_tblock_table<BY, NG, false, true>)
                     : (s.cnt ? k_tblock_table<BY, NG, true> : k_tblock_table<BY, NG, false>);
  for (long long it0 = 0; it0 < items; it0 += per_round) {
    ord.item0 = (int)it0;
    const unsigned n = (unsigned)std::min<long long>(per_round, items - it0);
    kern<<<n, dim3(32, BY + 1), smem, s.stream>>>(s.g, A, T, tmaps(s, BY), po, s.cur * 12, zc,
                                                  tiles_x, ord);
    CK(cudaGetLastError());
    ++*launches;
  }
  s.cur ^= 1;
  return THIIM_OK;
}

// Depth-3 TBLOCK pass (k_tblock3_tm, thiim_tblock3.cuh): whole-z slabs only.
template <int BY, int NG>
int launch_tblock3_t(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  if (s.deep || s.g.halo_lo || s.z1 < ctx->dims.nz || s.table)
    return fail(THIIM_ERR_CONFIG, "time_block 3 runs on whole-z contexts in the reference layout");
  const Arrays A = s.arrays(s.cur, s.cur ^ 1);
  int r = ensure_tmap(s, BY);
  if (r) return r;
  const size_t smem = sizeof(TmSmem<BY, NG>);
  static std::atomic<unsigned> attr_set{0};
  if (setup_needed(attr_set, s.device)) {
    CK(cudaFuncSetAttribute(k_tblock3_tm<BY, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    CK(cudaFuncSetAttribute(k_tblock3_tm<BY, NG, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    setup_done(attr_set, s.device);
  }
  constexpr int TX3 = 26, TY3 = BY - 6;
  const int tiles_x = (s.g.nx + TX3 - 1) / TX3, tiles_y = (s.g.ny + TY3 - 1) / TY3;
  const int nbt = tiles_x * tiles_y;
  int zc = ctx->opts.z_chunk;
  // a chunk start re-does ~3 planes of level work (prologues of three levels)
  if (zc <= 0) zc = tblock_zchunk(s, (long long)nbt, 3.0);
  const int nchunks = (s.g.nz + zc - 1) / zc;
  const long long items = (long long)nbt * nchunks;
  const int sms = sm_count(s.device);
  const bool one_launch = ctx->opts.schedule == 1;
  const long long rounds = one_launch ? 1 : (items + sms - 1) / sms;
  const long long per_round = (items + rounds - 1) / rounds;
  TileOrder ord;
  ord.nbt = nbt;
  ord.tiles_y = tiles_y;
  ord.band = one_launch ? tiles_x : tblock_band(tiles_x, (int)std::min<long long>(per_round, sms),
                                                 ctx->opts.band);
  const bool c = s.cnt != nullptr && !std::getenv("THIIM_SANITIZE_UNCOUNTED");
  auto kern = c ? k_tblock3_tm<BY, NG, true> : k_tblock3_tm<BY, NG, false>;
  for (long long it0 = 0; it0 < items; it0 += per_round) {
    ord.item0 = (int)it0;
    const unsigned n = (unsigned)std::min<long long>(per_round, items - it0);
    kern<<<n, dim3(32, BY + 1), smem, s.stream>>>(s.g, A, tmaps(s, BY), cur_slot(s), nf_slot(s), zc,
                                                   tiles_x, ord);
    CK(cudaGetLastError());
    ++*launches;
  }
  s.cur ^= 1;
  return THIIM_OK;
}

int launch_tblock3(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  CK(cudaSetDevice(s.device));
  return launch_tblock3_t<15, THIIM_TB_NG>(ctx, s, launches);
}

int launch_tblock2(thiim_gpu_ctx* ctx, Slab& s, long long* launches, const PeerOut& po) {
  CK(cudaSetDevice(s.device));
  if (s.table) return launch_tblock_table_t<15, 5>(ctx, s, launches, po);
  if (s.deep) return launch_tblock2_t<15, THIIM_TB_NG>(ctx, s, launches, po);
  switch (ctx->opts.tile_y) {  // CTA height incl. the 4 halo rows; ring depth fills the smem
    case 16: return launch_tblock2_t<16, 5>(ctx, s, launches, po);
    case 14: return launch_tblock2_t<14, 6>(ctx, s, launches, po);
    case 12: return launch_tblock2_t<12, 7>(ctx, s, launches, po);
    default: return launch_tblock2_t<15, THIIM_TB_NG>(ctx, s, launches, po);
  }
}

// TBLOCK without a second field set (BASELINE c3 in the reference layout:
// 40 arrays fit in HBM, the 52 of ping-pong TBLOCK do not).  Each field array
// has a gap of D = L + 2 planes above it (fstride = nz + 2 + D planes); at
// rest it sits at the bottom of its region (ip_pos = 0).  A pass sweeps z as
// sub-ranges [a, b) of L planes; each is one TBLOCK pass over the view of
// interior planes [a-1, b+1) plus the plane on either side (a z-slab whose
// halos hold the neighbours' current values -- here the not yet updated state
// itself; k_tblock_tm's view instances, DEEP = 2, sweep only the owned planes
// [a, b) of it) that stores its two-step outputs D planes away from its inputs:
//   even passes shift the array UP into the gap, sub-ranges top-down;
//   odd passes shift it back DOWN, sub-ranges bottom-up.
// Outputs of sub-range [a, b) land on padded planes [a+1, b] of the new
// position, which overlap only inputs of sub-ranges already swept (D = L + 2
// clears the sub-range's own window [a-1, b+2]), so nothing is copied back:
// 416 B/LUP plus the ~4 planes every view re-reads.  The sweep stores interior
// cells only, so the ghost ring of each output plane (only when some ring cell
// is non-zero: k_ring_nonzero) and the two ghost planes follow with small
// copies.  A call that ends on an odd pass moves the array back once (one
// copy), so every other entry point sees the canonical layout.
static int copy_ring(Slab& s, const Planes12& dst, const Planes12& src, int np, long long* launches) {
  k_copy_ring<<<dim3(8, np, 12), 256, 0, s.stream>>>(dst, src, np, s.g.nx, s.g.ny, s.g.px, s.g.pxy,
                                                      s.ring_nz);
  CK(cudaGetLastError());
  ++*launches;
  return THIIM_OK;
}

static Planes12 field_planes(const Slab& s, int phys) {
  Planes12 m;
  for (int k = 0; k < 12; ++k) m.p[k] = s.field(0, k) + (size_t)phys * s.g.pxy;
  return m;
}

static int copy_field_planes(Slab& s, int dst_phys, int src_phys, int np) {
  const size_t bytes = (size_t)np * s.g.pxy * sizeof(double2);
  for (int k = 0; k < 12; ++k)
    CK(cudaMemcpyAsync(s.field(0, k) + (size_t)dst_phys * s.g.pxy,
                       s.field(0, k) + (size_t)src_phys * s.g.pxy, bytes, cudaMemcpyDeviceToDevice,
                       s.stream));
  return THIIM_OK;
}

static int launch_tblock_inplace(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  const int nz = s.g.nz, L = s.ip_L, D = L + 2;
  const long long pxy = s.g.pxy;
  const int pin = s.ip_pos, pout = pin == 0 ? D : 0;
  const bool up = pout > pin;
  int r;
  // the ghost plane on the side the array moves towards goes first (its new
  // home is in the gap); the other one last (its new home is dead input)
  if (up && (r = copy_field_planes(s, pout + nz + 1, pin + nz + 1, 1))) return r;
  if (!up && (r = copy_field_planes(s, pout, pin, 1))) return r;
  // sub-ranges of equal length Lq <= L (a gap of D = L + 2 >= Lq + 2 planes
  // still clears each sub-range's window): 512 planes at L = 170 run as 4 x 128,
  // not 3 x 170 + 2
  const int nsub = (nz + L - 1) / L, Lq = (nz + nsub - 1) / nsub;
  for (int j = 0; j < nsub; ++j) {
    const int a = (up ? nsub - 1 - j : j) * Lq;
    const int b = std::min(nz, a + Lq);
    const int lo = a > 0 ? a - 1 : 0, hi = b < nz ? b + 1 : nz;
    Slab v = s;  // view: interior planes [lo, hi) of the same field region
    v.buf = s.buf + (size_t)(pin + lo) * pxy;
    v.cbuf = s.coeff(12) + (size_t)lo * pxy;
    v.g.nz = hi - lo;
    v.g.halo_lo = lo > 0 ? 1 : 0;
    v.deep = true;
    v.cur = 0;
    v.cnt = nullptr;
    for (auto& ok : v.maps_ok) ok = false;
    for (auto& row : v.maps_seg_ok)
      for (auto& ok : row) ok = false;
    PeerOut po{};
    po.st0 = a - lo;  // owned local planes [st0, st1) = global [a, b)
    po.st1 = b - lo;
    v.fo_base = s.buf + (size_t)(pout + lo) * pxy;  // the same planes at the new position
    v.fo_stride = (long long)s.fs();
    v.fo_shift = 0;
    if ((r = launch_tblock2(ctx, v, launches, po))) return r;
    // the ghost ring of the output planes (padded [a+1, b]) follows them
    if ((r = copy_ring(s, field_planes(s, pout + a + 1), field_planes(s, pin + a + 1), b - a,
                       launches)))
      return r;
  }
  if (up && (r = copy_field_planes(s, pout, pin, 1))) return r;
  if (!up && (r = copy_field_planes(s, pout + nz + 1, pin + nz + 1, 1))) return r;
  s.ip_pos = pout;
  return THIIM_OK;
}

// back to the canonical position (ip_pos 0) after a call that ended on an odd
// pass: planes [D, D + nz + 2) -> [0, nz + 2) in ascending chunks of D planes
// (each chunk's source and destination are disjoint)
static int inplace_restore(Slab& s) {
  if (s.ip_pos == 0) return THIIM_OK;
  const int D = s.ip_pos, np = s.g.nz + 2;
  int r;
  for (int p = 0; p < np; p += D)
    if ((r = copy_field_planes(s, p, p + D, std::min(D, np - p)))) return r;
  s.ip_pos = 0;
  return THIIM_OK;
}

template <int BY, int NG>
int launch_fused_table_t(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  static_assert(BY == 15, "material-id map box height is 15");
  const Arrays A = s.arrays(s.cur, s.cur ^ 1);
  const int cur = s.cur;
  GroupSeq S;
  seq_table(S, [&](int k) { return cur * 12 + k; });
  int r = ensure_tmap(s, BY, 32, true);
  if (r) return r;
  TableMaps maps;
  maps.f = tmaps(s, BY, 32, true);
  TableGrid T;
  T.mat = s.mat;
  T.mp = s.mp;
  T.mplane = s.mplane;
  T.table = s.tab;
  T.n_mat = s.n_mat;
  constexpr int TX = 30, TY = BY - 2;
  const size_t smem = sizeof(TableSmem<BY, NG>);
  static std::atomic<unsigned> attr_set{0};
  if (setup_needed(attr_set, s.device)) {
    CK(cudaFuncSetAttribute(k_fused_table<BY, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
    CK(cudaFuncSetAttribute(k_fused_table<BY, NG, true>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    setup_done(attr_set, s.device);
  }
  const int tiles_x = (s.g.nx + TX - 1) / TX, tiles_y = (s.g.ny + TY - 1) / TY;
  const int zc = balanced_zchunk(s, (long long)tiles_x * tiles_y, 1, ctx->opts.z_chunk);
  const dim3 grid(tiles_x * tiles_y, 1, (s.g.nz + zc - 1) / zc);
  (s.cnt ? k_fused_table<BY, NG, true> : k_fused_table<BY, NG, false>)<<<grid, dim3(32, BY + 1), smem,
                                                                        s.stream>>>(s.g, A, T, maps,
                                                                                    S, zc, tiles_x);
  CK(cudaGetLastError());
  s.cur ^= 1;
  ++*launches;
  return THIIM_OK;
}

int launch_fused(thiim_gpu_ctx* ctx, Slab& s, long long* launches) {
  CK(cudaSetDevice(s.device));
  if (s.table) return launch_fused_table_t<15, 5>(ctx, s, launches);
  if (ctx->opts.tile_y == 8) return launch_fused_tma_t<8, 12>(ctx, s, launches);
  if (ctx->opts.tile_y == 16) return launch_fused_tma_t<16, 5>(ctx, s, launches);
  if (ctx->opts.tile_y == 116) return launch_fused_tma_t<16, 2>(ctx, s, launches);  // stress: tiny ring
  return launch_fused_tma_t<15, 6>(ctx, s, launches);
}

bool valid_dims(const thiim_dims* d) {
  return d && d->nx >= 4 && d->ny >= 4 && d->nz >= 4 && d->ghost == 1;
}

}  // namespace

// ------------------------------------------------------------------ C-ABI

extern "C" {

int thiim_gpu_abi_version(void) { return THIIM_GPU_ABI_VERSION; }

const char* thiim_gpu_last_error(void) { return g_err.c_str(); }

void thiim_gpu_default_opts(thiim_gpu_opts* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->device = 0;
  o->n_gpus = 1;
  o->engine = THIIM_ENGINE_AUTO;
}

double thiim_gpu_balance_model(int engine, int time_block) {
  switch (engine) {
    case THIIM_ENGINE_SPLIT: return 1024.0;
    case THIIM_ENGINE_TBLOCK: return 832.0 / (time_block > 0 ? time_block : 2);
    // one TBLOCK pass per two steps, outputs shifted into the gap (no
    // copy-back; the ghost-ring copies add ~4 / nx of the bytes)
    case THIIM_ENGINE_TBLOCK_INPLACE: return 832.0 / 2;
    // table coefficient layout: 24 fields x 16 B + 1 B id per HBM pass of time_block steps
    case 100 + THIIM_COEFF_TABLE: return 385.0 / (time_block > 0 ? time_block : 1);
    default: return 832.0;
  }
}

// ---- device memory: the slab state comes from the device's stream-ordered
// pool with an unbounded release threshold, so destroying a context keeps the
// pages mapped for the next one (a caching allocator, like torch's): context
// create/destroy stay in the milliseconds, while cudaFree of a 14 GB state
// costs ~0.1 s.  Reserved-but-unused pool memory counts as available.
static cudaMemPool_t device_pool(int dev) {
  static std::atomic<unsigned> configured{0};
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) != cudaSuccess) return nullptr;
  if (setup_needed(configured, dev)) {
    uint64_t thr = UINT64_MAX;
    if (cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess)
      setup_done(configured, dev);
  }
  return pool;
}

static size_t device_available(int dev) {
  size_t freeb = 0, totalb = 0;
  cudaSetDevice(dev);
  cudaMemGetInfo(&freeb, &totalb);
  if (cudaMemPool_t pool = device_pool(dev)) {
    uint64_t reserved = 0, used = 0;
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    if (reserved > used) freeb += (size_t)(reserved - used);
  }
  return freeb;
}

static cudaError_t pool_alloc(void** p, size_t bytes, int dev, cudaStream_t st) {
  cudaError_t e = cudaMallocAsync(p, bytes, st);
  if (e == cudaErrorMemoryAllocation) {  // give cached pages back and retry once
    cudaGetLastError();
    cudaStreamSynchronize(st);
    if (cudaMemPool_t pool = device_pool(dev)) cudaMemPoolTrimTo(pool, 0);
    e = cudaMallocAsync(p, bytes, st);
  }
  return e;
}


// Shared by thiim_gpu_create (n_gpus slabs split like the reference's z_slab,
// reference_engines.cpp:26-30) and thiim_gpu_create_slab (one explicit slab).
// Longest TBLOCK-in-place sub-range a context created on this thread may take
// from free memory (run_batch lowers it so that all its contexts fit).
thread_local int g_ip_max_L = 128;

static int create_impl(const thiim_dims* dims, const thiim_gpu_opts* opts, bool ipc_alloc,
                       const std::vector<std::pair<int, int>>& ranges, thiim_gpu_ctx** out) {
  g_err.clear();
  if (!out) return fail(THIIM_ERR_CONFIG, "out pointer is null");
  *out = nullptr;
  if (!valid_dims(dims))
    return fail(THIIM_ERR_SETUP, "invalid grid dims (need nx,ny,nz >= 4, ghost = 1)");
  thiim_gpu_opts o;
  if (opts)
    o = *opts;
  else
    thiim_gpu_default_opts(&o);
  if (o.n_gpus < 1 || o.n_gpus > 8) return fail(THIIM_ERR_CONFIG, "n_gpus must be in 1..8");
  if (o.engine < THIIM_ENGINE_AUTO || o.engine > THIIM_ENGINE_TBLOCK_INPLACE)
    return fail(THIIM_ERR_CONFIG, "unknown engine");
  if ((o.engine == THIIM_ENGINE_TBLOCK || o.engine == THIIM_ENGINE_AUTO) && o.time_block != 0 &&
      o.time_block != 2 && o.time_block != 3)
    return fail(THIIM_ERR_CONFIG, "engine TBLOCK supports time_block 2 or 3");
  if (o.time_block == 3 && (o.n_gpus > 1 || o.coeff_layout != THIIM_COEFF_FULL))
    return fail(THIIM_ERR_CONFIG,
                "time_block 3 runs on one whole-z slab in the reference coefficient layout");
  const bool table = o.coeff_layout == THIIM_COEFF_TABLE;
  if (o.coeff_layout == THIIM_COEFF_AUTO_HOST)
    return fail(THIIM_ERR_CONFIG, "THIIM_COEFF_AUTO_HOST is resolved by the host adapters "
                                  "(thiim_coeff_compress), not by a context");
  if (o.coeff_layout != THIIM_COEFF_FULL && !table)
    return fail(THIIM_ERR_CONFIG, "unknown coefficient layout");
  if (table && (o.engine == THIIM_ENGINE_SPLIT || o.engine == THIIM_ENGINE_TBLOCK_INPLACE))
    return fail(THIIM_ERR_CONFIG, "the table coefficient layout runs on the fused or TBLOCK engine");
  if (table && (o.n_materials < 1 || o.n_materials > kMaxMaterials))
    return fail(THIIM_ERR_CONFIG, "n_materials must be in 1..16 for the table layout");
  for (const auto& r : ranges)
    if (r.first < 0 || r.second > dims->nz || r.second - r.first < 4)
      return fail(THIIM_ERR_CONFIG, "each z-slab needs at least 4 planes inside the grid");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
    return fail(THIIM_ERR_CUDA, "no CUDA device visible");
  // same_device = 1 (test knob): put every slab on opts->device, so the
  // multi-slab exchange paths can be exercised with one GPU
  const int dev_step = o.same_device == 1 ? 0 : 1;
  if (o.device < 0 || o.device + dev_step * ((int)ranges.size() - 1) >= ndev)
    return fail(THIIM_ERR_CONFIG, "device range exceeds visible devices");

  auto* ctx = new thiim_gpu_ctx;
  ctx->dims = *dims;
  ctx->opts = o;
  const long long pxy = ctx->pxy();
  const int n = (int)ranges.size();
  ctx->engine = o.engine;
  ctx->depth = o.time_block == 3 ? 3 : 2;
  const bool whole_z = n == 1 && ranges[0].first == 0 && ranges[0].second == dims->nz;
  // TBLOCK in place runs on a split (one field set) context plus spare planes
  const bool want_ip = o.engine == THIIM_ENGINE_TBLOCK_INPLACE;
  if (want_ip && !whole_z) {
    delete ctx;
    return fail(THIIM_ERR_CONFIG, "TBLOCK in place needs one whole-z slab");
  }
  if (want_ip) ctx->engine = THIIM_ENGINE_SPLIT;
  // AUTO: TBLOCK (two steps per HBM pass, odd remainders fused; z-slabs keep
  // deep two-plane halos exchanged per pass); the table layout has no split form
  if (table && o.engine == THIIM_ENGINE_AUTO) ctx->engine = THIIM_ENGINE_TBLOCK;
  if (o.engine == THIIM_ENGINE_AUTO && !table) {
    // TBLOCK needs the ping-pong field set (52 arrays); else split in place (40)
    ctx->engine = THIIM_ENGINE_TBLOCK;
    for (int s = 0; s < n; ++s) {
      const size_t freeb = device_available(o.device + dev_step * s);
      const size_t need = (size_t)(ranges[s].second - ranges[s].first + 2) * (size_t)pxy *
                          sizeof(double2) * 52 + ((size_t)256 << 20);
      if (need > freeb) ctx->engine = THIIM_ENGINE_SPLIT;
    }
  }
  const bool auto_split = o.engine == THIIM_ENGINE_AUTO && ctx->engine == THIIM_ENGINE_SPLIT;
  const int nf = ctx->engine == THIIM_ENGINE_SPLIT ? 1 : 2;
  for (int s = 0; s < n; ++s) {
    Slab sl;
    sl.device = o.device + dev_step * s;
    sl.own0 = ranges[s].first;
    sl.own1 = ranges[s].second;
    // TBLOCK slabs keep two-plane halos: one extended interior plane + the ghost
    sl.deep = ctx->engine == THIIM_ENGINE_TBLOCK && !whole_z;
    sl.ext_lo = sl.deep && sl.own0 > 0 ? 1 : 0;
    sl.ext_hi = sl.deep && sl.own1 < dims->nz ? 1 : 0;
    sl.z0 = sl.own0 - sl.ext_lo;
    sl.z1 = sl.own1 + sl.ext_hi;
    sl.g.nx = dims->nx;
    sl.g.ny = dims->ny;
    sl.g.nz = sl.z1 - sl.z0;
    sl.g.px = dims->nx + 2;
    sl.g.pxy = pxy;
    sl.g.halo_lo = sl.z0 > 0 ? 1 : 0;
    sl.nfield_sets = nf;
    sl.table = table;
    sl.n_mat = table ? o.n_materials : 0;
    sl.mp = (dims->nx + 2 + 15) / 16 * 16;
    sl.mplane = sl.mp * (dims->ny + 2);
    sl.stride = ((size_t)(sl.g.nz + 2) * (size_t)pxy + 15) / 16 * 16;
    ctx->slabs.push_back(sl);
  }
  if ((want_ip || auto_split) && whole_z && !table) {
    // TBLOCK in place: every field array gets a gap of D = L + 2 planes above it
    // (launch_tblock_inplace).  THIIM_INPLACE_TB=L forces the sub-range length
    // (0: plain split); default the most planes free memory holds, <= 128
    // (configs[2]: 64 -> 128 planes, 9.63 -> 9.87 GLUP/s; fewer halo re-reads
    // and round starts per pass)
    Slab& sl = ctx->slabs[0];
    const size_t plane = (size_t)pxy * sizeof(double2);
    const char* env = std::getenv("THIIM_INPLACE_TB");
    int L = env ? std::atoi(env) : -1;
    if (L < 0) {
      const size_t state = sl.stride * sizeof(double2) * 40, margin = (size_t)768 << 20;
      const size_t freeb = device_available(sl.device);
      L = freeb > state + margin
              ? (int)std::min<size_t>(g_ip_max_L + 2, (freeb - state - margin) / (12 * plane)) - 2
              : 0;
      if (!want_ip && L < 8) L = 0;  // too short to beat split
    }
    L = std::min(L, dims->nz);
    if (want_ip && !(L >= 2 || (L >= 1 && L == dims->nz))) {
      delete ctx;
      return fail(env ? THIIM_ERR_CONFIG : THIIM_ERR_SETUP,
                  env ? "TBLOCK in place needs sub-ranges of >= 2 planes (THIIM_INPLACE_TB=" +
                            std::to_string(L) + ")"
                      : std::string("TBLOCK in place: no device memory for the gap planes"));
    }
    if (L >= 2 || (L >= 1 && L == dims->nz)) {
      sl.ip_L = L;
      sl.fstride = ((size_t)(sl.g.nz + 2 + L + 2) * (size_t)pxy + 15) / 16 * 16;
    }
  }
  for (auto& sl : ctx->slabs) {
    // + tail slack: tile row copies may run past the last padded row; then 256 B
    // for the pass counter of multi-process peer stores
    const size_t tail = (size_t)(34 * (dims->nx + 2) + 256) * sizeof(double2);
    const size_t state_elems =
        sl.fs() * 12 * (size_t)sl.nfield_sets + (table ? 0 : sl.stride * 28);
    const size_t state_bytes = (state_elems * sizeof(double2) + tail + 255) / 256 * 256;
    size_t bytes = state_bytes + 256;
    sl.counter_offset = (long long)state_bytes;
    cudaError_t e = cudaSetDevice(sl.device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) {
      device_pool(sl.device);
      // slab contexts of a multi-process decomposition: cudaMalloc, so that
      // neighbours in other processes can map the state (thiim_gpu_slab_export).
      // Slabs of one context on different devices: cudaMalloc as well -- the
      // neighbours' kernels store into this slab's halos, and
      // cudaDeviceEnablePeerAccess (below) does not cover memory from a
      // stream-ordered pool (that would need cudaMemPoolSetAccess per pool)
      sl.ipc_buf = ipc_alloc || (n > 1 && dev_step != 0);
      e = sl.ipc_buf ? cudaMalloc(reinterpret_cast<void**>(&sl.buf), bytes)
                     : pool_alloc(reinterpret_cast<void**>(&sl.buf), bytes, sl.device, sl.stream);
      if (e != cudaSuccess && sl.fstride && !want_ip) {
        // AUTO: no room for the in-place gap after all -> plain split
        cudaGetLastError();
        sl.fstride = 0;
        sl.ip_L = 0;
        const size_t sb = (sl.stride * 40 * sizeof(double2) + tail + 255) / 256 * 256;
        bytes = sb + 256;
        sl.counter_offset = (long long)sb;
        e = pool_alloc(reinterpret_cast<void**>(&sl.buf), bytes, sl.device, sl.stream);
      }
      if (e == cudaSuccess) e = cudaMemsetAsync(sl.buf, 0, bytes, sl.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(sl.stream);
      if (e != cudaSuccess) sl.buf = nullptr;
      if (sl.buf)
        sl.counter = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(sl.buf) +
                                                           sl.counter_offset);
    }
    if (e == cudaSuccess && table) {
      const size_t mbytes = (size_t)sl.mplane * (sl.g.nz + 2) + 4096;
      // zero-fills on the slab stream: a legacy-stream cudaMemset does not order
      // against this non-blocking stream and raced the generator's id writes
      e = cudaMalloc(&sl.mat, mbytes);
      if (e == cudaSuccess) e = cudaMemsetAsync(sl.mat, 0, mbytes, sl.stream);
      if (e == cudaSuccess) e = cudaMalloc(&sl.tab, kMaxMaterials * 28 * sizeof(double2));
      if (e == cudaSuccess)
        e = cudaMemsetAsync(sl.tab, 0, kMaxMaterials * 28 * sizeof(double2), sl.stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(sl.stream);
    }
    if (e == cudaSuccess) e = cudaEventCreate(&sl.ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&sl.ev1);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&sl.ev_pass, cudaEventDisableTiming);
    if (e != cudaSuccess) {
      const std::string msg = std::string("device allocation of ") + std::to_string(bytes) +
                              " bytes failed: " + cudaGetErrorString(e);
      cudaGetLastError();
      thiim_gpu_destroy(ctx);
      return fail(THIIM_ERR_SETUP, msg);
    }
  }
  if (n > 1) {
    for (int s = 0; s + 1 < n; ++s)
      for (int d : {0, 1}) {
        const int a = ctx->slabs[s + d].device, b = ctx->slabs[s + 1 - d].device;
        if (a == b) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, a, b);
        if (can) {
          cudaSetDevice(a);
          cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        }
      }
  }
  // deep slabs write each other's halos from the kernel when every adjacent
  // pair shares a device or has peer access (else copy exchange per pass)
  if (n > 1 && ctx->slabs[0].deep) {
    bool ok = true;
    for (int k = 0; k + 1 < n; ++k) {
      const int a = ctx->slabs[k].device, b = ctx->slabs[k + 1].device;
      int ab = 0, ba = 0;
      if (a != b) {
        cudaDeviceCanAccessPeer(&ab, a, b);
        cudaDeviceCanAccessPeer(&ba, b, a);
        ok = ok && ab && ba;
      }
    }
    ctx->peer_stores = ok && std::getenv("THIIM_NO_PEER_STORES") == nullptr;
  }
  *out = ctx;
  return THIIM_OK;
}

int thiim_gpu_create(const thiim_dims* dims, const thiim_gpu_opts* opts, thiim_gpu_ctx** out) {
  const int n = opts ? opts->n_gpus : 1;
  std::vector<std::pair<int, int>> ranges;
  if (dims && n >= 1 && n <= 8) {
    const int base = dims->nz / n, rem = dims->nz % n;  // reference z_slab split
    for (int s = 0; s < n; ++s) {
      const int z0 = s * base + std::min(s, rem);
      ranges.push_back({z0, z0 + base + (s < rem ? 1 : 0)});
    }
  }
  return create_impl(dims, opts, false, ranges, out);
}

int thiim_gpu_create_slab(const thiim_dims* global, int z0, int z1, const thiim_gpu_opts* opts,
                          thiim_gpu_ctx** out) {
  thiim_gpu_opts o;
  if (opts)
    o = *opts;
  else
    thiim_gpu_default_opts(&o);
  o.n_gpus = 1;
  if (o.engine == THIIM_ENGINE_SPLIT && global && (z0 > 0 || z1 < global->nz)) {
    g_err = "slab contexts with halos need a fused engine (the split engine exchanges mid-step)";
    return THIIM_ERR_CONFIG;
  }
  return create_impl(global, &o, true, {{z0, z1}}, out);
}

int thiim_gpu_halo_view(thiim_gpu_ctx* ctx, int which, thiim_halo_view* v) {
  g_err.clear();
  if (!ctx || !v) return fail(THIIM_ERR_CONFIG, "null argument");
  if (ctx->slabs.size() != 1) return fail(THIIM_ERR_CONFIG, "halo views need a slab context");
  const Slab& sl = ctx->slabs[0];
  if (which < THIIM_HALO_SEND_DOWN || which > THIIM_HALO_RECV_UP)
    return fail(THIIM_ERR_CONFIG, "unknown halo view");
  if (sl.deep) {  // two contiguous planes of all 12 fields
    v->base = sl.field(sl.cur, 0) + (size_t)deep_first_plane(sl, which) * (size_t)sl.g.pxy;
    v->array_stride_bytes = (long long)(sl.stride * sizeof(double2));
    v->plane_bytes = 2 * (long long)(sl.g.pxy * sizeof(double2));
    v->n_arrays = 12;
    v->device = sl.device;
    return THIIM_OK;
  }
  int plane, n;
  switch (which) {
    case THIIM_HALO_SEND_DOWN: plane = 1; n = 6; break;             // E of my first plane
    case THIIM_HALO_RECV_DOWN: plane = 0; n = 10; break;            // E + Hxy..Hyz below me
    case THIIM_HALO_SEND_UP: plane = sl.g.nz; n = 10; break;        // E + Hxy..Hyz of my last plane
    case THIIM_HALO_RECV_UP: plane = sl.g.nz + 1; n = 6; break;     // E above me
    default: return fail(THIIM_ERR_CONFIG, "unknown halo view");
  }
  v->base = sl.field(sl.cur, 0) + (size_t)plane * (size_t)sl.g.pxy;
  v->array_stride_bytes = (long long)(sl.stride * sizeof(double2));
  v->plane_bytes = (long long)(sl.g.pxy * sizeof(double2));
  v->n_arrays = n;
  v->device = sl.device;
  return THIIM_OK;
}

int thiim_gpu_slab_info(thiim_gpu_ctx* ctx, thiim_slab_info* info) {
  g_err.clear();
  if (!ctx || !info) return fail(THIIM_ERR_CONFIG, "null argument");
  if (ctx->slabs.size() != 1) return fail(THIIM_ERR_CONFIG, "slab info needs a slab context");
  const Slab& sl = ctx->slabs[0];
  info->own_z0 = sl.own0;
  info->own_z1 = sl.own1;
  info->local_z0 = sl.z0;
  info->local_z1 = sl.z1;
  info->exchange_period = sl.deep ? 2 : 1;
  info->engine = ctx->engine;
  info->device_ordered = ctx->ipc_ordered ? 1 : 0;
  return THIIM_OK;
}

int thiim_gpu_slab_export(thiim_gpu_ctx* ctx, thiim_slab_export* out) {
  g_err.clear();
  if (!ctx || !out) return fail(THIIM_ERR_CONFIG, "null argument");
  if (ctx->slabs.size() != 1 || !ctx->slabs[0].ipc_buf)
    return fail(THIIM_ERR_CONFIG, "export needs a slab context (thiim_gpu_create_slab)");
  const Slab& sl = ctx->slabs[0];
  std::memset(out, 0, sizeof(*out));
  cudaIpcMemHandle_t h;
  CK(cudaSetDevice(sl.device));
  CK(cudaIpcGetMemHandle(&h, sl.buf));
  static_assert(sizeof(h) <= sizeof(out->ipc), "IPC handle size");
  std::memcpy(out->ipc, &h, sizeof(h));
  out->stride = (long long)sl.stride;
  out->nz_local = sl.g.nz;
  out->ext_lo = sl.ext_lo;
  out->ext_hi = sl.ext_hi;
  out->nfield_sets = sl.nfield_sets;
  out->device = sl.device;
  out->px = sl.g.px;
  out->pxy = sl.g.pxy;
  out->counter_offset = sl.counter_offset;
  return THIIM_OK;
}

int thiim_gpu_slab_import(thiim_gpu_ctx* ctx, int which, const thiim_slab_export* peer) {
  g_err.clear();
  if (!ctx || !peer) return fail(THIIM_ERR_CONFIG, "null argument");
  if (ctx->slabs.size() != 1) return fail(THIIM_ERR_CONFIG, "import needs a slab context");
  Slab& sl = ctx->slabs[0];
  if (!sl.deep || ctx->engine != THIIM_ENGINE_TBLOCK)
    return fail(THIIM_ERR_CONFIG, "peer stores need a deep-halo (TBLOCK) slab");
  if (which != THIIM_PEER_LOWER && which != THIIM_PEER_UPPER)
    return fail(THIIM_ERR_CONFIG, "unknown neighbour");
  if ((which == THIIM_PEER_LOWER && !sl.ext_lo) || (which == THIIM_PEER_UPPER && !sl.ext_hi))
    return fail(THIIM_ERR_CONFIG, "no neighbour on that side");
  if (peer->nfield_sets != sl.nfield_sets || peer->px != sl.g.px || peer->pxy != sl.g.pxy ||
      (which == THIIM_PEER_LOWER ? !peer->ext_hi : !peer->ext_lo))
    return fail(THIIM_ERR_CONFIG, "neighbour layout does not match");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, peer->ipc, sizeof(h));
  CK(cudaSetDevice(sl.device));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(THIIM_ERR_COMM, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
  }
  Slab::Peer& p = sl.peer[which == THIIM_PEER_LOWER ? 0 : 1];
  if (p.base) cudaIpcCloseMemHandle(p.base);
  p.base = static_cast<double2*>(base);
  p.stride = peer->stride;
  p.nz = peer->nz_local;
  p.ext_lo = peer->ext_lo;
  p.ext_hi = peer->ext_hi;
  p.counter = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) +
                                                    peer->counter_offset);
  // peer stores once every neighbour this slab has is mapped
  ctx->peer_stores = (!sl.ext_lo || sl.peer[0].base) && (!sl.ext_hi || sl.peer[1].base);
  // device-side ordering if the stream memory operations take the mapped
  // counters (probe: a wait that is already satisfied)
  ctx->ipc_ordered = false;
  if (ctx->peer_stores) {
    bool ok = stream_mem_ops() != nullptr;
    for (const Slab::Peer& q : sl.peer)
      if (ok && q.counter)
        ok = stream_wait_geq(sl.stream, q.counter, 0) == CUDA_SUCCESS;
    ok = ok && cudaStreamSynchronize(sl.stream) == cudaSuccess;
    cudaGetLastError();
    ctx->ipc_ordered = ok;
  }
  return THIIM_OK;
}

int thiim_gpu_slab_detach(thiim_gpu_ctx* ctx) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  for (auto& sl : ctx->slabs)
    for (auto& p : sl.peer) {
      if (p.base) cudaIpcCloseMemHandle(p.base);
      p = Slab::Peer{};
    }
  if (ctx->slabs.size() == 1) {
    ctx->peer_stores = false;
    ctx->ipc_ordered = false;
  }
  return THIIM_OK;
}

int thiim_gpu_sync(thiim_gpu_ctx* ctx) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
  }
  return THIIM_OK;
}

int thiim_gpu_release_cached(int device) {
  g_err.clear();
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(THIIM_ERR_CONFIG, "no such device");
  CK(cudaSetDevice(device));
  CK(cudaDeviceSynchronize());
  if (cudaMemPool_t pool = device_pool(device)) CK(cudaMemPoolTrimTo(pool, 0));
  return THIIM_OK;
}

void thiim_gpu_destroy(thiim_gpu_ctx* ctx) {
  if (!ctx) return;
  for (auto& sl : ctx->slabs) {
    cudaSetDevice(sl.device);
    if (sl.stream) cudaStreamSynchronize(sl.stream);
    for (auto& p : sl.peer)
      if (p.base) cudaIpcCloseMemHandle(p.base);
    if (sl.buf && sl.ipc_buf) {
      cudaFree(sl.buf);
    } else if (sl.buf) {  // back to the pool; the sync lets the next context reuse it at once
      cudaFreeAsync(sl.buf, sl.stream);
      cudaStreamSynchronize(sl.stream);
    }
    if (sl.cnt) cudaFree(sl.cnt);
    if (sl.cov_bad) cudaFree(sl.cov_bad);
    if (sl.ring_nz) cudaFree(sl.ring_nz);
    if (sl.mat) cudaFree(sl.mat);
    if (sl.tab) cudaFree(sl.tab);
    if (sl.ev0) cudaEventDestroy(sl.ev0);
    if (sl.ev1) cudaEventDestroy(sl.ev1);
    if (sl.ev_pass) cudaEventDestroy(sl.ev_pass);
    for (auto& gx : sl.pass_graph)
      if (gx) cudaGraphExecDestroy(gx);
    if (sl.stream) cudaStreamDestroy(sl.stream);
  }
  delete ctx;
}

static int upload_arrays(thiim_gpu_ctx* ctx, const thiim_c128* const* arrays, int first, int count,
                         int p0 = 0, bool sync = true) {
  const long long pxy = ctx->pxy();
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    // planes [z0, z1+2) of the global padded grid == local planes [0, nz+2);
    // the host arrays start at global padded plane p0
    if (sl.z0 < p0) return fail(THIIM_ERR_CONFIG, "host planes start above the slab");
    const size_t off = (size_t)(sl.z0 - p0) * (size_t)pxy;
    const size_t bytes = (size_t)(sl.g.nz + 2) * (size_t)pxy * sizeof(double2);
    for (int a = first; a < first + count; ++a) {
      if (!arrays[a - first]) return fail(THIIM_ERR_CONFIG, "null host array");
      const thiim_c128* src = arrays[a - first] + off;
      if (a < 12) {
        // one PCIe transfer; the ping-pong set gets a device-side copy
        CK(cudaMemcpyAsync(sl.field(0, a), src, bytes, cudaMemcpyHostToDevice, sl.stream));
        for (int set = 1; set < sl.nfield_sets; ++set)
          CK(cudaMemcpyAsync(sl.field(set, a), sl.field(0, a), bytes, cudaMemcpyDeviceToDevice,
                             sl.stream));
      } else {
        if (sl.table) return fail(THIIM_ERR_CONFIG, "table-layout context: use thiim_gpu_upload_table");
        CK(cudaMemcpyAsync(sl.coeff(a), src, bytes, cudaMemcpyHostToDevice, sl.stream));
      }
    }
  }
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    if (sync) CK(cudaStreamSynchronize(sl.stream));
    sl.cur = 0;
  }
  return THIIM_OK;
}

int thiim_gpu_upload(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12],
                     const thiim_c128* const t[12], const thiim_c128* const c[12],
                     const thiim_c128* const src[4]) {
  g_err.clear();
  if (!ctx || !fields || !t || !c || !src) return fail(THIIM_ERR_CONFIG, "null argument");
  int r;
  if ((r = upload_arrays(ctx, fields, 0, 12))) return r;
  if ((r = upload_arrays(ctx, t, 12, 12))) return r;
  if ((r = upload_arrays(ctx, c, 24, 12))) return r;
  if ((r = upload_arrays(ctx, src, 36, 4))) return r;
  ctx->loaded = true;
  return THIIM_OK;
}

int thiim_gpu_upload_fields(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12]) {
  g_err.clear();
  if (!ctx || !fields) return fail(THIIM_ERR_CONFIG, "null argument");
  return upload_arrays(ctx, fields, 0, 12);
}

void thiim_scheme_default(thiim_scheme* sp) {
  if (!sp) return;
  sp->omega = 0.4;  // SchemeParams defaults, coefficients.hpp:21-26
  sp->tau = 1.0;
  sp->delta = 1.0;
  sp->source_e = {1.0, 0.0};
  sp->source_h = {1.0, 0.0};
}

namespace {

// Update coefficients of a homogeneous vacuum cell (MaterialCell{}: eps = 1,
// mu = 1, sigma = sigma* = 0 -- coefficients.hpp:14-19), restating
// derive_coefficients (coefficients.cpp:25-55) for family H and for family E
// in Forward mode (select_mode picks Back only for Re(eps) < 0,
// coefficients.hpp:50-53), then fill_coefficients' folding of the finite-
// difference orientation (-1 for E) and the curl sign into c
// (coefficients.cpp:63-66; curl signs components.hpp:54-67).  The complex
// expressions keep the reference's structure and types, so libgcc's complex
// division and libm's cos / sin round exactly as in the reference build.
using cplx = std::complex<double>;

int vacuum_coefficients(const thiim_scheme& sp, BenchValues& out) {
  if (!(sp.tau > 0.0)) return fail(THIIM_ERR_CONFIG, "tau must be > 0");
  if (!(sp.delta > 0.0)) return fail(THIIM_ERR_CONFIG, "delta must be > 0");
  if (!(sp.omega * sp.tau <= 3.14159265358979323846 + 1e-12))
    return fail(THIIM_ERR_CONFIG, "omega*tau must be <= pi");
  const cplx eps(1.0, 0.0);
  const double mu = 1.0, sigma = 0.0, sigma_star = 0.0;
  const cplx src_e(sp.source_e.re, sp.source_e.im), src_h(sp.source_h.re, sp.source_h.im);
  auto expi = [](double ph) { return cplx(std::cos(ph), std::sin(ph)); };
  const double wt = sp.omega * sp.tau;
  // H: [e^{-i wt/2} H + (tau/mu) D + tau S_H] / (e^{i wt/2} + tau sigma*/mu)
  const cplx den_h = expi(wt / 2.0) + cplx(sp.tau * sigma_star / mu, 0.0);
  // E forward: [e^{-i wt} E + (tau/eps) e^{-i wt/2} D + tau e^{-i wt} S_E] / (1 + tau sigma/eps)
  const cplx den_e = cplx(1.0, 0.0) + sp.tau * sigma / eps;
  if (std::abs(den_h) == 0.0 || std::abs(den_e) == 0.0)
    return fail(THIIM_ERR_SETUP, "vanishing update denominator: resonant sigma/tau combination");
  const cplx t_h = expi(-wt / 2.0) / den_h;
  const cplx c_h = cplx(sp.tau / (mu * sp.delta), 0.0) / den_h;
  const cplx s_h = sp.tau * src_h / den_h;
  const cplx t_e = expi(-wt) / den_e;
  const cplx c_e = (sp.tau / (eps * sp.delta)) * expi(-wt / 2.0) / den_e;
  const cplx s_e = sp.tau * expi(-wt) * src_e / den_e;
  // per component: curl sign (components.hpp:54-67), orientation -1 for E
  static const double curl[12] = {+1, -1, -1, +1, +1, -1, -1, +1, +1, -1, -1, +1};
  auto put = [](double2& d, const cplx& v) { d = make_double2(v.real(), v.imag()); };
  for (int k = 0; k < 12; ++k) {
    const bool e = k < HXY;
    const double sign = (e ? -1.0 : 1.0) * curl[k];
    put(out.v[k], e ? t_e : t_h);
    put(out.v[12 + k], sign * (e ? c_e : c_h));
  }
  put(out.v[24 + SRC_EXZ], s_e);
  put(out.v[24 + SRC_EYZ], s_e);
  put(out.v[24 + SRC_HXZ], s_h);
  put(out.v[24 + SRC_HYZ], s_h);
  return THIIM_OK;
}

}  // namespace

int thiim_gpu_init_benchmark(thiim_gpu_ctx* ctx, const thiim_scheme* spp) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  thiim_scheme sp;
  thiim_scheme_default(&sp);
  if (spp) sp = *spp;
  BenchValues bv;
  int r = vacuum_coefficients(sp, bv);
  if (r) return r;
  const int zsrc = ctx->dims.nz / 4;  // source_plane_z, coefficients.hpp:70
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    Arrays A = sl.arrays(0, 0);
    if (sl.table) {
      if (sl.n_mat < 3) return fail(THIIM_ERR_CONFIG, "the benchmark problem has 3 materials");
      double2 tab[3 * 28];
      for (int m = 0; m < 3; ++m)
        for (int a = 0; a < 28; ++a)
          tab[m * 28 + a] = (m == 0 || (m == 1 && a >= 24)) ? make_double2(0.0, 0.0) : bv.v[a];
      CK(cudaMemcpyAsync(sl.tab, tab, sizeof(tab), cudaMemcpyHostToDevice, sl.stream));
      k_init_benchmark_table<<<8 * sm_count(sl.device), 256, 0, sl.stream>>>(
          sl.g, sl.z0, ctx->dims.nz, A, sl.mat, sl.mp, sl.mplane, zsrc);
    } else {
      k_init_benchmark<<<8 * sm_count(sl.device), 256, 0, sl.stream>>>(sl.g, sl.z0, ctx->dims.nz,
                                                                      A, bv, zsrc);
    }
    CK(cudaGetLastError());
    for (int set = 1; set < sl.nfield_sets; ++set)
      for (int k = 0; k < 12; ++k)
        CK(cudaMemsetAsync(sl.field(set, k), 0, sl.stride * sizeof(double2), sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
    sl.cur = 0;
  }
  ctx->loaded = true;
  return THIIM_OK;
}

int thiim_gpu_init_materials(thiim_gpu_ctx* ctx, const thiim_scheme* spp, const double* materials) {
  g_err.clear();
  if (!ctx || !materials) return fail(THIIM_ERR_CONFIG, "null argument");
  thiim_scheme sp;
  thiim_scheme_default(&sp);
  if (spp) sp = *spp;
  if (!(sp.tau > 0.0)) return fail(THIIM_ERR_CONFIG, "tau must be > 0");
  if (!(sp.delta > 0.0)) return fail(THIIM_ERR_CONFIG, "delta must be > 0");
  if (!(sp.omega * sp.tau <= 3.14159265358979323846 + 1e-12))
    return fail(THIIM_ERR_CONFIG, "omega*tau must be <= pi");
  if (ctx->slabs[0].table)
    return fail(THIIM_ERR_CONFIG, "material maps fill the full coefficient layout");
  const double wt = sp.omega * sp.tau;  // expi with the host's libm, as the reference
  SchemeDev sd;
  sd.tau = sp.tau;
  sd.delta = sp.delta;
  sd.ep_h = dcx{std::cos(wt / 2.0), std::sin(wt / 2.0)};
  sd.em_h = dcx{std::cos(-wt / 2.0), std::sin(-wt / 2.0)};
  sd.em_1 = dcx{std::cos(-wt), std::sin(-wt)};
  sd.ep_1 = dcx{std::cos(wt), std::sin(wt)};
  sd.src_e = dcx{sp.source_e.re, sp.source_e.im};
  sd.src_h = dcx{sp.source_h.re, sp.source_h.im};
  sd.zsrc = ctx->dims.nz / 4;  // source_plane_z, coefficients.hpp:70
  const size_t plane = (size_t)ctx->dims.nx * ctx->dims.ny * 5;
  unsigned long long worst = ~0ull;
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    // the map planes the slab holds: its interior plus halo planes inside the grid
    const int m0 = std::max(sl.z0 - 1, 0), m1 = std::min(sl.z1 + 1, ctx->dims.nz);
    double* dm = nullptr;
    unsigned long long* derr = nullptr;
    CK(cudaMallocAsync(&dm, std::max<size_t>(1, (size_t)(m1 - m0) * plane) * sizeof(double), sl.stream));
    CK(cudaMallocAsync(&derr, sizeof(unsigned long long), sl.stream));
    CK(cudaMemcpyAsync(dm, materials + (size_t)m0 * plane, (size_t)(m1 - m0) * plane * sizeof(double),
                       cudaMemcpyHostToDevice, sl.stream));
    CK(cudaMemsetAsync(derr, 0xff, sizeof(unsigned long long), sl.stream));
    Arrays A = sl.arrays(0, 0);
    k_init_materials<<<8 * sm_count(sl.device), 256, 0, sl.stream>>>(sl.g, sl.z0, ctx->dims.nz, A, dm,
                                                                    m0, sd, derr);
    CK(cudaGetLastError());
    for (int set = 1; set < sl.nfield_sets; ++set)
      for (int k = 0; k < 12; ++k)
        CK(cudaMemsetAsync(sl.field(set, k), 0, sl.stride * sizeof(double2), sl.stream));
    unsigned long long e = ~0ull;
    CK(cudaMemcpyAsync(&e, derr, sizeof(e), cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaFreeAsync(dm, sl.stream));
    CK(cudaFreeAsync(derr, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
    worst = std::min(worst, e);
    sl.cur = 0;
  }
  if (worst != ~0ull) {  // the reference's SetupError text (coefficients.cpp:14-21, 70-84)
    static const char* names[12] = {"Exy", "Exz", "Eyx", "Eyz", "Ezx", "Ezy",
                                    "Hxy", "Hxz", "Hyx", "Hyz", "Hzx", "Hzy"};
    const unsigned code = (unsigned)(worst & 7);
    const unsigned long long ncells = (unsigned long long)ctx->dims.nx * ctx->dims.ny * ctx->dims.nz;
    const unsigned long long key = worst >> 3;
    const int comp = (int)(key / ncells);
    const unsigned long long cell = key % ncells;
    const int x = (int)(cell % ctx->dims.nx), y = (int)(cell / ctx->dims.nx % ctx->dims.ny),
              z = (int)(cell / ((unsigned long long)ctx->dims.nx * ctx->dims.ny));
    ctx->loaded = false;
    if (code == 1) return fail(THIIM_ERR_SETUP, "mu must be nonzero");
    if (code == 2) return fail(THIIM_ERR_SETUP, "eps must be nonzero");
    char where[96];
    std::snprintf(where, sizeof where, " at cell (%d,%d,%d) component %s", x, y, z, names[comp]);
    return fail(THIIM_ERR_SETUP, std::string("vanishing update denominator (") +
                                     (comp < HXY ? "E" : "H") + (code == 4 ? ", back" : ", forward") +
                                     "): resonant sigma/tau combination" + where);
  }
  ctx->loaded = true;
  return THIIM_OK;
}

int thiim_gpu_selftest_cdiv(int n, const double* in, double* out) {
  g_err.clear();
  if (n < 0 || (n && (!in || !out))) return fail(THIIM_ERR_CONFIG, "bad arguments");
  if (n == 0) return THIIM_OK;
  double *din = nullptr, *dout = nullptr;
  CK(cudaMalloc(&din, (size_t)n * 4 * sizeof(double)));
  CK(cudaMalloc(&dout, (size_t)n * 2 * sizeof(double)));
  CK(cudaMemcpy(din, in, (size_t)n * 4 * sizeof(double), cudaMemcpyHostToDevice));
  k_selftest_cdiv<<<256, 256>>>(n, din, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpy(out, dout, (size_t)n * 2 * sizeof(double), cudaMemcpyDeviceToHost));
  cudaFree(din);
  cudaFree(dout);
  return THIIM_OK;
}

int thiim_gpu_init_generated(thiim_gpu_ctx* ctx, int kind, uint64_t seed) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  if (kind != THIIM_GEN_RANDOM && kind != THIIM_GEN_LAYERED)
    return fail(THIIM_ERR_CONFIG, "unknown generator kind");
  // per-layer coefficient table (config 3), same draws as the host generator
  double2 table[28 * 6];
  for (int a = 12; a < 40; ++a)
    for (int L = 0; L < 6; ++L) table[(a - 12) * 6 + L] = gen_disk(gen_key(seed, a), (uint64_t)L);
  if (ctx->slabs[0].table) {
    if (kind != THIIM_GEN_LAYERED)
      return fail(THIIM_ERR_CONFIG, "the table layout needs a piecewise-constant (layered) problem");
    if (ctx->slabs[0].n_mat < 6) return fail(THIIM_ERR_CONFIG, "layered problems have 6 materials");
    double2 tab[6 * 28];
    for (int L = 0; L < 6; ++L)
      for (int a = 12; a < 40; ++a) tab[L * 28 + (a - 12)] = table[(a - 12) * 6 + L];
    for (auto& sl : ctx->slabs) {
      CK(cudaSetDevice(sl.device));
      CK(cudaMemcpyAsync(sl.tab, tab, sizeof(tab), cudaMemcpyHostToDevice, sl.stream));
      Arrays A = sl.arrays(0, 0);
      k_generate_table<<<8 * sm_count(sl.device), 256, 0, sl.stream>>>(
          sl.g, sl.z0, ctx->dims.nz, A, seed, sl.mat, sl.mp, sl.mplane);
      CK(cudaGetLastError());
      for (int k = 0; k < 12; ++k)
        CK(cudaMemcpyAsync(sl.field(1, k), sl.field(0, k), sl.stride * sizeof(double2),
                           cudaMemcpyDeviceToDevice, sl.stream));
      CK(cudaStreamSynchronize(sl.stream));
      sl.cur = 0;
    }
    ctx->loaded = true;
    return THIIM_OK;
  }
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    double2* dtable = nullptr;
    CK(cudaMallocAsync(&dtable, sizeof(table), sl.stream));
    CK(cudaMemcpyAsync(dtable, table, sizeof(table), cudaMemcpyHostToDevice, sl.stream));
    // local plane 0 is global padded plane z0 (global interior z0-1)
    Arrays A = sl.arrays(0, 0);
    k_generate<<<8 * sm_count(sl.device), 256, 0, sl.stream>>>(sl.g, sl.z0, ctx->dims.nz, A,
                                                                 kind, seed, dtable);
    CK(cudaGetLastError());
    for (int set = 1; set < sl.nfield_sets; ++set)
      for (int k = 0; k < 12; ++k)
        CK(cudaMemcpyAsync(sl.field(set, k), sl.field(0, k), sl.stride * sizeof(double2),
                           cudaMemcpyDeviceToDevice, sl.stream));
    CK(cudaFreeAsync(dtable, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
    sl.cur = 0;
  }
  ctx->loaded = true;
  return THIIM_OK;
}

// tblock_pass: deep slabs store their owned planes only (the extended planes
// come from the neighbours), other passes every local interior plane
static int coverage_pass(thiim_gpu_ctx* ctx, bool tblock_pass = false) {
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    const bool owned = tblock_pass && sl.deep;
    const int r0 = owned ? sl.ext_lo : 0, r1 = owned ? sl.g.nz - sl.ext_hi : sl.g.nz;
    k_coverage<<<4 * sm_count(sl.device), 256, 0, sl.stream>>>(sl.g, sl.cnt, (long long)sl.stride,
                                                               r0, r1, sl.cov_bad);
    CK(cudaGetLastError());
  }
  ++ctx->cov_passes;
  return THIIM_OK;
}

int thiim_gpu_set_sanitize(thiim_gpu_ctx* ctx, int on) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  if (on && ctx->opts.engine == THIIM_ENGINE_TBLOCK_INPLACE)
    return fail(THIIM_ERR_CONFIG,
                "the sanitizer checks one-pass schedules; TBLOCK in place (sub-range passes with "
                "copy-back) is not instrumented -- use engine AUTO, which then runs SPLIT");
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
    if (sl.cnt) CK(cudaFree(sl.cnt));
    if (sl.cov_bad) CK(cudaFree(sl.cov_bad));
    sl.cnt = nullptr;
    sl.cov_bad = nullptr;
    if (on) {
      const size_t bytes = (size_t)12 * sl.stride * sizeof(unsigned);
      if (cudaMalloc(&sl.cnt, bytes) != cudaSuccess ||
          cudaMalloc(&sl.cov_bad, sizeof(unsigned long long)) != cudaSuccess) {
        cudaGetLastError();
        return fail(THIIM_ERR_SETUP, "sanitizer counters: device allocation failed");
      }
      CK(cudaMemsetAsync(sl.cnt, 0, bytes, sl.stream));
      CK(cudaMemsetAsync(sl.cov_bad, 0, sizeof(unsigned long long), sl.stream));
      CK(cudaStreamSynchronize(sl.stream));
    }
  }
  ctx->sanitize = on != 0;
  ctx->cov_passes = 0;
  return THIIM_OK;
}

int thiim_gpu_coverage(thiim_gpu_ctx* ctx, unsigned long long* passes,
                       unsigned long long* violations) {
  g_err.clear();
  if (!ctx || !passes || !violations) return fail(THIIM_ERR_CONFIG, "null argument");
  if (!ctx->sanitize) return fail(THIIM_ERR_STATE, "sanitizer not enabled");
  unsigned long long v = 0;
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    unsigned long long b = 0;
    CK(cudaMemcpyAsync(&b, sl.cov_bad, sizeof(b), cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
    v += b;
  }
  *passes = ctx->cov_passes;
  *violations = v;
  return THIIM_OK;
}

// Enqueues `steps` iterations on the context's stream(s) without waiting for
// them; host-side bookkeeping (current field set, graphs) advances at enqueue
// time, so calls on one context must stay in stream order.
// The engine a step call of `steps` runs: split contexts with spare planes run
// TBLOCK in place (two-step sub-range passes) unless the sanitizer is on; a
// call of fewer than 2 steps runs only the split remainder.
static int engine_ran(const thiim_gpu_ctx* ctx, int steps) {
  const bool ip = ctx->engine == THIIM_ENGINE_SPLIT && ctx->slabs.size() == 1 &&
                  ctx->slabs[0].ip_L > 0 && !ctx->sanitize && steps >= 2;
  return ip ? THIIM_ENGINE_TBLOCK_INPLACE : ctx->engine;
}

static int tb_depth(const thiim_gpu_ctx* ctx) {
  const bool whole = ctx->slabs.size() == 1 && !ctx->slabs[0].deep && !ctx->slabs[0].table &&
                     ctx->slabs[0].z0 == 0 && ctx->slabs[0].z1 == ctx->dims.nz;
  return whole ? ctx->depth : 2;
}

static int step_enqueue(thiim_gpu_ctx* ctx, int steps, long long* launches_out) {
  long long launches = 0;
  const bool multi = ctx->slabs.size() > 1;
  int r;
  int n = 0;
  if (ctx->engine == THIIM_ENGINE_TBLOCK) {
    // deep slabs: a pass (2 steps, or 1 fused remainder step) leaves the owned
    // planes current and the extended + ghost planes stale; the exchange after
    // it refreshes them from the neighbours' owned planes
    // with peer stores a pass writes the neighbours' halos itself: no
    // exchange step, only stream-event ordering between adjacent slabs
    const int ns = (int)ctx->slabs.size();
    std::vector<PeerOut> po(ns);
    // time-block depth of the passes: 3 on one whole-z slab when asked for
    // (thiim_tblock3.cuh), else 2
    const int depth = tb_depth(ctx);
    auto pass = [&](Slab& sl, long long* l, const PeerOut& p) {
      return depth == 3 ? launch_tblock3(ctx, sl, l) : launch_tblock2(ctx, sl, l, p);
    };
    // whole-z context: after one plain pass (one-time setup outside any capture),
    // cycles of two passes replay a captured graph
    if (ns == 1 && !multi && !ctx->slabs[0].deep && !ctx->sanitize && steps - n >= 3 * depth &&
        std::getenv("THIIM_NO_GRAPHS") == nullptr) {
      Slab& sl = ctx->slabs[0];
      const PeerOut po0 = peer_out(ctx, 0);
      if ((r = pass(sl, &launches, po0))) return r;
      n += depth;
      cudaGraphExec_t& gx = sl.pass_graph[sl.cur];
      if (!gx || sl.pass_graph_depth[sl.cur] != depth) {
        if (gx) cudaGraphExecDestroy(gx);
        gx = nullptr;
        const int cur0 = sl.cur;
        cudaGraph_t graph = nullptr;
        long long dummy = 0;
        CK(cudaStreamBeginCapture(sl.stream, cudaStreamCaptureModeThreadLocal));
        int rc = pass(sl, &dummy, po0);
        if (!rc) rc = pass(sl, &dummy, po0);
        sl.pass_graph_launches[cur0] = dummy;
        const cudaError_t ec = cudaStreamEndCapture(sl.stream, &graph);
        sl.cur = cur0;  // the capture ran no kernels; both launches flipped cur
        if (rc) return rc;
        CK(ec);
        const cudaError_t ei = cudaGraphInstantiate(&gx, graph, 0);
        cudaGraphDestroy(graph);
        CK(ei);
        sl.pass_graph_depth[cur0] = depth;
      }
      for (; n + 2 * depth <= steps; n += 2 * depth) {
        CK(cudaGraphLaunch(gx, sl.stream));
        launches += sl.pass_graph_launches[sl.cur];
      }
    }
    if (depth == 3) {
      Slab& sl = ctx->slabs[0];
      for (; n + 3 <= steps; n += 3) {
        if ((r = launch_tblock3(ctx, sl, &launches))) return r;
        if (ctx->sanitize && (r = coverage_pass(ctx, true))) return r;
      }
    }
    for (; n + 2 <= steps; n += 2) {
      for (int k = 0; k < ns; ++k) po[k] = peer_out(ctx, k);
      // every slab's pass waits for its neighbours' PREVIOUS pass (their halo
      // reads of the set this pass stores into, and their stores into this
      // slab's input halos): all waits are enqueued before any of this
      // iteration's records, or slab k+1 would wait for slab k's current pass
      // and the slabs would run one after another
      if (ctx->peer_stores && multi)
        for (int k = 0; k < ns; ++k)
          if ((r = wait_neighbours(ctx, k))) return r;
      if (ctx->ipc_ordered) {
        // neighbours in other processes: their pass counters reach n - 1
        Slab& sl = ctx->slabs[0];
        for (const Slab::Peer& q : sl.peer)
          if (q.counter && stream_wait_geq(sl.stream, q.counter, sl.passes) != CUDA_SUCCESS)
            return fail(THIIM_ERR_CUDA, "cuStreamWaitValue64 on a neighbour's pass counter failed");
      }
      for (int k = 0; k < ns; ++k) {
        if ((r = launch_tblock2(ctx, ctx->slabs[k], &launches, po[k]))) return r;
        if (multi) CK(cudaEventRecord(ctx->slabs[k].ev_pass, ctx->slabs[k].stream));
      }
      if (ctx->ipc_ordered) {
        Slab& sl = ctx->slabs[0];
        if (stream_write(sl.stream, sl.counter, ++sl.passes) != CUDA_SUCCESS)
          return fail(THIIM_ERR_CUDA, "cuStreamWriteValue64 of the pass counter failed");
      }
      if (ctx->sanitize && (r = coverage_pass(ctx, true))) return r;
      if (multi && !ctx->peer_stores && (r = exchange_deep(ctx))) return r;
    }
    if (ctx->ipc_ordered) {
      // a pass only waits for the neighbours' PREVIOUS pass; whatever follows
      // the last one -- the fused remainder step below, a download or the next
      // upload after the call returns -- needs the halos their LAST pass
      // stores: the stream ends on their counters reaching this slab's count
      // (every rank wrote its own counter before it waits: no cycle)
      Slab& sl = ctx->slabs[0];
      for (const Slab::Peer& q : sl.peer)
        if (q.counter && stream_wait_geq(sl.stream, q.counter, sl.passes) != CUDA_SUCCESS)
          return fail(THIIM_ERR_CUDA, "cuStreamWaitValue64 on a neighbour's pass counter failed");
    }
    for (; n < steps; ++n) {
      if (ctx->peer_stores && multi)
        for (int k = 0; k < ns; ++k)
          if ((r = wait_neighbours(ctx, k))) return r;
      for (int k = 0; k < ns; ++k)
        if ((r = launch_fused(ctx, ctx->slabs[k], &launches))) return r;
      if (ctx->sanitize && (r = coverage_pass(ctx, false))) return r;
      if (multi && (r = exchange_deep(ctx))) return r;
    }
  }
  if (ctx->engine == THIIM_ENGINE_SPLIT && !multi && ctx->slabs[0].ip_L > 0 && !ctx->sanitize) {
    // TBLOCK in place: two steps per sub-range sweep, an odd remainder split
    Slab& s0 = ctx->slabs[0];
    if (n + 2 <= steps) {  // do the ghost rings have to move with the array?
      if (!s0.ring_nz) CK(cudaMalloc(&s0.ring_nz, sizeof(unsigned)));
      CK(cudaMemsetAsync(s0.ring_nz, 0, sizeof(unsigned), s0.stream));
      const int np = (int)(s0.fs() / s0.g.pxy);  // array + gap planes
      k_ring_nonzero<<<dim3(8, std::min(np, 512), 12), 256, 0, s0.stream>>>(
          field_planes(s0, 0), np, s0.g.nx, s0.g.ny, s0.g.px, s0.g.pxy, s0.ring_nz);
      CK(cudaGetLastError());
      ++launches;
    }
    for (; n + 2 <= steps; n += 2)
      if ((r = launch_tblock_inplace(ctx, ctx->slabs[0], &launches))) return r;
    if ((r = inplace_restore(ctx->slabs[0]))) return r;
  }
  for (; n < steps; ++n) {
    if (ctx->engine == THIIM_ENGINE_SPLIT) {
      if (multi && (r = exchange(ctx, 0))) return r;
      for (auto& sl : ctx->slabs)
        if ((r = launch_split(ctx, sl, 0, &launches))) return r;
      if (multi && (r = exchange(ctx, 1))) return r;
      for (auto& sl : ctx->slabs)
        if ((r = launch_split(ctx, sl, 1, &launches))) return r;
    } else {
      if (multi && (r = exchange_fused(ctx))) return r;
      for (auto& sl : ctx->slabs)
        if ((r = launch_fused(ctx, sl, &launches))) return r;
    }
    if (ctx->sanitize && (r = coverage_pass(ctx))) return r;
  }
  *launches_out += launches;
  return THIIM_OK;
}

int thiim_gpu_step(thiim_gpu_ctx* ctx, int steps, thiim_gpu_stats* stats) {
  g_err.clear();
  if (!ctx) return fail(THIIM_ERR_CONFIG, "null context");
  if (steps < 0) return fail(THIIM_ERR_CONFIG, "steps must be >= 0");
  if (!ctx->loaded) return fail(THIIM_ERR_STATE, "no problem uploaded or generated");
  if (ctx->peer_stores && ctx->slabs.size() == 1 && !ctx->ipc_ordered && steps > 2)
    return fail(THIIM_ERR_CONFIG,
                "a slab with IPC peer stores advances <= 2 steps per call (barrier in between)");
  if (ctx->ipc_ordered && (steps % 2) && steps > 1)
    return fail(THIIM_ERR_CONFIG,
                "device-ordered IPC peer stores advance an even number of steps per call (the "
                "odd remainder step needs the view exchange)");
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaEventRecord(sl.ev0, sl.stream));
  }
  long long launches = 0;
  int r;
  if ((r = step_enqueue(ctx, steps, &launches))) return r;
  double secs = 0.0;
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaEventRecord(sl.ev1, sl.stream));
    CK(cudaEventSynchronize(sl.ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, sl.ev0, sl.ev1));
    secs = std::max(secs, (double)ms * 1e-3);
  }
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->seconds = secs;
    stats->kernel_seconds = secs;
    stats->steps = steps;
    stats->engine = engine_ran(ctx, steps);
    stats->n_gpus = (int)ctx->slabs.size();
    stats->kernel_launches = launches;
    stats->balance_model = ctx->slabs[0].table
                               ? thiim_gpu_balance_model(100 + THIIM_COEFF_TABLE,
                                                         ctx->engine == THIIM_ENGINE_TBLOCK ? 2 : 1)
                               : thiim_gpu_balance_model(stats->engine, ctx->opts.time_block);
    const double lups = (double)ctx->dims.nx * ctx->dims.ny * ctx->dims.nz * steps;
    stats->mlups = (steps > 0 && secs > 0) ? lups / secs / 1e6 : 0.0;
  }
  return THIIM_OK;
}

static int download_impl(thiim_gpu_ctx* ctx, int a, thiim_c128* dst, int hp0 = 0,
                         bool sync = true) {
  const long long pxy = ctx->pxy();
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    // owned interior planes, plus the global ghost plane(s) this slab borders
    const int p0 = sl.z0 == 0 ? 0 : 1 + sl.ext_lo;
    const int p1 = sl.z1 == ctx->dims.nz ? sl.g.nz + 2 : sl.g.nz + 1 - sl.ext_hi;
    if (sl.z0 + p0 < hp0) return fail(THIIM_ERR_CONFIG, "host planes start above the slab");
    const size_t off_host = (size_t)(sl.z0 + p0 - hp0) * (size_t)pxy;
    CK(cudaMemcpyAsync(dst + off_host, sl.array(a) + (size_t)p0 * pxy,
                       (size_t)(p1 - p0) * (size_t)pxy * sizeof(double2), cudaMemcpyDeviceToHost,
                       sl.stream));
  }
  if (!sync) return THIIM_OK;
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    CK(cudaStreamSynchronize(sl.stream));
  }
  return THIIM_OK;
}

int thiim_gpu_download_fields(thiim_gpu_ctx* ctx, thiim_c128* const fields[12]) {
  g_err.clear();
  if (!ctx || !fields) return fail(THIIM_ERR_CONFIG, "null argument");
  for (int k = 0; k < 12; ++k) {
    if (!fields[k]) return fail(THIIM_ERR_CONFIG, "null host array");
    int r = download_impl(ctx, k, fields[k]);
    if (r) return r;
  }
  return THIIM_OK;
}

int thiim_gpu_upload_planes(thiim_gpu_ctx* ctx, const thiim_c128* const arrays[40], int p0) {
  g_err.clear();
  if (!ctx || !arrays) return fail(THIIM_ERR_CONFIG, "null argument");
  int r;
  if ((r = upload_arrays(ctx, arrays, 0, 12, p0))) return r;
  if ((r = upload_arrays(ctx, arrays + 12, 12, 12, p0))) return r;
  if ((r = upload_arrays(ctx, arrays + 24, 24, 12, p0))) return r;
  if ((r = upload_arrays(ctx, arrays + 36, 36, 4, p0))) return r;
  ctx->loaded = true;
  return THIIM_OK;
}

int thiim_gpu_download_fields_planes(thiim_gpu_ctx* ctx, thiim_c128* const fields[12], int p0) {
  g_err.clear();
  if (!ctx || !fields) return fail(THIIM_ERR_CONFIG, "null argument");
  for (int k = 0; k < 12; ++k) {
    if (!fields[k]) return fail(THIIM_ERR_CONFIG, "null host array");
    int r = download_impl(ctx, k, fields[k], p0);
    if (r) return r;
  }
  return THIIM_OK;
}

// A stream of independent problems through `depth` device contexts: problem i
// uploads while problem i-1 computes and problem i-2 downloads.  Three event
// chains keep each resource in problem order (H2D copies, sweeps, D2H copies),
// so the PCIe directions and the SMs each work on one problem at a time, and a
// context is reused only after its previous problem's download (same stream).
}  // extern "C"

// The engine and pipeline depth a batch under AUTO runs (thiim_gpu_run_batch).
// Ping-pong TBLOCK holds 52 arrays per context, TBLOCK in place 40 plus a gap
// of 12 x (L + 2) planes.  When ping-pong fits fewer than two contexts but
// in place fits two or more, the stream can overlap problem i's PCIe copies
// with its neighbours' sweeps -- at in place's cost per sweep (measured 1.13x
// the ping-pong sweep at configs[2]: 2.77 vs 2.45 s).  Per problem:
//   one ping-pong context:  up + S + down           (serial)
//   k >= 2 in place:        max(f S, up + down)     (steady state; f = 1.04 at
//                                                    sub-ranges of 128 planes)
// with S = LUPs x 416 B / 4.5 TB/s (the sustained TBLOCK rate) and the copies
// at 50 GB/s (pinned PCIe Gen5 x16, measured 55 up / 52 down).  (Before the
// view instances of r02t f was 1.13: in place then lost to serial ping-pong
// beyond ~1,000 iterations per problem at configs[2]; now beyond ~3,000.)  Returns
// THIIM_ENGINE_TBLOCK_INPLACE with *depth and the sub-range cap *ip_L set, or
// THIIM_ENGINE_AUTO (keep the default).
static int batch_plan(const thiim_dims* dims, int device, int steps, int n_problems, int* depth,
                      int* ip_L) {
  const double pxy = (double)(dims->nx + 2) * (dims->ny + 2);
  const double arr = pxy * (dims->nz + 2) * 16.0, plane = pxy * 16.0;
  const double margin = 1.0e9;  // >= create's 768 MB reserve + the tails
  const double freeb = (double)device_available(device);
  const int n_pp = (int)std::min<double>(*depth, std::floor(freeb / (52 * arr + margin)));
  if (n_pp >= 2) return THIIM_ENGINE_AUTO;
  // in-place contexts with the longest sub-range (<= 128, >= 8) they all fit
  int k = std::min(*depth, n_problems);
  for (; k >= 2; --k) {
    const double per = freeb / k - 40 * arr - margin;
    const int L = (int)std::min<double>(g_ip_max_L + 2.0, std::floor(per / (12 * plane))) - 2;
    if (L >= std::min(8, dims->nz)) {
      *ip_L = L;
      break;
    }
  }
  if (k < 2) return THIIM_ENGINE_AUTO;
  const double lups = (double)dims->nx * dims->ny * dims->nz * steps;
  const double S = lups * 416.0 / 4.5e12, up = 40 * arr / 50e9, down = 12 * arr / 50e9;
  // in place: ~2% slower per plane than a whole-z pass plus the halo plane and
  // prologue of each sub-range view (measured r02t: 10.58 vs 11.0 GLUP/s at
  // L = 128, configs[2]; 1.04x)
  const double f = 1.02 * (*ip_L + 2.0) / *ip_L;
  const double t_serial = n_problems * (up + S + down);
  const double t_stream = up + (n_problems - 1) * std::max(f * S, up + down) + f * S + down;
  if (n_pp == 1 && t_stream >= t_serial) return THIIM_ENGINE_AUTO;
  *depth = k;
  return THIIM_ENGINE_TBLOCK_INPLACE;
}

extern "C" {

int thiim_gpu_run_batch(const thiim_dims* dims, const thiim_gpu_opts* opts, int n_problems,
                        const thiim_c128* const* inputs, thiim_c128* const* outputs, int steps,
                        int depth, thiim_gpu_batch_stats* stats) {
  g_err.clear();
  if (!dims || !inputs) return fail(THIIM_ERR_CONFIG, "null argument");
  if (n_problems < 0 || steps < 0) return fail(THIIM_ERR_CONFIG, "n_problems and steps must be >= 0");
  thiim_gpu_opts o;
  if (opts)
    o = *opts;
  else
    thiim_gpu_default_opts(&o);
  if (o.n_gpus != 1) return fail(THIIM_ERR_CONFIG, "run_batch drives one GPU (n_gpus = 1)");
  if (o.coeff_layout != THIIM_COEFF_FULL)
    return fail(THIIM_ERR_CONFIG, "run_batch takes the reference layout (40 arrays per problem)");
  if (depth <= 0) depth = 3;
  depth = std::max(1, std::min(depth, std::max(n_problems, 1)));
  const size_t bytes = (size_t)(dims->nx + 2) * (size_t)(dims->ny + 2) * (size_t)(dims->nz + 2) *
                       sizeof(thiim_c128);
  auto out_ptr = [&](int i, int k) -> thiim_c128* {
    return outputs ? outputs[(size_t)i * 12 + k] : const_cast<thiim_c128*>(inputs[(size_t)i * 40 + k]);
  };
  for (int i = 0; i < n_problems; ++i) {
    for (int a = 0; a < 40; ++a)
      if (!inputs[(size_t)i * 40 + a]) return fail(THIIM_ERR_CONFIG, "null host array");
    for (int k = 0; k < 12; ++k)
      if (!out_ptr(i, k)) return fail(THIIM_ERR_CONFIG, "null host array");
  }
  // problem i's download may run while problem j's upload reads its inputs:
  // outputs must not overlap another problem's inputs (shared outputs are fine,
  // downloads are serialised; writing back over the problem's own inputs is fine)
  // (all arrays have the same length, so input starts sorted once and a
  // window search per output keep this O(n log n) for distinct inputs)
  {
    struct In {
      uintptr_t start;
      int problem, array;
    };
    std::vector<In> ins;
    ins.reserve((size_t)n_problems * 40);
    for (int j = 0; j < n_problems; ++j)
      for (int a = 0; a < 40; ++a) ins.push_back({(uintptr_t)inputs[(size_t)j * 40 + a], j, a});
    std::sort(ins.begin(), ins.end(), [](const In& x, const In& y) { return x.start < y.start; });
    for (int i = 0; i < n_problems; ++i)
      for (int k = 0; k < 12; ++k) {
        const uintptr_t o0 = (uintptr_t)out_ptr(i, k);
        // inputs overlapping [o0, o0 + bytes) start in (o0 - bytes, o0 + bytes)
        const uintptr_t lo = o0 > bytes ? o0 - bytes : 0;
        auto it = std::upper_bound(ins.begin(), ins.end(), lo,
                                   [](uintptr_t v, const In& x) { return v < x.start; });
        for (; it != ins.end() && it->start < o0 + bytes; ++it) {
          if (it->problem == i) continue;
          char msg[160];
          std::snprintf(msg, sizeof msg,
                        "output field %d of problem %d overlaps input array %d of problem %d", k, i,
                        it->array, it->problem);
          return fail(THIIM_ERR_CONFIG, msg);
        }
      }
  }
  const auto t0 = std::chrono::steady_clock::now();
  // AUTO with fewer than two ping-pong contexts in device memory: two or more
  // TBLOCK-in-place contexts (one field set + a gap) when overlapping the PCIe
  // copies with the sweeps saves more than in place costs (batch_plan)
  int ip_cap = 0;
  if (o.engine == THIIM_ENGINE_AUTO && n_problems >= 2 && depth >= 2) {
    int dplan = depth;
    if (batch_plan(dims, o.device, steps, n_problems, &dplan, &ip_cap) == THIIM_ENGINE_TBLOCK_INPLACE) {
      o.engine = THIIM_ENGINE_TBLOCK_INPLACE;
      depth = dplan;
    }
  }
  std::vector<thiim_gpu_ctx*> ctxs(depth, nullptr);
  // per problem: upload, sweep and download brackets
  std::vector<cudaEvent_t> ev((size_t)n_problems * 6, nullptr);
  auto cleanup = [&]() {
    for (auto* c : ctxs)
      if (c) thiim_gpu_destroy(c);  // waits for the context's stream
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  };
  auto bail = [&](int rc) {
    const std::string msg = g_err;
    cleanup();
    g_err = msg;
    return rc;
  };
  int r;
  const int saved_L = g_ip_max_L;
  if (ip_cap > 0) g_ip_max_L = ip_cap;
  for (int d = 0; d < depth; ++d)
    if ((r = thiim_gpu_create(dims, &o, &ctxs[d]))) {
      g_ip_max_L = saved_L;
      // device memory for fewer contexts: a shallower pipeline (depth 1 still
      // runs, one problem at a time); any other failure is an error
      if (d == 0 || r != THIIM_ERR_SETUP) return bail(r);
      depth = d;
      ctxs.resize(d);
      g_err.clear();
      break;
    }
  g_ip_max_L = saved_L;
  {
    const cudaError_t e = cudaSetDevice(ctxs[0]->slabs[0].device);
    for (auto& x : ev)
      if (e != cudaSuccess || cudaEventCreate(&x) != cudaSuccess)
        return bail(fail(THIIM_ERR_CUDA, "cudaEventCreate failed"));
  }
  long long launches = 0;
  auto E = [&](int i, int k) { return ev[(size_t)i * 6 + k]; };
  auto ck = [&](cudaError_t e) { return e == cudaSuccess ? THIIM_OK : fail(THIIM_ERR_CUDA, cudaGetErrorString(e)); };
  auto enqueue_upload = [&](int i) {
    thiim_gpu_ctx* ctx = ctxs[i % depth];
    cudaStream_t st = ctx->slabs[0].stream;
    int rr;
    if (i > 0 && (rr = ck(cudaStreamWaitEvent(st, E(i - 1, 1), 0)))) return rr;
    if ((rr = ck(cudaEventRecord(E(i, 0), st)))) return rr;
    const thiim_c128* const* in = inputs + (size_t)i * 40;
    if ((rr = upload_arrays(ctx, in, 0, 12, 0, false)) || (rr = upload_arrays(ctx, in + 12, 12, 12, 0, false)) ||
        (rr = upload_arrays(ctx, in + 24, 24, 12, 0, false)) ||
        (rr = upload_arrays(ctx, in + 36, 36, 4, 0, false)))
      return rr;
    ctx->loaded = true;
    return ck(cudaEventRecord(E(i, 1), st));
  };
  // Enqueue order: the uploads of the next depth-1 problems (other contexts)
  // go in BEFORE problem i's sweep.  A sweep is thousands of launches and the
  // host blocks in cudaLaunchKernel once the launch queue is full -- until the
  // sweeps ahead of it have nearly finished -- so an upload enqueued after a
  // sweep would start only at that sweep's end instead of beside it.  (With
  // one context every phase shares one stream and keeps problem order.)
  const int ahead = depth - 1;
  int uploaded = 0;  // problems whose upload is enqueued
  for (int i = 0; i < n_problems; ++i) {
    while (uploaded < n_problems && uploaded <= i + ahead)
      if ((r = enqueue_upload(uploaded++))) return bail(r);
    thiim_gpu_ctx* ctx = ctxs[i % depth];
    cudaStream_t st = ctx->slabs[0].stream;
    if (i > 0 && (r = ck(cudaStreamWaitEvent(st, E(i - 1, 3), 0)))) return bail(r);
    if ((r = ck(cudaEventRecord(E(i, 2), st)))) return bail(r);
    if ((r = step_enqueue(ctx, steps, &launches))) return bail(r);
    if ((r = ck(cudaEventRecord(E(i, 3), st)))) return bail(r);
    if (i > 0 && (r = ck(cudaStreamWaitEvent(st, E(i - 1, 5), 0)))) return bail(r);
    if ((r = ck(cudaEventRecord(E(i, 4), st)))) return bail(r);
    for (int k = 0; k < 12; ++k)
      if ((r = download_impl(ctx, k, out_ptr(i, k), 0, false))) return bail(r);
    if ((r = ck(cudaEventRecord(E(i, 5), st)))) return bail(r);
  }
  for (auto* c : ctxs) {
    const cudaError_t e = cudaStreamSynchronize(c->slabs[0].stream);
    if (e != cudaSuccess) return bail(fail(THIIM_ERR_CUDA, cudaGetErrorString(e)));
  }
  double up = 0, sw = 0, down = 0, span = 0;
  for (int i = 0; i < n_problems; ++i) {
    float a = 0, b = 0, c = 0, w = 0;
    cudaEventElapsedTime(&a, E(i, 0), E(i, 1));
    cudaEventElapsedTime(&b, E(i, 2), E(i, 3));
    cudaEventElapsedTime(&c, E(i, 4), E(i, 5));
    up += a * 1e-3;
    sw += b * 1e-3;
    down += c * 1e-3;
    if (i == n_problems - 1) {
      cudaEventElapsedTime(&w, E(0, 0), E(i, 5));
      span = w * 1e-3;
    }
  }
  const int ran = ctxs[0] ? engine_ran(ctxs[0], steps) : o.engine;
  cleanup();
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  if (stats) {
    std::memset(stats, 0, sizeof(*stats));
    stats->seconds = secs;
    stats->device_seconds = span;
    stats->upload_seconds = up;
    stats->kernel_seconds = sw;
    stats->download_seconds = down;
    stats->kernel_launches = launches;
    stats->h2d_bytes = (long long)n_problems * 40 * (long long)bytes;
    stats->d2h_bytes = (long long)n_problems * 12 * (long long)bytes;
    stats->n_problems = n_problems;
    stats->depth = depth;
    stats->engine = ran;
    const double lups = (double)dims->nx * dims->ny * dims->nz * steps * n_problems;
    stats->mlups = secs > 0 ? lups / secs / 1e6 : 0.0;
  }
  return THIIM_OK;
}

int thiim_gpu_upload_table(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12],
                           const uint8_t* material_id, const thiim_c128* table) {
  g_err.clear();
  if (!ctx || !fields || !material_id || !table) return fail(THIIM_ERR_CONFIG, "null argument");
  if (!ctx->slabs[0].table) return fail(THIIM_ERR_CONFIG, "context uses the full coefficient layout");
  int r;
  if ((r = upload_arrays(ctx, fields, 0, 12))) return r;
  const long long pxy = ctx->pxy();
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    // padded host planes [z0, z1+2) -> pitched device rows
    CK(cudaMemcpy2DAsync(sl.mat, (size_t)sl.mp, material_id + (size_t)sl.z0 * pxy, (size_t)sl.g.px,
                         (size_t)sl.g.px, (size_t)(pxy / sl.g.px) * (sl.g.nz + 2),
                         cudaMemcpyHostToDevice, sl.stream));
    CK(cudaMemcpyAsync(sl.tab, table, (size_t)sl.n_mat * 28 * sizeof(double2),
                       cudaMemcpyHostToDevice, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
  }
  ctx->loaded = true;
  return THIIM_OK;
}

int thiim_gpu_download_table(thiim_gpu_ctx* ctx, uint8_t* material_id, thiim_c128* table) {
  g_err.clear();
  if (!ctx || !material_id || !table) return fail(THIIM_ERR_CONFIG, "null argument");
  if (!ctx->slabs[0].table) return fail(THIIM_ERR_CONFIG, "context uses the full coefficient layout");
  const long long pxy = ctx->pxy();
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    const int p0 = sl.z0 == 0 ? 0 : 1 + sl.ext_lo;
    const int p1 = sl.z1 == ctx->dims.nz ? sl.g.nz + 2 : sl.g.nz + 1 - sl.ext_hi;
    CK(cudaMemcpy2DAsync(material_id + (size_t)(sl.z0 + p0) * pxy, (size_t)sl.g.px,
                         sl.mat + (size_t)p0 * sl.mplane, (size_t)sl.mp, (size_t)sl.g.px,
                         (size_t)(pxy / sl.g.px) * (p1 - p0), cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaMemcpyAsync(table, sl.tab, (size_t)sl.n_mat * 28 * sizeof(double2),
                       cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
  }
  return THIIM_OK;
}

int thiim_gpu_download_array(thiim_gpu_ctx* ctx, int array_id, thiim_c128* dst) {
  g_err.clear();
  if (!ctx || !dst) return fail(THIIM_ERR_CONFIG, "null argument");
  if (array_id < 0 || array_id >= 40) return fail(THIIM_ERR_CONFIG, "array id out of range");
  if (array_id >= 12 && ctx->slabs[0].table)
    return fail(THIIM_ERR_CONFIG, "table-layout context: use thiim_gpu_download_table");
  return download_impl(ctx, array_id, dst);
}

int thiim_gpu_compare_fields(thiim_gpu_ctx* ctx, const thiim_c128* const ref[12],
                             thiim_gpu_diff* out) {
  g_err.clear();
  if (!ctx || !ref || !out) return fail(THIIM_ERR_CONFIG, "null argument");
  std::memset(out, 0, sizeof(*out));
  const long long pxy = ctx->pxy();
  double num[12] = {0}, den[12] = {0};
  for (auto& sl : ctx->slabs) {
    CK(cudaSetDevice(sl.device));
    // owned planes only (a deep slab's extended planes duplicate its neighbours')
    Grid go = sl.g;
    go.nz = sl.own1 - sl.own0;
    const size_t lofs = (size_t)sl.ext_lo * (size_t)pxy;
    const size_t elems = (size_t)(go.nz + 2) * (size_t)pxy;
    double2* dref = nullptr;
    double* acc = nullptr;
    unsigned long long* cnt = nullptr;
    CK(cudaMalloc(&dref, elems * sizeof(double2)));
    CK(cudaMalloc(&acc, 24 * sizeof(double)));
    CK(cudaMalloc(&cnt, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(acc, 0, 24 * sizeof(double), sl.stream));
    CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), sl.stream));
    for (int k = 0; k < 12; ++k) {
      CK(cudaMemcpyAsync(dref, ref[k] + (size_t)sl.own0 * pxy, elems * sizeof(double2),
                         cudaMemcpyHostToDevice, sl.stream));
      k_compare<<<4 * sm_count(sl.device), 256, 0, sl.stream>>>(go, sl.field(sl.cur, k) + lofs, dref,
                                                                acc + 2 * k, cnt);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(sl.stream));
    }
    double h[24];
    unsigned long long c = 0;
    CK(cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaMemcpyAsync(&c, cnt, sizeof(c), cudaMemcpyDeviceToHost, sl.stream));
    CK(cudaStreamSynchronize(sl.stream));
    for (int k = 0; k < 12; ++k) {
      num[k] += h[2 * k];
      den[k] += h[2 * k + 1];
    }
    out->differing_values += c;
    cudaFree(dref);
    cudaFree(acc);
    cudaFree(cnt);
  }
  for (int k = 0; k < 12; ++k) {
    out->rel_l2[k] = den[k] > 0 ? std::sqrt(num[k] / den[k]) : std::sqrt(num[k]);
    out->max_rel_l2 = std::max(out->max_rel_l2, out->rel_l2[k]);
  }
  return THIIM_OK;
}

int thiim_generate_host_planes(const thiim_dims* dims, int kind, uint64_t seed, int p0, int p1,
                               thiim_c128* const arrays[40]) {
  g_err.clear();
  if (!valid_dims(dims)) return fail(THIIM_ERR_SETUP, "invalid grid dims");
  if (!arrays) return fail(THIIM_ERR_CONFIG, "null arrays");
  if (kind != THIIM_GEN_RANDOM && kind != THIIM_GEN_LAYERED)
    return fail(THIIM_ERR_CONFIG, "unknown generator kind");
  if (p0 < 0 || p1 > dims->nz + 2 || p0 >= p1) return fail(THIIM_ERR_CONFIG, "bad plane range");
  const int nx = dims->nx, ny = dims->ny, nz = dims->nz;
  const long long px = nx + 2, pxy = px * (ny + 2);
  const long long n = pxy * (long long)(p1 - p0), base = pxy * (long long)p0;
  double2 table[28 * 6];
  for (int a = 12; a < 40; ++a)
    for (int L = 0; L < 6; ++L) table[(a - 12) * 6 + L] = gen_disk(gen_key(seed, a), (uint64_t)L);
  uint64_t keys[40];
  for (int a = 0; a < 40; ++a) keys[a] = gen_key(seed, a);
  for (int a = 0; a < 40; ++a)
    if (!arrays[a]) return fail(THIIM_ERR_CONFIG, "null host array");
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < n; ++q) {
    const long long p = base + q;  // global padded index = generator counter
    const int zp = (int)(p / pxy);
    const long long r = p - (long long)zp * pxy;
    const int yp = (int)(r / px), xp = (int)(r - (long long)yp * px);
    const int x = xp - 1, y = yp - 1, z = zp - 1;
    const bool interior = x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz;
    const int L = (interior && kind == THIIM_GEN_LAYERED) ? gen_layer(seed, nx, nz, x, y, z) : 0;
    for (int a = 0; a < 40; ++a) {
      double2 v = make_double2(0.0, 0.0);
      if (interior) {
        if (a < 12)
          v = gen_field(keys[a], (uint64_t)p);
        else if (kind == THIIM_GEN_LAYERED)
          v = table[(a - 12) * 6 + L];
        else
          v = gen_disk(keys[a], (uint64_t)p);
      }
      arrays[a][q].re = v.x;
      arrays[a][q].im = v.y;
    }
  }
  return THIIM_OK;
}

int thiim_generate_host(const thiim_dims* dims, int kind, uint64_t seed,
                        thiim_c128* const arrays[40]) {
  if (!valid_dims(dims)) {
    g_err = "invalid grid dims";
    return THIIM_ERR_SETUP;
  }
  return thiim_generate_host_planes(dims, kind, seed, 0, dims->nz + 2, arrays);
}

int thiim_coeff_compress(const thiim_dims* dims, const thiim_c128* const coeffs[28],
                         int max_materials, uint8_t* material_id, thiim_c128* table,
                         int* n_materials) {
  g_err.clear();
  if (!valid_dims(dims)) return fail(THIIM_ERR_SETUP, "invalid grid dims");
  if (!coeffs || !material_id || !table || !n_materials) return fail(THIIM_ERR_CONFIG, "null argument");
  for (int k = 0; k < 28; ++k)
    if (!coeffs[k]) return fail(THIIM_ERR_CONFIG, "null coefficient array");
  if (max_materials < 1 || max_materials > kMaxMaterials)
    return fail(THIIM_ERR_CONFIG, "max_materials must be in 1..16");
  *n_materials = 0;
  const long long px = dims->nx + 2, pxy = px * (dims->ny + 2), nz = dims->nz;
  // a cell's coefficient row: 28 complex values = 56 words, compared bitwise
  typedef unsigned long long u64;
  auto word = [&](int k, long long i, int h) -> u64 {
    u64 w;
    std::memcpy(&w, reinterpret_cast<const char*>(coeffs[k] + i) + 8 * h, 8);
    return w;
  };
  auto same = [&](long long i, const u64* row) {
    for (int k = 0; k < 28; ++k)
      if (word(k, i, 0) != row[2 * k] || word(k, i, 1) != row[2 * k + 1]) return false;
    return true;
  };
  // pass 1: per thread, over a contiguous range of interior planes, the
  // distinct rows in order of first appearance; material_id holds the local
  // row index for now
  int nth = 1;
#pragma omp parallel
  {
#pragma omp single
    nth = omp_get_num_threads();
  }
  nth = (int)std::max<long long>(1, std::min<long long>(nth, nz));
  std::vector<std::vector<u64>> rows(nth);  // 56 words per row
  std::vector<int> overflow(nth, 0);
#pragma omp parallel for schedule(static, 1) num_threads(nth)
  for (int t = 0; t < nth; ++t) {
    const long long z0 = 1 + nz * t / nth, z1 = 1 + nz * (t + 1) / nth;
    std::vector<u64>& R = rows[t];
    int last = -1;
    for (long long z = z0; z < z1 && !overflow[t]; ++z)
      for (long long y = 1; y <= dims->ny && !overflow[t]; ++y) {
        const long long i0 = z * pxy + y * px;
        for (long long i = i0 + 1; i <= i0 + dims->nx; ++i) {
          int id = -1;
          if (last >= 0 && same(i, &R[56 * (size_t)last])) id = last;
          for (int r = 0; id < 0 && r < (int)(R.size() / 56); ++r)
            if (r != last && same(i, &R[56 * (size_t)r])) id = r;
          if (id < 0) {
            if ((int)(R.size() / 56) == max_materials) {
              overflow[t] = 1;
              break;
            }
            id = (int)(R.size() / 56);
            for (int k = 0; k < 28; ++k) {
              R.push_back(word(k, i, 0));
              R.push_back(word(k, i, 1));
            }
          }
          material_id[i] = (uint8_t)id;
          last = id;
        }
      }
  }
  for (int t = 0; t < nth; ++t)
    if (overflow[t]) return THIIM_OK;  // more than max_materials rows: not compressible
  // merge in plane order: global ids by first appearance along the interior
  std::vector<u64> G;
  std::vector<std::vector<uint8_t>> remap(nth);
  for (int t = 0; t < nth; ++t) {
    const int nloc = (int)(rows[t].size() / 56);
    for (int r = 0; r < nloc; ++r) {
      const u64* row = &rows[t][56 * (size_t)r];
      int gid = -1;
      for (int q = 0; gid < 0 && q < (int)(G.size() / 56); ++q)
        if (std::memcmp(row, &G[56 * (size_t)q], 56 * sizeof(u64)) == 0) gid = q;
      if (gid < 0) {
        if ((int)(G.size() / 56) == max_materials) return THIIM_OK;
        gid = (int)(G.size() / 56);
        G.insert(G.end(), row, row + 56);
      }
      remap[t].push_back((uint8_t)gid);
    }
  }
  // pass 2: local -> global ids; ghost cells 0
#pragma omp parallel for schedule(static, 1) num_threads(nth)
  for (int t = 0; t < nth; ++t) {
    const long long z0 = 1 + nz * t / nth, z1 = 1 + nz * (t + 1) / nth;
    for (long long z = z0; z < z1; ++z)
      for (long long y = 1; y <= dims->ny; ++y) {
        const long long i0 = z * pxy + y * px;
        for (long long i = i0 + 1; i <= i0 + dims->nx; ++i) material_id[i] = remap[t][material_id[i]];
      }
  }
  std::memset(material_id, 0, (size_t)pxy);  // ghost planes
  std::memset(material_id + (nz + 1) * pxy, 0, (size_t)pxy);
#pragma omp parallel for schedule(static) num_threads(nth)
  for (long long z = 1; z <= nz; ++z) {  // ghost rows and columns
    uint8_t* m = material_id + z * pxy;
    std::memset(m, 0, (size_t)px);
    std::memset(m + (dims->ny + 1) * px, 0, (size_t)px);
    for (long long y = 1; y <= dims->ny; ++y) m[y * px] = m[y * px + px - 1] = 0;
  }
  const int n = (int)(G.size() / 56);
  std::memcpy(table, G.data(), G.size() * sizeof(u64));
  *n_materials = n;
  return THIIM_OK;
}

int thiim_gpu_pin_host(void* ptr, size_t bytes) {
  g_err.clear();
  CK(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault));
  return THIIM_OK;
}

int thiim_gpu_unpin_host(void* ptr) {
  g_err.clear();
  CK(cudaHostUnregister(ptr));
  return THIIM_OK;
}

}  // extern "C"
#include "thiim_tune.cuh"
