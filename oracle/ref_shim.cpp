// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (oracle + CPU baseline arm).
//
// A thin C-ABI around the UNMODIFIED reference library.  oracle/Makefile
// compiles this file together with the reference sources where they lie
// (/root/reference/proj/src/*.cpp, never copied into this repo) into
// oracle/_ref/libthiim_ref.so.  tests/ use it to pin the C restatement
// (thiim_oracle.c) bitwise and to run the reference's own known-answer tests;
// bench.py's cpu_baseline leg and `--impl reference` time the reference's
// run_naive / run_spatial_blocked / run_mwd through it.
//
// Arrays cross as 40 pointers to interleaved complex128 in the reference's
// padded layout (grid.hpp:12-48) in ProblemState order (state.hpp:49-66):
// [0..11] fields, [12..23] t, [24..35] c, [36..39] src.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "thiim/bandwidth.hpp"
#include "thiim/coefficients.hpp"
#include "thiim/kernels.hpp"
#include "thiim/mwd.hpp"
#include "thiim/reference_engines.hpp"
#include "thiim/verifier.hpp"

using namespace thiim;

namespace {

thread_local std::string g_err;

ProblemState make_state(int nx, int ny, int nz, double* const* arrays) {
  ProblemState s = allocate_state(GridDims(nx, ny, nz));
  const std::size_t bytes = s.dims.padded_cells() * sizeof(ComplexScalar);
  for (int i = 0; i < 12; ++i) {
    std::memcpy(s.fields[i].data(), arrays[i], bytes);
    std::memcpy(s.coeff_t[i].data(), arrays[12 + i], bytes);
    std::memcpy(s.coeff_c[i].data(), arrays[24 + i], bytes);
  }
  for (int i = 0; i < 4; ++i) std::memcpy(s.coeff_src[i].data(), arrays[36 + i], bytes);
  return s;
}

void export_all(const ProblemState& s, double* const* arrays) {
  const std::size_t bytes = s.dims.padded_cells() * sizeof(ComplexScalar);
  for (int i = 0; i < 12; ++i) {
    std::memcpy(arrays[i], s.fields[i].data(), bytes);
    std::memcpy(arrays[12 + i], s.coeff_t[i].data(), bytes);
    std::memcpy(arrays[24 + i], s.coeff_c[i].data(), bytes);
  }
  for (int i = 0; i < 4; ++i) std::memcpy(arrays[36 + i], s.coeff_src[i].data(), bytes);
}

void export_fields(const ProblemState& s, double* const* arrays) {
  const std::size_t bytes = s.dims.padded_cells() * sizeof(ComplexScalar);
  for (int i = 0; i < 12; ++i) std::memcpy(arrays[i], s.fields[i].data(), bytes);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SetupError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ---- seeded synthetic inputs, restated here
// so the CPU baseline arm generates its problem without loading any other
// library; bitwise equal to oracle/thiim_oracle.c (tests/test_oracle.py).
std::uint64_t sm64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
std::uint64_t gen_key(std::uint64_t seed, int array_id) {
  return sm64(sm64(seed) ^ ((std::uint64_t)(array_id + 1) * 0x9E3779B97F4A7C15ull));
}
double gen_u(std::uint64_t key, std::uint64_t counter, int draw) {
  return (double)(sm64(key + (counter << 8) + (std::uint64_t)draw) >> 11) * 0x1.0p-53;
}
ComplexScalar gen_field(std::uint64_t key, std::uint64_t i) {
  return {2.0 * gen_u(key, i, 0) - 1.0, 2.0 * gen_u(key, i, 1) - 1.0};
}
ComplexScalar gen_disk(std::uint64_t key, std::uint64_t i) {
  const double r = 0.45;
  for (int k = 0; k < 64; ++k) {
    const double re = r * (2.0 * gen_u(key, i, 2 * k) - 1.0);
    const double im = r * (2.0 * gen_u(key, i, 2 * k + 1) - 1.0);
    if (re * re + im * im <= r * r) return {re, im};
  }
  return {0.0, 0.0};
}
int gen_layer(std::uint64_t seed, int nx, int nz, int x, int y, int z) {
  const std::uint64_t c = (std::uint64_t)y * (std::uint64_t)nx + (std::uint64_t)x;
  int layer = 0;
  for (int k = 1; k <= 5; ++k) {
    const std::uint64_t b = sm64(gen_key(seed, 64 + k) + (c << 8));
    const int h = (int)((b >> 11) % 17ull) - 8;
    if (z >= k * nz / 6 + h) ++layer;
  }
  return layer;
}

ComplexScalar* array_of(ProblemState& s, int a) {
  return a < 12 ? s.fields[a].data()
         : a < 24 ? s.coeff_t[a - 12].data()
         : a < 36 ? s.coeff_c[a - 24].data()
                  : s.coeff_src[a - 36].data();
}

void generate_into(ProblemState& s, std::uint64_t seed, bool layered, int threads) {
  const int nx = s.dims.nx, ny = s.dims.ny, nz = s.dims.nz;
  std::uint64_t key[40];
  for (int a = 0; a < 40; ++a) key[a] = gen_key(seed, a);
  ComplexScalar table[28][6];
  for (int a = 12; a < 40; ++a)
    for (int L = 0; L < 6; ++L) table[a - 12][L] = gen_disk(key[a], (std::uint64_t)L);
  ComplexScalar* arr[40];
  for (int a = 0; a < 40; ++a) arr[a] = array_of(s, a);
  auto work = [&](int w, int nw) {
    for (int z = w; z < nz; z += nw)
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
          const std::size_t i = s.dims.linear_index(x, y, z);
          const int L = layered ? gen_layer(seed, nx, nz, x, y, z) : 0;
          for (int a = 0; a < 40; ++a)
            arr[a][i] = a < 12 ? gen_field(key[a], i)
                        : layered ? table[a - 12][L]
                                  : gen_disk(key[a], i);
        }
  };
  threads = std::max(1, std::min(threads, nz));
  std::vector<std::thread> pool;
  for (int w = 1; w < threads; ++w) pool.emplace_back(work, w, threads);
  work(0, threads);
  for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// build_benchmark_problem (coefficients.cpp:94-111) exported as 40 arrays.
int ref_build_benchmark_problem(int nx, int ny, int nz, double omega, double tau, double delta,
                                double* const* arrays) {
  return guarded([&] {
    SchemeParams sp;
    sp.omega = omega;
    sp.tau = tau;
    sp.delta = delta;
    ProblemState s = build_benchmark_problem(GridDims(nx, ny, nz), sp);
    export_all(s, arrays);
  });
}

// build_problem_from_voxels (coefficients.cpp:112-141) on a voxel-map file.
int ref_build_problem_from_voxels(int nx, int ny, int nz, double omega, double tau, double delta,
                                  const char* path, double* const* arrays) {
  return guarded([&] {
    SchemeParams sp;
    sp.omega = omega;
    sp.tau = tau;
    sp.delta = delta;
    ProblemState s = build_problem_from_voxels(GridDims(nx, ny, nz), sp, path);
    export_all(s, arrays);
  });
}

// derive_coefficients (coefficients.cpp:25-55); out = {t.re,t.im,c.re,c.im,src.re,src.im}.
int ref_derive_coefficients(double eps_re, double eps_im, double mu, double sigma,
                            double sigma_star, double omega, double tau, double delta,
                            int family, int back_mode, double* out) {
  return guarded([&] {
    MaterialCell m;
    m.eps = {eps_re, eps_im};
    m.mu = mu;
    m.sigma = sigma;
    m.sigma_star = sigma_star;
    SchemeParams sp;
    sp.omega = omega;
    sp.tau = tau;
    sp.delta = delta;
    const UpdateCoefficients uc =
        derive_coefficients(m, sp, family == 0 ? Family::E : Family::H,
                            back_mode ? IterationMode::Back : IterationMode::Forward);
    out[0] = uc.t.real();
    out[1] = uc.t.imag();
    out[2] = uc.c.real();
    out[3] = uc.c.imag();
    out[4] = uc.src.real();
    out[5] = uc.src.imag();
  });
}

// update_component_region (kernels.cpp:12-69) on one region; fields written back.
int ref_update_component_region(int nx, int ny, int nz, double* const* arrays, int comp, int x0,
                                int x1, int y0, int y1, int z0, int z1) {
  return guarded([&] {
    ProblemState s = make_state(nx, ny, nz, arrays);
    Region r{x0, x1, y0, y1, z0, z1, descriptor(Component(comp)).family, 0};
    update_component_region(s, descriptor(Component(comp)), r);
    export_fields(s, arrays);
  });
}

// run_naive (reference_engines.cpp:34-67).  *seconds = RunReport.seconds.
int ref_run_naive(int nx, int ny, int nz, double* const* arrays, int steps, int threads,
                  double* seconds) {
  return guarded([&] {
    ProblemState s = make_state(nx, ny, nz, arrays);
    const RunReport r = run_naive(s, steps, threads);
    if (seconds) *seconds = r.seconds;
    export_fields(s, arrays);
  });
}

// run_spatial_blocked (reference_engines.cpp:69-140).
int ref_run_spatial(int nx, int ny, int nz, double* const* arrays, int steps, int block_y,
                    int block_x, int threads, double* seconds) {
  return guarded([&] {
    ProblemState s = make_state(nx, ny, nz, arrays);
    const RunReport r = run_spatial_blocked(s, steps, block_y, block_x, threads);
    if (seconds) *seconds = r.seconds;
    export_fields(s, arrays);
  });
}

// run_mwd (mwd.cpp:129-248).  Steps are padded to a multiple of dw/2 by the
// reference (tiling.hpp:54-57); *steps_executed reports the padded count.
int ref_run_mwd(int nx, int ny, int nz, double* const* arrays, int steps, int dw, int bz,
                int tgz, int tgx, int tgc, int threads, double* seconds, int* steps_executed) {
  return guarded([&] {
    ProblemState s = make_state(nx, ny, nz, arrays);
    ThreadGroupShape shape;
    shape.tgz = tgz;
    shape.tgx = tgx;
    shape.tgc = tgc;
    const MwdResult r = run_mwd(s, steps, dw, bz, shape, threads);
    if (seconds) *seconds = r.report.seconds;
    if (steps_executed) *steps_executed = r.report.steps_executed;
    export_fields(s, arrays);
  });
}

// compare_states (verifier.cpp:13-44) over two 40-array states.
// out_i = {bitwise_equal, differing_values, first_component, x, y, z}.
int ref_compare_states(int nx, int ny, int nz, double* const* a, double* const* b,
                       long long* out_i, double* max_abs_diff) {
  return guarded([&] {
    ProblemState sa = make_state(nx, ny, nz, a);
    ProblemState sb = make_state(nx, ny, nz, b);
    const StateDiff d = compare_states(sa, sb);
    out_i[0] = d.bitwise_equal;
    out_i[1] = (long long)d.differing_values;
    out_i[2] = (long long)d.first_component;
    out_i[3] = d.x;
    out_i[4] = d.y;
    out_i[5] = d.z;
    *max_abs_diff = d.max_abs_diff;
  });
}

// ---- a reference ProblemState held by the shim (no copies per call): the
// CPU baseline arm and the full-size parity tests run the reference on
// 87-174 GB states, which must not be duplicated in host memory.
void* ref_state_new(int nx, int ny, int nz) {
  ProblemState* p = nullptr;
  const int rc = guarded([&] { p = new ProblemState(allocate_state(GridDims(nx, ny, nz))); });
  return rc ? nullptr : p;
}

void ref_state_free(void* h) { delete static_cast<ProblemState*>(h); }

int ref_state_generate(void* h, unsigned long long seed, int layered, int threads) {
  return guarded([&] { generate_into(*static_cast<ProblemState*>(h), seed, layered != 0, threads); });
}

int ref_state_run_naive(void* h, int steps, int threads, double* seconds) {
  return guarded([&] {
    const RunReport r = run_naive(*static_cast<ProblemState*>(h), steps, threads);
    if (seconds) *seconds = r.seconds;
  });
}

int ref_state_run_spatial(void* h, int steps, int block_y, int block_x, int threads,
                          double* seconds) {
  return guarded([&] {
    const RunReport r =
        run_spatial_blocked(*static_cast<ProblemState*>(h), steps, block_y, block_x, threads);
    if (seconds) *seconds = r.seconds;
  });
}

int ref_state_run_mwd(void* h, int steps, int dw, int bz, int tgz, int tgx, int tgc, int threads,
                      double* seconds, int* steps_executed) {
  return guarded([&] {
    ThreadGroupShape shape;
    shape.tgz = tgz;
    shape.tgx = tgx;
    shape.tgc = tgc;
    const MwdResult r = run_mwd(*static_cast<ProblemState*>(h), steps, dw, bz, shape, threads);
    if (seconds) *seconds = r.report.seconds;
    if (steps_executed) *steps_executed = r.report.steps_executed;
  });
}

// copy array a (0..39, ProblemState order) of the held state out / in
int ref_state_get(void* h, int a, double* out) {
  return guarded([&] {
    ProblemState& s = *static_cast<ProblemState*>(h);
    std::memcpy(out, array_of(s, a), s.dims.padded_cells() * sizeof(ComplexScalar));
  });
}

int ref_state_set(void* h, int a, const double* in) {
  return guarded([&] {
    ProblemState& s = *static_cast<ProblemState*>(h);
    std::memcpy(array_of(s, a), in, s.dims.padded_cells() * sizeof(ComplexScalar));
  });
}

// compare_states' field loop (verifier.cpp:13-44) between the held state's
// fields and 12 host field arrays: out_i = {differing_values, first_component,
// x, y, z} (first_component -1 when equal), *max_abs_diff.
int ref_state_compare_fields(void* h, double* const* fields, long long* out_i,
                             double* max_abs_diff) {
  return guarded([&] {
    const ProblemState& s = *static_cast<ProblemState*>(h);
    long long n = 0;
    double mx = 0.0;
    out_i[1] = -1;
    for (int c = 0; c < 12; ++c) {
      const ComplexScalar* a = s.fields[c].data();
      const ComplexScalar* b = reinterpret_cast<const ComplexScalar*>(fields[c]);
      for (int z = 0; z < s.dims.nz; ++z)
        for (int y = 0; y < s.dims.ny; ++y)
          for (int x = 0; x < s.dims.nx; ++x) {
            const std::size_t i = s.dims.linear_index(x, y, z);
            if (std::memcmp(&a[i], &b[i], sizeof(ComplexScalar)) != 0) {
              if (n == 0) {
                out_i[1] = c;
                out_i[2] = x;
                out_i[3] = y;
                out_i[4] = z;
              }
              ++n;
              mx = std::max(mx, std::max(std::abs(a[i].re - b[i].re), std::abs(a[i].im - b[i].im)));
            }
          }
    }
    out_i[0] = n;
    *max_abs_diff = mx;
  });
}

double ref_code_balance_naive() { return code_balance_naive(); }

// the reference's host triad (bandwidth.cpp:12-44; the CLI's `bandwidth`
// subcommand, tools/main.cpp:433-436), GB/s best of five
int ref_measure_bandwidth(int threads, unsigned long long cache_bytes, double* gbs) {
  return guarded([&] { *gbs = measure_bandwidth(threads, cache_bytes); });
}

}  // extern "C"
