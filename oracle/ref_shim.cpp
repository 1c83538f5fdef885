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

#include <cstring>
#include <exception>
#include <string>

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

double ref_code_balance_naive() { return code_balance_naive(); }

// the reference's host triad (bandwidth.cpp:12-44; the CLI's `bandwidth`
// subcommand, tools/main.cpp:433-436), GB/s best of five
int ref_measure_bandwidth(int threads, unsigned long long cache_bytes, double* gbs) {
  return guarded([&] { *gbs = measure_bandwidth(threads, cache_bytes); });
}

}  // extern "C"
