// test_run_gpu.cpp -- reference-style tests of thiim::run_gpu (needs a GPU).
//
// Mirrors the reference's engine-equivalence tests: the GPU engine is checked
// against run_naive with compare_states (verifier.cpp:13-44), bitwise, the way
// test_reference_engines.cpp:32-55 and test_mwd.cpp:14-26 check their engines.
// Built by adapter/Makefile against the UNMODIFIED reference library objects
// (oracle/_ref/obj) into build/test_run_gpu; run by tests/test_gpu_slabs.py.
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "thiim/coefficients.hpp"
#include "thiim/reference_engines.hpp"
#include "thiim/verifier.hpp"
#include "thiim_gpu_engine.hpp"

using namespace thiim;

namespace {

int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(cond)) {                                                         \
      ++g_fail;                                                            \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                      \
  } while (0)

template <class E, class F>
bool throws_as(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// Seeded synthetic state through the engine's host generator (the reference
// has no generator; config.cpp:49 parses a seed nothing consumes).
ProblemState random_state(const GridDims& d, uint64_t seed, int kind = THIIM_GEN_RANDOM) {
  ProblemState s = allocate_state(d);
  thiim_c128* a[40];
  for (int i = 0; i < 12; ++i) {
    a[i] = reinterpret_cast<thiim_c128*>(s.fields[i].data());
    a[12 + i] = reinterpret_cast<thiim_c128*>(s.coeff_t[i].data());
    a[24 + i] = reinterpret_cast<thiim_c128*>(s.coeff_c[i].data());
  }
  for (int i = 0; i < 4; ++i) a[36 + i] = reinterpret_cast<thiim_c128*>(s.coeff_src[i].data());
  thiim_dims dd{d.nx, d.ny, d.nz, d.ghost};
  if (thiim_generate_host(&dd, kind, seed, a) != THIIM_OK) throw SetupError("generator failed");
  return s;
}

void test_matches_run_naive_random() {
  for (GridDims d : {GridDims(12, 16, 20), GridDims(33, 7, 9), GridDims(64, 64, 64)}) {
    for (int engine : {THIIM_ENGINE_SPLIT, THIIM_ENGINE_FUSED, THIIM_ENGINE_TBLOCK}) {
      ProblemState a = random_state(d, 42);
      ProblemState b = clone_state(a);
      run_naive(a, 6, 4);
      GpuOptions o;
      o.engine = engine;
      const RunReport r = run_gpu(b, 6, o);
      const StateDiff diff = compare_states(a, b);
      CHECK(diff.bitwise_equal);
      CHECK(r.steps == 6 && r.threads == 1 && r.mlups.has_value());
      CHECK(r.balance_model == (engine == THIIM_ENGINE_SPLIT    ? 1024.0
                                : engine == THIIM_ENGINE_FUSED ? 832.0
                                                               : 416.0));
    }
  }
}

void test_matches_run_naive_benchmark_problem() {
  // build_benchmark_problem (coefficients.cpp:94-111): vacuum + source plane
  SchemeParams sp;
  const GridDims d(48, 48, 48);
  ProblemState a = build_benchmark_problem(d, sp);
  ProblemState b = clone_state(a);
  run_naive(a, 16, 8);
  run_gpu(b, 16);
  CHECK(compare_states(a, b).bitwise_equal);
}

void test_matches_spatial_and_mwd() {
  // the reference's own tuned engines are bitwise-equal to naive, hence to GPU
  const GridDims d(32, 32, 32);
  ProblemState a = random_state(d, 3);
  ProblemState b = clone_state(a);
  ProblemState c = clone_state(a);
  run_spatial_blocked(a, 4, 8, 0, 4);
  ThreadGroupShape shape;
  run_mwd(b, 4, 8, 1, shape, 1);  // 4 steps = 1 diamond pass at dw 8
  run_gpu(c, 4);
  CHECK(compare_states(a, c).bitwise_equal);
  CHECK(compare_states(b, c).bitwise_equal);
}

void test_empty_run_and_validation() {
  // test_reference_engines.cpp:7-16 and :60-67
  const GridDims d(8, 8, 8);
  SchemeParams sp;
  ProblemState s = build_benchmark_problem(d, sp);
  ProblemState before = clone_state(s);
  const RunReport r = run_gpu(s, 0);
  CHECK(compare_states(before, s).bitwise_equal);
  CHECK(!r.mlups.has_value());
  CHECK(throws_as<ConfigError>([&] { run_gpu(s, -1); }));
  GpuOptions bad;
  bad.n_gpus = 0;
  CHECK(throws_as<ConfigError>([&] { run_gpu(s, 1, bad); }));
}

void test_single_cell_kat() {
  // test_kernels.cpp:27-43, on a whole step: Hyz = 0.5*2 + 1*0.25 + 0.1 = 1.35
  const GridDims d(4, 4, 4);
  ProblemState s = allocate_state(d);
  const ComponentDescriptor& desc = descriptor(Component::Hyz);
  const std::size_t i = d.linear_index(1, 1, 1), j = d.linear_index(1, 1, 2);
  s.field(desc.id)[i] = {2.0, 0.0};
  s.t_of(desc.id)[i] = {0.5, 0.0};
  s.c_of(desc.id)[i] = {1.0, 0.0};
  s.coeff_src[source_index(desc.id)][i] = {0.1, 0.0};
  s.field(desc.operand_a)[j] = {0.25, 0.0};
  run_gpu(s, 1);
  CHECK(std::abs(s.field(desc.id)[i].re - 1.35) <= 1e-15 * 1.35);
  CHECK(s.field(desc.id)[i].im == 0.0);
}

void test_layered_material() {
  const GridDims d(40, 30, 60);
  ProblemState a = random_state(d, 5, THIIM_GEN_LAYERED);
  ProblemState b = clone_state(a);
  run_naive(a, 5, 4);
  run_gpu(b, 5);
  CHECK(compare_states(a, b).bitwise_equal);
}

void test_batch_matches_run_naive() {
  // a stream of distinct problems, each == run_naive on its own copy
  const GridDims d(40, 33, 24);
  std::vector<ProblemState> want, got;
  for (int k = 0; k < 4; ++k) {
    want.push_back(random_state(d, 100 + k, k % 2 ? THIIM_GEN_LAYERED : THIIM_GEN_RANDOM));
    got.push_back(clone_state(want.back()));
  }
  for (auto& s : want) run_naive(s, 5, 4);
  std::vector<ProblemState*> ptrs;
  for (auto& s : got) ptrs.push_back(&s);
  const RunReport r = run_gpu_batch(ptrs, 5);
  for (int k = 0; k < 4; ++k) CHECK(compare_states(want[k], got[k]).bitwise_equal);
  CHECK(r.steps == 5 && r.mlups.has_value() && r.engine == "gpu-tblock");
  // the same state twice would be read while being written back
  std::vector<ProblemState*> twice{&got[0], &got[0]};
  CHECK(throws_as<ConfigError>([&] { run_gpu_batch(twice, 1); }));
  CHECK(throws_as<ConfigError>([&] { run_gpu_batch(ptrs, -1); }));
}

}  // namespace

void test_auto_table_layout() {
  // coeff_layout = THIIM_COEFF_AUTO_HOST: a piecewise-constant medium (the
  // layered stack, the vacuum benchmark problem) runs in the compressed TABLE
  // layout, a random one in the reference layout -- all bitwise run_naive
  SchemeParams sp;
  struct Case {
    ProblemState s;
    bool table;
  };
  std::vector<Case> cases;
  cases.push_back({random_state(GridDims(40, 33, 24), 5, THIIM_GEN_LAYERED), true});
  cases.push_back({build_benchmark_problem(GridDims(32, 32, 32), sp), true});
  cases.push_back({random_state(GridDims(20, 18, 16), 6), false});
  for (Case& c : cases) {
    ProblemState a = clone_state(c.s);
    run_naive(a, 6, 4);
    GpuOptions o;
    o.coeff_layout = THIIM_COEFF_AUTO_HOST;
    const RunReport r = run_gpu(c.s, 6, o);
    CHECK(compare_states(a, c.s).bitwise_equal);
    const bool table = r.engine.size() > 6 && r.engine.compare(r.engine.size() - 6, 6, "-table") == 0;
    CHECK(table == c.table);
    CHECK(r.balance_model == (c.table ? 192.5 : 416.0));
  }
}

int main() {
  const std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"run_gpu matches run_naive (random states, split + fused)", test_matches_run_naive_random},
      {"run_gpu matches run_naive (benchmark problem)", test_matches_run_naive_benchmark_problem},
      {"run_gpu matches run_spatial_blocked and run_mwd", test_matches_spatial_and_mwd},
      {"empty run and argument validation", test_empty_run_and_validation},
      {"single-cell known answer 1.35", test_single_cell_kat},
      {"layered thin-film material", test_layered_material},
      {"run_gpu_batch: stream of problems == run_naive each", test_batch_matches_run_naive},
      {"coeff_layout AUTO_HOST: compressed table layout for piecewise-constant media",
       test_auto_table_layout},
  };
  for (const auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception: %s\n", e.what());
    }
    std::printf("[%s] %s\n", g_fail == before ? "PASS" : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
