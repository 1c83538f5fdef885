// thiim_gpu_bench.cpp -- repo-local driver for the GPU engine with the
// reference CLI's semantics: `thiim-bench run` / `tune`
// (/root/reference/proj/tools/main.cpp:78-151, 165-208) with `--engine gpu`.
//
//   thiim-gpu-bench run  [--config F] [--grid N|NXxNYxNZ] [--steps S]
//                        [--engine gpu|gpu-tblock|gpu-tblock-inplace|gpu-fused|gpu-split]
//                        [--threads G] [--time-block K] [--tile-y R] [--z-chunk Z]
//                        [--band B] [--schedule S] [--bandwidth GBs]
//                        [--report-dir D] [--check] [--sanitize]
//   thiim-gpu-bench tune [--config F] [--grid ..] [--steps S] [--bandwidth GBs]
//                        [--trials N] [--min-seconds T] [--table tune_trials.csv]
//                        [--winner W.json]
//
// The problem is the reference's build_benchmark_problem (coefficients.cpp:94-111)
// for the configured grid and scheme; `--threads` is the number of GPUs (z-slabs
// of one context).  run prints the reference's report line (main.cpp:63-76),
// checks against run_naive like check_against_naive (main.cpp:43-61: `--check`,
// or automatically for grids up to 96^3), runs the exactly-once coverage
// sanitizer with `--sanitize`, and appends the run to <report-dir>/reports.jsonl
// and reports.csv through the reference's emit_reports.  tune is the library's
// thiim_gpu_tune (the reference's enumerate_candidates + tune,
// autotuner.cpp:15-142, over time block x tile height x z-chunk x band x
// schedule, ranked by the GPU models): it times the model's best candidates,
// writes the trial table CSV -- trial_table_csv's layout (autotuner.cpp:165-177)
// with the GPU's knobs and model columns -- and the winner JSON; the winner is
// verified bitwise by the library against the fused engine and here, on the
// reference's benchmark problem, against run_naive (grids up to 96^3).  The
// `--bandwidth` default is MEASURED_PEAKS.json's hbm_gbs when that file is in
// the working directory.  Exit codes follow main.cpp: 0 ok, 1 verification /
// sanitizer failure or other error, 2 bad configuration.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "thiim/coefficients.hpp"
#include "thiim/config.hpp"
#include "thiim/perf_models.hpp"
#include "thiim/reference_engines.hpp"
#include "thiim/report.hpp"
#include "thiim/verifier.hpp"
#include "thiim_gpu.h"
#include "thiim_gpu_engine.hpp"

namespace {

using namespace thiim;

struct Args {
  BenchConfig cfg;
  std::string engine = "gpu";
  int tile_y = 0, z_chunk = 0, time_block = 0, band = 0, schedule = 0;
  int trials = 8;
  double min_seconds = 0.5;
  bool check = false, sanitize = false;
  std::string table = "tune_trials.csv", winner;
};

[[noreturn]] void usage(const char* msg, int code = 2) {
  std::fprintf(stderr,
               "%s%susage: thiim-gpu-bench run|tune [--config F] [--grid N|NXxNYxNZ] "
               "[--steps S] [--engine gpu|gpu-tblock|gpu-tblock-inplace|gpu-fused|gpu-split] "
               "[--threads G] [--time-block K] [--tile-y R] [--z-chunk Z] [--band B] "
               "[--schedule S] [--bandwidth GBs] [--report-dir D] [--check] [--sanitize] "
               "[--trials N] [--min-seconds T] [--table CSV] [--winner JSON]\n",
               msg ? msg : "", msg ? "\n" : "");
  std::exit(code);
}

int engine_id(const std::string& e) {
  if (e == "gpu") return THIIM_ENGINE_AUTO;
  if (e == "gpu-tblock") return THIIM_ENGINE_TBLOCK;
  if (e == "gpu-tblock-inplace") return THIIM_ENGINE_TBLOCK_INPLACE;
  if (e == "gpu-fused") return THIIM_ENGINE_FUSED;
  if (e == "gpu-split") return THIIM_ENGINE_SPLIT;
  throw ConfigError("unknown engine: " + e +
                    " (gpu | gpu-tblock | gpu-tblock-inplace | gpu-fused | gpu-split)");
}

// the reference's report line (tools/main.cpp:63-76)
void print_report(const RunReport& r) {
  std::printf("engine=%s grid=%dx%dx%d steps=%d(executed %d) threads=%d", r.engine.c_str(),
              r.dims.nx, r.dims.ny, r.dims.nz, r.steps, r.steps_executed, r.threads);
  std::printf(" seconds=%.4f", r.seconds);
  if (r.mlups) std::printf(" mlups=%.2f", *r.mlups);
  std::printf(" balance_model=%.2f", r.balance_model);
  if (r.predicted_mlups) std::printf(" predicted_mlups=%.2f", *r.predicted_mlups);
  std::printf("\n");
}

int host_threads() {
  const unsigned n = std::thread::hardware_concurrency();
  return n ? (int)n : 1;
}

// check_against_naive (tools/main.cpp:43-61)
bool check_against_naive(const ProblemState& before, const ProblemState& after, int steps,
                         RunReport& report) {
  ProblemState ref = clone_state(before);
  run_naive(ref, steps, host_threads());
  const StateDiff diff = compare_states(ref, after);
  if (diff.bitwise_equal) {
    report.verification = "bitwise-equal";
    std::printf("verification: bitwise-equal\n");
    return true;
  }
  report.verification = "failed";
  std::fprintf(stderr,
               "verification FAILED: max |diff| = %.17g, first at %s (%d,%d,%d), %llu values "
               "differ\n",
               diff.max_abs_diff, std::string(component_name(diff.first_component)).c_str(),
               diff.x, diff.y, diff.z, (unsigned long long)diff.differing_values);
  return false;
}

GpuOptions gpu_options(const Args& a, int engine, int tile_y) {
  GpuOptions o;
  o.n_gpus = a.cfg.threads;
  o.engine = engine;
  o.tile_y = tile_y;
  o.z_chunk = a.z_chunk;
  o.time_block = a.time_block;
  o.band = a.band;
  o.schedule = a.schedule;
  o.sanitize = a.sanitize;
  o.hbm_gbs = a.cfg.profile.bandwidth_gbs;
  return o;
}

int do_run(const Args& a) {
  const BenchConfig& cfg = a.cfg;
  ProblemState state = build_benchmark_problem(cfg.grid, cfg.scheme);
  const bool auto_check = cfg.steps > 0 && cfg.grid.interior_cells() <= 96ull * 96 * 96;
  const bool do_check = a.check || auto_check;
  ProblemState before = do_check ? clone_state(state) : ProblemState{};
  GpuRunExtras ex;
  RunReport report = run_gpu(state, cfg.steps, gpu_options(a, engine_id(a.engine), a.tile_y), &ex);
  report.predicted_mlups = predict_mlups(cfg.profile.bandwidth_gbs, report.balance_model);
  int rc = 0;
  if (do_check && cfg.steps > 0 && !check_against_naive(before, state, cfg.steps, report)) rc = 1;
  if (a.sanitize) {
    const bool ok = ex.coverage_violations == 0 && ex.coverage_passes > 0;
    std::printf("sanitizer: exactly-once coverage %s (%llu passes, %llu violations)\n",
                ok ? "OK" : "VIOLATED", ex.coverage_passes, ex.coverage_violations);
    if (!ok) rc = 1;
  }
  print_report(report);
  emit_reports({report}, cfg.report_dir);
  return rc;
}

// tune (autotuner.cpp:62-142) over the GPU knobs: thiim_gpu_tune ranks the
// candidates by the GPU models, times the best, verifies the winner against
// the fused engine; here the winner is also checked against run_naive on the
// reference's benchmark problem (grids up to 96^3, like check_against_naive).
int do_tune(const Args& a) {
  const BenchConfig& cfg = a.cfg;
  if (cfg.steps < 1) throw ConfigError("tune needs --steps >= 1");
  if (cfg.threads != 1) throw ConfigError("tune runs on one GPU (--threads 1)");
  const thiim_dims d{cfg.grid.nx, cfg.grid.ny, cfg.grid.nz, cfg.grid.ghost};
  thiim_gpu_opts base;
  thiim_gpu_default_opts(&base);
  std::vector<thiim_gpu_trial> table((std::size_t)a.trials + 2);
  int n = 0, verified = 0;
  thiim_gpu_opts w;
  const int rc = thiim_gpu_tune(&d, &base, cfg.steps, a.min_seconds, a.trials, table.data(),
                                (int)table.size(), &n, &w, &verified);
  if (rc == THIIM_ERR_CONFIG) throw ConfigError(thiim_gpu_last_error());
  if (rc) throw std::runtime_error(std::string("thiim_gpu_tune: ") + thiim_gpu_last_error());
  {
    std::ofstream out(a.table);
    if (!out) throw ConfigError("cannot write " + a.table);
    out << "engine,time_block,tile_y,z_chunk,band,schedule,tiles,rounds,balance_model,"
           "model_bytes_per_lup,model_mlups,l2_set_bytes,steps,seconds,mlups,ok,note\n";
    for (int i = 0; i < n; ++i) {
      const thiim_gpu_trial& t = table[i];
      const thiim_gpu_candidate& c = t.cand;
      out << "gpu-tblock," << c.time_block << ',' << c.tile_y << ',' << c.z_chunk << ','
          << c.band << ',' << c.schedule << ',' << c.tiles << ',' << c.rounds << ','
          << c.balance_model << ',' << c.model_bytes_per_lup << ',' << c.model_mlups << ','
          << c.l2_set_bytes << ',' << t.steps << ',' << t.seconds << ',' << t.mlups << ','
          << t.ok << ',' << t.note << '\n';
    }
  }
  double best = 0.0;
  for (int i = 0; i < n; ++i)
    if (table[i].ok && table[i].cand.time_block == w.time_block && table[i].cand.tile_y == w.tile_y &&
        table[i].cand.z_chunk == w.z_chunk && table[i].cand.band == w.band &&
        table[i].cand.schedule == w.schedule)
      best = table[i].mlups;
  std::string verification = verified ? "bitwise-equal vs gpu-fused" : "failed";
  if (verified && cfg.grid.interior_cells() <= 96ull * 96 * 96) {
    const ProblemState base_state = build_benchmark_problem(cfg.grid, cfg.scheme);
    ProblemState got = clone_state(base_state), ref = clone_state(base_state);
    GpuOptions go;
    go.engine = THIIM_ENGINE_TBLOCK;
    go.time_block = w.time_block;
    go.tile_y = w.tile_y;
    go.z_chunk = std::min(w.z_chunk, cfg.grid.nz);
    go.band = w.band;
    go.schedule = w.schedule;
    run_gpu(got, cfg.steps, go);
    run_naive(ref, cfg.steps, host_threads());
    verification = compare_states(ref, got).bitwise_equal ? "bitwise-equal vs naive" : "failed";
  }
  char js[512];
  std::snprintf(js, sizeof js,
                "{\"engine\":\"gpu-tblock\",\"time_block\":%d,\"tile_y\":%d,\"z_chunk\":%d,"
                "\"band\":%d,\"schedule\":%d,\"balance_model\":%g,\"mlups\":%.2f,"
                "\"trials\":%d}",
                w.time_block, w.tile_y, w.z_chunk, w.band, w.schedule,
                thiim_gpu_balance_model(THIIM_ENGINE_TBLOCK, w.time_block), best, n);
  std::printf("winner: %s (verification: %s)\n", js, verification.c_str());
  if (!a.winner.empty()) {
    std::ofstream out(a.winner);
    out << js << '\n';
  }
  return verification == "failed" ? 1 : 0;
}

// MEASURED_PEAKS.json hbm_gbs (driver-written, in the working directory), else
// 6536 GB/s (the measured B200 copy peak of this pool)
double measured_hbm_gbs() {
  std::ifstream f("MEASURED_PEAKS.json");
  std::string s((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  const std::size_t k = s.find("\"hbm_gbs\"");
  if (k != std::string::npos) {
    const std::size_t c = s.find(':', k);
    if (c != std::string::npos) {
      const double v = std::atof(s.c_str() + c + 1);
      if (v > 0) return v;
    }
  }
  return 6536.0;
}

Args parse(int argc, char** argv) {
  Args a;
  a.cfg.engine = "gpu";
  std::string config_path, grid_spec;
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) usage(("missing value for " + k).c_str());
      return argv[++i];
    };
    if (k == "--config") config_path = val();
    else if (k == "--grid") grid_spec = val();
    else if (k == "--steps") a.cfg.steps = std::stoi(val());
    else if (k == "--engine") a.engine = val();
    else if (k == "--threads") a.cfg.threads = std::stoi(val());
    else if (k == "--tile-y") a.tile_y = std::stoi(val());
    else if (k == "--time-block") a.time_block = std::stoi(val());
    else if (k == "--band") a.band = std::stoi(val());
    else if (k == "--schedule") a.schedule = std::stoi(val());
    else if (k == "--trials") a.trials = std::stoi(val());
    else if (k == "--min-seconds") a.min_seconds = std::stod(val());
    else if (k == "--z-chunk") a.z_chunk = std::stoi(val());
    else if (k == "--bandwidth") a.cfg.profile.bandwidth_gbs = std::stod(val());
    else if (k == "--report-dir") a.cfg.report_dir = val();
    else if (k == "--table") a.table = val();
    else if (k == "--winner") a.winner = val();
    else if (k == "--check") a.check = true;
    else if (k == "--sanitize") a.sanitize = true;
    else usage(("unknown option " + k).c_str());
  }
  if (!config_path.empty()) {  // file values, then the flags given (main.cpp:383-411)
    Args f = a;
    f.cfg = BenchConfig::from_file(config_path);
    if (a.cfg.steps != BenchConfig{}.steps) f.cfg.steps = a.cfg.steps;
    if (a.cfg.threads != BenchConfig{}.threads) f.cfg.threads = a.cfg.threads;
    if (a.cfg.report_dir != BenchConfig{}.report_dir) f.cfg.report_dir = a.cfg.report_dir;
    a = f;
  }
  if (!grid_spec.empty()) a.cfg.grid = parse_grid(grid_spec);
  // (no THIIM_THREADS override: --threads counts GPUs here)
  if (a.cfg.profile.bandwidth_gbs == MachineProfile{}.bandwidth_gbs)
    a.cfg.profile.bandwidth_gbs = measured_hbm_gbs();
  if (a.cfg.threads < 1) throw ConfigError("--threads must be >= 1");
  return a;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) usage(nullptr);
  const std::string cmd = argv[1];
  if (cmd == "--help" || cmd == "-h") usage(nullptr, 0);
  try {
    const Args a = parse(argc, argv);
    if (cmd == "run") return do_run(a);
    if (cmd == "tune") return do_tune(a);
    usage(("unknown subcommand " + cmd).c_str());
  } catch (const ConfigError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const SetupError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
