// thiim_gpu_engine.cpp -- thiim::run_gpu over the C-ABI (include/thiim_gpu.h).
#include "thiim_gpu_engine.hpp"

#include <stdexcept>
#include <string>
#include <vector>

namespace thiim {

namespace {

void check(int rc, const char* what) {
  if (rc == THIIM_OK) return;
  const std::string msg = std::string(what) + ": " + thiim_gpu_last_error();
  if (rc == THIIM_ERR_CONFIG) throw ConfigError(msg);
  if (rc == THIIM_ERR_SETUP) throw SetupError(msg);
  throw std::runtime_error(msg);
}

const char* engine_name(int e) {
  switch (e) {
    case THIIM_ENGINE_SPLIT: return "gpu-split";
    case THIIM_ENGINE_TBLOCK: return "gpu-tblock";
    case THIIM_ENGINE_TBLOCK_INPLACE: return "gpu-tblock-inplace";
    default: return "gpu-fused";
  }
}

void apply(const GpuOptions& opts, thiim_gpu_opts& o) {
  o.device = opts.device;
  o.n_gpus = opts.n_gpus;
  o.engine = opts.engine;
  o.time_block = opts.time_block;
  o.z_chunk = opts.z_chunk;
  o.tile_y = opts.tile_y;
  o.band = opts.band;
  o.schedule = opts.schedule;
}

// RAII over the page-lock of the 40 host arrays.
struct PinGuard {
  std::vector<void*> pinned;
  void pin(void* p, std::size_t bytes) {
    if (thiim_gpu_pin_host(p, bytes) == THIIM_OK) pinned.push_back(p);
  }
  ~PinGuard() {
    for (void* p : pinned) thiim_gpu_unpin_host(p);
  }
};

struct CtxGuard {
  thiim_gpu_ctx* ctx = nullptr;
  ~CtxGuard() { thiim_gpu_destroy(ctx); }
};

}  // namespace

RunReport run_gpu(ProblemState& state, int steps, const GpuOptions& opts) {
  return run_gpu(state, steps, opts, nullptr);
}

RunReport run_gpu(ProblemState& state, int steps, const GpuOptions& opts, GpuRunExtras* extras) {
  if (steps < 0) throw ConfigError("steps must be >= 0");  // reference_engines.cpp:35
  RunReport report;
  report.dims = state.dims;
  report.steps = report.steps_executed = steps;
  report.threads = opts.n_gpus;

  thiim_dims d{state.dims.nx, state.dims.ny, state.dims.nz, state.dims.ghost};
  thiim_gpu_opts o;
  thiim_gpu_default_opts(&o);
  apply(opts, o);

  // THIIM_COEFF_AUTO_HOST: piecewise-constant media (<= 16 distinct rows)
  // run in the compressed TABLE layout, bitwise the same results
  std::vector<uint8_t> mid;
  std::vector<thiim_c128> tab;
  if (opts.coeff_layout == THIIM_COEFF_AUTO_HOST) {
    const thiim_c128* co[28];
    for (int i = 0; i < kNumComponents; ++i) {
      co[i] = reinterpret_cast<const thiim_c128*>(state.coeff_t[i].data());
      co[12 + i] = reinterpret_cast<const thiim_c128*>(state.coeff_c[i].data());
    }
    for (int i = 0; i < kNumSourceComponents; ++i)
      co[24 + i] = reinterpret_cast<const thiim_c128*>(state.coeff_src[i].data());
    mid.resize(state.dims.padded_cells());
    tab.resize(16 * 28);
    int n = 0;
    check(thiim_coeff_compress(&d, co, 16, mid.data(), tab.data(), &n), "thiim_coeff_compress");
    if (n > 0) {
      o.coeff_layout = THIIM_COEFF_TABLE;
      o.n_materials = n;
    } else {
      mid.clear();
    }
  } else {
    o.coeff_layout = opts.coeff_layout;
  }
  const bool packed = !mid.empty();

  CtxGuard g;
  check(thiim_gpu_create(&d, &o, &g.ctx), "thiim_gpu_create");
  if (opts.sanitize) check(thiim_gpu_set_sanitize(g.ctx, 1), "thiim_gpu_set_sanitize");

  const std::size_t bytes = state.dims.padded_cells() * sizeof(ComplexScalar);
  const thiim_c128* f[12];
  const thiim_c128* t[12];
  const thiim_c128* c[12];
  const thiim_c128* s[4];
  PinGuard pins;
  for (int i = 0; i < kNumComponents; ++i) {
    f[i] = reinterpret_cast<const thiim_c128*>(state.fields[i].data());
    t[i] = reinterpret_cast<const thiim_c128*>(state.coeff_t[i].data());
    c[i] = reinterpret_cast<const thiim_c128*>(state.coeff_c[i].data());
    if (opts.pin_host) {
      pins.pin(state.fields[i].data(), bytes);
      pins.pin(state.coeff_t[i].data(), bytes);
      pins.pin(state.coeff_c[i].data(), bytes);
    }
  }
  for (int i = 0; i < kNumSourceComponents; ++i) {
    s[i] = reinterpret_cast<const thiim_c128*>(state.coeff_src[i].data());
    if (opts.pin_host) pins.pin(state.coeff_src[i].data(), bytes);
  }
  if (packed)
    check(thiim_gpu_upload_table(g.ctx, f, mid.data(), tab.data()), "thiim_gpu_upload_table");
  else
    check(thiim_gpu_upload(g.ctx, f, t, c, s), "thiim_gpu_upload");

  thiim_gpu_stats st{};
  check(thiim_gpu_step(g.ctx, steps, &st), "thiim_gpu_step");
  if (extras) {
    extras->kernel_launches = st.kernel_launches;
    if (opts.sanitize)
      check(thiim_gpu_coverage(g.ctx, &extras->coverage_passes, &extras->coverage_violations),
            "thiim_gpu_coverage");
  }

  thiim_c128* out[12];
  for (int i = 0; i < kNumComponents; ++i)
    out[i] = reinterpret_cast<thiim_c128*>(state.fields[i].data());
  check(thiim_gpu_download_fields(g.ctx, out), "thiim_gpu_download_fields");

  report.engine = std::string(engine_name(st.engine)) + (packed ? "-table" : "");
  report.seconds = st.seconds;
  report.balance_model = st.balance_model;
  if (steps > 0 && st.seconds > 0.0)  // reference_engines.cpp:19-23
    report.mlups = double(state.dims.interior_cells()) * steps / st.seconds / 1e6;
  if (opts.hbm_gbs > 0.0) report.predicted_mlups = opts.hbm_gbs * 1e3 / st.balance_model;
  report.verification = "skipped";
  return report;
}

RunReport run_gpu_batch(const std::vector<ProblemState*>& states, int steps, const GpuOptions& opts) {
  if (steps < 0) throw ConfigError("steps must be >= 0");
  if (opts.n_gpus != 1) throw ConfigError("run_gpu_batch drives one GPU (n_gpus = 1)");
  RunReport report;
  report.steps = report.steps_executed = steps;
  report.threads = 1;
  if (states.empty()) return report;
  const GridDims dims = states[0]->dims;
  report.dims = dims;
  const std::size_t bytes = dims.padded_cells() * sizeof(ComplexScalar);
  std::vector<const thiim_c128*> in;
  in.reserve(states.size() * 40);
  PinGuard pins;
  auto add = [&](const FieldArray& a) {
    in.push_back(reinterpret_cast<const thiim_c128*>(a.data()));
    if (opts.pin_host) pins.pin(const_cast<ComplexScalar*>(a.data()), bytes);
  };
  for (ProblemState* st : states) {
    if (!st) throw ConfigError("null state");
    if (st->dims.nx != dims.nx || st->dims.ny != dims.ny || st->dims.nz != dims.nz)
      throw ConfigError("all problems of a batch need the same grid dims");
    for (int i = 0; i < kNumComponents; ++i) add(st->fields[i]);
    for (int i = 0; i < kNumComponents; ++i) add(st->coeff_t[i]);
    for (int i = 0; i < kNumComponents; ++i) add(st->coeff_c[i]);
    for (int i = 0; i < kNumSourceComponents; ++i) add(st->coeff_src[i]);
  }
  thiim_dims d{dims.nx, dims.ny, dims.nz, dims.ghost};
  thiim_gpu_opts o;
  thiim_gpu_default_opts(&o);
  apply(opts, o);
  o.n_gpus = 1;
  thiim_gpu_batch_stats bs{};
  check(thiim_gpu_run_batch(&d, &o, int(states.size()), in.data(), nullptr, steps, 0, &bs),
        "thiim_gpu_run_batch");
  report.engine = engine_name(bs.engine);
  report.seconds = bs.seconds;
  report.balance_model = thiim_gpu_balance_model(bs.engine, opts.time_block);
  if (steps > 0 && bs.seconds > 0.0) report.mlups = bs.mlups;
  report.verification = "skipped";
  return report;
}

}  // namespace thiim
