// thiim_gpu_engine.hpp -- the reference-side binding of libthiim_gpu.so.
//
// A maintainer drops this header (and thiim_gpu_engine.cpp) next to the
// reference engines (/root/reference/proj/include/thiim/reference_engines.hpp)
// and gets a GPU time loop with run_naive's contract:
//
//   RunReport run_naive(ProblemState&, int steps, int threads = 1, UpdateLog* = nullptr);
//                                   -- reference_engines.hpp:12-13
//   RunReport run_gpu(ProblemState&, int steps, const GpuOptions& = {});
//                                   -- this file
//
// Same semantics: `steps` x step_reference (kernels.cpp:105-113) applied to
// state.fields in place, coefficients read-only, ghosts never written,
// results bitwise equal to run_naive.  Errors are the reference's:
// ConfigError (bad arguments), SetupError (dims, allocation), std::runtime_error
// (CUDA / device).  See INTEGRATION.md for the CLI branch (tools/main.cpp:106-126).
#pragma once

#include "thiim/report.hpp"
#include "thiim/state.hpp"
#include "thiim_gpu.h"

#include <vector>

namespace thiim {

struct GpuOptions {
  int device = 0;                  // first CUDA device
  int n_gpus = 1;                  // z-slabs, one per device (single process)
  int engine = THIIM_ENGINE_AUTO;  // THIIM_ENGINE_SPLIT / FUSED / TBLOCK
  int time_block = 0;              // TBLOCK: steps per HBM pass (0 = auto)
  int z_chunk = 0;                 // planes per CTA along z (0 = auto)
  int tile_y = 0;                  // CTA height in rows (0 = the engine default)
  int band = 0;                    // TBLOCK rounds: tile columns per band (0 = auto)
  int schedule = 0;                // TBLOCK CTA schedule (0 = rounds, 1 = one launch)
  bool sanitize = false;           // exactly-once store coverage check per pass
  bool pin_host = true;            // page-lock the 40 arrays during the copies
  // coefficient storage on the device: THIIM_COEFF_FULL (the reference
  // layout) or THIIM_COEFF_AUTO_HOST: compress the state's coefficients on the
  // host (thiim_coeff_compress) and run the TABLE layout when the medium has
  // <= 16 distinct coefficient rows (layered stacks), else FULL
  int coeff_layout = THIIM_COEFF_FULL;
  double hbm_gbs = 0.0;            // if > 0: predicted_mlups = hbm_gbs / balance
};

// Upload `state`, run `steps` THIIM iterations on the GPU(s), download the 12
// fields back into `state`.  RunReport: engine "gpu-split|gpu-fused|gpu-tblock|
// gpu-tblock-inplace" (+ "-table" when the compressed layout ran),
// threads = #GPUs, seconds = device time of the step loop (CUDA events),
// mlups = interior*steps/seconds/1e6, balance_model = algorithmic bytes/LUP.
RunReport run_gpu(ProblemState& state, int steps, const GpuOptions& opts = {});

// What a run measured beyond RunReport.
struct GpuRunExtras {
  unsigned long long coverage_passes = 0;      // sanitize: passes checked
  unsigned long long coverage_violations = 0;  // sanitize: (component, cell) violations
  long long kernel_launches = 0;
};
RunReport run_gpu(ProblemState& state, int steps, const GpuOptions& opts, GpuRunExtras* extras);

// A stream of independent problems of one shape (e.g. the paper's sweep over
// wavelengths): every state advanced `steps` iterations in place, each bitwise
// == run_naive(*state, steps).  One GPU; uploads, sweeps and downloads of
// consecutive problems overlap (thiim_gpu_run_batch).  The states must be
// distinct objects (ConfigError otherwise).  RunReport of the whole stream:
// seconds = wall clock of the call (copies included), mlups =
// states x interior x steps / seconds, threads = 1.
RunReport run_gpu_batch(const std::vector<ProblemState*>& states, int steps,
                        const GpuOptions& opts = {});

}  // namespace thiim
