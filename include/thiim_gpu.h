/*
 * thiim_gpu.h -- C-ABI of the B200 THIIM sweep engine (libthiim_gpu.so).
 *
 * The drop-in boundary for the reference's hot path.  The reference
 * (arXiv 1510.05218 THIIM, /root/reference/proj) exposes a C++ driver API:
 *
 *   ProblemState build/fill   include/thiim/coefficients.hpp:66-79, state.hpp:49-66
 *   time loop                 RunReport run_naive(ProblemState&, int steps,
 *                                                 int threads, UpdateLog*)
 *                             include/thiim/reference_engines.hpp:12-13
 *   readback                  ProblemState::fields / field(Component) state.hpp:51-57
 *
 * This header replaces the time loop with a GPU engine.  No C++ or torch types
 * cross it: plain pointers and sizes, status codes instead of exceptions.  The
 * C++ adapter thiim::run_gpu(ProblemState&, int, const GpuOptions&) in
 * adapter/thiim_gpu_engine.hpp is the reference-side binding; INTEGRATION.md
 * shows how a maintainer wires it next to run_naive.
 *
 * Semantics: thiim_gpu_step(ctx, n) == n calls of step_reference
 * (kernels.cpp:105-113): per step the six H components (kHOrder), then the
 * six E components (kEOrder), over the full interior, ghosts never written.
 * Results are BITWISE equal to the reference built without FMA contraction
 * (kernels are compiled with -fmad=false and use explicit round-to-nearest
 * intrinsics in the reference's per-cell operation order, kernels.cpp:43-51).
 *
 * Threading: calls on one context are synchronous and not reentrant, like the
 * reference engines (worker_pool.hpp:39-64).  Distinct contexts are
 * independent.
 */
#ifndef THIIM_GPU_H
#define THIIM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define THIIM_GPU_ABI_VERSION 2

/* == thiim::ComplexScalar (include/thiim/complex.hpp:11-20). */
typedef struct { double re, im; } thiim_c128;

/* == thiim::GridDims (include/thiim/grid.hpp:12-48); ghost must be 1,
 * n >= 4 per axis (GridDims::valid, grid.hpp:21).  Every array is
 * (nx+2)*(ny+2)*(nz+2) elements, x unit-stride, z slowest. */
typedef struct { int nx, ny, nz, ghost; } thiim_dims;

/* Status codes.  The C++ adapter maps CONFIG -> thiim::ConfigError and
 * SETUP -> thiim::SetupError (grid.hpp:50-60), the rest -> std::runtime_error,
 * mirroring the CLI's exit-code split (tools/main.cpp:438-450). */
enum {
  THIIM_OK = 0,
  THIIM_ERR_CONFIG = 2, /* bad argument (negative steps, bad engine, ...) */
  THIIM_ERR_SETUP = 3,  /* invalid dims, device allocation failure */
  THIIM_ERR_CUDA = 4,   /* CUDA runtime error or no device */
  THIIM_ERR_COMM = 5,   /* halo exchange / peer access failure */
  THIIM_ERR_STATE = 6   /* call order (step before upload, ...) */
};

/* Engines (all bitwise-equal to step_reference).  AUTO picks TBLOCK (two steps
 * per HBM pass, 416 B/LUP; odd remainders run one fused step) when the
 * ping-pong state fits, else SPLIT. */
enum {
  THIIM_ENGINE_AUTO = 0,
  THIIM_ENGINE_SPLIT = 1, /* H sweep + E sweep, in place, z-streamed: 1024 B/LUP */
  THIIM_ENGINE_FUSED = 2, /* one z-streamed H->E sweep per step, ping-pong fields: 832 B/LUP */
  THIIM_ENGINE_TBLOCK = 3, /* temporally blocked fused sweep, `time_block` steps per pass */
  /* TBLOCK on one field set (state that fits in place but not twice): every
   * field array gets a gap of L + 2 planes; a pass sweeps z sub-ranges of L
   * planes and stores their outputs L + 2 planes away, alternately up and
   * down, so nothing is copied back: 416 B/LUP.  One whole-z slab; AUTO picks
   * it over SPLIT when >= 8 gap planes fit.  THIIM_INPLACE_TB=L (env) sets L,
   * 0 disables it under AUTO. */
  THIIM_ENGINE_TBLOCK_INPLACE = 4
};

/* Synthetic problem kinds for thiim_gpu_init_generated / thiim_generate_host
 * (BASELINE.json configs). */
enum {
  THIIM_GEN_RANDOM = 0,  /* fields U[-1,1]^2, 28 coefficient arrays uniform in |z|<=0.45 */
  THIIM_GEN_LAYERED = 1  /* config 3: 6 z-layers, seeded +-8-cell interface height maps */
};

typedef struct {
  int device;       /* CUDA device ordinal of the first slab */
  int n_gpus;       /* z-slabs driven by this context (1..8), one device each */
  int engine;       /* THIIM_ENGINE_* */
  int tile_x;       /* 0 = auto */
  int tile_y;       /* 0 = auto */
  int z_chunk;      /* planes per CTA along the z-stream, 0 = auto */
  int time_block;   /* TBLOCK: steps per HBM pass, 0 = auto */
  int schedule;     /* TBLOCK CTA schedule: 0 = auto (rounds of <= one CTA per SM,
                       tiles in bands, so neighbouring tiles stream the same planes at
                       the same time), 1 = one launch of all tiles (x-fastest order) */
  int band;         /* TBLOCK rounds: tile columns per band, 0 = auto */
  int same_device;  /* test knob: 1 places every slab on `device` (exercises the
                       multi-slab paths on one GPU) */
  int reserved[4];  /* 0 */
  int coeff_layout; /* THIIM_COEFF_FULL (28 arrays) or THIIM_COEFF_TABLE (material ids) */
  int n_materials;  /* THIIM_COEFF_TABLE: rows of the coefficient table (<= 64) */
} thiim_gpu_opts;

/* Coefficient storage.  FULL is the reference layout (28 domain arrays).
 * TABLE is the compressed layout for piecewise-constant media:
 * a uint8 material id per cell plus a [n_materials][28] table (t x12, c x12,
 * src x4, ProblemState order); the fused sweep then moves 385 instead of
 * 832 B/LUP.  Results are bitwise those of the equivalent FULL problem; the
 * figure is reported separately from the reference-layout roofline. */
enum { THIIM_COEFF_FULL = 0, THIIM_COEFF_TABLE = 1 };
/* Not a context layout: host-side adapters (thiim::run_gpu, Python run_gpu)
 * take it to mean "TABLE when thiim_coeff_compress finds <= 16 rows, else FULL". */
enum { THIIM_COEFF_AUTO_HOST = 2 };

/* Host-side compression of a reference-layout problem into the TABLE form
 * (for callers that hold the reference's ProblemState of a piecewise-
 * constant medium, e.g. the paper's layered thin-film stacks): when the
 * INTERIOR cells carry at most max_materials (<= 16) distinct coefficient
 * rows (t x12, c x12, src x4 compared bit for bit), writes material_id
 * (padded layout, (nx+2)(ny+2)(nz+2) bytes, ghosts 0) and table
 * [n][28] in order of first appearance along the linear interior index,
 * and sets *n_materials = n; otherwise *n_materials = 0 (outputs undefined).
 * Ghost-cell coefficients are never read by any engine and are ignored.
 * coeffs[k] = ProblemState array 12 + k.  OpenMP over z-planes; no device. */
int thiim_coeff_compress(const thiim_dims* dims, const thiim_c128* const coeffs[28],
                         int max_materials, uint8_t* material_id, thiim_c128* table,
                         int* n_materials);

typedef struct {
  double seconds;          /* device time of the whole step loop (CUDA events) */
  double mlups;            /* interior*steps/seconds/1e6 (reference_engines.cpp:19-23) */
  double balance_model;    /* algorithmic bytes per LUP of the engine that ran */
  double kernel_seconds;   /* device time summed over the sweep kernels only */
  long long kernel_launches;
  int steps;
  int engine;              /* engine that actually ran (AUTO resolved) */
  int n_gpus;
  int reserved[5];
} thiim_gpu_stats;

typedef struct thiim_gpu_ctx thiim_gpu_ctx;

void thiim_gpu_default_opts(thiim_gpu_opts* opts);

/* Allocates device state for `dims` (reference padded layout).  Fields and
 * coefficients start zeroed, like allocate_state (state.cpp:5-16). */
int thiim_gpu_create(const thiim_dims* dims, const thiim_gpu_opts* opts, thiim_gpu_ctx** out);

/* Uploads a full ProblemState: 12 fields (Component order, components.hpp:17-30),
 * 12 t, 12 c (same order), 4 src (source_index order, components.hpp:89-97).
 * Host arrays are (nx+2)(ny+2)(nz+2) elements, ghosts included. */
int thiim_gpu_upload(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12],
                     const thiim_c128* const t[12], const thiim_c128* const c[12],
                     const thiim_c128* const src[4]);

/* Uploads the 12 field arrays only (coefficients unchanged). */
int thiim_gpu_upload_fields(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12]);

/* Generates a synthetic problem directly in HBM (no PCIe traffic); bitwise
 * identical to thiim_generate_host with the same (kind, seed). */
int thiim_gpu_init_generated(thiim_gpu_ctx* ctx, int kind, uint64_t seed);

/* The reference's benchmark problem built on the device:
 * build_benchmark_problem (coefficients.cpp:94-111) -- homogeneous vacuum
 * medium, Dirichlet ghosts, plane-wave source layer at z = nz/4, fields zero --
 * for scheme parameters `sp` (SchemeParams, coefficients.hpp:21-34).  The 28
 * per-component coefficient values are the closed forms of derive_coefficients
 * (coefficients.cpp:25-55) evaluated once on the host with the reference's
 * complex arithmetic; the device broadcasts them, so the 40 arrays never cross
 * PCIe and the result is bitwise the reference's.  Table-layout contexts get
 * material ids (interior 1, source plane 2) and the 3-row table.  Errors:
 * CONFIG for invalid parameters (SchemeParams::validate), SETUP for a vanishing
 * update denominator. */
typedef struct {
  double omega, tau, delta;
  thiim_c128 source_e, source_h;
} thiim_scheme;
void thiim_scheme_default(thiim_scheme* sp); /* omega 0.4, tau 1, delta 1, sources 1+0i */
int thiim_gpu_init_benchmark(thiim_gpu_ctx* ctx, const thiim_scheme* sp);

/* build_problem_from_voxels (coefficients.cpp:112-141) on the device: `materials`
 * holds nx*ny*nz records of 5 doubles (eps_re, eps_im, mu, sigma, sigma_star),
 * x fastest -- the reference's voxel-map layout; 40 B/cell cross PCIe instead of
 * the 448 B/cell of coefficients.  The per-cell closed forms run on the GPU
 * with the host build's complex arithmetic (libgcc's division restated), so the
 * coefficients are bitwise the reference's.  Fields zero, source on plane nz/4.
 * Errors: CONFIG (parameters, table layout), SETUP with the reference's message
 * ("mu must be nonzero", "eps must be nonzero", "vanishing update denominator
 * ... at cell (x,y,z) component C") for the first failing (component, cell). */
int thiim_gpu_init_materials(thiim_gpu_ctx* ctx, const thiim_scheme* sp, const double* materials);

/* Verification entry: n complex divisions (a+ib)/(c+id), in = {a,b,c,d}[n],
 * out = {re,im}[n], with the device restatement of libgcc's __divdc3. */
int thiim_gpu_selftest_cdiv(int n, const double* in, double* out);

/* Advances `steps` THIIM iterations (== steps x step_reference).  Blocking.
 * steps < 0 -> THIIM_ERR_CONFIG (run_naive, reference_engines.cpp:35). */
int thiim_gpu_step(thiim_gpu_ctx* ctx, int steps, thiim_gpu_stats* stats);

/* Copies the 12 current field arrays back (ghosts included). */
int thiim_gpu_download_fields(thiim_gpu_ctx* ctx, thiim_c128* const fields[12]);

/* Copies one of the 40 arrays back: 0..11 fields, 12..23 t, 24..35 c, 36..39 src. */
int thiim_gpu_download_array(thiim_gpu_ctx* ctx, int array_id, thiim_c128* dst);

/* On-device comparison of the current fields against 12 host arrays (interior
 * only, like compare_states, verifier.cpp:13-44): bitwise mismatch count plus
 * the worst per-component relative L2 error ||a-b||/||b||. */
typedef struct {
  unsigned long long differing_values;
  double max_rel_l2;
  double rel_l2[12];
} thiim_gpu_diff;
int thiim_gpu_compare_fields(thiim_gpu_ctx* ctx, const thiim_c128* const ref_fields[12],
                             thiim_gpu_diff* out);

/* A stream of independent problems on one GPU (e.g. the paper's sweep over
 * wavelengths): for each problem i, == run_naive(problem i, steps)
 * (reference_engines.cpp:34-67) with the result's 12 fields written to
 * outputs[12*i .. 12*i+11] (NULL outputs: back into the problem's own field
 * arrays, in place like run_naive).  inputs[40*i .. 40*i+39] are problem i's
 * arrays in thiim_gpu_upload order (12 fields, 12 t, 12 c, 4 src).
 * Problems are pipelined over `depth` device contexts (<= 0: 3; fewer when
 * device memory holds fewer, stats->depth says how many ran): problem i
 * uploads while i-1 computes and i-2 downloads, each resource in problem
 * order.  Under THIIM_ENGINE_AUTO, when device memory holds fewer than two
 * ping-pong TBLOCK contexts but two or more TBLOCK-in-place ones (one field
 * set each), the batch runs in place whenever overlapping the copies with the
 * sweeps wins by the library's model (stats->engine, stats->depth).  Host
 * buffers should be pinned (thiim_gpu_pin_host) for the copies to overlap.
 * An output may be shared by several problems but must not overlap another
 * problem's inputs (THIIM_ERR_CONFIG).  Blocking; reference layout,
 * n_gpus = 1. */
typedef struct {
  double seconds;          /* host wall clock of the whole call, contexts included */
  double device_seconds;   /* first upload start .. last download end (device events) */
  double upload_seconds;   /* sums over problems of each phase's device time */
  double kernel_seconds;
  double download_seconds;
  double mlups;            /* n_problems x interior cells x steps / seconds / 1e6 */
  long long kernel_launches;
  long long h2d_bytes, d2h_bytes;
  int n_problems, depth, engine;
  int reserved[5];
} thiim_gpu_batch_stats;
int thiim_gpu_run_batch(const thiim_dims* dims, const thiim_gpu_opts* opts, int n_problems,
                        const thiim_c128* const* inputs, thiim_c128* const* outputs, int steps,
                        int depth, thiim_gpu_batch_stats* stats);

/* Host-side generator for the same synthetic problem (for CPU oracles and for
 * uploading); arrays must be zeroed or are fully overwritten (ghosts -> 0). */
int thiim_generate_host(const thiim_dims* dims, int kind, uint64_t seed,
                        thiim_c128* const arrays[40]);

/* Page-locks (cudaHostRegister) / unlocks a host buffer so uploads and
 * downloads run at full PCIe rate.  Optional. */
int thiim_gpu_pin_host(void* ptr, size_t bytes);
int thiim_gpu_unpin_host(void* ptr);

void thiim_gpu_destroy(thiim_gpu_ctx* ctx);

/* ---- z-slab decomposition, one process per GPU (multi-rank drivers) ----
 *
 * A slab context owns global interior planes [z0, z1) of the grid `global`
 * on opts->device.  Its local ghost planes are global ghosts at the grid
 * boundary and HALO copies of the neighbour slab's boundary planes inside.
 * Uploads and downloads take GLOBAL-size host arrays and touch only the
 * slab's planes.  Between steps the driver moves, per interface:
 *   lower rank SEND_UP (E x6 + Hxy,Hxz,Hyx,Hyz of its last plane)
 *        -> upper rank RECV_DOWN (its plane below z0)
 *   upper rank SEND_DOWN (E x6 of its first plane)
 *        -> lower rank RECV_UP (its plane above z1-1)
 * The upper rank recomputes H_new on the received plane, so a step needs no
 * mid-step exchange (engine FUSED).
 *
 * Engine TBLOCK (default for AUTO) makes a DEEP-halo slab: two steps per HBM
 * pass need two-plane halos, so the slab also holds one extended interior
 * plane per internal interface (recomputed redundantly, refreshed by the
 * exchange) and every view is two contiguous planes of all 12 fields:
 *   SEND_DOWN: owned planes z0, z0+1      -> lower rank's RECV_UP
 *   RECV_DOWN: ghost z0-2, extended z0-1  <- lower rank's SEND_UP
 *   SEND_UP:   owned planes z1-2, z1-1    -> upper rank's RECV_DOWN
 *   RECV_UP:   extended z1, ghost z1+1    <- upper rank's SEND_DOWN
 * Driver loop for both kinds (thiim_gpu_slab_info gives the period):
 *   k = min(period, remaining); thiim_gpu_step(ctx, k); exchange;
 * (the uploaded halos are valid for the first pass).  Downloads and compares
 * touch the owned planes only. */
int thiim_gpu_create_slab(const thiim_dims* global, int z0, int z1, const thiim_gpu_opts* opts,
                          thiim_gpu_ctx** out);

enum {
  THIIM_HALO_SEND_DOWN = 0,
  THIIM_HALO_RECV_DOWN = 1,
  THIIM_HALO_SEND_UP = 2,
  THIIM_HALO_RECV_UP = 3
};

/* One halo plane set: n_arrays array-planes of plane_bytes each, the k-th at
 * base + k*array_stride_bytes (device memory of `device`).  Valid until the
 * next thiim_gpu_step (the fused engines ping-pong their field buffers). */
typedef struct {
  void* base;
  long long array_stride_bytes;
  long long plane_bytes;
  int n_arrays;
  int device;
} thiim_halo_view;
int thiim_gpu_halo_view(thiim_gpu_ctx* ctx, int which, thiim_halo_view* view);

/* Plane ranges and exchange period of a slab context. */
typedef struct {
  int own_z0, own_z1;      /* owned global interior planes [own_z0, own_z1) */
  int local_z0, local_z1;  /* planes held as local interior (incl. extended planes) */
  int exchange_period;     /* steps per exchange: 1 (FUSED), 2 (TBLOCK deep halo) */
  int engine;              /* THIIM_ENGINE_* the context runs */
  int device_ordered;      /* IPC peer stores ordered by device pass counters */
} thiim_slab_info;
int thiim_gpu_slab_info(thiim_gpu_ctx* ctx, thiim_slab_info* info);

/* Multi-process peer stores (ranks on one node, NVLink / NVSwitch): each rank
 * exports its slab (CUDA IPC handle + layout), imports its neighbours' exports,
 * and from then on every TBLOCK pass stores its boundary planes straight into
 * the neighbours' halo planes -- no halo exchange after 2-step passes.
 * Ordering between the ranks' passes is on the devices: every slab keeps a
 * pass counter in its own (exported) allocation; before pass n a slab's stream
 * waits until both neighbours' counters reach n-1 (their reads of the halo set
 * pass n stores into are done, and their stores into this slab's input halos
 * have landed), and after the pass it writes n (stream memory operations,
 * preceded by a system-scope fence).  So thiim_gpu_step(ctx, k) may advance
 * any even k in one call with no host synchronisation between passes, and the
 * call's stream ends on the neighbours' counters reaching this slab's pass
 * count: when thiim_gpu_step returns, the neighbours' last stores into this
 * slab's halos have landed (the remainder step, a download or a new upload may
 * follow);
 * thiim_slab_info.device_ordered says so (0: the stream memory operations were
 * unavailable for the mapped counters, and the caller must barrier all ranks
 * after every 2-step call).  The caller still barriers all ranks once after an
 * upload / generate (they write both field sets, halos included).  Odd
 * remainder steps (k = 1) use the view exchange.  TBLOCK deep-halo slabs only. */
typedef struct {
  unsigned char ipc[64]; /* cudaIpcMemHandle_t of the slab state */
  long long stride;      /* elements per array */
  int nz_local, ext_lo, ext_hi, nfield_sets, device;
  int px;
  long long pxy;
  long long counter_offset; /* byte offset of the pass counter in the allocation */
} thiim_slab_export;
enum { THIIM_PEER_LOWER = 0, THIIM_PEER_UPPER = 1 };
int thiim_gpu_slab_export(thiim_gpu_ctx* ctx, thiim_slab_export* out);
int thiim_gpu_slab_import(thiim_gpu_ctx* ctx, int which, const thiim_slab_export* peer);
/* Unmaps imported neighbours: back to exchange after every pass. */
int thiim_gpu_slab_detach(thiim_gpu_ctx* ctx);

/* Plane-range variants for rank-local host buffers: the host arrays hold the
 * global padded planes [p0, ...) only (plane p = global interior z p-1); a
 * slab reads padded planes [local_z0, local_z1 + 2) and writes back its owned
 * planes (plus the global ghost planes it borders). */
int thiim_gpu_upload_planes(thiim_gpu_ctx* ctx, const thiim_c128* const arrays[40], int p0);
int thiim_gpu_download_fields_planes(thiim_gpu_ctx* ctx, thiim_c128* const fields[12], int p0);
int thiim_generate_host_planes(const thiim_dims* global, int kind, uint64_t seed, int p0, int p1,
                               thiim_c128* const arrays[40]);

/* THIIM_COEFF_TABLE contexts: upload fields, per-cell material ids (padded
 * layout, (nx+2)(ny+2)(nz+2) bytes, ghosts ignored) and the coefficient table
 * ([n_materials][28] complex128). */
int thiim_gpu_upload_table(thiim_gpu_ctx* ctx, const thiim_c128* const fields[12],
                           const uint8_t* material_id, const thiim_c128* table);
/* Reads back the material ids and the table of a THIIM_COEFF_TABLE context. */
int thiim_gpu_download_table(thiim_gpu_ctx* ctx, uint8_t* material_id, thiim_c128* table);

/* Sanitizer (the reference's exactly-once coverage check, tools/main.cpp:20-41,
 * for the GPU schedules): while on, the default kernels count every output
 * store per (component, cell) and after every pass (one launch of the fused /
 * TBLOCK engines, an H+E launch pair of the split engine) a check kernel
 * demands exactly one store per interior cell of every slab -- extended
 * planes of deep slabs included -- and none on ghosts.  Costs ~48 B/cell of
 * device memory and atomics on every store: a debug mode. */
int thiim_gpu_set_sanitize(thiim_gpu_ctx* ctx, int on);
/* Passes checked and (component, cell) violations since thiim_gpu_set_sanitize. */
int thiim_gpu_coverage(thiim_gpu_ctx* ctx, unsigned long long* passes,
                       unsigned long long* violations);

/* Blocks until all work queued on the context's streams has finished. */
int thiim_gpu_sync(thiim_gpu_ctx* ctx);

/* One-GPU contexts take their state from the device's stream-ordered memory pool
 * and give it back on destroy (slabs that a peer device or process writes into --
 * n_gpus > 1 on distinct devices, thiim_gpu_create_slab -- are plain cudaMalloc
 * allocations: peer access and CUDA IPC do not cover pool memory); the pool
 * keeps the pages for the next context
 * (creating a 14 GB context costs ~2 ms instead of a fresh allocation).  This
 * returns the cached, unused pages of `device`'s pool to the driver, e.g.
 * before another library allocates device memory. */
int thiim_gpu_release_cached(int device);

/* ---- auto-tuner (the reference's tune, autotuner.cpp:15-142, for the GPU
 * knobs).  Candidates: time_block {2, 3} x tile_y x z-chunk count x band x
 * schedule of the TBLOCK engine.  A GPU re-parameterisation of the
 * reference's models ranks them: Eq. 12's code balance becomes the DRAM bytes
 * per LUP of a candidate (832 / time_block, plus the tile-overlap rows the L2
 * does not share across round / band edges and the chunk-start re-reads) times
 * its wave quantisation; Eq. 11's cache-fit test becomes the L2 working set of
 * the evict_last coefficient planes one round keeps for the deeper levels,
 * which must fit 60% of the L2.  Sorted by model MLUP/s, best first. */
typedef struct {
  int time_block, tile_y, z_chunk, band, schedule;
  int tiles, rounds;            /* CTAs and launches (rounds) per pass */
  double balance_model;         /* 832 / time_block */
  double model_bytes_per_lup;   /* incl. overlap re-fetch and chunk starts */
  double quantization;          /* useful / scheduled CTA-planes */
  double model_mlups;           /* hbm_gbs / model_bytes_per_lup * quantization */
  double l2_set_bytes;          /* coefficient planes held in L2 by one round */
} thiim_gpu_candidate;
int thiim_gpu_enumerate_candidates(const thiim_dims* dims, const thiim_gpu_opts* base,
                                   double hbm_gbs, thiim_gpu_candidate* out, int cap, int* n);

typedef struct {
  thiim_gpu_candidate cand;
  int steps, ok;
  double seconds, mlups;  /* device time of the timed runs, steps x interior / seconds */
  char note[96];
} thiim_gpu_trial;
/* Times the `max_trials` best-ranked candidates (plus the default schedule)
 * on the seeded random problem of `dims` (generated on the device), `steps`
 * iterations per run, repeated until `min_seconds` of device time; the winner
 * is the deepest time_block within 2% of the best (then the fastest), and is
 * verified bitwise against the FUSED engine (one step per pass, an
 * independent schedule) on `dims` if it has <= 2^24 cells, else on a
 * 120 x 100 x 48 grid.  *verified = 1 if equal.  winner: base with the
 * winning knobs. */
int thiim_gpu_tune(const thiim_dims* dims, const thiim_gpu_opts* base, int steps,
                   double min_seconds, int max_trials, thiim_gpu_trial* table, int cap,
                   int* n_trials, thiim_gpu_opts* winner, int* verified);

/* Message of the last failing call on this thread ("" if none). */
const char* thiim_gpu_last_error(void);

/* Algorithmic bytes per LUP of an engine (832 / time_block for TBLOCK);
   engine 100 + THIIM_COEFF_TABLE: the table layout, 385 / time_block. */
double thiim_gpu_balance_model(int engine, int time_block);

int thiim_gpu_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* THIIM_GPU_H */
