// thiim_tune.cuh -- the GPU auto-tuner: candidate enumeration with a model
// (the reference's enumerate_candidates + perf models, autotuner.cpp:15-50,
// perf_models.cpp:22-38) and timed trials with a verified winner (tune,
// autotuner.cpp:62-142).  Host code over the library's own C-ABI; included
// once, at the end of thiim_gpu.cu.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

namespace {

// Element counts of the level-1 boxes of one tile-plane (BoxGeom shapes) and
// of the rows / columns a neighbouring tile re-reads (its overlap), for a
// 32 x BY thread tile whose output tile is (32 - 2k) x (BY - 2k).
struct TileTraffic {
  double box;      // level-1 box elements per tile-plane (40 arrays)
  double y_edge;   // elements shared with the tile above (y-overlap)
  double x_edge;   // elements shared with the tile to the right (x-overlap)
  double coef;     // level-1 coefficient box elements (28 arrays) per tile-plane
};

TileTraffic tile_traffic(int by, int k) {
  // arrays per box kind (thiim_producer.cuh produce_plane_ct)
  const int n[5] = {6, 6, 7, 7, 14};  // A, B, BX, BY, C
  const int w[5] = {32, 31, 31, 30, 30};
  const int h[5] = {by, by - 1, by - 2, by - 1, by - 2};
  const int ncoef[5] = {0, 4, 5, 5, 14};  // t, c (, src) per H box kind; E coefficients
  const int tx = 32 - 2 * k, ty = by - 2 * k;
  TileTraffic t{0, 0, 0, 0};
  for (int b = 0; b < 5; ++b) {
    t.box += (double)n[b] * w[b] * h[b];
    t.y_edge += (double)n[b] * w[b] * std::max(0, h[b] - ty);
    t.x_edge += (double)n[b] * h[b] * std::max(0, w[b] - tx);
    t.coef += (double)ncoef[b] * w[b] * h[b];
  }
  return t;
}

// DRAM bytes per cell of a synchronised wave of exact tiles beyond the
// algorithmic 832 (sector granularity, L2 misses of shared overlap rows):
// measured 1.08x on 252 x 176 grids (profiles/r01h_traffic_probe.md)
constexpr double kExactTileFloor = 1.08;

// SM-side bound: every level of a pass runs the whole 32 x BY thread tile, so a
// LUP costs 32 * BY / (output tile area) thread-level updates whatever the
// depth.  Calibrated on the depth-3 kernel, which is SM-bound (issue slots,
// dependent FP64, CTA barriers; profiles/r02_depth3.md): 8.43 GLUP/s x 2.05 =
// 17.3 G thread-level updates/s.  It puts depth 2 at 15 rows at 11.1 GLUP/s --
// where its pattern-only ceiling and the product sit.
constexpr double kThreadUpdatesPerSec = 17.3e9;

thiim_gpu_candidate model_candidate(const thiim_dims& d, int sms, double l2_bytes, double hbm_gbs,
                                    int k, int by, int nchunks, int band_mode, int schedule) {
  thiim_gpu_candidate c{};
  c.time_block = k;
  c.tile_y = by;
  c.schedule = schedule;
  const int tx = 32 - 2 * k, ty = by - 2 * k;
  const int tiles_x = (d.nx + tx - 1) / tx, tiles_y = (d.ny + ty - 1) / ty;
  const int zc = (d.nz + nchunks - 1) / nchunks;
  nchunks = (d.nz + zc - 1) / zc;
  c.z_chunk = zc;
  c.tiles = tiles_x * tiles_y * nchunks;
  const long long items = c.tiles;
  const long long rounds = schedule == 1 ? 1 : (items + sms - 1) / sms;
  const long long per_round = (items + rounds - 1) / rounds;
  c.rounds = (int)rounds;
  // band: 0 auto (tblock_band), 1 whole rows (band = tiles_x), 2 half the auto width
  const int auto_band = tblock_band(tiles_x, (int)std::min<long long>(per_round, sms), 0);
  const int band = band_mode == 1 ? tiles_x : band_mode == 2 ? std::max(1, auto_band / 2) : auto_band;
  c.band = schedule == 1 ? 0 : band_mode == 0 ? 0 : band;
  const TileTraffic tt = tile_traffic(by, k);
  // overlap rows the L2 does not share: across round / band edges (rounds),
  // or every tile row boundary (one launch: y-neighbours start tiles_x / SMs of
  // a CTA lifetime apart and miss each other in L2)
  double y_edges, x_edges;
  if (schedule == 1) {
    y_edges = (double)tiles_x * (tiles_y - 1);
    x_edges = 0.0;
  } else {
    const int nbands = (tiles_x + band - 1) / band;
    y_edges = (double)rounds / nchunks * band;  // one ragged edge per round
    x_edges = (double)(nbands - 1) * tiles_y;
  }
  const double cells = (double)d.nx * d.ny;
  const double reads = kExactTileFloor * (cells * 40.0 + y_edges * tt.y_edge + x_edges * tt.x_edge);
  const double writes = cells * 12.0;
  // a chunk start re-runs k - 1 level-1 planes below the chunk
  const double restart = 1.0 + (k - 1.0) / zc;
  c.balance_model = 832.0 / k;
  c.model_bytes_per_lup = 16.0 * (reads * restart + writes) / cells / k;
  // wave quantisation: SM-plane slots of all rounds (idle SMs included) x
  // (planes + k prologue planes)
  const double useful = (double)tiles_x * tiles_y * d.nz;
  const double waves = schedule == 1 ? std::ceil((double)items / sms) : (double)rounds;
  const double slots = waves * sms * (zc + k);
  c.quantization = std::min(1.0, useful / slots);
  // the slower of the memory bound (Eq. 12 analogue) and the SM-side bound
  const double mem_mlups = hbm_gbs * 1e3 / c.model_bytes_per_lup;
  const double sm_mlups = kThreadUpdatesPerSec / (32.0 * by / ((double)tx * ty)) / 1e6;
  c.model_mlups = std::min(mem_mlups, sm_mlups) * c.quantization;
  // Eq. 11 analogue: coefficient planes kept evict_last for the k - 1 deeper
  // levels by the CTAs of one round
  c.l2_set_bytes = 16.0 * tt.coef * (k - 1) * (double)std::min<long long>(per_round, sms);
  (void)l2_bytes;
  return c;
}

}  // namespace

extern "C" {

int thiim_gpu_enumerate_candidates(const thiim_dims* dims, const thiim_gpu_opts* base,
                                   double hbm_gbs, thiim_gpu_candidate* out, int cap, int* n) {
  g_err.clear();
  if (!valid_dims(dims)) return fail(THIIM_ERR_SETUP, "invalid grid dims");
  if (!n) return fail(THIIM_ERR_CONFIG, "null count");
  thiim_gpu_opts o;
  if (base)
    o = *base;
  else
    thiim_gpu_default_opts(&o);
  if (hbm_gbs <= 0) hbm_gbs = 6536.0;
  int dev = o.device, sms = 148, l2 = 126 << 20;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  const bool whole = o.n_gpus == 1 && o.coeff_layout == THIIM_COEFF_FULL;
  std::vector<thiim_gpu_candidate> all;
  for (int k : {2, 3}) {
    if (k == 3 && !whole) continue;
    for (int by : {15, 14, 12, 16}) {
      if (k == 3 && by != 15) continue;  // depth 3: tile height 15 only
      for (int nch : {1, 2, 3, 4, 6, 8}) {
        if (dims->nz / nch < 4 * k) continue;
        for (int sched : {0, 1})
          for (int bm : {0, 1, 2}) {
            if (sched == 1 && bm != 0) continue;
            thiim_gpu_candidate c = model_candidate(*dims, sms, l2, hbm_gbs, k, by, nch, bm, sched);
            // Eq. 11 analogue: the deeper levels' coefficient planes must stay in L2
            if (c.l2_set_bytes > 0.6 * l2) continue;
            bool dup = false;
            for (const auto& e : all)
              dup = dup || (e.time_block == c.time_block && e.tile_y == c.tile_y &&
                            e.z_chunk == c.z_chunk && e.band == c.band && e.schedule == c.schedule);
            if (!dup) all.push_back(c);
          }
      }
    }
  }
  // best model MLUP/s first; within 0.5% (the SM-side bound ties them), fewer
  // DRAM bytes first (less power at the board's cap)
  std::stable_sort(all.begin(), all.end(), [](const thiim_gpu_candidate& a,
                                              const thiim_gpu_candidate& b) {
    if (std::fabs(a.model_mlups - b.model_mlups) > 0.005 * std::max(a.model_mlups, b.model_mlups))
      return a.model_mlups > b.model_mlups;
    return a.model_bytes_per_lup < b.model_bytes_per_lup;
  });
  *n = (int)all.size();
  if (out)
    for (int i = 0; i < std::min(cap, *n); ++i) out[i] = all[i];
  return THIIM_OK;
}

int thiim_gpu_tune(const thiim_dims* dims, const thiim_gpu_opts* base, int steps,
                   double min_seconds, int max_trials, thiim_gpu_trial* table, int cap,
                   int* n_trials, thiim_gpu_opts* winner, int* verified) {
  g_err.clear();
  if (!valid_dims(dims)) return fail(THIIM_ERR_SETUP, "invalid grid dims");
  if (steps < 1) return fail(THIIM_ERR_CONFIG, "tune needs steps >= 1");
  if (!n_trials || !winner || !verified) return fail(THIIM_ERR_CONFIG, "null output");
  thiim_gpu_opts o;
  if (base)
    o = *base;
  else
    thiim_gpu_default_opts(&o);
  if (o.n_gpus != 1) return fail(THIIM_ERR_CONFIG, "tune runs on one GPU (n_gpus = 1)");
  int n = 0;
  int r = thiim_gpu_enumerate_candidates(dims, &o, 0.0, nullptr, 0, &n);
  if (r) return r;
  std::vector<thiim_gpu_candidate> cands(n);
  if ((r = thiim_gpu_enumerate_candidates(dims, &o, 0.0, cands.data(), n, &n))) return r;
  if (max_trials < 1) max_trials = 8;
  // the model's best candidate of every (time_block, tile_y), then the next
  // best overall, plus the library default (the tuner must be able to keep it)
  std::vector<thiim_gpu_candidate> trials;
  auto same = [](const thiim_gpu_candidate& a, const thiim_gpu_candidate& b) {
    return a.time_block == b.time_block && a.tile_y == b.tile_y && a.z_chunk == b.z_chunk &&
           a.band == b.band && a.schedule == b.schedule;
  };
  for (const auto& c : cands) {
    bool seen = false;
    for (const auto& t : trials) seen = seen || (t.time_block == c.time_block && t.tile_y == c.tile_y);
    if (!seen && (int)trials.size() < max_trials) trials.push_back(c);
  }
  for (const auto& c : cands) {
    if ((int)trials.size() >= max_trials) break;
    bool dup = false;
    for (const auto& t : trials) dup = dup || same(t, c);
    if (!dup) trials.push_back(c);
  }
  {
    // the library default: depth 2, 15 rows, rounds, auto band, and the z-chunk
    // count tblock_zchunk picks (modelled with that count, run with z_chunk 0)
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, o.device);
    cudaGetLastError();
    const long long nbt = (long long)((dims->nx + 27) / 28) * ((dims->ny + 10) / 11);
    double best_t = 1e300;
    int best_c = 1;
    for (int c = 1; c <= std::max(1, dims->nz / 8); ++c) {
      const double t = (double)((nbt * c + sms - 1) / sms) * ((dims->nz + c - 1) / c + 4.5);
      if (t < best_t - 1e-9) {
        best_t = t;
        best_c = c;
      }
    }
    thiim_gpu_candidate def = model_candidate(*dims, sms, 0.0, 6536.0, 2, 15, best_c, 0, 0);
    def.z_chunk = 0;  // run it as the library would
    trials.push_back(def);
  }
  std::vector<thiim_gpu_trial> done;
  for (const auto& c : trials) {
    thiim_gpu_trial t{};
    t.cand = c;
    t.steps = std::max(steps, 2 * c.time_block);
    thiim_gpu_opts to = o;
    to.engine = THIIM_ENGINE_TBLOCK;
    to.time_block = c.time_block;
    to.tile_y = c.tile_y;
    to.z_chunk = c.z_chunk;
    to.band = c.band;
    to.schedule = c.schedule;
    thiim_gpu_ctx* ctx = nullptr;
    int rc = thiim_gpu_create(dims, &to, &ctx);
    if (!rc) rc = thiim_gpu_init_generated(ctx, THIIM_GEN_RANDOM, 1);
    thiim_gpu_stats st;
    if (!rc) rc = thiim_gpu_step(ctx, t.steps, &st);  // warm-up: tensor maps, graphs
    double secs = 0.0;
    long long runs = 0;
    while (!rc && (secs < min_seconds || runs == 0)) {
      rc = thiim_gpu_step(ctx, t.steps, &st);
      secs += st.seconds;
      ++runs;
    }
    if (rc) {
      std::snprintf(t.note, sizeof t.note, "%s", g_err.c_str());
      for (char* p = t.note; *p; ++p)
        if (*p == ',' || *p == '\n') *p = ';';
    } else {
      t.ok = 1;
      t.seconds = secs;
      t.mlups = (double)dims->nx * dims->ny * dims->nz * t.steps * runs / secs / 1e6;
    }
    if (ctx) thiim_gpu_destroy(ctx);
    done.push_back(t);
  }
  *n_trials = (int)done.size();
  if (table)
    for (int i = 0; i < std::min(cap, *n_trials); ++i) table[i] = done[i];
  // winner: the deepest time_block within 2% of the best, then the fastest
  // (the reference prefers the widest diamond in its 2% window)
  double best = 0.0;
  for (const auto& t : done)
    if (t.ok) best = std::max(best, t.mlups);
  const thiim_gpu_trial* w = nullptr;
  for (const auto& t : done) {
    if (!t.ok || t.mlups < 0.98 * best) continue;
    if (!w || t.cand.time_block > w->cand.time_block ||
        (t.cand.time_block == w->cand.time_block && t.mlups > w->mlups))
      w = &t;
  }
  if (!w) return fail(THIIM_ERR_CONFIG, "tuner: no candidate ran");
  *winner = o;
  winner->engine = THIIM_ENGINE_TBLOCK;
  winner->time_block = w->cand.time_block;
  winner->tile_y = w->cand.tile_y;
  winner->z_chunk = w->cand.z_chunk;
  winner->band = w->cand.band;
  winner->schedule = w->cand.schedule;
  // verification: the winner vs the fused engine (one step per pass), bitwise
  thiim_dims vd = *dims;
  if ((double)vd.nx * vd.ny * vd.nz > (double)(1 << 24)) vd = thiim_dims{120, 100, 48, 1};
  thiim_gpu_opts wv = *winner, fv = o;
  wv.z_chunk = std::min(wv.z_chunk, vd.nz);
  fv.engine = THIIM_ENGINE_FUSED;
  fv.time_block = 0;
  fv.z_chunk = 0;
  const int vsteps = 2 * w->cand.time_block + 1;  // full passes + a remainder
  const size_t np = (size_t)(vd.nx + 2) * (vd.ny + 2) * (vd.nz + 2);
  std::vector<thiim_c128> host(12 * np);
  thiim_c128* fields[12];
  for (int k = 0; k < 12; ++k) fields[k] = host.data() + k * np;
  thiim_gpu_ctx* a = nullptr;
  thiim_gpu_ctx* b = nullptr;
  *verified = 0;
  r = thiim_gpu_create(&vd, &fv, &a);
  if (!r) r = thiim_gpu_init_generated(a, THIIM_GEN_RANDOM, 7);
  if (!r) r = thiim_gpu_step(a, vsteps, nullptr);
  if (!r) r = thiim_gpu_download_fields(a, fields);
  if (!r) r = thiim_gpu_create(&vd, &wv, &b);
  if (!r) r = thiim_gpu_init_generated(b, THIIM_GEN_RANDOM, 7);
  if (!r) r = thiim_gpu_step(b, vsteps, nullptr);
  thiim_gpu_diff diff{};
  if (!r) r = thiim_gpu_compare_fields(b, fields, &diff);
  if (a) thiim_gpu_destroy(a);
  if (b) thiim_gpu_destroy(b);
  if (r) return r;
  *verified = diff.differing_values == 0 ? 1 : 0;
  return THIIM_OK;
}

}  // extern "C"
