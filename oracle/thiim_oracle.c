/*
 * thiim_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker; see thiim_oracle.h).
 *
 * A plain-C restatement of the reference THIIM sweep.  Every function cites
 * the reference file:line (relative to /root/reference/proj) it follows.
 * Compiled with -O2 -ffp-contract=off so no multiply-add is ever contracted,
 * matching the reference's default x86-64 build.
 */
#include "thiim_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <string.h>

/* kComponentTable, include/thiim/components.hpp:54-67:
 * {id, family, shift_axis, shift_sign, operand_a, operand_b, curl_sign, has_source} */
const orc_desc orc_component_table[12] = {
    {ORC_EXY, ORC_FAM_E, ORC_AXIS_Y, -1, ORC_HZX, ORC_HZY, +1, 0},
    {ORC_EXZ, ORC_FAM_E, ORC_AXIS_Z, -1, ORC_HYX, ORC_HYZ, -1, 1},
    {ORC_EYX, ORC_FAM_E, ORC_AXIS_X, -1, ORC_HZX, ORC_HZY, -1, 0},
    {ORC_EYZ, ORC_FAM_E, ORC_AXIS_Z, -1, ORC_HXY, ORC_HXZ, +1, 1},
    {ORC_EZX, ORC_FAM_E, ORC_AXIS_X, -1, ORC_HYX, ORC_HYZ, +1, 0},
    {ORC_EZY, ORC_FAM_E, ORC_AXIS_Y, -1, ORC_HXY, ORC_HXZ, -1, 0},
    {ORC_HXY, ORC_FAM_H, ORC_AXIS_Y, +1, ORC_EZX, ORC_EZY, -1, 0},
    {ORC_HXZ, ORC_FAM_H, ORC_AXIS_Z, +1, ORC_EYX, ORC_EYZ, +1, 1},
    {ORC_HYX, ORC_FAM_H, ORC_AXIS_X, +1, ORC_EZX, ORC_EZY, +1, 0},
    {ORC_HYZ, ORC_FAM_H, ORC_AXIS_Z, +1, ORC_EXY, ORC_EXZ, -1, 1},
    {ORC_HZX, ORC_FAM_H, ORC_AXIS_X, +1, ORC_EYX, ORC_EYZ, -1, 0},
    {ORC_HZY, ORC_FAM_H, ORC_AXIS_Y, +1, ORC_EXY, ORC_EXZ, +1, 0},
};

/* kHOrder / kEOrder, components.hpp:73-86 */
static const int kHOrder[6] = {ORC_HXY, ORC_HXZ, ORC_HYX, ORC_HYZ, ORC_HZX, ORC_HZY};
static const int kEOrder[6] = {ORC_EXY, ORC_EXZ, ORC_EYX, ORC_EYZ, ORC_EZX, ORC_EZY};

int orc_source_index(int comp) { /* components.hpp:89-97 */
  switch (comp) {
    case ORC_EXZ: return 0;
    case ORC_EYZ: return 1;
    case ORC_HXZ: return 2;
    case ORC_HYZ: return 3;
    default: return -1;
  }
}

size_t orc_padded_cells(int nx, int ny, int nz) { /* grid.hpp:23-29 */
  return (size_t)(nx + 2) * (size_t)(ny + 2) * (size_t)(nz + 2);
}

size_t orc_linear_index(int nx, int ny, int x, int y, int z) { /* grid.hpp:39-43 */
  const size_t px = (size_t)nx + 2, py = (size_t)ny + 2;
  return (size_t)(z + 1) * px * py + (size_t)(y + 1) * px + (size_t)(x + 1);
}

/* update_component_region, kernels.cpp:12-69.  Exact per-cell op order of
 * kernels.cpp:43-51 (sourced) / :56-64 (unsourced). */
void orc_update_component_region(orc_state* s, int comp, int x0, int x1, int y0, int y1,
                                 int z0, int z1) {
  const orc_desc* d = &orc_component_table[comp];
  const ptrdiff_t px = s->nx + 2, py = s->ny + 2;
  ptrdiff_t shift = d->shift_axis == ORC_AXIS_X ? 1 : d->shift_axis == ORC_AXIS_Y ? px : px * py;
  shift *= d->shift_sign;
  orc_c128* f = s->a[comp];
  const orc_c128* tc = s->a[12 + comp];
  const orc_c128* cc = s->a[24 + comp];
  const orc_c128* a = s->a[d->operand_a];
  const orc_c128* b = s->a[d->operand_b];
  const int si = orc_source_index(comp);
  const orc_c128* src = si >= 0 ? s->a[36 + si] : NULL;
  for (int z = z0; z < z1; ++z)
    for (int y = y0; y < y1; ++y) {
      const size_t row = orc_linear_index(s->nx, s->ny, x0, y, z);
      for (size_t i = row; i < row + (size_t)(x1 - x0); ++i) {
        const size_t j = (size_t)((ptrdiff_t)i + shift);
        const double dr = (a[j].re + b[j].re) - (a[i].re + b[i].re);
        const double di = (a[j].im + b[j].im) - (a[i].im + b[i].im);
        const double fr = f[i].re, fi = f[i].im;
        const double tr = tc[i].re * fr - tc[i].im * fi;
        const double ti = tc[i].re * fi + tc[i].im * fr;
        const double cr = cc[i].re * dr - cc[i].im * di;
        const double ci = cc[i].re * di + cc[i].im * dr;
        if (src) {
          f[i].re = tr + cr + src[i].re;
          f[i].im = ti + ci + src[i].im;
        } else {
          f[i].re = tr + cr;
          f[i].im = ti + ci;
        }
      }
    }
}

/* step_reference, kernels.cpp:105-113 */
void orc_step_reference(orc_state* s) {
  for (int k = 0; k < 6; ++k)
    orc_update_component_region(s, kHOrder[k], 0, s->nx, 0, s->ny, 0, s->nz);
  for (int k = 0; k < 6; ++k)
    orc_update_component_region(s, kEOrder[k], 0, s->nx, 0, s->ny, 0, s->nz);
}

/* One step of a z-slab whose plane below z = 0 is a halo copy of the
 * neighbour's last plane (halo_lo = 1): H is also updated on that plane
 * (z = -1) so E at z = 0 sees H_new there, exactly as the neighbour computes
 * it.  Models the decomposition of paper_1510_05218_b200/distributed.py. */
void orc_step_slab(orc_state* s, int halo_lo) {
  for (int k = 0; k < 6; ++k)
    orc_update_component_region(s, kHOrder[k], 0, s->nx, 0, s->ny, halo_lo ? -1 : 0, s->nz);
  for (int k = 0; k < 6; ++k)
    orc_update_component_region(s, kEOrder[k], 0, s->nx, 0, s->ny, 0, s->nz);
}

/* run_naive serial branch, reference_engines.cpp:44-46 */
void orc_run_naive(orc_state* s, int steps) {
  for (int n = 0; n < steps; ++n) orc_step_reference(s);
}

/* ---- threaded run_naive: static z slabs + barrier per half-step
 *      (reference_engines.cpp:26-30, 48-63) ---- */
typedef struct {
  orc_state* s;
  int steps, threads, w;
  pthread_barrier_t* bar;
} orc_worker;

static void* orc_worker_main(void* p) {
  orc_worker* wk = (orc_worker*)p;
  const int nz = wk->s->nz, n = wk->threads, w = wk->w;
  const int base = nz / n, rem = nz % n;
  const int z0 = w * base + (w < rem ? w : rem);
  const int z1 = z0 + base + (w < rem ? 1 : 0);
  for (int st = 0; st < wk->steps; ++st) {
    for (int fam = 0; fam < 2; ++fam) {
      const int* order = fam == 0 ? kHOrder : kEOrder;
      if (z0 < z1)
        for (int k = 0; k < 6; ++k)
          orc_update_component_region(wk->s, order[k], 0, wk->s->nx, 0, wk->s->ny, z0, z1);
      pthread_barrier_wait(wk->bar);
    }
  }
  return NULL;
}

void orc_run_naive_threads(orc_state* s, int steps, int threads) {
  if (threads <= 1) { orc_run_naive(s, steps); return; }
  pthread_barrier_t bar;
  pthread_barrier_init(&bar, NULL, (unsigned)threads);
  pthread_t tid[256];
  orc_worker wk[256];
  if (threads > 256) threads = 256;
  for (int w = 0; w < threads; ++w) {
    wk[w].s = s; wk[w].steps = steps; wk[w].threads = threads; wk[w].w = w; wk[w].bar = &bar;
    pthread_create(&tid[w], NULL, orc_worker_main, &wk[w]);
  }
  for (int w = 0; w < threads; ++w) pthread_join(tid[w], NULL);
  pthread_barrier_destroy(&bar);
}

/* compare_states, verifier.cpp:13-44: memcmp per value over the interior. */
uint64_t orc_compare_fields(const orc_state* a, const orc_state* b, int* first_comp,
                            int* fx, int* fy, int* fz, double* max_abs_diff) {
  uint64_t n = 0;
  double mx = 0.0;
  if (first_comp) *first_comp = -1;
  for (int ci = 0; ci < 12; ++ci)
    for (int z = 0; z < a->nz; ++z)
      for (int y = 0; y < a->ny; ++y)
        for (int x = 0; x < a->nx; ++x) {
          const size_t i = orc_linear_index(a->nx, a->ny, x, y, z);
          if (memcmp(&a->a[ci][i], &b->a[ci][i], sizeof(orc_c128)) != 0) {
            if (n == 0 && first_comp) {
              *first_comp = ci; *fx = x; *fy = y; *fz = z;
            }
            ++n;
            const double dr = fabs(a->a[ci][i].re - b->a[ci][i].re);
            const double di = fabs(a->a[ci][i].im - b->a[ci][i].im);
            if (dr > mx) mx = dr;
            if (di > mx) mx = di;
          }
        }
  if (max_abs_diff) *max_abs_diff = mx;
  return n;
}

/* ---- coefficient closed forms, coefficients.cpp:25-55 ---- */
void orc_default_scheme(orc_scheme* sp) { /* coefficients.hpp:21-26 */
  sp->omega = 0.4; sp->tau = 1.0; sp->delta = 1.0;
  sp->src_e_re = 1.0; sp->src_e_im = 0.0;
  sp->src_h_re = 1.0; sp->src_h_im = 0.0;
}

static double complex mkc(double re, double im) { return CMPLX(re, im); }
static double complex expi(double p) { return CMPLX(cos(p), sin(p)); } /* :12 */
/* std::complex<double> operator*(double, complex): both parts scaled, no cross terms */
static double complex rscale(double complex z, double k) { return CMPLX(creal(z) * k, cimag(z) * k); }

int orc_derive_coefficients(const orc_material* m, const orc_scheme* sp, int family,
                            int back_mode, orc_c128* t, orc_c128* c, orc_c128* src) {
  const double wt = sp->omega * sp->tau;
  const double complex eps = mkc(m->eps_re, m->eps_im);
  double complex ot, oc, os;
  if (family == ORC_FAM_H) { /* :29-36 */
    const double complex denom = expi(wt / 2.0) + mkc(sp->tau * m->sigma_star / m->mu, 0.0);
    if (cabs(denom) == 0.0) return -1;
    ot = expi(-wt / 2.0) / denom;
    oc = mkc(sp->tau / (m->mu * sp->delta), 0.0) / denom;
    /* tau * source_h: std::complex operator*(double, complex) scales re and im */
    os = rscale(mkc(sp->src_h_re, sp->src_h_im), sp->tau) / denom;
  } else if (!back_mode) { /* :37-45 */
    /* 1 + tau*sigma/eps parses as complex(1,0) + complex(tau*sigma,0)/eps */
    const double complex denom = mkc(1.0, 0.0) + mkc(sp->tau * m->sigma, 0.0) / eps;
    if (cabs(denom) == 0.0) return -1;
    ot = expi(-wt) / denom;
    /* (tau / (eps*delta)) * expi(-wt/2) / denom; complex*double scales both parts */
    const double complex ed = rscale(eps, sp->delta);
    oc = (mkc(sp->tau, 0.0) / ed) * expi(-wt / 2.0) / denom;
    /* tau * expi(-wt) * source_e / denom */
    os = (rscale(expi(-wt), sp->tau) * mkc(sp->src_e_re, sp->src_e_im)) / denom;
  } else { /* :46-53 */
    const double complex denom = mkc(1.0 / sp->tau, 0.0) - mkc(m->sigma, 0.0) / eps;
    if (cabs(denom) == 0.0) return -1;
    ot = expi(wt) / rscale(denom, sp->tau);
    const double complex ed = rscale(eps, sp->delta);
    oc = -(mkc(1.0, 0.0) / ed) * expi(wt / 2.0) / denom;
    os = -mkc(sp->src_e_re, sp->src_e_im) / denom;
  }
  t->re = creal(ot); t->im = cimag(ot);
  c->re = creal(oc); c->im = cimag(oc);
  src->re = creal(os); src->im = cimag(os);
  return 0;
}

/* n complex divisions with the host compiler's C99 complex division (libgcc
 * __divdc3, as std::complex<double> in the reference): in = {a,b,c,d}[n]. */
void orc_cdiv_batch(int n, const double* in, double* out) {
  for (int i = 0; i < n; ++i) {
    const double complex q = mkc(in[4 * i], in[4 * i + 1]) / mkc(in[4 * i + 2], in[4 * i + 3]);
    out[2 * i] = creal(q);
    out[2 * i + 1] = cimag(q);
  }
}

/* fill_coefficients, coefficients.cpp:57-92, homogeneous material. */
int orc_fill_coefficients_uniform(orc_state* s, const orc_scheme* sp, const orc_material* m) {
  for (int ci = 0; ci < 12; ++ci) {
    const orc_desc* d = &orc_component_table[ci];
    const int si = orc_source_index(ci);
    const double orient = d->family == ORC_FAM_E ? -1.0 : 1.0; /* :64-66 */
    const double sign = orient * (double)d->curl_sign;
    /* select_mode, coefficients.hpp:42-45 */
    const int back = d->family == ORC_FAM_E && m->eps_re < 0.0;
    orc_c128 t, c, src;
    if (orc_derive_coefficients(m, sp, d->family, back, &t, &c, &src)) return -1;
    /* from_std(sign * uc.c): double * complex scales both parts */
    const orc_c128 cs = {sign * c.re, sign * c.im};
    for (int z = 0; z < s->nz; ++z)
      for (int y = 0; y < s->ny; ++y)
        for (int x = 0; x < s->nx; ++x) {
          const size_t i = orc_linear_index(s->nx, s->ny, x, y, z);
          s->a[12 + ci][i] = t;
          s->a[24 + ci][i] = cs;
          if (si >= 0) s->a[36 + si][i] = src;
        }
  }
  return 0;
}

/* build_benchmark_problem, coefficients.cpp:94-111 (state pre-zeroed). */
int orc_build_benchmark_problem(orc_state* s, const orc_scheme* sp) {
  const orc_material vac = {1.0, 0.0, 1.0, 0.0, 0.0}; /* MaterialCell{} defaults */
  if (orc_fill_coefficients_uniform(s, sp, &vac)) return -1;
  const int zsrc = s->nz / 4; /* source_plane_z, coefficients.hpp:70 */
  for (int si = 0; si < 4; ++si)
    for (int z = 0; z < s->nz; ++z) {
      if (z == zsrc) continue;
      for (int y = 0; y < s->ny; ++y)
        for (int x = 0; x < s->nx; ++x) {
          orc_c128* p = &s->a[36 + si][orc_linear_index(s->nx, s->ny, x, y, z)];
          p->re = 0.0; p->im = 0.0;
        }
    }
  return 0;
}

/* ---- seeded synthetic inputs ---- */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

static uint64_t orc_bits(uint64_t seed, int array_id, uint64_t counter, int draw) {
  const uint64_t key =
      orc_splitmix64(orc_splitmix64(seed) ^ ((uint64_t)(array_id + 1) * 0x9E3779B97F4A7C15ull));
  return orc_splitmix64(key + (counter << 8) + (uint64_t)draw);
}

double orc_uniform(uint64_t seed, int array_id, uint64_t counter, int draw) {
  return (double)(orc_bits(seed, array_id, counter, draw) >> 11) * 0x1.0p-53;
}

static orc_c128 orc_field_value(uint64_t seed, int array_id, uint64_t counter) {
  orc_c128 v;
  v.re = 2.0 * orc_uniform(seed, array_id, counter, 0) - 1.0;
  v.im = 2.0 * orc_uniform(seed, array_id, counter, 1) - 1.0;
  return v;
}

static orc_c128 orc_disk_value(uint64_t seed, int array_id, uint64_t counter) {
  const double r = 0.45;
  for (int k = 0; k < 64; ++k) {
    const double re = r * (2.0 * orc_uniform(seed, array_id, counter, 2 * k) - 1.0);
    const double im = r * (2.0 * orc_uniform(seed, array_id, counter, 2 * k + 1) - 1.0);
    if (re * re + im * im <= r * r) {
      orc_c128 v = {re, im};
      return v;
    }
  }
  orc_c128 z = {0.0, 0.0};
  return z;
}

/* Every value is a pure function of (seed, array, padded index), so the
   planes are filled in parallel (OpenMP; same values for any thread count). */
void orc_generate_random(orc_state* s, uint64_t seed) {
  for (int a = 0; a < 40; ++a)
#pragma omp parallel for schedule(static)
    for (int z = 0; z < s->nz; ++z)
      for (int y = 0; y < s->ny; ++y)
        for (int x = 0; x < s->nx; ++x) {
          const size_t i = orc_linear_index(s->nx, s->ny, x, y, z);
          s->a[a][i] = a < 12 ? orc_field_value(seed, a, i) : orc_disk_value(seed, a, i);
        }
}

static int orc_layer_of(uint64_t seed, int nx, int nz, int x, int y, int z) {
  int layer = 0;
  for (int k = 1; k <= 5; ++k) {
    const int h = (int)((orc_bits(seed, 64 + k, (uint64_t)y * (uint64_t)nx + (uint64_t)x, 0) >> 11) %
                        17ull) - 8;
    if (z >= k * nz / 6 + h) ++layer;
  }
  return layer;
}

void orc_generate_layered(orc_state* s, uint64_t seed) {
  orc_c128 table[28][6];
  for (int a = 12; a < 40; ++a)
    for (int L = 0; L < 6; ++L) table[a - 12][L] = orc_disk_value(seed, a, (uint64_t)L);
#pragma omp parallel for schedule(static)
  for (int z = 0; z < s->nz; ++z)
    for (int y = 0; y < s->ny; ++y)
      for (int x = 0; x < s->nx; ++x) {
        const size_t i = orc_linear_index(s->nx, s->ny, x, y, z);
        const int L = orc_layer_of(seed, s->nx, s->nz, x, y, z);
        for (int a = 0; a < 12; ++a) s->a[a][i] = orc_field_value(seed, a, i);
        for (int a = 12; a < 40; ++a) s->a[a][i] = table[a - 12][L];
      }
}
