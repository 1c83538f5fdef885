// thiim_complex.cuh -- complex arithmetic of the host reference build, on the
// device, bit for bit (for derive_coefficients, coefficients.cpp:25-55, run per
// cell on the GPU).
//
// The reference computes its update coefficients with std::complex<double>
// under g++ (no -ffast-math, no FMA on x86-64):
//   * division goes to libgcc's __divdc3 (GCC >= 12: Smith's method with the
//     overflow / underflow guards of the 2021 rework -- scale by 1/2 near
//     DBL_MAX, by 1/DBL_EPSILON when operands are tiny, alternate evaluation
//     order when the ratio is subnormal, NaN+iNaN recovery of infinities and
//     zeros), restated in cdiv below from the published algorithm;
//   * multiplication is GCC's inline (ac - bd) + i(ad + bc) (__muldc3 only
//     repairs NaN+iNaN results, which finite materials never produce);
//   * double (op) complex scales or promotes componentwise.
// Built with -fmad=false, so no product is fused.  Pinned by
// tests/test_gpu_materials.py against host libgcc on random and edge operands.
// Attribution: the division algorithm (Smith 1962, with the scaling guards of
// GCC's 2021 rework) is the one GCC ships in libgcc2.c (GPL-3.0 with the GCC
// Runtime Library Exception); cdiv is an independent restatement of that
// published algorithm in CUDA, not a copy of the libgcc source.
#pragma once

#include <cfloat>
#include <cmath>

namespace thiim_gpu {

struct dcx {
  double re, im;
};

__device__ __forceinline__ dcx cx(double re, double im) { return dcx{re, im}; }
__device__ __forceinline__ dcx cadd(dcx a, dcx b) { return dcx{a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ dcx csub(dcx a, dcx b) { return dcx{a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ dcx cneg(dcx a) { return dcx{-a.re, -a.im}; }
__device__ __forceinline__ dcx cscale(double s, dcx a) { return dcx{s * a.re, s * a.im}; }
__device__ __forceinline__ dcx cmul(dcx x, dcx y) {
  return dcx{x.re * y.re - x.im * y.im, x.re * y.im + x.im * y.re};
}

// libgcc __divdc3 (GCC >= 12), (a + ib) / (c + id)
__device__ __forceinline__ dcx cdiv(dcx n, dcx dd) {
  constexpr double RBIG = DBL_MAX / 2.0;
  constexpr double RMIN = DBL_MIN;
  constexpr double RMIN2 = DBL_EPSILON;
  constexpr double RMINSCAL = 1.0 / DBL_EPSILON;
  constexpr double RMAX2 = RBIG * RMIN2;
  double a = n.re, b = n.im, c = dd.re, d = dd.im;
  double denom, ratio, x, y;
  if (fabs(c) < fabs(d)) {
    if (fabs(d) >= RBIG) {
      a = a / 2;
      b = b / 2;
      c = c / 2;
      d = d / 2;
    }
    if (fabs(d) < RMIN2) {
      a = a * RMINSCAL;
      b = b * RMINSCAL;
      c = c * RMINSCAL;
      d = d * RMINSCAL;
    } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(d) < RMAX2)) ||
               ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(d) < RMAX2))) {
      a = a * RMINSCAL;
      b = b * RMINSCAL;
      c = c * RMINSCAL;
      d = d * RMINSCAL;
    }
    ratio = c / d;
    denom = (c * ratio) + d;
    if (fabs(ratio) > RMIN) {
      x = ((a * ratio) + b) / denom;
      y = ((b * ratio) - a) / denom;
    } else {
      x = ((c * (a / d)) + b) / denom;
      y = ((c * (b / d)) - a) / denom;
    }
  } else {
    if (fabs(c) >= RBIG) {
      a = a / 2;
      b = b / 2;
      c = c / 2;
      d = d / 2;
    }
    if (fabs(c) < RMIN2) {
      a = a * RMINSCAL;
      b = b * RMINSCAL;
      c = c * RMINSCAL;
      d = d * RMINSCAL;
    } else if (((fabs(a) < RMIN) && (fabs(b) < RMAX2) && (fabs(c) < RMAX2)) ||
               ((fabs(b) < RMIN) && (fabs(a) < RMAX2) && (fabs(c) < RMAX2))) {
      a = a * RMINSCAL;
      b = b * RMINSCAL;
      c = c * RMINSCAL;
      d = d * RMINSCAL;
    }
    ratio = d / c;
    denom = (d * ratio) + c;
    if (fabs(ratio) > RMIN) {
      x = ((b * ratio) + a) / denom;
      y = (b - (a * ratio)) / denom;
    } else {
      x = (a + (d * (b / c))) / denom;
      y = (b - (d * (a / c))) / denom;
    }
  }
  if (isnan(x) && isnan(y)) {  // recover infinities and zeros
    if (c == 0.0 && d == 0.0 && (!isnan(a) || !isnan(b))) {
      x = copysign(INFINITY, c) * a;
      y = copysign(INFINITY, c) * b;
    } else if ((isinf(a) || isinf(b)) && isfinite(c) && isfinite(d)) {
      a = copysign(isinf(a) ? 1.0 : 0.0, a);
      b = copysign(isinf(b) ? 1.0 : 0.0, b);
      x = INFINITY * (a * c + b * d);
      y = INFINITY * (b * c - a * d);
    } else if ((isinf(c) || isinf(d)) && isfinite(a) && isfinite(b)) {
      c = copysign(isinf(c) ? 1.0 : 0.0, c);
      d = copysign(isinf(d) ? 1.0 : 0.0, d);
      x = 0.0 * (a * c + b * d);
      y = 0.0 * (b * c - a * d);
    }
  }
  return dcx{x, y};
}

}  // namespace thiim_gpu
