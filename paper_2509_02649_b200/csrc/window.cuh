// window.cuh -- device helpers shared by the spreading (type-1) and gather (type-2) kernels:
// sample position on a fine grid and the cubic B-spline window taps.
#pragma once
#include "fk_internal.cuh"

namespace fk {
namespace {

// cubic B-spline taps at cells c-1, c, c+1, c+2 for fractional offset f in [0,1), scaled by K*6
// and rounded to integers; i2 closes the partition of unity exactly (sum = S).
__device__ __forceinline__ void bs3_fixed(float f, float K, int S, int& i0, int& i1, int& i2, int& i3) {
  const float g = 1.0f - f;
  const float f2 = f * f, f3 = f2 * f, g3 = g * g * g;
  i0 = __float_as_int(fmaf(g3, K, FK_MAGIC)) - FK_MAGIC_BITS;
  i3 = __float_as_int(fmaf(f3, K, FK_MAGIC)) - FK_MAGIC_BITS;
  const float w1 = fmaf(f3, 3.0f * K, fmaf(f2, -6.0f * K, 4.0f * K));
  i1 = __float_as_int(w1 + FK_MAGIC) - FK_MAGIC_BITS;
  i2 = S - i0 - i1 - i3;
}

__device__ __forceinline__ void bs3_exact(float f, double* w) {
  const double fd = f, g = 1.0 - fd;
  w[0] = g * g * g / 6.0;
  w[3] = fd * fd * fd / 6.0;
  w[1] = (3.0 * fd * fd * fd - 6.0 * fd * fd + 4.0) / 6.0;
  w[2] = 1.0 - w[0] - w[1] - w[3];
}

// Position of one sample on both grids.  p = X * nf_mu / (4L) is the offset (in moment-grid
// cells) from the grid centre; the rhs grid has half the cells, so its offset is p / 2.
template <bool EXACT>
__device__ __forceinline__ void pos_f32(float x, float a_hi, float a_lo, int nqA, int nqB, int& tA, int& tB, float& fA,
                                        float& fB) {
  float p = x * a_hi;
  float fl = floorf(p);
  float f = p - fl;
  float pB = p * 0.5f;
  float flB = floorf(pB);
  float fb = pB - flB;
  if (!EXACT) {  // compensated product: p_true = p + e exactly up to fp32 rounding of e
    const float e = fmaf(x, a_hi, -p) + x * a_lo;
    f += e;
    if (f < 0.0f) { f += 1.0f; fl -= 1.0f; }
    if (f >= 1.0f) { f -= 1.0f; fl += 1.0f; }
    fb += 0.5f * e;
    if (fb < 0.0f) { fb += 1.0f; flB -= 1.0f; }
    if (fb >= 1.0f) { fb -= 1.0f; flB += 1.0f; }
  }
  tA = (__float_as_int(fl + FK_MAGIC) - FK_MAGIC_BITS) + nqA;
  tB = (__float_as_int(flB + FK_MAGIC) - FK_MAGIC_BITS) + nqB;
  fA = f;
  fB = fb;
}

__device__ __forceinline__ void pos_f64(double x, double a, int nqA, int nqB, int& tA, int& tB, float& fA, float& fB) {
  const double p = x * a;
  double fl = floor(p);
  float f = (float)(p - fl);
  if (f >= 1.0f) { f = 0.0f; fl += 1.0; }
  const double pB = 0.5 * p;
  double flB = floor(pB);
  float fb = (float)(pB - flB);
  if (fb >= 1.0f) { fb = 0.0f; flB += 1.0; }
  // clamp before the int conversion so NaN / huge values land out of range
  const double lim = 4.0e8;
  tA = (int)fmin(fmax(fl, -lim), lim) + nqA;
  tB = (int)fmin(fmax(flB, -lim), lim) + nqB;
  if (p != p) tA = -1;
  fA = f;
  fB = fb;
}



// Single-grid position: first tap t (local index, = floor(p) + nq) and offset f for p = x * a.
template <bool EXACT>
__device__ __forceinline__ void pos1_f32(float x, float a_hi, float a_lo, int nq, int& t, float& f) {
  const float p = x * a_hi;
  float fl = floorf(p);
  f = p - fl;
  if (!EXACT) {
    const float e = fmaf(x, a_hi, -p) + x * a_lo;
    f += e;
    if (f < 0.0f) { f += 1.0f; fl -= 1.0f; }
    if (f >= 1.0f) { f -= 1.0f; fl += 1.0f; }
  }
  t = (__float_as_int(fl + FK_MAGIC) - FK_MAGIC_BITS) + nq;
}

__device__ __forceinline__ void bs3_float(float f, float* w) {
  const float g = 1.0f - f;
  const float f2 = f * f, f3 = f2 * f;
  w[0] = g * g * g * (1.0f / 6.0f);
  w[3] = f3 * (1.0f / 6.0f);
  w[1] = fmaf(f3, 0.5f, fmaf(f2, -1.0f, 2.0f / 3.0f));
  w[2] = 1.0f - w[0] - w[1] - w[3];
}

}  // namespace
}  // namespace fk
