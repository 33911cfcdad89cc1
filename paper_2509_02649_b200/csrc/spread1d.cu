// spread1d.cu -- the d = 1 type-1 pass over all samples (sec. 2.3):
//   mu_q = sum_j exp(-i q t_j),  |q| <= 2m      r_k = sum_j Y_j exp(-i k t_j),  |k| <= m
// computed as: spread every sample onto an oversampled periodic fine grid on t in [-pi, pi)
// (points occupy its middle half), FFT the grid, deconvolve by the window transform and keep
// the needed modes.  DESIGN.md §"Kernels" derives the design; summary:
//
//   fp32 path (eps >= 1e-7): cubic B-spline window (4 taps, no transcendental), moment grid
//     nf_mu ~ sigma (4m+1) with sigma ~ 16, rhs grid nf_r = nf_mu / 2; both grids' occupied
//     halves live in ONE CTA's shared memory as int32 fixed point (native ATOMS.ADD; fp32 smem
//     atomics are CAS loops on sm_100a).  Partition of unity is exact in fixed point.  A cell
//     that reaches 2^29 in magnitude is drained into an fp64 global carry grid (atomicExch), so no
//     periodic flush is needed.  No overflow: after a cell crosses 2^29 each of the CTA's 1024
//     threads can add at most once more (<= 2/3 x 2^21 each) before it drains, 2^29 + 1024 x 1.4e6
//     < 2^31 (tests/test_gpu_d1.py: 10^4 identical samples in one CTA).  The rhs channel uses a per-CTA power-of-two
//     scale from the CTA's first 4096 |Y|; |Y| outliers (and NaN) take an exact fp64 slow path.
//   fp64 mode (eps < 1e-7): septic B-spline window (8 taps, sigma ~ 11 at 1e-10), one channel per
//     pass, 64-bit fixed point held as int32 pairs in shared memory (pair_add_n) -- k_spread1d_bs7.
//     When a grid does not fit a CTA (large m, eps < 1e-13): the exponential-of-semicircle window
//     (sigma = 2, w ~ log10(1/eps) + 2) in the same fixed point (k_spread1d_esx), else fp64
//     global atomics (k_spread1d_es).
//
// X and Y are streamed once from HBM with 128-bit evict-first loads, software-pipelined one
// iteration ahead; CTAs are persistent (1-2 per SM) over contiguous sample ranges.
#include <cmath>
#include <type_traits>

#include "fk_internal.cuh"
#include "window.cuh"

namespace fk {
namespace {

constexpr float kSA = 2097152.0f;  // 2^21: density fixed-point scale (tap weights <= 2/3)
constexpr double kInvSA = 1.0 / 2097152.0;
constexpr int kYProbe = 4096;      // samples used to pick a CTA's rhs scale

__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }

__device__ __noinline__ void drain_cells(int* G, int t0, double* carry, double inv_scale) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int v = atomicExch(G + t0 + k, 0);
    if (v) atomicAdd(carry + t0 + k, (double)v * inv_scale);
  }
}

__device__ __noinline__ void rhs_slow(float y, float fB, double* carryB, int tB0) {
  double w[4];
  bs3_exact(fB, w);
#pragma unroll
  for (int k = 0; k < 4; ++k) atomicAdd(carryB + tB0 + k, w[k] * (double)y);
}

struct Bs3Args {
  int64_t n, stride, per;
  float a_hi, a_lo;
  double a_d;
  int nqA, GA, nqB, GB;
  int* partA;
  int* partB;
  int* escale;
  double* carryA;
  double* carryB;
  int* d_status;
};

template <bool MU, bool R>
__device__ __forceinline__ void bs3_sample(int* __restrict__ A, int* __restrict__ B, const Bs3Args& g, int tA, int tB, float fA,
                                           float fB, float y, float SY, float invSY_unused, double invSY, bool& bad) {
  if ((unsigned)tA > (unsigned)(g.GA - 4)) {  // |X| > L (beyond rounding) or NaN: skip, flag
    bad = true;
    return;
  }
  if (MU) {
    int i0, i1, i2, i3;
    bs3_fixed(fA, kSA * (1.0f / 6.0f), (int)kSA, i0, i1, i2, i3);
    int* c = A + tA;
    const int o0 = atomicAdd(c, i0), o1 = atomicAdd(c + 1, i1), o2 = atomicAdd(c + 2, i2), o3 = atomicAdd(c + 3, i3);
    if ((o0 | o1 | o2 | o3) & 0x60000000) drain_cells(A, tA, g.carryA, kInvSA);  // some cell >= 2^29
  }
  if (R) {
    const float ys = y * SY;
    if (fabsf(ys) < 2097152.0f) {
      int j0, j1, j2, j3;
      const int jS = __float_as_int(ys + FK_MAGIC) - FK_MAGIC_BITS;
      bs3_fixed(fB, ys * (1.0f / 6.0f), jS, j0, j1, j2, j3);
      int* c = B + tB;
      const unsigned p0 = (unsigned)atomicAdd(c, j0), p1 = (unsigned)atomicAdd(c + 1, j1);
      const unsigned p2 = (unsigned)atomicAdd(c + 2, j2), p3 = (unsigned)atomicAdd(c + 3, j3);
      const unsigned T = 1u << 29;  // |cell| >= 2^29  <=>  cell + 2^29 outside [0, 2^30)
      if (((p0 + T) | (p1 + T) | (p2 + T) | (p3 + T)) & 0xC0000000u) drain_cells(B, tB, g.carryB, invSY);
    } else {
      rhs_slow(y, fB, g.carryB, tB);
    }
  }
}

template <typename XT, bool MU, bool R, bool VEC, bool EXACT>
__global__ void __launch_bounds__(1024, 1) k_spread1d_bs3(const XT* __restrict__ X, const XT* __restrict__ Y, Bs3Args g) {
  extern __shared__ int sm[];
  int* A = sm;
  int* B = sm + (MU ? g.GA : 0);
  const int nsm = (MU ? g.GA : 0) + (R ? g.GB : 0);
  for (int i = threadIdx.x; i < nsm; i += blockDim.x) sm[i] = 0;

  const int64_t beg = (int64_t)blockIdx.x * g.per;
  const int64_t end = min(g.n, beg + g.per);

  // rhs scale of this CTA: 2^E with max|Y| 2^E in [2^19, 2^20) over its first kYProbe samples
  float SY = 0.0f;
  double invSY = 0.0;
  int E = 19;
  if (R) {
    __shared__ float red[32];
    __shared__ int sE;
    float mx = 0.0f;
    const int64_t cnt = max((int64_t)0, min(end - beg, (int64_t)kYProbe));
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) mx = fmaxf(mx, fabsf((float)Y[beg + i]));
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.0f;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmaxf(t, red[w]);
      int e2 = 0;
      int Eloc = 19;
      if (t > 0.0f && t <= 3.0e38f) {
        frexpf(t, &e2);  // t = mant * 2^e2, mant in [0.5, 1)
        Eloc = 20 - e2;
      }
      Eloc = max(-100, min(110, Eloc));
      sE = Eloc;
      g.escale[blockIdx.x] = Eloc;
    }
    __syncthreads();
    E = sE;
    SY = ldexpf(1.0f, E);
    invSY = ldexp(1.0, -E);
  }
  __syncthreads();

  bool bad = false;
  if (VEC) {
    // 4 samples per thread per step; float4 streaming loads, prefetched one step ahead
    const float4* X4 = reinterpret_cast<const float4*>(X);
    const float4* Y4 = reinterpret_cast<const float4*>(Y);
    const int64_t b4 = beg >> 2, e4 = end >> 2;
    int64_t i = b4 + threadIdx.x;
    float4 xv = make_float4(0, 0, 0, 0), yv = make_float4(0, 0, 0, 0);
    if (i < e4) {
      xv = ld_stream(X4 + i);
      if (R) yv = ld_stream(Y4 + i);
    }
    while (i < e4) {
      const int64_t inx = i + blockDim.x;
      float4 xn = make_float4(0, 0, 0, 0), yn = make_float4(0, 0, 0, 0);
      if (inx < e4) {
        xn = ld_stream(X4 + inx);
        if (R) yn = ld_stream(Y4 + inx);
      }
      const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
      const float ys[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int tA, tB;
        float fA, fB;
        pos_f32<EXACT>(xs[q], g.a_hi, g.a_lo, g.nqA, g.nqB, tA, tB, fA, fB);
        bs3_sample<MU, R>(A, B, g, tA, tB, fA, fB, ys[q], SY, 0.f, invSY, bad);
      }
      xv = xn;
      yv = yn;
      i = inx;
    }
    // tail (< 4 samples, last CTA only)
    for (int64_t j = (e4 << 2) + threadIdx.x; j < end; j += blockDim.x) {
      if (j < beg) continue;
      int tA, tB;
      float fA, fB;
      pos_f32<EXACT>((float)X[j], g.a_hi, g.a_lo, g.nqA, g.nqB, tA, tB, fA, fB);
      bs3_sample<MU, R>(A, B, g, tA, tB, fA, fB, R ? (float)Y[j] : 0.f, SY, 0.f, invSY, bad);
    }
  } else {
    for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
      int tA, tB;
      float fA, fB;
      if (sizeof(XT) == 8) pos_f64((double)X[j * g.stride], g.a_d, g.nqA, g.nqB, tA, tB, fA, fB);
      else pos_f32<EXACT>((float)X[j * g.stride], g.a_hi, g.a_lo, g.nqA, g.nqB, tA, tB, fA, fB);
      bs3_sample<MU, R>(A, B, g, tA, tB, fA, fB, R ? (float)Y[j] : 0.f, SY, 0.f, invSY, bad);
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  if (MU) {
    int* dst = g.partA + (int64_t)blockIdx.x * g.GA;
    for (int i = threadIdx.x; i < g.GA; i += blockDim.x) dst[i] = A[i];
  }
  if (R) {
    int* dst = g.partB + (int64_t)blockIdx.x * g.GB;
    for (int i = threadIdx.x; i < g.GB; i += blockDim.x) dst[i] = B[i];
  }
}

// ------------------------------------------------------------------------------------------
// fallback path (grids beyond a CTA's shared memory): exponential-of-semicircle window, fp64
// accumulation in global memory (k_spread1d_es) or, in fp64 mode with the grids in shared memory,
// 64-bit fixed point (k_spread1d_esx below)
// ------------------------------------------------------------------------------------------
struct EsArgs {
  int64_t n, stride, per;
  double a;  // nf_mu / (4L)
  int w;
  double beta;
  int nfA, offA, GA, nfB, offB, GB;
  double* partA;
  double* partB;
  double* carryA;  // fixed-point fp64-mode kernel (k_spread1d_esx): drained hi words
  double* carryB;
  int* d_status;
};

__device__ __forceinline__ void es_spread(double* G, double ul, int w, double beta, double c) {
  const int l0 = (int)ceil(ul - 0.5 * w);
  const double inv = 2.0 / w;
  for (int i = 0; i < w; ++i) {
    const double z = ((double)(l0 + i) - ul) * inv;
    const double v = 1.0 - z * z;
    const double psi = v > 0.0 ? exp(beta * (sqrt(v) - 1.0)) : 0.0;
    atomicAdd(G + l0 + i, c * psi);
  }
}

template <typename XT, bool MU, bool R, bool SMEM>
__global__ void __launch_bounds__(1024, 1) k_spread1d_es(const XT* __restrict__ X, const XT* __restrict__ Y, EsArgs g) {
  extern __shared__ double smd[];
  double* A = SMEM ? smd : g.partA;
  double* B = SMEM ? smd + (MU ? g.GA : 0) : g.partB;
  if (SMEM) {
    const int nsm = (MU ? g.GA : 0) + (R ? g.GB : 0);
    for (int i = threadIdx.x; i < nsm; i += blockDim.x) smd[i] = 0.0;
    __syncthreads();
  }
  const int64_t beg = (int64_t)blockIdx.x * g.per;
  const int64_t end = min(g.n, beg + g.per);
  bool bad = false;
  for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
    const double x = (double)X[j * g.stride];
    const double u = x * g.a + 0.5 * g.nfA;  // moment-grid coordinate (cells), t = -pi at 0
    const double ulA = u - g.offA;
    const int l0 = (int)ceil(ulA - 0.5 * g.w);
    if (!(ulA == ulA) || l0 < 0 || l0 + g.w > g.GA) {
      bad = true;
      continue;
    }
    if (MU) es_spread(A, ulA, g.w, g.beta, 1.0);
    if (R) es_spread(B, 0.5 * u - g.offB, g.w, g.beta, (double)Y[j]);
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  if (SMEM) {
    __syncthreads();
    if (MU) {
      double* dst = g.partA + (int64_t)blockIdx.x * g.GA;
      for (int i = threadIdx.x; i < g.GA; i += blockDim.x) dst[i] = A[i];
    }
    if (R) {
      double* dst = g.partB + (int64_t)blockIdx.x * g.GB;
      for (int i = threadIdx.x; i < g.GB; i += blockDim.x) dst[i] = B[i];
    }
  }
}

// fp64-accuracy mode (eps < 1e-7), shared-memory grids: ES taps as polynomials from a
// constant-memory table (es_horner_table; slot W, uploaded once) instead of exp + sqrt per tap, and
// 64-bit fixed-point accumulation (below).  Measured at C2 shape, n = 1e9, eps = 1e-10: 79 ms with
// exp taps + fp64 CAS atomics, 77 ms now -- the instruction mix moved (ncu: the 360 coefficient
// loads per sample became the MIO limiter) but the rate did not; the gain is that the result is
// now order-independent (bitwise deterministic) like the fp32 path.
__constant__ double c_es_coef[kHornerSlots][kHornerSlot];  // slot W: the W x (W + 3) Horner table (horner_slot)

// tap i of a point at ul from the constant-memory table
template <int W>
__device__ __forceinline__ double es_tap_const(double sv, int i) {
  constexpr int NP = W + 3;
  double acc = c_es_coef[W][i * NP + NP - 1];
#pragma unroll
  for (int q = NP - 2; q >= 0; --q) acc = fma(acc, sv, c_es_coef[W][i * NP + q]);
  return acc;
}

// fp64-accuracy accumulation in 64-bit fixed point held as two int32 words per cell (lo
// unsigned, hi signed): an add is one native ATOMS.ADD on lo, the carry is read off its return
// value, and hi gets (v >> 32) + carry only when that is non-zero.  3.1x the rate of fp64
// shared-memory atomicAdd (a CAS loop on sm_100a; scratch microbenchmark 1.31e12 vs 4.2e11 tap
// adds/s).  Tap weights x 2^40 (rounding 2^-41, far below the 1e-10 target); a hi word that
// reaches 2^29 in magnitude is drained (atomicExch) into an fp64 carry grid, so no overflow.
template <typename XT, bool MU, bool R, int W>
__global__ void __launch_bounds__(1024, 1) k_spread1d_esx(const XT* __restrict__ X, const XT* __restrict__ Y, EsArgs g) {
  extern __shared__ unsigned smx[];
  unsigned* Alo = smx;
  int* Ahi = (int*)(smx + (MU ? g.GA : 0));
  unsigned* Blo = smx + (MU ? 2 * g.GA : 0);
  int* Bhi = (int*)(Blo + (R ? g.GB : 0));
  const int nsm = (MU ? 2 * g.GA : 0) + (R ? 2 * g.GB : 0);
  for (int i = threadIdx.x; i < nsm; i += blockDim.x) smx[i] = 0u;
  const int64_t beg = (int64_t)blockIdx.x * g.per;
  const int64_t end = min(g.n, beg + g.per);
  // rhs scale 2^E with max |Y| 2^E in [2^19, 2^20) over the CTA's first 4096 samples
  int E = 0;
  if (R) {
    __shared__ double red[32];
    __shared__ int sE;
    double mx = 0.0;
    const int64_t cnt = max((int64_t)0, min(end - beg, (int64_t)kYProbe));
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double a = fabs((double)Y[beg + i]);
      if (a == a) mx = fmax(mx, a);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
      int e2 = 0;
      int Eloc = 19;
      if (t > 0.0 && t < 1e300) {
        frexp(t, &e2);
        Eloc = 20 - e2;
      }
      sE = max(-900, min(900, Eloc));
    }
    __syncthreads();
    E = sE;
  }
  __syncthreads();
  const double sy = R ? ldexp(1.0, E) : 0.0;           // Y -> |Y sy| < 2^20
  const double unitA = 1.0 / kSX * 4294967296.0;       // value of one hi unit, mu grid (2^-8)
  const double unitB = R ? ldexp(4294967296.0, -(E + 20)) : 0.0;
  bool bad = false;
  for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
    const double x = (double)X[j * g.stride];
    const double u = x * g.a + 0.5 * g.nfA;  // moment-grid coordinate (cells), t = -pi at 0
    const double ulA = u - g.offA;
    const int l0 = (int)ceil(ulA - 0.5 * W);
    if (!(ulA == ulA) || l0 < 0 || l0 + W > g.GA) {
      bad = true;
      continue;
    }
    if (MU) {
      const double sv = 2.0 * (ulA - l0 - 0.5 * W + 1.0) - 1.0;
#pragma unroll
      for (int i = 0; i < W; ++i) pair_add(Alo, Ahi, l0 + i, __double2ll_rn(es_tap_const<W>(sv, i) * kSX), g.carryA, unitA);
    }
    if (R) {
      const double y = (double)Y[j];
      const double ulB = 0.5 * u - g.offB;
      const int b0 = (int)ceil(ulB - 0.5 * W);
      const double sv = 2.0 * (ulB - b0 - 0.5 * W + 1.0) - 1.0;
      const double ys = y * sy;
      if (fabs(ys) < 2097152.0) {  // |y 2^E| < 2^21: |v| < 2^41, hi stays small
#pragma unroll
        for (int i = 0; i < W; ++i)
          pair_add(Blo, Bhi, b0 + i, __double2ll_rn(es_tap_const<W>(sv, i) * ys * 1048576.0), g.carryB, unitB);
      } else {  // |Y| outlier or NaN: exact fp64 into the carry grid
#pragma unroll 1
        for (int i = 0; i < W; ++i) atomicAdd(g.carryB + b0 + i, y * es_tap_const<W>(sv, i));
      }
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  // per-CTA partials as fp64 values (exact integers times a power of two, rounded once)
  if (MU) {
    double* dst = g.partA + (int64_t)blockIdx.x * g.GA;
    const double sc = 1.0 / kSX;
    for (int i = threadIdx.x; i < g.GA; i += blockDim.x) dst[i] = ((double)Ahi[i] * 4294967296.0 + (double)Alo[i]) * sc;
  }
  if (R) {
    double* dst = g.partB + (int64_t)blockIdx.x * g.GB;
    const double sc = ldexp(1.0, -(E + 20));
    for (int i = threadIdx.x; i < g.GB; i += blockDim.x) dst[i] = ((double)Bhi[i] * 4294967296.0 + (double)Blo[i]) * sc;
  }
}

// ------------------------------------------------------------------------------------------
// fp64 mode, septic B-spline (plan KER_BS7): one channel per pass (CH = 0 moments, 1 rhs), the
// channel's occupied grid in shared memory as 64-bit fixed point (int32 pairs, pair_add), tap
// weights by the uniform Cox-de Boor recursion in fp64 (28 steps, constants 1/j only).  Taps at
// cells floor(p) - 3 .. floor(p) + 4 relative to the grid centre; transform sinc^8 (deconvolved in dft1d.cu).
// Moments: the 8 integer weights are closed to 2^40 exactly (partition of unity: mu_0 = n).
// ------------------------------------------------------------------------------------------
// The 8 weights are degree-7 polynomials in f (the pieces of the cardinal B-spline M_8, exact
// rational coefficients, from the uniform Cox-de Boor recursion): taps 0..3 are P_0..P_3 at f and,
// by symmetry, taps 7..4 are P_0..P_3 at 1 - f (exact in fp64).  Horner from constant memory:
// 56 DFMA per sample instead of the recursion's ~140 fp64 operations.
__constant__ double c_bs7[4][8] = {
    {1.0 / 5040, -1.0 / 720, 1.0 / 240, -1.0 / 144, 1.0 / 144, -1.0 / 240, 1.0 / 720, -1.0 / 5040},
    {1.0 / 42, -7.0 / 90, 1.0 / 10, -1.0 / 18, 0.0, 1.0 / 60, -1.0 / 120, 1.0 / 720},
    {397.0 / 1680, -49.0 / 144, 1.0 / 16, 19.0 / 144, -1.0 / 16, -1.0 / 48, 1.0 / 48, -1.0 / 240},
    {151.0 / 315, 0.0, -1.0 / 3, 0.0, 1.0 / 9, 0.0, -1.0 / 36, 1.0 / 144}};

__device__ __forceinline__ void bs7_weights(double f, double* N) {
  const double g = 1.0 - f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double a = c_bs7[i][7], b = c_bs7[i][7];
#pragma unroll
    for (int k = 6; k >= 0; --k) {
      a = fma(a, f, c_bs7[i][k]);
      b = fma(b, g, c_bs7[i][k]);
    }
    N[i] = a;
    N[7 - i] = b;
  }
}

// round(v) for |v| < 2^51 as a two's-complement int64 by the 1.5 x 2^52 shift: one DFMA (folded
// with the scaling) and a 64-bit subtract instead of F2I.S64.F64
__device__ __forceinline__ long long round_fma(double w, double scale) {
  return __double_as_longlong(fma(w, scale, 6755399441055744.0)) - 0x4338000000000000LL;
}

// 8 consecutive 64-bit fixed-point taps (int32 pairs) of one sample, branch-free: the 8 low-word
// atomics, the carries read off their return values with add.cc/addc (2 instructions per tap),
// then the 8 high-word atomics UNCONDITIONALLY (adding 0 where the high part and carry are 0) and
// one test of all 8 new high words for the rare drain (|hi| >= 2^29 -> fp64 carry grid).  ncu of
// the per-tap-branch version (pair_add_n): the BSSY/BRA/BSYNC around each conditional high-word
// atomic were ~20 % of the fp64 kernel's issued instructions (ptxas turns a predicated atom into a
// branch), while an always-issued high-word atomic costs only atomic-unit time (5 of 8 taps need
// it anyway).
__device__ __forceinline__ void pair_add8(unsigned* __restrict__ lo, int* __restrict__ hi, int c0, const unsigned* l, const int* h,
                                          double* carry, double hi_unit) {
  unsigned o[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) o[i] = atomicAdd(lo + c0 + i, l[i]);
  unsigned any = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int hc;
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.s32 %0, %3, 0;\n\t}" : "=r"(hc) : "r"(o[i]), "r"(l[i]), "r"(h[i]));
    const int old = atomicAdd(hi + c0 + i, hc);
    any |= (unsigned)(old + hc + (1 << 29));  // >= 2^30 iff the new high word is >= 2^29 in magnitude
  }
  if (any >= (1u << 30)) {
#pragma unroll 1
    for (int i = 0; i < 8; ++i) {
      const int t = atomicExch(hi + c0 + i, 0);  // drain (the OR test is conservative: any of the 8)
      if (t) atomicAdd(carry + c0 + i, (double)t * hi_unit);
    }
  }
}

// round(w S) as the two int32 words of a two's-complement int64 (|w S| < 2^51) via the 1.5 x 2^52
// shift: the low word is the double's low word, the high word its high word minus 0x43380000
__device__ __forceinline__ void split_fma(double w, double scale, unsigned& l, int& h) {
  const double d = fma(w, scale, 6755399441055744.0);
  l = (unsigned)__double2loint(d);
  h = __double2hiint(d) - 0x43380000;
}

struct Bs7Args {
  int64_t n, stride, per;
  double a;  // nf / (4L) of the channel's grid (moment grid: nf_mu; rhs grid: nf_r)
  // fixed-point scale of a weight: moments 2^34 for eps >= 1e-10 (then a tap's value fits the low
  // word unless it exceeds 1/4: ~5 high-word atomics per sample instead of ~7 at 2^40; rounding
  // 2^-35 relative per tap, worst case 8 x 2^-35 = 2.3e-10 of mu_0 per mode); the rhs always 2^40
  // (its l2 norm can be ~sqrt(n) times smaller than sum |Y|: 2^34 gave 2.6e-10 l2 at n = 2e4 and
  // 2^37 1.6e-10 at n = 10, eps = 1e-11); 2^40 for both below eps = 1e-10
  double S;
  int nq, G;
  double* part;
  double* carry;
  int* d_status;
};

template <typename XT, int CH>
__global__ void __launch_bounds__(1024, 1) k_spread1d_bs7(const XT* __restrict__ X, const XT* __restrict__ Y, Bs7Args g) {
  extern __shared__ unsigned sm7[];
  unsigned* lo = sm7;
  int* hi = (int*)(sm7 + g.G);
  for (int i = threadIdx.x; i < 2 * g.G; i += blockDim.x) sm7[i] = 0u;
  const int64_t beg = (int64_t)blockIdx.x * g.per;
  const int64_t end = min(g.n, beg + g.per);
  int E = 0;
  if (CH == 1) {  // rhs scale 2^E with max |Y| 2^E in [2^19, 2^20) over the CTA's first samples
    __shared__ double red[32];
    __shared__ int sE;
    double mx = 0.0;
    const int64_t cnt = max((int64_t)0, min(end - beg, (int64_t)kYProbe));
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double a = fabs((double)Y[beg + i]);
      if (a == a) mx = fmax(mx, a);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = fmax(t, red[w]);
      int e2 = 0, Eloc = 19;
      if (t > 0.0 && t < 1e300) {
        frexp(t, &e2);
        Eloc = 20 - e2;
      }
      sE = max(-900, min(900, Eloc));
    }
    __syncthreads();
    E = sE;
  }
  __syncthreads();
  const double sy = CH == 1 ? ldexp(1.0, E) : 0.0;
  // rhs: |Y 2^E| < 2^21 on the fast path, so Y 2^E x S 2^-21 keeps a tap below S
  const double Rm = g.S * (1.0 / 2097152.0);
  const double unit = CH == 0 ? 4294967296.0 / g.S : 4294967296.0 / (ldexp(1.0, E) * Rm);
  const long long S64 = (long long)g.S;  // the closure total as two words
  const unsigned S_lo = (unsigned)S64;
  const int S_hi = (int)(S64 >> 32);
  bool bad = false;
  // software pipeline: the next sample's X (and Y) are loaded one iteration ahead
  int64_t j = beg + threadIdx.x;
  XT xn = j < end ? X[j * g.stride] : (XT)0;
  XT yn = (CH == 1 && j < end) ? Y[j] : (XT)0;
  for (; j < end; j += blockDim.x) {
    const XT xc = xn, yc = yn;
    if (j + blockDim.x < end) {
      xn = X[(j + blockDim.x) * g.stride];
      if (CH == 1) yn = Y[j + blockDim.x];
    }
    const double p = (double)xc * g.a;
    const double fl = floor(p);
    const double f = p - fl;
    const int t0 = (p == p && fabs(p) < 1e9) ? (int)fl + g.nq : -1;
    if ((unsigned)t0 > (unsigned)(g.G - 8)) {
      bad = true;
      continue;
    }
    double wv[8];
    bs7_weights(f, wv);
    if (CH == 0) {
      unsigned l[8];
      int h[8];
      unsigned sl = 0;
      int sh = 0;
#pragma unroll
      for (int i = 0; i < 7; ++i) {
        split_fma(wv[i], g.S, l[i], h[i]);
        asm("add.cc.u32 %0, %0, %2;\n\taddc.s32 %1, %1, %3;" : "+r"(sl), "+r"(sh) : "r"(l[i]), "r"(h[i]));
      }
      // partition of unity closed in integers: tap 7 = S - sum of taps 0..6 (64-bit, as two words)
      asm("sub.cc.u32 %0, %2, %3;\n\tsubc.s32 %1, %4, %5;" : "=r"(l[7]), "=r"(h[7]) : "r"(S_lo), "r"(sl), "r"(S_hi), "r"(sh));
      pair_add8(lo, hi, t0, l, h, g.carry, unit);
    } else {
      const double y = (double)yc;
      const double ys = y * sy;
      if (fabs(ys) < 2097152.0) {
        const double ysr = ys * Rm;
        unsigned l[8];
        int h[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) split_fma(wv[i], ysr, l[i], h[i]);
        pair_add8(lo, hi, t0, l, h, g.carry, unit);
      } else {  // |Y| outlier or NaN: exact fp64 into the carry grid (unrolled: a runtime index
                // would put wv in local memory, stored on every sample -- ncu showed the STLs)
#pragma unroll
        for (int i = 0; i < 8; ++i) atomicAdd(g.carry + t0 + i, y * wv[i]);
      }
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  double* dst = g.part + (int64_t)blockIdx.x * g.G;
  const double sc = CH == 0 ? 1.0 / g.S : 1.0 / (ldexp(1.0, E) * Rm);
  for (int i = threadIdx.x; i < g.G; i += blockDim.x) dst[i] = ((double)hi[i] * 4294967296.0 + (double)lo[i]) * sc;
}

struct Ws1 {
  void* partA = nullptr;
  void* partB = nullptr;
  int* escale = nullptr;
  double* carryA = nullptr;
  double* carryB = nullptr;
  double* tabA = nullptr;
  double* tabB = nullptr;
  void* dftws = nullptr;
  size_t dft_bytes = 0;
};

// the grids of a pass in the order dft1d_run takes them (moments first)
static int dft_grids(const Plan1& p, bool mu, bool r, const Ws1& w, const Type1Out* out, Dft1Grid* g) {
  const int nparts = p.smem ? p.ctas : 1;
  int k = 0;
  for (int ch = 0; ch < 2; ++ch) {
    if ((ch == 0 && !mu) || (ch == 1 && !r)) continue;
    const Geo& gg = ch == 0 ? p.gA : p.gB;
    Dft1Grid d;
    d.nf = gg.nf;
    d.off = gg.off;
    d.G = gg.G;
    d.K = ch == 0 ? 2 * p.m : p.m;
    d.nparts = nparts;
    void* part = ch == 0 ? w.partA : w.partB;
    if (p.fp64) d.part_d = (const double*)part;
    else d.part_i = (const int*)part;
    d.escale = (ch == 1 && !p.fp64) ? w.escale : nullptr;
    d.inv_scale = kInvSA;
    d.carry = ch == 0 ? w.carryA : w.carryB;
    d.phihat = ch == 0 ? w.tabA : w.tabB;
    d.out = out ? (ch == 0 ? out->mu : out->r) : nullptr;
    g[k++] = d;
  }
  return k;
}

static fk_status layout1(const Plan1& p, bool mu, bool r, Bump& b, Ws1& w) {
  const size_t esz = p.fp64 ? 8 : 4;
  const int nparts = p.smem ? p.ctas : 1;
  if (mu) {
    w.partA = b.take((size_t)nparts * p.gA.G * esz);
    if (!p.fp64 || p.smem) w.carryA = (double*)b.take((size_t)p.gA.G * 8);
    if (p.ker == KER_ES) w.tabA = (double*)b.take((size_t)(2 * p.m + 1) * 8);
  }
  if (r) {
    w.partB = b.take((size_t)nparts * p.gB.G * esz);
    if (!p.fp64 || p.smem) w.carryB = (double*)b.take((size_t)p.gB.G * 8);
    if (!p.fp64) w.escale = (int*)b.take((size_t)p.ctas * 4);
    if (p.ker == KER_ES) w.tabB = (double*)b.take((size_t)(p.m + 1) * 8);
  }
  Dft1Grid g[2];
  const int ng = dft_grids(p, mu, r, w, nullptr, g);
  w.dft_bytes = dft1d_ws_bytes(g, ng);
  if (w.dft_bytes == 0) return fail(FK_E_UNSUPPORTED, "type-1 pass: no DFT factorisation for this grid size");
  w.dftws = b.take(w.dft_bytes);
  return FK_OK;
}

template <typename XT, bool MU, bool R>
static void launch_bs3(const Plan1& p, const XT* X, const XT* Y, const Bs3Args& a, bool vec, bool exact, cudaStream_t s) {
  auto run = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
    prof_spread_begin(s);
    kern<<<p.ctas, p.threads, p.smem_bytes, s>>>(X, Y, a);
    prof_spread_end(s);
    count_launch();
  };
  if (sizeof(XT) == 8) {
    run(k_spread1d_bs3<XT, MU, R, false, false>);
  } else if (vec) {
    if (exact) run(k_spread1d_bs3<XT, MU, R, true, true>);
    else run(k_spread1d_bs3<XT, MU, R, true, false>);
  } else {
    if (exact) run(k_spread1d_bs3<XT, MU, R, false, true>);
    else run(k_spread1d_bs3<XT, MU, R, false, false>);
  }
}

template <typename XT, bool MU, bool R>
static void launch_es(const Plan1& p, const XT* X, const XT* Y, const EsArgs& a, cudaStream_t s) {
  if (p.smem && p.es.w >= 9 && (!MU || a.carryA) && (!R || a.carryB) && horner_slot(c_es_coef, p.es.w, p.es.beta) == FK_OK) {
    const size_t smem = p.smem_bytes;  // 2 x int32 per cell = the fp64 grid's bytes
    auto go = [&](auto wtag) {
      constexpr int WW = decltype(wtag)::value;
      auto k = k_spread1d_esx<XT, MU, R, WW>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      prof_spread_begin(s);
      k<<<p.ctas, p.threads, smem, s>>>(X, Y, a);
      prof_spread_end(s);
    };
    switch (p.es.w) {
      case 9: go(std::integral_constant<int, 9>{}); break;
      case 10: go(std::integral_constant<int, 10>{}); break;
      case 11: go(std::integral_constant<int, 11>{}); break;
      case 12: go(std::integral_constant<int, 12>{}); break;
      case 13: go(std::integral_constant<int, 13>{}); break;
      case 14: go(std::integral_constant<int, 14>{}); break;
      case 15: go(std::integral_constant<int, 15>{}); break;
      default: go(std::integral_constant<int, 16>{}); break;
    }
    count_launch();
    return;
  }
  if (p.smem) {
    auto k = k_spread1d_es<XT, MU, R, true>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem_bytes);
    prof_spread_begin(s);
    k<<<p.ctas, p.threads, p.smem_bytes, s>>>(X, Y, a);
    prof_spread_end(s);
  } else {
    prof_spread_begin(s);
    k_spread1d_es<XT, MU, R, false><<<p.ctas, p.threads, 0, s>>>(X, Y, a);
    prof_spread_end(s);
  }
  count_launch();
}

template <typename XT>
static fk_status spread_dispatch(const Plan1& p, const fk_points& Xp, const void* Yv, double L, bool mu, bool r, const Ws1& w,
                                 int* d_status, cudaStream_t s) {
  const XT* X = (const XT*)Xp.ptr;
  const XT* Y = (const XT*)Yv;
  const int64_t n = Xp.n;
  if (p.ker == KER_BS7) {  // one pass per channel
    for (int ch = 0; ch < 2; ++ch) {
      if ((ch == 0 && !mu) || (ch == 1 && !r)) continue;
      Bs7Args a{};
      a.n = n;
      a.stride = Xp.stride_n;
      a.per = (n + p.ctas - 1) / p.ctas;
      const Geo& gg = ch == 0 ? p.gA : p.gB;
      a.a = (double)gg.nf / (4.0 * L);
      a.nq = gg.nf / 4;
      a.G = gg.G;
      a.part = (double*)(ch == 0 ? w.partA : w.partB);
      a.carry = ch == 0 ? w.carryA : w.carryB;
      a.d_status = d_status;
      a.S = (p.eps >= 1e-10 && ch == 0) ? 17179869184.0 : 1099511627776.0;  // 2^34 / 2^40 (Bs7Args)
      const size_t smem = (size_t)gg.G * 8;
      auto k = ch == 0 ? k_spread1d_bs7<XT, 0> : k_spread1d_bs7<XT, 1>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      prof_spread_begin(s);
      k<<<p.ctas, p.threads, smem, s>>>(X, Y, a);
      prof_spread_end(s);
      count_launch();
    }
    FK_CUDA_TRY(cudaGetLastError());
    return FK_OK;
  }
  if (!p.fp64) {
    Bs3Args a{};
    a.n = n;
    a.stride = Xp.stride_n;
    const double ad = (double)p.nf_mu / (4.0 * L);
    a.a_d = ad;
    a.a_hi = (float)ad;
    a.a_lo = (float)(ad - (double)a.a_hi);
    int ex = 0;
    const bool exact = (std::frexp(ad, &ex) == 0.5);  // power of two: X * a is exact in fp32
    a.nqA = p.nf_mu / 4;
    a.nqB = p.nf_r / 4;
    a.GA = p.gA.G;
    a.GB = p.gB.G;
    const bool vec = sizeof(XT) == 4 && Xp.stride_n == 1 && ((uintptr_t)X % 16 == 0) && (!r || ((uintptr_t)Y % 16 == 0));
    int64_t per = (n + p.ctas - 1) / p.ctas;
    per = (per + 3) & ~(int64_t)3;
    a.per = per;
    a.partA = (int*)w.partA;
    a.partB = (int*)w.partB;
    a.escale = w.escale;
    a.carryA = w.carryA;
    a.carryB = w.carryB;
    a.d_status = d_status;
    if (mu && r) launch_bs3<XT, true, true>(p, X, Y, a, vec, exact, s);
    else if (mu) launch_bs3<XT, true, false>(p, X, Y, a, vec, exact, s);
    else launch_bs3<XT, false, true>(p, X, Y, a, vec, exact, s);
  } else {
    EsArgs a{};
    a.n = n;
    a.stride = Xp.stride_n;
    a.a = (double)p.nf_mu / (4.0 * L);
    a.w = p.es.w;
    a.beta = p.es.beta;
    a.nfA = p.nf_mu;
    a.offA = p.gA.off;
    a.GA = p.gA.G;
    a.nfB = p.nf_r;
    a.offB = p.gB.off;
    a.GB = p.gB.G;
    a.per = (n + p.ctas - 1) / p.ctas;
    a.partA = (double*)w.partA;
    a.partB = (double*)w.partB;
    a.carryA = w.carryA;
    a.carryB = w.carryB;
    a.d_status = d_status;
    if (mu && r) launch_es<XT, true, true>(p, X, Y, a, s);
    else if (mu) launch_es<XT, true, false>(p, X, Y, a, s);
    else launch_es<XT, false, true>(p, X, Y, a, s);
  }
  FK_CUDA_TRY(cudaGetLastError());
  return FK_OK;
}

}  // namespace

size_t type1_ws_bytes(const Plan1& p, bool need_mu, bool need_r) {
  Bump b(nullptr, 0);
  Ws1 w;
  if (layout1(p, need_mu, need_r, b, w) != FK_OK) return 0;
  return b.used + 256;
}

fk_status type1_run(const Plan1& p, const fk_points& X, const void* Y, double L, const Type1Out& out, void* ws, size_t ws_bytes,
                    int* d_status, cudaStream_t s) {
  const bool mu = out.mu != nullptr, r = out.r != nullptr;
  Bump b(ws, ws_bytes);
  Ws1 w;
  FK_TRY(layout1(p, mu, r, b, w));
  if (!b.ok()) return fail(FK_E_WORKSPACE, "workspace too small: need " + std::to_string(b.used + 256) + " bytes");
  // zero what is accumulated globally
  if (!p.fp64 || p.smem) {
    if (mu) FK_CUDA_TRY(cudaMemsetAsync(w.carryA, 0, (size_t)p.gA.G * 8, s));
    if (r) FK_CUDA_TRY(cudaMemsetAsync(w.carryB, 0, (size_t)p.gB.G * 8, s));
  }
  if (p.fp64 && !p.smem) {
    if (mu) FK_CUDA_TRY(cudaMemsetAsync(w.partA, 0, (size_t)p.gA.G * 8, s));
    if (r) FK_CUDA_TRY(cudaMemsetAsync(w.partB, 0, (size_t)p.gB.G * 8, s));
  }
  if (X.n > 0) {
    if (X.dtype == FK_F32) FK_TRY(spread_dispatch<float>(p, X, Y, L, mu, r, w, d_status, s));
    else FK_TRY(spread_dispatch<double>(p, X, Y, L, mu, r, w, d_status, s));
  } else if (!p.fp64 || p.smem) {
    // no samples: partials are all zero
    const size_t esz = p.fp64 ? 8 : 4;
    if (mu) FK_CUDA_TRY(cudaMemsetAsync(w.partA, 0, (size_t)p.ctas * p.gA.G * esz, s));
    if (r) FK_CUDA_TRY(cudaMemsetAsync(w.partB, 0, (size_t)p.ctas * p.gB.G * esz, s));
    if (r && w.escale) FK_CUDA_TRY(cudaMemsetAsync(w.escale, 0, (size_t)p.ctas * 4, s));
  }
  // reduce the partials, pruned DFT at the needed modes, deconvolve: dft1d.cu (no cuFFT)
  if (mu && p.ker == KER_ES) FK_TRY(es_phihat_table(p.es, p.nf_mu, 2 * p.m, w.tabA, s));
  if (r && p.ker == KER_ES) FK_TRY(es_phihat_table(p.es, p.nf_r, p.m, w.tabB, s));
  Dft1Grid g[2];
  const int ng = dft_grids(p, mu, r, w, &out, g);
  FK_TRY(dft1d_run(g, ng, p.ker, out.accumulate ? 1 : 0, w.dftws, w.dft_bytes, s));
  return FK_OK;
}

}  // namespace fk
