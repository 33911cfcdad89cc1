// predict.cu -- prediction by the type-2 sum (additive :463-468):
//   f(x) = Re sum_{|k|<=m} theta_k exp(+i k t(x))
// Since only the real part is returned, theta is replaced by its Hermitian part
// h_k = (theta_k + conj theta_{-k}) / 2, so the fine grid
//   g_l = sum_k h_k (-1)^k / psi-hat(k/nf) exp(+2 pi i k l / nf)
// is real (hand-written inverse DFT evaluated only on the occupied cells: dft1d.cu for d = 1 /
// additive, dft2d.cu for d = 2; no cuFFT), and f(x) = sum_l g_l psi(u(x) - l) is a w-tap gather
// from the occupied half of the grid, held in shared memory (fp32 path: cubic B-spline, 4 taps,
// d = 2: ES window; fp64 path: septic B-spline or ES window).
// The gather streams Xq once and writes f once: 8 B per query in fp32 (HBM-bound).
#include <cmath>
#include <type_traits>

#include <cstdlib>

#include "fk_internal.cuh"
#include "window.cuh"

namespace fk {
namespace {

struct PredPlan {
  int d, m, nfeat;
  bool additive;
  KerKind ker;
  bool fp64;
  EsParams es;
  int nf;
  Geo g;
  size_t smem;
  bool in_smem;
};

static double bs3_sigma_p(double eps) { return std::max(4.0, 0.5 * (std::pow(1.0 / eps, 0.25) + 1.0)); }

static fk_status make_pred_plan(int d, int m, double eps, int additive, PredPlan* p) {
  PredPlan q{};
  q.d = d;
  q.m = m;
  q.additive = additive != 0;
  q.nfeat = q.additive ? d : 1;
  if (!q.additive && d > 2) return fail(FK_E_UNSUPPORTED, "fk_predict_type2: d <= 2 (or additive) in this build");
  q.fp64 = eps < 1e-7;
  int smem_cap = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_cap, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (!q.additive && d == 2) {  // 2-D: ES window on a sigma = 2 grid (the B-spline grid would be ~8x larger per dim)
    q.ker = KER_ES;
    int w = (int)std::ceil(std::log10(1.0 / eps)) + (q.fp64 ? 2 : 1);
    w = std::min(16, std::max(4, w));
    q.es.w = w;
    q.es.beta = 2.30 * w;
    q.nf = fft_friendly(std::max(2 * (2 * m + 1), 2 * w + 8));  // grid must not wrap (small m)
    q.g = {q.nf, q.nf / 4 - w / 2 - 2, q.nf / 2 + w + 4};
    q.smem = (size_t)q.g.G * q.g.G * (q.fp64 ? 8 : 4);
  } else if (!q.fp64) {
    q.ker = KER_BS3;
    q.nf = fft_friendly((int)std::ceil(bs3_sigma_p(eps) * (2 * m + 1)));
    q.g = {q.nf, q.nf / 4 - 1, q.nf / 2 + 4};
    q.smem = (size_t)q.nfeat * q.g.G * 4;
  } else {
    // fp64: septic B-spline (8 taps, Cox-de Boor weights, sinc^8 transform) when its grids fit in
    // shared memory, as in the type-1 fp64 mode; else the ES window
    const double s7 = std::max(4.0, 0.5 * (std::pow(4.0 / std::max(eps, 1e-300), 0.125) + 1.0));
    const int nf7 = fft_friendly((int)std::ceil(s7 * (2 * m + 1)));
    const size_t b7 = (size_t)q.nfeat * (nf7 / 2 + 8) * 8;
    if (eps >= 1e-13 && b7 <= (size_t)smem_cap) {
      q.ker = KER_BS7;
      q.nf = nf7;
      q.g = {q.nf, q.nf / 4 - 3, q.nf / 2 + 8};
      q.smem = b7;
    } else {
      q.ker = KER_ES;
      int w = (int)std::ceil(std::log10(1.0 / eps)) + 2;
      w = std::min(16, std::max(4, w));
      q.es.w = w;
      q.es.beta = 2.30 * w;
      q.nf = fft_friendly(std::max(2 * (2 * m + 1), 2 * w + 8));  // grid must not wrap (small m)
      q.g = {q.nf, q.nf / 4 - w / 2 - 2, q.nf / 2 + w + 4};
      q.smem = (size_t)q.nfeat * q.g.G * 8;
    }
  }
  q.in_smem = q.smem <= (size_t)smem_cap;
  if (!q.in_smem) q.smem = 0;
  *p = q;
  return FK_OK;
}

__global__ void k_pred_prep(const double2* __restrict__ theta, int nfeat, int m, int nf, int ker, const double* __restrict__ tab,
                            double2* __restrict__ H) {
  const int half = nf / 2 + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)nfeat * half) return;
  const int f = (int)(t / half), k = (int)(t % half);
  double2 h = make_double2(0.0, 0.0);
  if (k <= m) {
    const double2 a = theta[(int64_t)f * (2 * m + 1) + m + k];
    const double2 b = theta[(int64_t)f * (2 * m + 1) + m - k];
    double ph;
    if (ker == KER_BS3 || ker == KER_BS7) {
      const double s = sinc_pi((double)k / nf);
      ph = (s * s) * (s * s);
      if (ker == KER_BS7) ph *= ph;
    } else {
      ph = tab[k];
    }
    const double sc = 0.5 * ((k & 1) ? -1.0 : 1.0) / ph;
    h = make_double2((a.x + b.x) * sc, (a.y - b.y) * sc);
    if (k == 0) h.y = 0.0;
  }
  H[t] = h;
}

template <typename XT, bool EXACT>
__global__ void __launch_bounds__(512) k_gather_bs3(const XT* __restrict__ Xq, int64_t n, int nfeat, int64_t sn, int64_t sd,
                                                   const double* __restrict__ grid, int nf, int off, int G, float a_hi,
                                                   float a_lo, double a_d, int in_smem, XT* __restrict__ out,
                                                   int* __restrict__ d_status) {
  extern __shared__ float sg[];
  const float* gs = sg;
  if (in_smem) {
    for (int64_t i = threadIdx.x; i < (int64_t)nfeat * G; i += blockDim.x) {
      const int f = (int)(i / G), c = (int)(i % G);
      sg[i] = (float)grid[(int64_t)f * nf + off + c];
    }
    __syncthreads();
  }
  const int nq = nf / 4;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    bool ok = true;
    for (int f = 0; f < nfeat; ++f) {
      int t;
      float fr;
      if (sizeof(XT) == 8) {
        const double p = (double)Xq[j * sn + f * sd] * a_d;
        const double fl = floor(p);
        fr = (float)(p - fl);
        t = (p == p && fabs(p) < 1e9) ? (int)fl + nq : -1;
        if (fr >= 1.0f) { fr = 0.0f; t += 1; }
      } else {
        pos1_f32<EXACT>((float)Xq[j * sn + f * sd], a_hi, a_lo, nq, t, fr);
      }
      if ((unsigned)t > (unsigned)(G - 4)) {
        ok = false;
        continue;
      }
      float w[4];
      bs3_float(fr, w);
      if (in_smem) {
        const float* c = gs + (int64_t)f * G + t;
        acc += w[0] * c[0] + w[1] * c[1] + w[2] * c[2] + w[3] * c[3];
      } else {
        const double* c = grid + (int64_t)f * nf + off + t;
        acc += w[0] * (float)c[0] + w[1] * (float)c[1] + w[2] * (float)c[2] + w[3] * (float)c[3];
      }
    }
    if (!ok) bad = true;
    out[j] = ok ? (XT)acc : (XT)NAN;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// fp32, any layout (additive: nfeat grids), grids in shared memory as overlapping float2 pairs
// (2 LDS.64 per feature instead of 4 LDS.32), 1024-thread CTAs
template <bool EXACT>
__global__ void __launch_bounds__(1024) k_gather_bs3_pairs(const float* __restrict__ Xq, int64_t n, int nfeat, int64_t sn, int64_t sd,
                                                         const double* __restrict__ grid, int nf, int off, int G, float a_hi,
                                                         float a_lo, float* __restrict__ out, int* __restrict__ d_status) {
  extern __shared__ float2 sgq[];
  for (int64_t i = threadIdx.x; i < (int64_t)nfeat * G; i += blockDim.x) {
    const int f = (int)(i / G), c = (int)(i % G);
    const double* gf = grid + (int64_t)f * nf + off;
    sgq[i] = make_float2((float)gf[c], c + 1 < G ? (float)gf[c + 1] : 0.0f);
  }
  __syncthreads();
  const int nq = nf / 4;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.0f;
    bool ok = true;
    for (int f = 0; f < nfeat; ++f) {
      int t;
      float fr;
      pos1_f32<EXACT>(Xq[j * sn + f * sd], a_hi, a_lo, nq, t, fr);
      if ((unsigned)t > (unsigned)(G - 4)) {
        ok = false;
        continue;
      }
      float w[4];
      bs3_float(fr, w);
      const float2* c = sgq + (int64_t)f * G + t;
      const float2 lo = c[0], hi = c[2];
      acc += w[0] * lo.x + w[1] * lo.y + w[2] * hi.x + w[3] * hi.y;
    }
    if (!ok) bad = true;
    out[j] = ok ? acc : NAN;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// d = 1, fp32, contiguous 16-byte-aligned Xq / out, grid in smem: 4 queries per thread per step,
// 128-bit streaming loads and stores (the scalar kernel above handles every other case)
template <bool EXACT>
__global__ void __launch_bounds__(512) k_gather_bs3_vec(const float4* __restrict__ Xq4, int64_t n4, const double* __restrict__ grid,
                                                       int nf, int off, int G, float a_hi, float a_lo, float4* __restrict__ out4,
                                                       int* __restrict__ d_status) {
  extern __shared__ float sgv[];
  for (int i = threadIdx.x; i < G; i += blockDim.x) sgv[i] = (float)grid[off + i];
  __syncthreads();
  const int nq = nf / 4;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
    const float4 xv = __ldcs(Xq4 + j);
    const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
    float r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int t;
      float fr;
      pos1_f32<EXACT>(xs[q], a_hi, a_lo, nq, t, fr);
      const bool ok = (unsigned)t <= (unsigned)(G - 4);
      bad |= !ok;
      t = ok ? t : 0;
      float w[4];
      bs3_float(fr, w);
      const float* c = sgv + t;
      r[q] = ok ? (w[0] * c[0] + w[1] * c[1] + w[2] * c[2] + w[3] * c[3]) : NAN;
    }
    __stcs(out4 + j, make_float4(r[0], r[1], r[2], r[3]));
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// Same with the grid held as overlapping pairs P[i] = (g[i], g[i+1]) (8 B per cell): the 4 taps
// of a query are 2 LDS.64 instead of 4 LDS.32, half the shared-memory wavefronts per query
// under random addresses (the gather is bound by them, not by HBM, with the 4-byte layout).
template <bool EXACT>
__global__ void __launch_bounds__(1024) k_gather_bs3_pair(const float4* __restrict__ Xq4, int64_t n4, const double* __restrict__ grid,
                                                        int nf, int off, int G, float a_hi, float a_lo, float4* __restrict__ out4,
                                                        int* __restrict__ d_status) {
  extern __shared__ float2 sgp[];
  for (int i = threadIdx.x; i < G; i += blockDim.x)
    sgp[i] = make_float2((float)grid[off + i], i + 1 < G ? (float)grid[off + i + 1] : 0.0f);
  __syncthreads();
  const int nq = nf / 4;
  bool bad = false;
  auto one = [&](float x) {
    int t;
    float fr;
    pos1_f32<EXACT>(x, a_hi, a_lo, nq, t, fr);
    const bool ok = (unsigned)t <= (unsigned)(G - 4);
    bad |= !ok;
    t = ok ? t : 0;
    float w[4];
    bs3_float(fr, w);
    const float2 lo = sgp[t], hi = sgp[t + 2];
    return ok ? (w[0] * lo.x + w[1] * lo.y + w[2] * hi.x + w[3] * hi.y) : NAN;
  };
  // U float4 per thread per step (4U queries in flight)
  constexpr int U = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; j + (U - 1) * stride < n4; j += U * stride) {
    float4 xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = __ldcs(Xq4 + j + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out4 + j + u * stride, make_float4(one(xv[u].x), one(xv[u].y), one(xv[u].z), one(xv[u].w)));
  }
  for (; j < n4; j += stride) {
    const float4 xa = __ldcs(Xq4 + j);
    __stcs(out4 + j, make_float4(one(xa.x), one(xa.y), one(xa.z), one(xa.w)));
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// fp64 gather with the septic B-spline (d = 1 or additive, grids in shared memory)
__device__ __forceinline__ void bs7_w(double f, double* N) {
  N[0] = 1.0;
#pragma unroll
  for (int j = 1; j <= 7; ++j) {
    const double invj = 1.0 / j;
    double saved = 0.0;
#pragma unroll
    for (int r = 0; r < j; ++r) {
      const double temp = N[r] * invj;
      N[r] = fma((double)(r + 1) - f, temp, saved);
      saved = ((double)(j - r - 1) + f) * temp;
    }
    N[j] = saved;
  }
}

template <typename XT>
__global__ void __launch_bounds__(512) k_gather_bs7(const XT* __restrict__ Xq, int64_t n, int nfeat, int64_t sn, int64_t sd,
                                                   const double* __restrict__ grid, int nf, int off, int G, double a,
                                                   XT* __restrict__ out, int* __restrict__ d_status) {
  extern __shared__ double sg7[];
  for (int64_t i = threadIdx.x; i < (int64_t)nfeat * G; i += blockDim.x) {
    const int f = (int)(i / G), c = (int)(i % G);
    sg7[i] = grid[(int64_t)f * nf + off + c];
  }
  __syncthreads();
  const int nq = nf / 4;
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    bool ok = true;
    for (int f = 0; f < nfeat; ++f) {
      const double p = (double)Xq[j * sn + f * sd] * a;
      const double fl = floor(p);
      const int t0 = (p == p && fabs(p) < 1e9) ? (int)fl + nq : -1;
      if ((unsigned)t0 > (unsigned)(G - 8)) {
        ok = false;
        continue;
      }
      double w[8];
      bs7_w(p - fl, w);
      const double* c = sg7 + (int64_t)f * G + t0;
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fma(w[i], c[i], acc);
    }
    bad |= !ok;
    out[j] = ok ? (XT)acc : (XT)NAN;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// fp64 gather, d = 1 or additive, grid in shared memory: compile-time width, taps as polynomials
// from a constant-memory table (es_horner_table) instead of exp + sqrt per tap
__constant__ double c_pred_coef[kHornerSlots][kHornerSlot];  // slot W (horner_slot)

template <typename XT, int W>
__global__ void __launch_bounds__(512) k_gather_es_h(const XT* __restrict__ Xq, int64_t n, int nfeat, int64_t sn, int64_t sd,
                                                    const double* __restrict__ grid, int nf, int off, int G, double a,
                                                    XT* __restrict__ out, int* __restrict__ d_status) {
  constexpr int NP = W + 3;
  extern __shared__ double sgh[];
  for (int64_t i = threadIdx.x; i < (int64_t)nfeat * G; i += blockDim.x) {
    const int f = (int)(i / G), c = (int)(i % G);
    sgh[i] = grid[(int64_t)f * nf + off + c];
  }
  __syncthreads();
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    bool ok = true;
    for (int f = 0; f < nfeat; ++f) {
      const double ul = (double)Xq[j * sn + f * sd] * a + 0.5 * nf - off;
      const int l0 = (int)ceil(ul - 0.5 * W);
      if (!(ul == ul) || l0 < 0 || l0 + W > G) {
        ok = false;
        continue;
      }
      const double sv = 2.0 * (ul - l0 - 0.5 * W + 1.0) - 1.0;
      const double* c = sgh + (int64_t)f * G + l0;
#pragma unroll
      for (int i = 0; i < W; ++i) {
        double psi = c_pred_coef[W][i * NP + NP - 1];
#pragma unroll
        for (int q = NP - 2; q >= 0; --q) psi = fma(psi, sv, c_pred_coef[W][i * NP + q]);
        acc = fma(psi, c[i], acc);
      }
    }
    bad |= !ok;
    out[j] = ok ? (XT)acc : (XT)NAN;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

template <typename XT>
__global__ void __launch_bounds__(512) k_gather_es(const XT* __restrict__ Xq, int64_t n, int nfeat, int64_t sn, int64_t sd,
                                                  const double* __restrict__ grid, int nf, int off, int G, double a, int w,
                                                  double beta, int in_smem, XT* __restrict__ out, int* __restrict__ d_status) {
  extern __shared__ double sgd[];
  if (in_smem) {
    for (int64_t i = threadIdx.x; i < (int64_t)nfeat * G; i += blockDim.x) {
      const int f = (int)(i / G), c = (int)(i % G);
      sgd[i] = grid[(int64_t)f * nf + off + c];
    }
    __syncthreads();
  }
  bool bad = false;
  const double inv = 2.0 / w;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    bool ok = true;
    for (int f = 0; f < nfeat; ++f) {
      const double ul = (double)Xq[j * sn + f * sd] * a + 0.5 * nf - off;
      const int l0 = (int)ceil(ul - 0.5 * w);
      if (!(ul == ul) || l0 < 0 || l0 + w > G) {
        ok = false;
        continue;
      }
      const double* c = in_smem ? sgd + (int64_t)f * G : grid + (int64_t)f * nf + off;
      for (int i = 0; i < w; ++i) {
        const double z = ((double)(l0 + i) - ul) * inv;
        const double v = 1.0 - z * z;
        if (v > 0.0) acc += exp(beta * (sqrt(v) - 1.0)) * c[l0 + i];
      }
    }
    if (!ok) bad = true;
    out[j] = ok ? (XT)acc : (XT)NAN;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

// ---- d = 2: Hc[(k0 + m)(m + 1) + k1] = c_k1 (-1)^(k0+k1) (theta_k + conj theta_-k) / 2 / (psi-hat psi-hat),
// |k0| <= m, 0 <= k1 <= m, c_0 = 1, c_k1>0 = 2: the half spectrum idft2d_run turns into the grid ----
__global__ void k_pred_prep2d(const double2* __restrict__ theta, int m, const double* __restrict__ tab, double2* __restrict__ H) {
  const int side = 2 * m + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)side * (m + 1)) return;
  const int k0 = (int)(t / (m + 1)) - m, k1 = (int)(t % (m + 1));
  const double2 a = theta[(int64_t)(k0 + m) * side + (k1 + m)];
  const double2 b = theta[(int64_t)(-k0 + m) * side + (-k1 + m)];
  const double sc = (k1 > 0 ? 1.0 : 0.5) * (((k0 + k1) & 1) ? -1.0 : 1.0) / (tab[k0 < 0 ? -k0 : k0] * tab[k1]);
  H[t] = make_double2((a.x + b.x) * sc, (a.y - b.y) * sc);
}

template <typename GT>
__device__ __forceinline__ GT es_eval(double beta, GT v);
template <>
__device__ __forceinline__ float es_eval<float>(double beta, float v) { return __expf((float)beta * (sqrtf(v) - 1.0f)); }
template <>
__device__ __forceinline__ double es_eval<double>(double beta, double v) { return exp(beta * (sqrt(v) - 1.0)); }

// one coordinate on an ES grid: first tap (local index) and the offset f of the point
__device__ __forceinline__ void es_place(double x, double a, int K, int w, int& l0, double& f) {
  const double p = x * a;
  const double P = floor(p);
  f = p - P;
  const int d0 = (w & 1) ? (f > 0.5 ? 1 : 0) - (w >> 1) : (f > 0.0 ? 1 : 0) - (w >> 1);
  l0 = (fabs(p) < 1e8) ? (int)P + K + d0 : -1000000;
  f = f - d0;  // tap i sits at offset (i - f) cells
}

template <typename XT, typename GT, int W>
__global__ void __launch_bounds__(1024) k_gather2d(const XT* __restrict__ Xq, int64_t n, int64_t sn, int64_t sd,
                                                 const double* __restrict__ grid, int nf, int off, int G, int K, double a, int w_unused,
                                                 double beta, int in_smem, XT* __restrict__ out, int* __restrict__ d_status) {
  constexpr int w = W;
  extern __shared__ unsigned char sgraw[];
  GT* sg = reinterpret_cast<GT*>(sgraw);
  if (in_smem) {
    for (int64_t i = threadIdx.x; i < (int64_t)G * G; i += blockDim.x) {
      const int r = (int)(i / G), c = (int)(i % G);
      sg[i] = (GT)grid[(int64_t)(off + r) * nf + off + c];
    }
    __syncthreads();
  }
  bool bad = false;
  const GT inv = (GT)2.0 / (GT)w;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    int l0, l1;
    double f0, f1;
    es_place((double)Xq[j * sn], a, K, w, l0, f0);
    es_place((double)Xq[j * sn + sd], a, K, w, l1, f1);
    if (l0 < 0 || l1 < 0 || l0 + w > G || l1 + w > G) {
      bad = true;
      out[j] = (XT)NAN;
      continue;
    }
    GT px[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const GT z = ((GT)i - (GT)f1) * inv;
      const GT v = (GT)1 - z * z;
      px[i] = v > (GT)0 ? es_eval<GT>(beta, v) : (GT)0;
    }
    GT acc = 0;
#pragma unroll
    for (int r = 0; r < W; ++r) {
      const GT z = ((GT)r - (GT)f0) * inv;
      const GT v = (GT)1 - z * z;
      const GT wy = v > (GT)0 ? es_eval<GT>(beta, v) : (GT)0;
      GT racc = 0;
      if (in_smem) {
        const GT* row = sg + (int64_t)(l0 + r) * G + l1;
#pragma unroll
        for (int c = 0; c < W; ++c) racc += px[c] * row[c];
      } else {
        const double* row = grid + (int64_t)(off + l0 + r) * nf + off + l1;
#pragma unroll
        for (int c = 0; c < W; ++c) racc += px[c] * (GT)row[c];
      }
      acc += wy * racc;
    }
    out[j] = (XT)acc;
  }
  if (bad && d_status) atomicOr(d_status, (int)FK_E_RANGE);
}

struct PredWs {
  double2* H;
  double* grid;
  double* tab;
  void* work;
  size_t work_bytes;
};

static bool is2d(const PredPlan& p) { return !p.additive && p.d == 2; }

static fk_status pred_layout(const PredPlan& p, Bump& b, PredWs& w) {
  FftPlan fp;
  if (is2d(p)) {  // d = 2: the hand-written 2-D inverse DFT (dft2d.cu) fills the occupied block
    fp.work = idft2d_ws_bytes(p.nf, p.g.G, p.m);
    w.H = (double2*)b.take((size_t)(2 * p.m + 1) * (p.m + 1) * 16);
    w.grid = (double*)b.take((size_t)p.nf * p.nf * 8);
  } else {  // d = 1 / additive: the hand-written inverse DFT (dft1d.cu) fills the occupied cells
    fp.work = idft1d_ws_bytes(p.nf, p.m, p.nfeat);
    if (fp.work == 0) return fail(FK_E_UNSUPPORTED, "fk_predict_type2: no DFT factorisation of the fine grid");
    w.H = (double2*)b.take((size_t)p.nfeat * (p.nf / 2 + 1) * 16);
    w.grid = (double*)b.take((size_t)p.nfeat * p.nf * 8);
  }
  w.tab = (double*)b.take((size_t)(p.m + 1) * 8);
  w.work = b.take(std::max<size_t>(fp.work, 256));
  w.work_bytes = std::max<size_t>(fp.work, 256);
  return FK_OK;
}

template <typename XT>
static fk_status gather2d(const PredPlan& p, const fk_points& Xq, double L, const PredWs& w, void* out, int* d_status, cudaStream_t s) {
  const int sms = device_sm_count();
  const double a = (double)p.nf / (4.0 * L);
  const int K = p.nf / 2 - p.g.off;
  // 1024-thread CTAs, as many per SM as the grid copy allows (2 at m = 64): the gather is bound by
  // the latency of its w^2 random shared-memory loads, so occupancy is what matters (256-thread
  // CTAs left 16 warps per SM: 3.4e10 queries/s at C3's m)
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  const int per_sm = p.smem ? std::max(1, std::min(2, (int)(optin / (p.smem + 1024)))) : 2;
  auto go = [&](auto k) {
    if (p.smem) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    k<<<sms * per_sm, 1024, p.smem, s>>>((const XT*)Xq.ptr, Xq.n, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off, p.g.G, K, a,
                                         p.es.w, p.es.beta, p.in_smem ? 1 : 0, (XT*)out, d_status);
  };
  auto byw = [&](auto wtag) {
    constexpr int WW = decltype(wtag)::value;
    if (p.fp64) go(k_gather2d<XT, double, WW>);
    else go(k_gather2d<XT, float, WW>);
  };
  switch (p.es.w) {
    case 4: byw(std::integral_constant<int, 4>{}); break;
    case 5: byw(std::integral_constant<int, 5>{}); break;
    case 6: byw(std::integral_constant<int, 6>{}); break;
    case 7: byw(std::integral_constant<int, 7>{}); break;
    case 8: byw(std::integral_constant<int, 8>{}); break;
    case 9: byw(std::integral_constant<int, 9>{}); break;
    case 10: byw(std::integral_constant<int, 10>{}); break;
    case 11: byw(std::integral_constant<int, 11>{}); break;
    case 12: byw(std::integral_constant<int, 12>{}); break;
    case 13: byw(std::integral_constant<int, 13>{}); break;
    case 14: byw(std::integral_constant<int, 14>{}); break;
    case 15: byw(std::integral_constant<int, 15>{}); break;
    default: byw(std::integral_constant<int, 16>{}); break;
  }
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  return FK_OK;
}

template <typename XT>
static fk_status gather(const PredPlan& p, const fk_points& Xq, double L, const PredWs& w, void* out, int* d_status, cudaStream_t s) {
  const int sms = device_sm_count();
  const double a = (double)p.nf / (4.0 * L);
  if (p.ker == KER_BS3) {
    const float a_hi = (float)a, a_lo = (float)(a - (double)a_hi);
    int ex = 0;
    const bool exact = std::frexp(a, &ex) == 0.5;
    const int per_sm = p.smem ? std::max(1, std::min(4, (int)(200000 / (p.smem + 1024)))) : 4;
    const bool vec = sizeof(XT) == 4 && p.nfeat == 1 && p.in_smem && Xq.stride_n == 1 && ((uintptr_t)Xq.ptr % 16 == 0) &&
                     ((uintptr_t)out % 16 == 0) && Xq.n >= 4;
    if (vec) {
      const int64_t n4 = Xq.n / 4;
      const size_t pair_smem = (size_t)p.g.G * 8;
      int optin = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      // pair layout + 16 queries in flight per thread: 5.08e11 -> 6.06e11 queries/s at m = 1000
      // (0.62 -> 0.74 of the measured copy bandwidth, bench_rows predict)
      bool pair = pair_smem <= (size_t)optin;
      if (const char* e = getenv("FK_PRED_PAIR")) pair = pair && e[0] == '1';  // experiments
      if (pair) {
        auto kv = exact ? k_gather_bs3_pair<true> : k_gather_bs3_pair<false>;
        cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair_smem);
        const int ps = std::max(1, std::min(2, (int)(optin / (pair_smem + 1024))));
        kv<<<sms * ps, 1024, pair_smem, s>>>((const float4*)Xq.ptr, n4, w.grid, p.nf, p.g.off, p.g.G, a_hi, a_lo, (float4*)out,
                                             d_status);
      } else {
        auto kv = exact ? k_gather_bs3_vec<true> : k_gather_bs3_vec<false>;
        cudaFuncSetAttribute(kv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        kv<<<sms * per_sm, 512, p.smem, s>>>((const float4*)Xq.ptr, n4, w.grid, p.nf, p.g.off, p.g.G, a_hi, a_lo, (float4*)out,
                                             d_status);
      }
      FK_CUDA_TRY(cudaGetLastError());
      count_launch();
      if (n4 * 4 == Xq.n) return FK_OK;
      // tail (< 4 queries) through the scalar kernel
      fk_points tail = Xq;
      tail.ptr = (const float*)Xq.ptr + n4 * 4;
      tail.n = Xq.n - n4 * 4;
      auto ks = exact ? k_gather_bs3<float, true> : k_gather_bs3<float, false>;
      cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      ks<<<1, 512, p.smem, s>>>((const float*)tail.ptr, tail.n, 1, 1, 1, w.grid, p.nf, p.g.off, p.g.G, a_hi, a_lo, a, 1,
                                (float*)out + n4 * 4, d_status);
      FK_CUDA_TRY(cudaGetLastError());
      count_launch();
      return FK_OK;
    }
    if (sizeof(XT) == 4 && p.in_smem) {
      const size_t pair_smem = (size_t)p.nfeat * p.g.G * 8;
      int optin = 0, dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
      if (pair_smem <= (size_t)optin) {
        auto kp = exact ? k_gather_bs3_pairs<true> : k_gather_bs3_pairs<false>;
        cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pair_smem);
        const int ps = std::max(1, std::min(2, (int)(optin / (pair_smem + 1024))));
        kp<<<sms * ps, 1024, pair_smem, s>>>((const float*)Xq.ptr, Xq.n, p.nfeat, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off,
                                             p.g.G, a_hi, a_lo, (float*)out, d_status);
        FK_CUDA_TRY(cudaGetLastError());
        count_launch();
        return FK_OK;
      }
    }
    auto k = exact ? k_gather_bs3<XT, true> : k_gather_bs3<XT, false>;
    if (p.smem) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    k<<<sms * per_sm, 512, p.smem, s>>>((const XT*)Xq.ptr, Xq.n, p.nfeat, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off, p.g.G,
                                        a_hi, a_lo, a, p.in_smem ? 1 : 0, (XT*)out, d_status);
  } else if (p.ker == KER_BS7) {
    auto k = k_gather_bs7<XT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    const int per_sm = std::max(1, std::min(4, (int)(200000 / (p.smem + 1024))));
    k<<<sms * per_sm, 512, p.smem, s>>>((const XT*)Xq.ptr, Xq.n, p.nfeat, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off, p.g.G, a,
                                        (XT*)out, d_status);
  } else {
    if (p.in_smem && p.es.w >= 9 && p.es.w <= 14 && horner_slot(c_pred_coef, p.es.w, p.es.beta) == FK_OK) {
      const int per_sm = std::max(1, std::min(4, (int)(200000 / (p.smem + 1024))));
      auto go = [&](auto wtag) {
        constexpr int WW = decltype(wtag)::value;
        auto k = k_gather_es_h<XT, WW>;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        k<<<sms * per_sm, 512, p.smem, s>>>((const XT*)Xq.ptr, Xq.n, p.nfeat, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off, p.g.G, a,
                                            (XT*)out, d_status);
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
      FK_CUDA_TRY(cudaGetLastError());
      count_launch();
      return FK_OK;
    }
    auto k = k_gather_es<XT>;
    if (p.smem) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
    const int per_sm = p.smem ? std::max(1, std::min(4, (int)(200000 / (p.smem + 1024)))) : 4;
    k<<<sms * per_sm, 512, p.smem, s>>>((const XT*)Xq.ptr, Xq.n, p.nfeat, Xq.stride_n, Xq.stride_d, w.grid, p.nf, p.g.off, p.g.G, a,
                                        p.es.w, p.es.beta, p.in_smem ? 1 : 0, (XT*)out, d_status);
  }
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  return FK_OK;
}

}  // namespace

size_t predict_ws_bytes(int d, int m, double eps, int additive) {
  PredPlan p;
  if (make_pred_plan(d, m, eps, additive, &p) != FK_OK) return 0;
  Bump b(nullptr, 0);
  PredWs w;
  if (pred_layout(p, b, w) != FK_OK) return 0;
  return b.used + 256;
}

fk_status predict_run(const double* theta, int d, int m, double L, int additive, const fk_points& Xq, double eps, void* out, void* ws,
                      size_t ws_bytes, int* d_status, cudaStream_t s) {
  PredPlan p;
  FK_TRY(make_pred_plan(d, m, eps, additive, &p));
  Bump b(ws, ws_bytes);
  PredWs w;
  FK_TRY(pred_layout(p, b, w));
  if (!b.ok()) return fail(FK_E_WORKSPACE, "fk_predict_type2: workspace too small");
  if (p.ker == KER_ES) FK_TRY(es_phihat_table(p.es, p.nf, p.m, w.tab, s));
  if (is2d(p)) {
    const int64_t tot2 = (int64_t)(2 * m + 1) * (m + 1);
    k_pred_prep2d<<<(unsigned)((tot2 + 255) / 256), 256, 0, s>>>((const double2*)theta, m, w.tab, w.H);
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
    FK_TRY(idft2d_run(w.H, m, p.nf, p.g.off, p.g.G, w.grid, p.nf, w.work, w.work_bytes, s));
    if (Xq.n == 0) return FK_OK;
    if (Xq.dtype == FK_F32) return gather2d<float>(p, Xq, L, w, out, d_status, s);
    return gather2d<double>(p, Xq, L, w, out, d_status, s);
  }
  const int64_t tot = (int64_t)p.nfeat * (p.nf / 2 + 1);
  k_pred_prep<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>((const double2*)theta, p.nfeat, m, p.nf, p.ker, w.tab, w.H);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  FK_TRY(idft1d_run(w.H, p.nf / 2 + 1, p.nfeat, p.nf, m, p.g.off, p.g.G, w.grid, p.nf, w.work, w.work_bytes, s));
  if (Xq.n == 0) return FK_OK;
  if (Xq.dtype == FK_F32) return gather<float>(p, Xq, L, w, out, d_status, s);
  return gather<double>(p, Xq, L, w, out, d_status, s);
}

}  // namespace fk
