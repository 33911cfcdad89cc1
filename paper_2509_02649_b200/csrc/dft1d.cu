// dft1d.cu -- the d = 1 type-1 pass after the spreading: CTA partial grids -> one fine grid ->
// the window-convolved grid's DFT at the needed modes only -> deconvolution (PAPER.md:203-220,
// sec. 2.3: the NUFFT's FFT step).  Hand-written, no cuFFT; three launches for BOTH grids of a
// pass (moments and rhs):
//
//   k_reduce_occ  per occupied fine cell, the sum over the CTA partials (moments: int64, exact and
//                 order-free; rhs: per-CTA power-of-two scales, fp64 in fixed CTA order) + the
//                 drained carries -> fp64 grid of the occupied cells only (G of nf cells)
//   k_dft_s1      pruned two-level DFT, stage 1: nf = N1 N2, l = l1 + N1 l2, q = q2 + N2 q1;
//                   T[q2][l1] = w_nf^(q2 l1) sum_l2 g[l1 + N1 l2] w_N2^(q2 l2)
//                 one CTA per (l1, grid), thread q2; only the l2 of occupied cells are summed
//                 (about half), twiddles exact from a per-CTA table (integer index arithmetic)
//   k_dft_s2      stage 2 + deconvolution: F_q = sum_l1 T[q mod N2][l1] w_N1^((q / N2) l1) for the
//                 K + 1 modes q = 0..K only (K = 2m moments, m rhs); one warp per q; then
//                 out_{+-q} = (-1)^q F_q / psi-hat(q / nf) (conjugate for -q: the grid is real)
//
// w_N = exp(-2 pi i / N).  A full FFT would produce nf/2 + 1 modes of which the fit needs K + 1
// (C2: 2001 of 32769 for the moments): the pruned DFT does (K+1) N1 + N1 N2 G/nf complex
// multiply-adds, ~10^7 at C2 -- microseconds -- and reads the fine grid once.
#include <cmath>

#include "fk_internal.cuh"

namespace fk {
namespace {

constexpr int kMaxN2 = 512;
constexpr int kMaxN1 = 8192;

__device__ __forceinline__ double2 tw(int a, int N) {  // w_N^a = exp(-2 pi i a / N), 0 <= a < N
  double s, c;
  sincospi(2.0 * (double)a / (double)N, &s, &c);
  return make_double2(c, -s);
}

struct RedArgs {
  const int* part_i[2];     // int32 fixed-point partials (fp32 path), or
  const double* part_d[2];  // fp64 partials (fp64 modes)
  const int* escale[2];     // per-CTA power-of-two exponents of an int32 grid (rhs), or null
  const double* carry[2];
  double inv_scale[2];      // value of one fixed-point unit when escale is null
  int G[2];
  int nparts[2];
  double* out[2];
};

// occupied cells of both grids.  A 256-thread block takes 32 consecutive cells; its 8 warps split the
// partials (warp k sums partials k, k + 8, ...), so 8x more loads are in flight than with one thread
// per cell, then warp 0 combines the 8 sums in fixed order.  Uniform-scale int32 grids sum in int64
// (exact, so order-free); per-CTA-scaled and fp64 partials in a fixed order (bitwise reproducible).
constexpr int kRedSplit = 8;  // warps per block, each a share of the partials

// V cells per thread (V = 4: int4 loads, needs G % 4 == 0 -- the fp32 path's grids -- so every
// partial row starts 16-byte aligned); block = 32 V consecutive cells x kRedSplit warps
template <int V>
__global__ void __launch_bounds__(256) k_reduce_occ(RedArgs a) {
  __shared__ double sd[kRedSplit][32 * V];
  __shared__ long long sl[kRedSplit][32 * V];
  const int ch = blockIdx.y;
  const int lane = threadIdx.x & 31, k = threadIdx.x >> 5;
  const int G = a.G[ch];
  const int i0 = blockIdx.x * 32 * V + lane * V;
  if (blockIdx.x * 32 * V >= G) return;
  const int64_t st = G;
  const int np = a.nparts[ch];
  const bool ok = i0 < G;
  const bool fixed = !a.part_d[ch] && !a.escale[ch];
  if (a.part_d[ch]) {  // fp64 partials (V == 1 only)
    const double* __restrict__ p = a.part_d[ch] + i0;
    double s = 0.0;
    if (ok)
#pragma unroll 4
      for (int c = k; c < np; c += kRedSplit) s += __ldcg(p + c * st);
    sd[k][lane] = s;
  } else {
    const int* __restrict__ p = a.part_i[ch] + i0;
    const int* __restrict__ e = a.escale[ch];
    long long si[V];
    double sf[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      si[v] = 0;
      sf[v] = 0.0;
    }
    if (ok) {
#pragma unroll 4
      for (int c = k; c < np; c += kRedSplit) {
        int x[V];
        if (V == 4) {
          const int4 q = __ldcg(reinterpret_cast<const int4*>(p + c * st));
          x[0] = q.x;
          x[V > 1 ? 1 : 0] = q.y;
          x[V > 2 ? 2 : 0] = q.z;
          x[V > 3 ? 3 : 0] = q.w;
        } else {
          x[0] = __ldcg(p + c * st);
        }
        if (e) {
          const double sc = pow2(-__ldg(e + c));
#pragma unroll
          for (int v = 0; v < V; ++v) sf[v] += (double)x[v] * sc;
        } else {
#pragma unroll
          for (int v = 0; v < V; ++v) si[v] += x[v];  // exact: at most nparts x 2^31 in magnitude
        }
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      sd[k][lane * V + v] = sf[v];
      sl[k][lane * V + v] = si[v];
    }
  }
  __syncthreads();
  if (k != 0 || !ok) return;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int i = i0 + v;
    if (i >= G) break;
    double val;
    if (fixed) {
      long long t = 0;
#pragma unroll
      for (int q = 0; q < kRedSplit; ++q) t += sl[q][lane * V + v];
      val = (double)t * a.inv_scale[ch];
    } else {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < kRedSplit; ++q) t += sd[q][lane * V + v];
      val = t;
    }
    if (a.carry[ch]) val += a.carry[ch][i];
    a.out[ch][i] = val;
  }
}

struct S1Args {
  const double* g[2];  // occupied cells: g[i] = cell off + i, i < G
  int nf[2], N1[2], N2[2], off[2], G[2], nq2[2];
  double2* T[2];       // [q2][l1], q2 < nq2
};

__global__ void __launch_bounds__(kMaxN2) k_dft_s1(S1Args a) {
  __shared__ double col[kMaxN2];
  __shared__ double2 tab[kMaxN2];
  const int ch = blockIdx.y;
  const int N1 = a.N1[ch], N2 = a.N2[ch], nf = a.nf[ch], off = a.off[ch], G = a.G[ch];
  const int l1 = blockIdx.x;
  if (l1 >= N1) return;
  // l2 range with occupied cells: off <= l1 + N1 l2 < off + G
  const int lo2 = max(0, (off - l1 + N1 - 1) / N1);
  const int hi2 = min(N2 - 1, (off + G - 1 - l1) / N1);
  for (int k = threadIdx.x; k < N2; k += blockDim.x) {
    tab[k] = tw(k, N2);
    const int i = l1 + N1 * k - off;
    col[k] = (i >= 0 && i < G) ? a.g[ch][i] : 0.0;
  }
  __syncthreads();
  for (int q2 = threadIdx.x; q2 < a.nq2[ch]; q2 += blockDim.x) {
    // four independent accumulation chains (l2 = lo2 + 4 j + u); chain u's twiddle starts exact from
    // the table and advances by the complex rotation w_N2^(4 q2) (a table lookup per term would hit
    // shared-memory bank conflicts at the index stride q2; ~N2/8 rotations per chain: ~1e-14)
    double re[4] = {0.0, 0.0, 0.0, 0.0}, im[4] = {0.0, 0.0, 0.0, 0.0};
    double2 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = tab[(q2 * (lo2 + u)) % N2];
    const double2 r4 = tab[(4 * q2) % N2];
    int l2 = lo2;
    for (; l2 + 3 <= hi2; l2 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double v = col[l2 + u];
        re[u] = fma(v, t[u].x, re[u]);
        im[u] = fma(v, t[u].y, im[u]);
        const double tx = t[u].x * r4.x - t[u].y * r4.y;
        t[u].y = fma(t[u].x, r4.y, t[u].y * r4.x);
        t[u].x = tx;
      }
    }
    for (int u = 0; l2 <= hi2; ++l2, ++u) {
      const double v = col[l2];
      re[u] = fma(v, t[u].x, re[u]);
      im[u] = fma(v, t[u].y, im[u]);
    }
    const double r0 = (re[0] + re[1]) + (re[2] + re[3]), i0 = (im[0] + im[1]) + (im[2] + im[3]);
    const double2 w = tw((q2 * l1) % nf, nf);
    a.T[ch][(int64_t)q2 * N1 + l1] = make_double2(r0 * w.x - i0 * w.y, r0 * w.y + i0 * w.x);
  }
}

struct S2Args {
  const double2* T[2];
  int nf[2], N1[2], N2[2], K[2];
  int ker;
  const double* tab[2];  // KER_ES: psi-hat(q / nf), q = 0..K
  double2* out[2];       // 2K + 1 modes, index K + q
  int acc;
};

// one warp per mode q >= 0 of grid blockIdx.y; lanes stride over l1; w_N1 table in shared memory
constexpr int kS2Tab = 2048;

__global__ void __launch_bounds__(256) k_dft_s2(S2Args a) {
  __shared__ double2 tab[kS2Tab];
  const int ch = blockIdx.y;
  const int K = a.K[ch];
  const int N1 = a.N1[ch], N2 = a.N2[ch], nf = a.nf[ch];
  if (blockIdx.x * 8 > K) return;
  const bool use_tab = N1 <= kS2Tab;
  if (use_tab)
    for (int k = threadIdx.x; k < N1; k += blockDim.x) tab[k] = tw(k, N1);
  __syncthreads();
  const int q = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (q > K) return;
  const int q2 = q % N2, q1 = q / N2;
  const double2* __restrict__ T = a.T[ch] + (int64_t)q2 * N1;
  double re = 0.0, im = 0.0;
  if (q1 == 0) {
    for (int l1 = lane; l1 < N1; l1 += 32) {
      const double2 t = T[l1];
      re += t.x;
      im += t.y;
    }
  } else {
    int idx = (q1 * lane) % N1;
    const int step = (q1 * 32) % N1;
    for (int l1 = lane; l1 < N1; l1 += 32) {
      const double2 t = T[l1];
      const double2 w = use_tab ? tab[idx] : tw(idx, N1);
      re = fma(t.x, w.x, fma(-t.y, w.y, re));
      im = fma(t.x, w.y, fma(t.y, w.x, im));
      idx += step;
      if (idx >= N1) idx -= N1;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane != 0) return;
  double ph;
  if (a.ker == KER_BS3) {
    const double s = sinc_pi((double)q / nf);
    ph = (s * s) * (s * s);
  } else if (a.ker == KER_BS7) {
    const double s = sinc_pi((double)q / nf);
    const double s2 = s * s, s4 = s2 * s2;
    ph = s4 * s4;
  } else {
    ph = a.tab[ch][q];
  }
  const double sc = ((q & 1) ? -1.0 : 1.0) / ph;
  const double2 v = make_double2(re * sc, im * sc);
  double2* o = a.out[ch];
  if (a.acc) {
    o[K + q].x += v.x;
    o[K + q].y += v.y;
    if (q > 0) {
      o[K - q].x += v.x;
      o[K - q].y -= v.y;
    }
  } else {
    o[K + q] = v;
    if (q > 0) o[K - q] = make_double2(v.x, -v.y);
  }
}

// ---- type-2 direction (predict): the occupied cells of the real fine grid from its half spectrum
// out[l] = H_0 + 2 Re sum_{k=1..m} H_k w^(-k l) (cuFFT Z2D semantics, H_0 real), l in [off, off+G),
// with the same factorisation (k = k2 + N2 k1, l = l1 + N1 l2; w^(-1) = exp(+2 pi i / nf)):
//   U[k2][l1] = w_nf^(-k2 l1) sum_k1 H'_(k2 + N2 k1) w_N1^(-k1 l1)      (H'_0 = H_0 / 2)
//   out[l1 + N1 l2] = 2 Re sum_k2 U[k2][l1] w_N2^(-k2 l2)
struct I1Args {
  const double2* H;  // nfeat half spectra, row stride hstride
  int64_t hstride;
  int nf, N1, N2, m, off, G, K2;  // K2 = min(N2, m + 1) k2 values carry a coefficient
  double2* U;        // [feat][k2][l1]
  double* out;       // [feat][nf] (only [off, off + G) written)
  int64_t ostride;
};

__global__ void __launch_bounds__(256) k_idft_s1(I1Args a) {
  const int f = blockIdx.y;
  const int l1 = blockIdx.x;
  const double2* __restrict__ H = a.H + f * a.hstride;
  for (int k2 = threadIdx.x; k2 < a.K2; k2 += blockDim.x) {
    double re = 0.0, im = 0.0;
    for (int k1 = 0, k = k2; k <= a.m; ++k1, k += a.N2) {
      double2 h = H[k];
      if (k == 0) h.x *= 0.5;
      const double2 t = tw((k1 * l1) % a.N1, a.N1);  // w^(+) -> conjugate below
      re += h.x * t.x + h.y * t.y;                   // h * conj(t)
      im += h.y * t.x - h.x * t.y;
    }
    const double2 w = tw((int)(((long long)k2 * l1) % a.nf), a.nf);
    a.U[((int64_t)f * a.K2 + k2) * a.N1 + l1] = make_double2(re * w.x + im * w.y, im * w.x - re * w.y);  // x conj(w)
  }
}

__global__ void __launch_bounds__(256) k_idft_s2(I1Args a) {
  __shared__ double2 tab[kMaxN2];
  __shared__ double2 ucol[kMaxN2];
  const int f = blockIdx.y;
  const int l1 = blockIdx.x;
  const int N1 = a.N1, N2 = a.N2;
  for (int k = threadIdx.x; k < N2; k += blockDim.x) {
    const double2 t = tw(k, N2);
    tab[k] = make_double2(t.x, -t.y);  // w_N2^(-k)
    ucol[k] = k < a.K2 ? a.U[((int64_t)f * a.K2 + k) * N1 + l1] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int lo2 = max(0, (a.off - l1 + N1 - 1) / N1);
  const int hi2 = min(N2 - 1, (a.off + a.G - 1 - l1) / N1);
  for (int l2 = lo2 + threadIdx.x; l2 <= hi2; l2 += blockDim.x) {
    // four chains over k2 = 4 j + u, twiddles w_N2^(-k2 l2) advanced by rotation (exact start)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    double2 t[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) t[u] = tab[(u * l2) % N2];
    const double2 r4 = tab[(4 * l2) % N2];
    int k2 = 0;
    for (; k2 + 3 < a.K2; k2 += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double2 c = ucol[k2 + u];
        acc[u] += c.x * t[u].x - c.y * t[u].y;  // Re(c t)
        const double tx = t[u].x * r4.x - t[u].y * r4.y;
        t[u].y = fma(t[u].x, r4.y, t[u].y * r4.x);
        t[u].x = tx;
      }
    }
    for (int u = 0; k2 < a.K2; ++k2, ++u) {
      const double2 c = ucol[k2];
      acc[u] += c.x * t[u].x - c.y * t[u].y;
    }
    a.out[f * a.ostride + l1 + (int64_t)N1 * l2] = 2.0 * ((acc[0] + acc[1]) + (acc[2] + acc[3]));
  }
}

}  // namespace

// N2: the divisor of nf closest to sqrt(nf) with N2 <= 512 and nf / N2 <= 8192
fk_status dft1d_factor(int nf, int* N1, int* N2) {
  int best = 0;
  const double r = std::sqrt((double)nf);
  for (int d = 1; d <= kMaxN2 && d <= nf; ++d)
    if (nf % d == 0 && nf / d <= kMaxN1 && (best == 0 || std::fabs(std::log(d / r)) < std::fabs(std::log(best / r)))) best = d;
  if (best == 0) return fail(FK_E_UNSUPPORTED, "dft1d: no N1 x N2 factorisation of nf = " + std::to_string(nf));
  *N2 = best;
  *N1 = nf / best;
  return FK_OK;
}

size_t dft1d_ws_bytes(const Dft1Grid* g, int ngrids) {
  Bump b(nullptr, 0);
  for (int k = 0; k < ngrids; ++k) {
    int N1 = 0, N2 = 0;
    if (dft1d_factor(g[k].nf, &N1, &N2) != FK_OK) return 0;
    b.take((size_t)g[k].G * 8);                        // occupied fine grid
    b.take((size_t)std::min(N2, g[k].K + 1) * N1 * 16);  // stage-1 output
  }
  return b.used + 256;
}

fk_status dft1d_run(const Dft1Grid* g, int ngrids, int ker, int acc, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (ngrids < 1 || ngrids > 2) return fail(FK_E_ARG, "dft1d: 1 or 2 grids");
  Bump b(ws, ws_bytes);
  RedArgs ra{};
  S1Args s1{};
  S2Args s2{};
  int maxG = 0, maxN1 = 0, maxK = 0, maxN2 = 0;
  for (int k = 0; k < ngrids; ++k) {
    int N1 = 0, N2 = 0;
    FK_TRY(dft1d_factor(g[k].nf, &N1, &N2));
    double* fine = (double*)b.take((size_t)g[k].G * 8);
    const int nq2 = std::min(N2, g[k].K + 1);
    double2* T = (double2*)b.take((size_t)nq2 * N1 * 16);
    ra.part_i[k] = g[k].part_i;
    ra.part_d[k] = g[k].part_d;
    ra.escale[k] = g[k].escale;
    ra.nparts[k] = g[k].nparts;
    ra.carry[k] = g[k].carry;
    ra.inv_scale[k] = g[k].inv_scale;
    ra.G[k] = g[k].G;
    ra.out[k] = fine;
    s1.g[k] = fine;
    s1.nf[k] = g[k].nf;
    s1.N1[k] = N1;
    s1.N2[k] = N2;
    s1.off[k] = g[k].off;
    s1.G[k] = g[k].G;
    s1.nq2[k] = nq2;
    s1.T[k] = T;
    s2.T[k] = T;
    s2.nf[k] = g[k].nf;
    s2.N1[k] = N1;
    s2.N2[k] = N2;
    s2.K[k] = g[k].K;
    s2.tab[k] = g[k].phihat;
    s2.out[k] = (double2*)g[k].out;
    maxG = std::max(maxG, g[k].G);
    maxN1 = std::max(maxN1, N1);
    maxN2 = std::max(maxN2, nq2);
    maxK = std::max(maxK, g[k].K);
  }
  if (!b.ok()) return fail(FK_E_WORKSPACE, "dft1d: workspace too small");
  s2.ker = ker;
  s2.acc = acc;
  bool vec4 = true;  // int32 partials with G % 4 == 0 in every grid
  for (int k = 0; k < ngrids; ++k) vec4 = vec4 && g[k].part_i && g[k].G % 4 == 0;
  if (vec4) k_reduce_occ<4><<<dim3((maxG + 127) / 128, ngrids), 256, 0, s>>>(ra);
  else k_reduce_occ<1><<<dim3((maxG + 31) / 32, ngrids), 256, 0, s>>>(ra);
  const int t1 = std::min(kMaxN2, (maxN2 + 31) / 32 * 32);
  k_dft_s1<<<dim3(maxN1, ngrids), t1, 0, s>>>(s1);
  k_dft_s2<<<dim3((maxK + 1 + 7) / 8, ngrids), 256, 0, s>>>(s2);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(3);
  return FK_OK;
}

}  // namespace fk

namespace fk {

size_t idft1d_ws_bytes(int nf, int m, int nfeat) {
  int N1 = 0, N2 = 0;
  if (dft1d_factor(nf, &N1, &N2) != FK_OK) return 0;
  return (size_t)nfeat * std::min(N2, m + 1) * N1 * 16 + 256;
}

fk_status idft1d_run(const double2* H, int64_t hstride, int nfeat, int nf, int m, int off, int G, double* out, int64_t ostride, void* ws,
                     size_t ws_bytes, cudaStream_t s) {
  int N1 = 0, N2 = 0;
  FK_TRY(dft1d_factor(nf, &N1, &N2));
  if (ws_bytes < idft1d_ws_bytes(nf, m, nfeat)) return fail(FK_E_WORKSPACE, "idft1d: workspace too small");
  I1Args a{};
  a.H = H;
  a.hstride = hstride;
  a.nf = nf;
  a.N1 = N1;
  a.N2 = N2;
  a.m = m;
  a.off = off;
  a.G = G;
  a.K2 = std::min(N2, m + 1);
  a.U = (double2*)ws;
  a.out = out;
  a.ostride = ostride;
  k_idft_s1<<<dim3(N1, nfeat), 256, 0, s>>>(a);
  k_idft_s2<<<dim3(N1, nfeat), 256, 0, s>>>(a);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(2);
  return FK_OK;
}

}  // namespace fk
