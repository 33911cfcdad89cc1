// dft2d.cu -- the FFT step of the d = 2 type-1 passes and of the additive cross moments
// (PAPER.md:203-220 sec. 2.3 with d-level moments; :505-512), hand-written, no cuFFT.
//
// Only the (2K+1)^2 modes |q|_inf <= K of the window-convolved fine grid are needed (C3 moments:
// 257^2 of 540^2), and the grid is non-zero only on its occupied G x G block (rows and columns
// [off, off + G)).  So the DFT is two small complex matrix products with generated twiddles
// (w = exp(-2 pi i / nf)), batched over grids (the 45 cross-moment pairs):
//   stage A (along columns)  H[r][q1]  = sum_c g[off + r][off + c] w^(q1 (off + c)),  q1 = -K..K
//   stage B (along rows)     F[q0][q1] = sum_r H[r][q1] w^(q0 (off + r)),             q0 = 0..K
// (q0 < 0 by Hermitian symmetry of a real grid), then the deconvolution
//   out[q0][q1] = (-1)^(q0+q1) F[q0][q1] / (psi-hat(q0/nf) psi-hat(q1/nf)).
// One tiled kernel does both stages: C[b][i][j] = sum_k D[b][i][k] w^(((j + jbase) (off + k)) mod nf)
// with 32 x 32 output tiles, 2 x 2 per thread, 32-wide k chunks staged in shared memory (D and the
// twiddles from a per-call w^t table).  C3: ~8e7 fp64 multiply-adds; C5: ~7e8 over the 45 pairs.
//
// The type-2 direction (idft2d_run, the d = 2 predict grid, round 2: replaces cuFFT Z2D) is the same
// two products with conjugate twiddles, evaluated only on the occupied block:
//   P[k1][r]  = sum_{k0=-m..m} c_k1 Hf[k0][k1] w^(-k0 (off + r)),         k1 = 0..m
//   g[r][c]   = Re sum_{k1=0..m} P[k1][r] w^(-k1 (off + c))
// (Hf Hermitian, c_0 = 1, c_k1 = 2 folded into the input), i.e. exactly the real inverse transform
// of the half spectrum on the cells the gather reads.
#include <cmath>

#include "fk_internal.cuh"

namespace fk {
namespace {

constexpr int TT = 32;  // output tile (i and j) and k chunk

__global__ void k_twtab(int nf, double2* tab, double sign) {  // tab[t] = exp(sign 2 pi i t / nf)
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nf) return;
  double s, c;
  sincospi(2.0 * (double)t / (double)nf, &s, &c);
  tab[t] = make_double2(c, sign * s);
}

struct TwArgs {
  const void* D;              // real (double) or complex (double2) input
  int64_t d_b, d_i, d_k;      // element strides of D: batch, row i, contraction k
  int M, N, Kd;               // C is M x N per batch item, contraction length Kd
  int jbase;                  // frequency of column j: q = j + jbase
  int off, nf;                // fine-grid index of k: off + k
  const double2* tab;         // w^t, t = 0..nf-1
  void* C;                    // double2, or double (the real part) when REALOUT
  int64_t c_b, c_i, c_j;      // element strides of C
};

template <bool CPLX, bool REALOUT = false>
__global__ void __launch_bounds__(256) k_twdft(TwArgs a) {
  __shared__ double2 Ds[TT][TT + 1];  // [i][k]
  __shared__ double2 Ws[TT][TT + 1];  // [k][j]
  const int b = blockIdx.z;
  const int i0 = blockIdx.y * TT, j0 = blockIdx.x * TT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // thread owns rows i0 + ty, i0 + ty + 16; cols j0 + tx, j0 + tx + 16
  double2 acc[2][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) acc[u][v] = make_double2(0.0, 0.0);
  const int nf = a.nf;
  for (int k0 = 0; k0 < a.Kd; k0 += TT) {
    // stage the D tile and the twiddle tile (each thread 4 entries of each)
    for (int e = threadIdx.x; e < TT * TT; e += blockDim.x) {
      const int r = e / TT, c = e % TT;
      const int gi = i0 + r, gk = k0 + c;
      double2 dv = make_double2(0.0, 0.0);
      if (gi < a.M && gk < a.Kd) {
        const int64_t idx = b * a.d_b + gi * a.d_i + gk * a.d_k;
        if (CPLX) dv = reinterpret_cast<const double2*>(a.D)[idx];
        else dv.x = reinterpret_cast<const double*>(a.D)[idx];
      }
      Ds[r][c] = dv;
      const int kk = k0 + r, jj = j0 + c;  // twiddle tile: row = k, col = j
      double2 wv = make_double2(0.0, 0.0);
      if (kk < a.Kd && jj < a.N) {
        const int q = jj + a.jbase;  // |q (off + k)| < nf^2 < 2^31 for nf < 46341
        int t = (q * (a.off + kk)) % nf;
        if (t < 0) t += nf;
        wv = __ldg(a.tab + t);
      }
      Ws[r][c] = wv;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < TT; ++k) {
      const double2 d0 = Ds[ty][k], d1 = Ds[ty + 16][k];
      const double2 w0 = Ws[k][tx], w1 = Ws[k][tx + 16];
      if (CPLX) {
        acc[0][0].x = fma(d0.x, w0.x, fma(-d0.y, w0.y, acc[0][0].x));
        acc[0][0].y = fma(d0.x, w0.y, fma(d0.y, w0.x, acc[0][0].y));
        acc[0][1].x = fma(d0.x, w1.x, fma(-d0.y, w1.y, acc[0][1].x));
        acc[0][1].y = fma(d0.x, w1.y, fma(d0.y, w1.x, acc[0][1].y));
        acc[1][0].x = fma(d1.x, w0.x, fma(-d1.y, w0.y, acc[1][0].x));
        acc[1][0].y = fma(d1.x, w0.y, fma(d1.y, w0.x, acc[1][0].y));
        acc[1][1].x = fma(d1.x, w1.x, fma(-d1.y, w1.y, acc[1][1].x));
        acc[1][1].y = fma(d1.x, w1.y, fma(d1.y, w1.x, acc[1][1].y));
      } else {
        acc[0][0].x = fma(d0.x, w0.x, acc[0][0].x);
        acc[0][0].y = fma(d0.x, w0.y, acc[0][0].y);
        acc[0][1].x = fma(d0.x, w1.x, acc[0][1].x);
        acc[0][1].y = fma(d0.x, w1.y, acc[0][1].y);
        acc[1][0].x = fma(d1.x, w0.x, acc[1][0].x);
        acc[1][0].y = fma(d1.x, w0.y, acc[1][0].y);
        acc[1][1].x = fma(d1.x, w1.x, acc[1][1].x);
        acc[1][1].y = fma(d1.x, w1.y, acc[1][1].y);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int gi = i0 + ty + 16 * u, gj = j0 + tx + 16 * v;
      if (gi < a.M && gj < a.N) {
        const int64_t o = b * a.c_b + gi * a.c_i + gj * a.c_j;
        if (REALOUT) reinterpret_cast<double*>(a.C)[o] = acc[u][v].x;
        else reinterpret_cast<double2*>(a.C)[o] = acc[u][v];
      }
    }
}

// FT[b][j][q0] = F[q0][q1 = j - K] for q0 = 0..K  ->  out[b][(q0 + K)(2K+1) + q1 + K], q0, q1 = -K..K
__global__ void k_deconv2d_t(const double2* __restrict__ FT, int K, const double* __restrict__ tab, double2* __restrict__ out, int acc,
                             int batch) {
  const int side = 2 * K + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)side * side * batch) return;
  const int bi = (int)(t / ((int64_t)side * side));
  const int rem = (int)(t % ((int64_t)side * side));
  const int q0 = rem / side - K, q1 = rem % side - K;
  const double2* Fb = FT + (int64_t)bi * side * (K + 1);
  double2 v;
  if (q0 >= 0) {
    v = Fb[(int64_t)(q1 + K) * (K + 1) + q0];
  } else {  // real grid: F[-q0][-q1] = conj F[q0][q1]
    v = Fb[(int64_t)(-q1 + K) * (K + 1) + (-q0)];
    v.y = -v.y;
  }
  const double sc = (((q0 + q1) & 1) ? -1.0 : 1.0) / (tab[q0 < 0 ? -q0 : q0] * tab[q1 < 0 ? -q1 : q1]);
  v.x *= sc;
  v.y *= sc;
  double2* o = out + t;
  if (acc) {
    o->x += v.x;
    o->y += v.y;
  } else {
    *o = v;
  }
}

}  // namespace

size_t dft2d_ws_bytes(int nf, int G, int K, int batch) {
  Bump b(nullptr, 0);
  b.take((size_t)nf * 16);                              // twiddle table
  b.take((size_t)batch * G * (2 * K + 1) * 16);         // H
  b.take((size_t)batch * (2 * K + 1) * (K + 1) * 16);   // F^T
  return b.used + 256;
}

// fine: batch x nf x nf full-period grids (zero outside the occupied block), phihat: psi-hat(q / nf)
// for q = 0..K; out: batch x (2K+1)^2 modes (accumulated when acc)
fk_status dft2d_run(const double* fine, int nf, int off, int G, int K, int batch, const double* phihat, double* out, int acc, void* ws,
                    size_t ws_bytes, cudaStream_t s) {
  if (off < 0 || off + G > nf) return fail(FK_E_ARG, "dft2d: occupied block outside the grid");
  if (nf >= 46341) return fail(FK_E_UNSUPPORTED, "dft2d: fine grid too large (nf >= 46341)");
  Bump bp(ws, ws_bytes);
  double2* tab = (double2*)bp.take((size_t)nf * 16);
  double2* H = (double2*)bp.take((size_t)batch * G * (2 * K + 1) * 16);
  double2* FT = (double2*)bp.take((size_t)batch * (2 * K + 1) * (K + 1) * 16);
  if (!bp.ok()) return fail(FK_E_WORKSPACE, "dft2d: workspace too small");
  k_twtab<<<(nf + 255) / 256, 256, 0, s>>>(nf, tab, -1.0);
  const int side = 2 * K + 1;
  // stage A: H[b][r][j] = sum_c fine[b][off + r][off + c] w^((j - K)(off + c))
  TwArgs A{};
  A.D = fine + (int64_t)off * nf + off;
  A.d_b = (int64_t)nf * nf;
  A.d_i = nf;
  A.d_k = 1;
  A.M = G;
  A.N = side;
  A.Kd = G;
  A.jbase = -K;
  A.off = off;
  A.nf = nf;
  A.tab = tab;
  A.C = H;
  A.c_b = (int64_t)G * side;
  A.c_i = side;
  A.c_j = 1;
  k_twdft<false><<<dim3((side + TT - 1) / TT, (G + TT - 1) / TT, batch), 256, 0, s>>>(A);
  // stage B: FT[b][j][q0] = sum_r H[b][r][j] w^(q0 (off + r)), q0 = 0..K  (D = H^T: row j, contraction r)
  TwArgs B{};
  B.D = H;
  B.d_b = (int64_t)G * side;
  B.d_i = 1;
  B.d_k = side;
  B.M = side;
  B.N = K + 1;
  B.Kd = G;
  B.jbase = 0;
  B.off = off;
  B.nf = nf;
  B.tab = tab;
  B.C = FT;
  B.c_b = (int64_t)side * (K + 1);
  B.c_i = K + 1;
  B.c_j = 1;
  k_twdft<true><<<dim3((K + 1 + TT - 1) / TT, (side + TT - 1) / TT, batch), 256, 0, s>>>(B);
  const int64_t nout = (int64_t)side * side * batch;
  k_deconv2d_t<<<(unsigned)((nout + 255) / 256), 256, 0, s>>>(FT, K, phihat, (double2*)out, acc, batch);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(4);
  return FK_OK;
}

size_t idft2d_ws_bytes(int nf, int G, int m) {
  Bump b(nullptr, 0);
  b.take((size_t)nf * 16);             // conjugate twiddle table
  b.take((size_t)(m + 1) * G * 16);    // P
  return b.used + 256;
}

// Hc: (2m+1) x (m+1) complex, Hc[(k0 + m)(m+1) + k1] = c_k1 Hf[k0][k1] (deconvolved, Hermitian part);
// grid: row-major with leading dimension ldg, cells [off, off + G)^2 written (the rest untouched)
fk_status idft2d_run(const double2* Hc, int m, int nf, int off, int G, double* grid, int64_t ldg, void* ws, size_t ws_bytes, cudaStream_t s) {
  if (off < 0 || off + G > nf) return fail(FK_E_ARG, "idft2d: occupied block outside the grid");
  if (nf >= 46341) return fail(FK_E_UNSUPPORTED, "idft2d: fine grid too large (nf >= 46341)");
  Bump bp(ws, ws_bytes);
  double2* tab = (double2*)bp.take((size_t)nf * 16);
  double2* P = (double2*)bp.take((size_t)(m + 1) * G * 16);
  if (!bp.ok()) return fail(FK_E_WORKSPACE, "idft2d: workspace too small");
  k_twtab<<<(nf + 255) / 256, 256, 0, s>>>(nf, tab, 1.0);
  // stage A: P[k1][r] = sum_k Hc[k][k1] w^(-(off + r)(k - m))   (i = k1, j = r, contraction k = k0 + m)
  TwArgs A{};
  A.D = Hc;
  A.d_b = 0;
  A.d_i = 1;
  A.d_k = m + 1;
  A.M = m + 1;
  A.N = G;
  A.Kd = 2 * m + 1;
  A.jbase = off;
  A.off = -m;
  A.nf = nf;
  A.tab = tab;
  A.C = P;
  A.c_b = 0;
  A.c_i = G;
  A.c_j = 1;
  k_twdft<true><<<dim3((G + TT - 1) / TT, (m + 1 + TT - 1) / TT, 1), 256, 0, s>>>(A);
  // stage B: g[off + r][off + c] = Re sum_k1 P[k1][r] w^(-(off + c) k1)   (i = r, j = c, contraction k1)
  TwArgs B{};
  B.D = P;
  B.d_b = 0;
  B.d_i = 1;
  B.d_k = G;
  B.M = G;
  B.N = G;
  B.Kd = m + 1;
  B.jbase = off;
  B.off = 0;
  B.nf = nf;
  B.tab = tab;
  B.C = grid + (int64_t)off * ldg + off;
  B.c_b = 0;
  B.c_i = ldg;
  B.c_j = 1;
  k_twdft<true, true><<<dim3((G + TT - 1) / TT, (G + TT - 1) / TT, 1), 256, 0, s>>>(B);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(3);
  return FK_OK;
}

}  // namespace fk
