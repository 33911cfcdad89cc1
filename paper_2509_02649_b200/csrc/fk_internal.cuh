// fk_internal.cuh -- internal declarations of libfk (not installed; include/fk.h is the ABI).
#pragma once

#include <cuda_runtime.h>
#include <cufft.h>
#include <cstdint>
#include <cstddef>
#include <string>

#include "../../include/fk.h"

namespace fk {

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
void set_error(const std::string& msg);
fk_status fail(fk_status st, const std::string& msg);
#define FK_CUDA_TRY(expr)                                                                       \
  do {                                                                                          \
    cudaError_t _e = (expr);                                                                    \
    if (_e != cudaSuccess)                                                                      \
      return ::fk::fail(FK_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)
#define FK_CUFFT_TRY(expr)                                                                      \
  do {                                                                                          \
    cufftResult _r = (expr);                                                                    \
    if (_r != CUFFT_SUCCESS) return ::fk::fail(FK_E_CUDA, std::string(#expr) + ": cufft error " + std::to_string((int)_r)); \
  } while (0)
#define FK_TRY(expr)                  \
  do {                                \
    fk_status _s = (expr);            \
    if (_s != FK_OK) return _s;       \
  } while (0)

int device_sm_count();

// diagnostics: kernel-launch counter and spreading-kernel event brackets (fk_profile_*)
void count_launch(int k = 1);
void prof_spread_begin(cudaStream_t s);
void prof_spread_end(cudaStream_t s);

// ------------------------------------------------------------------------------------------
// workspace: a bump allocator over the caller's buffer (256-byte aligned slices)
// ------------------------------------------------------------------------------------------
struct Bump {
  char* base;
  size_t used = 0;
  size_t cap;
  explicit Bump(void* b, size_t c) : base((char*)b), cap(c) {}
  void* take(size_t bytes) {
    size_t off = (used + 255) & ~(size_t)255;
    used = off + bytes;
    return base ? (void*)(base + off) : nullptr;
  }
  bool ok() const { return used <= cap; }
};

// ------------------------------------------------------------------------------------------
// spreading plans
// ------------------------------------------------------------------------------------------
enum KerKind { KER_BS3 = 0, KER_ES = 1, KER_BS7 = 2 };  // BS7: septic B-spline, fp64 mode (spread1d.cu)

// One fine grid of one channel along one dimension: period nf, cells [off, off + G) held locally.
struct Geo {
  int nf = 0;
  int off = 0;
  int G = 0;
};

struct EsParams {
  int w = 0;
  double beta = 0.0;
};

// Plan of a type-1 pass: window, precision and the two fine grids (moments: modes 4m+1,
// rhs: modes 2m+1, nf_r = nf_mu / 2 so the rhs cell is the moment cell halved).
struct Plan1 {
  int d = 1;
  int m = 0;
  KerKind ker = KER_BS3;
  bool fp64 = false;      // fp64 accumulation path (ES window)
  EsParams es;
  int nf_mu = 0, nf_r = 0;  // per dimension
  Geo gA, gB;             // per-dimension geometry of the moment / rhs grids
  bool smem = true;       // grids held in shared memory (else global accumulation)
  int threads = 1024;
  int ctas = 0;
  size_t smem_bytes = 0;
  double eps = 1e-6;      // the requested accuracy (fp64-mode fixed-point scale)
};

fk_status make_plan1(int d, int m, double eps, bool need_mu, bool need_r, Plan1* p);
int fft_friendly(int n);  // smallest 2^a 3^b 5^c >= n, even, multiple of 8

// ES taps as degree-P polynomials in s in (-1, 1] (plan.cu): coef[i * (P + 1) + q], device memory,
// built once per (device, w, beta).
inline int es_horner_degree(int w) { return w + 2; }
fk_status es_horner_table(const EsParams& es, const double** d_coef);
// Constant-memory copies of the tables, one slot per width w (the ES shape is beta = 2.30 w on every
// path, so slot w never changes): a kernel of width W reads slot W.  horner_slot uploads slot w of
// `symbol` (a __constant__ double[kHornerSlots][kHornerSlot] of the calling translation unit) once
// per device -- no per-call copy, so concurrent calls on different streams cannot overwrite a
// table another kernel is reading.  FK_E_UNSUPPORTED if beta is not 2.30 w (then the caller uses
// its exp-based taps).
constexpr int kHornerSlots = 17;
constexpr int kHornerSlot = 16 * 19;
fk_status horner_slot(const void* symbol, int w, double beta);

// ES window Fourier transform table phihat[k] = psi-hat(k / nf), k = 0..K (computed on device).
fk_status es_phihat_table(const EsParams& es, int nf, int K, double* d_tab, cudaStream_t s);

// cuFFT plan cache (plans own no memory; the work area comes from the workspace)
struct FftPlan {
  cufftHandle h = 0;
  size_t work = 0;
};
fk_status fft_plan(int rank, const int* dims, int batch, cufftType type, FftPlan* out);
fk_status fft_exec_d2z(const FftPlan& p, double* in, cufftDoubleComplex* out, void* work, cudaStream_t s);
fk_status fft_exec_z2d(const FftPlan& p, cufftDoubleComplex* in, double* out, void* work, cudaStream_t s);

// ------------------------------------------------------------------------------------------
// d = 1 pass (spread1d.cu)
// ------------------------------------------------------------------------------------------
struct Type1Out {
  double* mu;  // (4m+1)^d complex or null
  double* r;   // (2m+1)^d complex or null
  bool accumulate;
};
size_t type1_ws_bytes(const Plan1& p, bool need_mu, bool need_r);

// hand-written reduce + pruned DFT + deconvolution of a d = 1 pass (dft1d.cu), up to two grids
// per launch set.  out[K + q], q = -K..K: (-1)^q F_q / psi-hat(q / nf) with F the DFT of the
// full-period grid whose occupied cells [off, off + G) are the summed partials + carries.
struct Dft1Grid {
  int nf = 0, off = 0, G = 0, K = 0;
  const int* part_i = nullptr;     // nparts x G int32 partials, or
  const double* part_d = nullptr;  // nparts x G fp64 partials
  int nparts = 0;
  const int* escale = nullptr;     // per-partial exponent: value = int x 2^-escale (else x inv_scale)
  double inv_scale = 1.0;
  const double* carry = nullptr;   // G fp64 drained values, or null
  const double* phihat = nullptr;  // KER_ES: psi-hat(q / nf), q = 0..K
  double* out = nullptr;           // 2K + 1 complex128
};
fk_status dft1d_factor(int nf, int* N1, int* N2);
size_t dft1d_ws_bytes(const Dft1Grid* g, int ngrids);
fk_status dft1d_run(const Dft1Grid* g, int ngrids, int ker, int acc, void* ws, size_t ws_bytes, cudaStream_t s);
// the type-2 direction (predict, dft1d.cu): cells [off, off + G) of nfeat real grids from their half
// spectra H (coefficients k = 0..m; Z2D semantics), no cuFFT
size_t idft1d_ws_bytes(int nf, int m, int nfeat);
fk_status idft1d_run(const double2* H, int64_t hstride, int nfeat, int nf, int m, int off, int G, double* out, int64_t ostride, void* ws,
                     size_t ws_bytes, cudaStream_t s);

// hand-written DFT of batch d = 2 fine grids (dft2d.cu): the (2K+1)^2 modes of full-period nf x nf
// grids non-zero on [off, off + G)^2, deconvolved by phihat (psi-hat(q / nf), q = 0..K) per dimension
size_t dft2d_ws_bytes(int nf, int G, int K, int batch);
fk_status dft2d_run(const double* fine, int nf, int off, int G, int K, int batch, const double* phihat, double* out, int acc, void* ws,
                    size_t ws_bytes, cudaStream_t s);
// the type-2 direction for the d = 2 predict grid (dft2d.cu): Hc (2m+1) x (m+1) half spectrum
// (k1 >= 0, the k1 > 0 entries doubled) -> the real grid on the occupied block [off, off + G)^2
size_t idft2d_ws_bytes(int nf, int G, int m);
fk_status idft2d_run(const double2* Hc, int m, int nf, int off, int G, double* grid, int64_t ldg, void* ws, size_t ws_bytes, cudaStream_t s);
fk_status type1_run(const Plan1& p, const fk_points& X, const void* Y, double L, const Type1Out& out, void* ws, size_t ws_bytes,
                    int* d_status, cudaStream_t s);

// ------------------------------------------------------------------------------------------
// solve (solve.cu), predict (predict.cu), additive (additive.cu)
// ------------------------------------------------------------------------------------------
size_t solve_ws_bytes(int d, int m, int kind);
size_t chol_ws_bytes(int N);
// the state chol_tiles resets before its kernel (side buffer to the sentinel, flags / ticket / info
// to zero): a caller that already launches a kernel before it can do the reset there (chol_reset)
// and pass preset = true, saving the memset nodes on the solve's latency chain
struct CholReset {
  unsigned long long* ld;  // side buffer, filled with all-ones
  int64_t n_ld;            // 8-byte words
  int* zero;               // flags + ticket (+ uflags when used), zeroed
  int64_t n_zero;
  int* info;               // zeroed
};
CholReset chol_reset_args(int N, void* ws, int* info);
__device__ __forceinline__ void chol_reset(const CholReset& c, int64_t t, int64_t stride) {
  for (int64_t i = t; i < c.n_ld; i += stride) c.ld[i] = ~0ULL;
  for (int64_t i = t; i < c.n_zero; i += stride) c.zero[i] = 0;
  if (t == 0) *c.info = 0;
}
fk_status chol_tiles(double* M, int64_t ld, int N, int* info, void* ws, cudaStream_t s, unsigned long long* trace = nullptr,
                     bool preset = false);
size_t solve_path_ws_bytes(int d, int m, int kind, int nlam);
fk_status solve_path_run(const fk_problem* P, const double* lambdas, int nlam, double* theta, int* info, void* ws, size_t ws_bytes,
                         cudaStream_t s);
size_t path_validate_ws_bytes(int d, int m, int kind, int nlam);
fk_status path_validate_run(const fk_problem* Pv, const double* theta, int nlam, double sum_y2, double* risk_out, void* ws,
                            size_t ws_bytes, cudaStream_t s);
fk_status solve_run(const fk_problem* P, double* theta, fk_solve_report* rep, void* ws, size_t ws_bytes, cudaStream_t s);

size_t predict_ws_bytes(int d, int m, double eps, int additive);
fk_status predict_run(const double* theta, int d, int m, double L, int additive, const fk_points& Xq, double eps, void* out,
                      void* ws, size_t ws_bytes, int* d_status, cudaStream_t s);

size_t cross_ws_bytes(int d, int m, double eps, int64_t n, int dtype);
size_t type1_2d_ws_bytes(int m, double eps, bool mu, bool r, int dtype);
fk_status type1_2d_run(int m, double eps, const fk_points& X, const void* Y, double L, double* mu_out, double* r_out, bool acc, void* ws,
                       size_t ws_bytes, int* d_status, cudaStream_t s);
fk_status cross_run(const fk_points& X, double L, int m, double eps, double* G, bool accumulate, void* ws, size_t ws_bytes,
                    int* d_status, cudaStream_t s);

// ------------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------------
#define FK_MAGIC 12582912.0f        // 1.5 * 2^23: x + MAGIC rounds x to an integer in the low mantissa bits
#define FK_MAGIC_BITS 0x4B400000

// 64-bit fixed point held as two int32 words per cell (lo unsigned, hi signed) in shared memory:
// an add is one native ATOMS.ADD on lo, the carry is read off its return value, and hi gets
// (v >> 32) + carry only when that is non-zero -- 3.1x the rate of fp64 shared-memory atomicAdd
// (a CAS loop on sm_100a).  A hi word that reaches 2^29 in magnitude is drained (atomicExch) into
// an fp64 carry cell (hi_unit = value of one hi unit), so no overflow.  Used by the fp64 modes.
constexpr double kSX = 1099511627776.0;  // 2^40: tap weights in [0, 1] -> 2^-41 rounding

__device__ __forceinline__ void pair_add(unsigned* __restrict__ lo, int* __restrict__ hi, int c, long long v, double* carry,
                                         double hi_unit) {
  const unsigned l = (unsigned)v;
  const int h = (int)(v >> 32);
  const unsigned o = atomicAdd(lo + c, l);
  const int hc = h + ((o + l) < o ? 1 : 0);
  if (hc != 0) {
    const int oh = atomicAdd(hi + c, hc);
    if ((unsigned)(oh + hc + (1 << 29)) >= (1u << 30)) {
      const int t = atomicExch(hi + c, 0);
      if (t) atomicAdd(carry + c, (double)t * hi_unit);
    }
  }
}

// pair_add over N consecutive cells c0 .. c0+N-1 with values vf(i), in groups of up to 8 whose
// atomics are issued phase by phase (all low words, then the high words, then the rare drains):
// one tap's high-word update needs its low word's old value, so tap-by-tap pair_add waits ~2
// shared-atomic round trips per tap; grouped, 3 round trips per 8 taps.
template <int N, class VF>
__device__ __forceinline__ void pair_add_n(unsigned* __restrict__ lo, int* __restrict__ hi, int c0, VF vf, double* carry,
                                           double hi_unit) {
#pragma unroll
  for (int g0 = 0; g0 < N; g0 += 8) {
    constexpr int B = 8;
    unsigned o[B], l[B];
    int h[B];
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (g0 + i < N) {
        const long long v = vf(g0 + i);
        l[i] = (unsigned)v;
        h[i] = (int)(v >> 32);
        o[i] = atomicAdd(lo + c0 + g0 + i, l[i]);
      }
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (g0 + i < N) {
        h[i] += (o[i] + l[i]) < o[i] ? 1 : 0;  // carry out of the low word
        o[i] = h[i] != 0 ? (unsigned)atomicAdd(hi + c0 + g0 + i, h[i]) : 0u;
      }
#pragma unroll
    for (int i = 0; i < B; ++i)
      if (g0 + i < N && h[i] != 0 && (unsigned)((int)o[i] + h[i] + (1 << 29)) >= (1u << 30)) {
        const int t = atomicExch(hi + c0 + g0 + i, 0);
        if (t) atomicAdd(carry + c0 + g0 + i, (double)t * hi_unit);
      }
  }
}

// N consecutive cells c0.. of one row, values round(wy x[b]) (|wy x[b]| < 2^51), branch-free: the
// 1.5 x 2^52 shift gives both int32 words of each value, then the N low-word atomics, the carries by
// add.cc/addc, the N high-word atomics unconditionally (ptxas turns any conditional atomic into
// BSSY/BRA/BSYNC -- 3 issue slots per tap -- and in the 2-D fp64 kernels nearly every tap carries
// anyway: sum_ab w_a w_b ~ (W/2)^2 low-word wraps per sample), and one drain test per row.
template <int N>
__device__ __forceinline__ void pair_add_row(unsigned* __restrict__ lo, int* __restrict__ hi, int c0, double wy, const double* x,
                                             double* carry, double hi_unit) {
  unsigned l[N], o[N];
  int h[N];
#pragma unroll
  for (int b = 0; b < N; ++b) {
    const double d = fma(wy, x[b], 6755399441055744.0);
    l[b] = (unsigned)__double2loint(d);
    h[b] = __double2hiint(d) - 0x43380000;
  }
#pragma unroll
  for (int b = 0; b < N; ++b) o[b] = atomicAdd(lo + c0 + b, l[b]);
  unsigned any = 0;
#pragma unroll
  for (int b = 0; b < N; ++b) {
    int hc;
    asm("{\n\t.reg .u32 t;\n\tadd.cc.u32 t, %1, %2;\n\taddc.s32 %0, %3, 0;\n\t}" : "=r"(hc) : "r"(o[b]), "r"(l[b]), "r"(h[b]));
    const int old = atomicAdd(hi + c0 + b, hc);
    any |= (unsigned)(old + hc + (1 << 29));
  }
  if (any >= (1u << 30)) {
#pragma unroll 1
    for (int b = 0; b < N; ++b) {
      const int t = atomicExch(hi + c0 + b, 0);
      if (t) atomicAdd(carry + c0 + b, (double)t * hi_unit);
    }
  }
}

// exact 2^e for |e| < 1000 without the libm ldexp call
__device__ inline double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

__host__ __device__ inline double sinc_pi(double x) {  // sin(pi x) / (pi x)
  if (x == 0.0) return 1.0;
  const double a = 3.14159265358979323846 * x;
  return sin(a) / a;
}

}  // namespace fk
