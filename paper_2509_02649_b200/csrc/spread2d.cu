// spread2d.cu -- d = 2 type-1 passes (PAPER.md:212-220 d-level moments, :203-208 rhs) and the
// additive model's cross moments (2-D unit-weight sums at (X_l1, -X_l2)).
//
// Window: exponential of semicircle psi(z) = exp(beta (sqrt(1 - z^2) - 1)), sigma = 2 (fine grid
// nf >= 2 x modes per dimension), w = ceil(log10 1/eps) + 1 taps per dimension (+1 in fp64),
// beta = 2.30 w.  A 2-D grid's occupied quarter does not fit one CTA at C3 (299^2 + 155^2
// cells), so the occupied rows are split into T row tiles ("binned subproblems"): tile t owns
// the samples whose first tap row lies in its row range and keeps those rows plus a (w-1)-row
// halo in shared memory; CTA (chunk, t) streams its chunk of samples and spreads the ones it
// owns.  Accumulation: int32 fixed point (weights x 2^21, rhs with a per-CTA power-of-two scale,
// native ATOMS.ADD, drain-at-2^29 into fp64 carry grids) on the fp32 path; on the fp64 path
// 64-bit fixed point held as int32 pairs (pair_add: ATOMS.ADD on the low word, the carry read off
// its return value, the high word when non-zero; high words drained at 2^29 into fp64 carry
// grids), weights from a Chebyshev-fitted Horner table.  Partials are reduced per fine-grid cell in a fixed CTA order, FFT'd (cuFFT 2-D
// D2Z, batched over pairs) and deconvolved by psi-hat(q0) psi-hat(q1).
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "fk_internal.cuh"

namespace fk {
namespace {

constexpr int kW = 16;  // max taps per dimension
// 2^20: a tap weight is <= 1, so after a cell crosses the drain threshold 2^29 the CTA's 1024
// threads add at most 1024 x 2^20 more before one of them drains it: < 2^31, no overflow
constexpr float kS2 = 1048576.0f;
constexpr double kInvS2 = 1.0 / 1048576.0;

// Exact position of a coordinate on a grid: p = x * a (compensated when a is not a power of
// two), P = floor(p), f = p - P in [0,1).  The first tap of a w-tap ES window centred at the
// point is P + d0 where d0 = 1 - w/2 (w even, f > 0) / -w/2 (w even, f = 0) / etc., and tap i
// sits at offset (d0 + i - f) cells from the point -- exact in fp32.
struct P1 {
  int P;
  float f;
};

template <bool EXACT>
__device__ __forceinline__ P1 place_f32(float x, float a_hi, float a_lo) {
  float p = x * a_hi;
  float fl = floorf(p);
  float f = p - fl;
  if (!EXACT) {
    const float e = fmaf(x, a_hi, -p) + x * a_lo;
    f += e;
    if (f < 0.0f) { f += 1.0f; fl -= 1.0f; }
    if (f >= 1.0f) { f -= 1.0f; fl += 1.0f; }
  }
  P1 r;
  r.P = (__float_as_int(fl + FK_MAGIC) - FK_MAGIC_BITS);
  r.f = f;
  return r;
}

__device__ __forceinline__ P1 halve(P1 a, float e_unused) {  // position on the half-resolution grid
  P1 r;
  const int odd = a.P & 1;
  r.P = (a.P - odd) / 2;  // floor(P/2) for any sign
  if (a.P < 0 && odd) r.P = (a.P - 1) / 2;
  r.f = 0.5f * (a.f + (float)odd);
  return r;
}

// first-tap offset d0 so that taps d0..d0+w-1 cover [f - w/2, f + w/2]
__device__ __forceinline__ int first_tap(float f, int w) {
  // ceil(f - w/2) with f in [0,1)
  return (w & 1) ? (f > 0.5f ? 1 : 0) - (w >> 1) : (f > 0.0f ? 1 : 0) - (w >> 1);
}

__device__ __forceinline__ int first_tap_d(double f, int w) {
  return (w & 1) ? (f > 0.5 ? 1 : 0) - (w >> 1) : (f > 0.0 ? 1 : 0) - (w >> 1);
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// ES taps in fp32: psi = 2^(beta log2(e) (sqrt(1 - z^2) - 1)); the taps cover |z| <= 1 by
// construction (v is clamped at 0 against rounding), so no branch; 2 MUFU + 3 FMA per tap.
// betal2 = beta * log2(e).
template <int W>
__device__ __forceinline__ void es_taps_f32(float f, int d0, float betal2, float* psi) {
  const float inv = 2.0f / (float)W;
  const float z0 = ((float)d0 - f) * inv;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const float z = fmaf((float)i, inv, z0);
    const float v = fmaxf(fmaf(-z, z, 1.0f), 0.0f);
    psi[i] = ex2_approx(fmaf(betal2, sqrt_approx(v), -betal2));
  }
}

template <int W>
__device__ __forceinline__ void es_taps_f64(double f, int d0, double beta, double* psi) {
  const double inv = 2.0 / (double)W;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const double z = ((double)(d0 + i) - f) * inv;
    const double v = 1.0 - z * z;
    psi[i] = v > 0.0 ? exp(beta * (sqrt(v) - 1.0)) : 0.0;
  }
}

// fp64-accuracy taps of both dimensions by Horner's rule on the launch's Chebyshev-fitted table
// (es_horner_table: W polynomials of degree W + 2 in s in [-1, 1], the same table the 1-D fp64
// kernel uses) instead of 2W fp64 exp + sqrt; each coefficient serves both dimensions.  The
// first tap d0 = first_tap_d(f, W) puts u = f - d0 in [W/2 - 1, W/2], the table's interval.
__constant__ double c_es2_coef[kHornerSlots][kHornerSlot];  // slot W (horner_slot)

template <int W>
__device__ __forceinline__ void es_taps2_horner(double fy, int dy, double fx, int dx, double* py, double* px) {
  constexpr int NP = W + 3;
  const double sy = 2.0 * (fy - dy - 0.5 * W + 1.0) - 1.0;
  const double sx = 2.0 * (fx - dx - 0.5 * W + 1.0) - 1.0;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    double ay = c_es2_coef[W][i * NP + NP - 1], ax = ay;
#pragma unroll
    for (int q = NP - 2; q >= 0; --q) {
      const double c = c_es2_coef[W][i * NP + q];
      ay = fma(ay, sy, c);
      ax = fma(ax, sx, c);
    }
    py[i] = ay;
    px[i] = ax;
  }
}

static fk_status upload_es2_table(int w, double beta, cudaStream_t) {
  const fk_status st = horner_slot(c_es2_coef, w, beta);
  return st == FK_OK ? FK_OK : fail(st, "fp64 ES Horner table unavailable for w = " + std::to_string(w));
}

__device__ __noinline__ void drain_row(int* row, int w, double* carry_row, double inv_scale) {
  for (int b = 0; b < w; ++b) {
    const int v = atomicExch(row + b, 0);
    if (v) atomicAdd(carry_row + b, (double)v * inv_scale);
  }
}

// One 2-D tile of one grid: rows [r0, r0 + rows) of the occupied G x G region, in smem.
struct Tile {
  int G;     // occupied cells per dimension (local coordinates 0..G-1)
  int K;     // local index of the grid centre offset: local = P + K (+ tap offset)
  int R;     // rows owned per tile
  int rows;  // rows stored = R + w - 1
};

// fixed-point spread of one sample into a tile (fp32 path); returns false if out of range
template <bool SIGNED, int W>
__device__ __forceinline__ void spread_fixed(int* T, const Tile& g, int lr /*local first row*/, int lc, const float* py,
                                             const float* px, float scale, double* carry, int tile_r0, double inv_scale) {
  int* row = T + (lr - tile_r0) * g.G + lc;
  unsigned orr = 0;
#pragma unroll
  for (int a = 0; a < W; ++a) {
    const float wy = py[a] * scale;
#pragma unroll
    for (int b = 0; b < W; ++b) {
      const int v = __float_as_int(fmaf(wy, px[b], FK_MAGIC)) - FK_MAGIC_BITS;
      const unsigned o = (unsigned)atomicAdd(row + a * g.G + b, v);
      orr |= SIGNED ? (o + (1u << 29)) : o;
    }
  }
  if (SIGNED ? (orr & 0xC0000000u) : (orr & 0x60000000u))  // some cell >= 2^29 in magnitude
    for (int a = 0; a < W; ++a) drain_row(row + a * g.G, W, carry + (int64_t)(lr + a) * g.G + lc, inv_scale);
}

template <int W>
__device__ __forceinline__ void spread_f64(double* T, const Tile& g, int lr, int lc, const double* py, const double* px, double c,
                                           int tile_r0) {
#pragma unroll
  for (int a = 0; a < W; ++a) {
    double* row = T + (lr - tile_r0 + a) * g.G + lc;
    const double wy = py[a] * c;
#pragma unroll
    for (int b = 0; b < W; ++b) atomicAdd(row + b, wy * px[b]);
  }
}

struct Args2 {
  int64_t n, sn, sd, per;
  int aos2;  // sn == 2, sd == 1 and X 8-byte aligned (float2 loads)
  int w;
  float beta_f;
  double beta_d;
  float a_hi, a_lo;  // nf_mu / (4L)
  double a_d;
  int T;             // row tiles
  Tile gA, gB;
  int KA, KB;        // centre offsets (local index of the grid centre)
  void* partA;
  void* partB;
  int* escale;
  double* carryA;
  double* carryB;
  int* d_status;
  int* gsync;  // per chunk: blocks completed by the chunk's T tile CTAs (lockstep streaming), or null
};

// The T tile CTAs of a chunk stream the SAME samples; each keeps the ~1/T it owns.  Left alone
// they drift apart by more than the L2 can cover (C3: ncu measured 19.1 B/sample of DRAM traffic
// for 12 algorithmic, 1.6x), so every kSyncEvery blocks of blockDim samples a CTA waits until the
// other CTAs of its chunk have finished the previous step: the group reads each block from HBM
// once and hits L2 for the other T - 1 reads (working set: chunks x 2 steps x 384 KB ~ 40 MB).
// The wait affects only locality, never the result: a spin that outlives its 20 ms watchdog (the
// group's CTAs not co-resident, e.g. SMs taken by another stream's kernel) proceeds and the CTA
// stops waiting for the rest of the launch.
constexpr int kSyncEvery = 32;

__device__ __forceinline__ void group_lockstep(int* gsync, int chunk, int T, int64_t step, int* s_off) {
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicAdd(gsync + chunk, 1);
    if (!*s_off) {
      const long long target = (long long)T * (step - 1);
      unsigned long long t0, t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      for (;;) {
        int v;
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(gsync + chunk) : "memory");
        if ((long long)v >= target) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t0 > 20000000ULL) {
          *s_off = 1;
          break;
        }
      }
    }
  }
  __syncthreads();
}

// moments (grid A) and rhs (grid B) of d = 2 points, fp32 fixed-point path
template <int W, bool MU, bool R, bool EXACT>
__global__ void __launch_bounds__(1024) k_spread2d_fixed(const float* __restrict__ X, const float* __restrict__ Y, Args2 g) {
  extern __shared__ int sm2[];
  int* A = sm2;
  int* B = sm2 + (MU ? g.gA.rows * g.gA.G : 0);
  const int tile = blockIdx.x % g.T;
  const int chunk = blockIdx.x / g.T;
  const int nsm = (MU ? g.gA.rows * g.gA.G : 0) + (R ? g.gB.rows * g.gB.G : 0);
  for (int i = threadIdx.x; i < nsm; i += blockDim.x) sm2[i] = 0;
  const int64_t beg = (int64_t)chunk * g.per;
  const int64_t end = min(g.n, beg + g.per);
  float SY = 0.f;
  double invSY = 0.0;
  if (R) {
    __shared__ float red[32];
    __shared__ int sE;
    float mx = 0.0f;
    const int64_t cnt = max((int64_t)0, min(end - beg, (int64_t)4096));
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) mx = fmaxf(mx, fabsf(Y[beg + i]));
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      float t = 0.0f;
      for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmaxf(t, red[i]);
      int e2 = 0, E = 19;
      if (t > 0.0f && t <= 3.0e38f) {
        frexpf(t, &e2);
        E = 20 - e2;
      }
      E = max(-100, min(110, E));
      sE = E;
      g.escale[blockIdx.x] = E;
    }
    __syncthreads();
    SY = ldexpf(1.0f, sE);
    invSY = ldexp(1.0, -sE);
  }
  __syncthreads();
  const int rA0 = tile * g.gA.R, rB0 = tile * g.gB.R;
  bool bad = false;
  float px[W], py[W];
  // A tile owns ~1/T of the samples it reads; spreading them straight from the read loop would
  // run every 49-atomic spread with ~1/T of the lanes active.  Owned samples are therefore
  // compacted into a per-warp queue (ballot + popc) and spread 32 at a time.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  float2* qa = reinterpret_cast<float2*>(sm2 + ((nsm + 3) & ~3)) + warp * 64;
  float2* qb = reinterpret_cast<float2*>(sm2 + ((nsm + 3) & ~3)) + nwarps * 64 + warp * 64;
  float* qy = reinterpret_cast<float*>(reinterpret_cast<float2*>(sm2 + ((nsm + 3) & ~3)) + 2 * nwarps * 64) + warp * 64;
  int cA = 0, cB = 0;
  auto spreadA = [&](float x0, float x1) {
    const P1 q0 = place_f32<EXACT>(x0, g.a_hi, g.a_lo), q1 = place_f32<EXACT>(x1, g.a_hi, g.a_lo);
    const int d00 = first_tap(q0.f, W), d01 = first_tap(q1.f, W);
    es_taps_f32<W>(q0.f, d00, g.beta_f, py);
    es_taps_f32<W>(q1.f, d01, g.beta_f, px);
    spread_fixed<false, W>(A, g.gA, q0.P + g.KA + d00, q1.P + g.KA + d01, py, px, kS2, g.carryA, rA0, kInvS2);
  };
  auto spreadB = [&](float x0, float x1, float y) {
    const P1 h0 = halve(place_f32<EXACT>(x0, g.a_hi, g.a_lo), 0.f), h1 = halve(place_f32<EXACT>(x1, g.a_hi, g.a_lo), 0.f);
    const int e0 = first_tap(h0.f, W), e1 = first_tap(h1.f, W);
    const int lrB = h0.P + g.KB + e0, lcB = h1.P + g.KB + e1;
    es_taps_f32<W>(h0.f, e0, g.beta_f, py);
    es_taps_f32<W>(h1.f, e1, g.beta_f, px);
    const float ys = y * SY;
    if (fabsf(ys) < 1048576.0f) {
      spread_fixed<true, W>(B, g.gB, lrB, lcB, py, px, ys, g.carryB, rB0, invSY);
    } else {  // outlier / NaN: exact fp64 path straight into the carry grid
      for (int a = 0; a < W; ++a)
        for (int b = 0; b < W; ++b) atomicAdd(g.carryB + (int64_t)(lrB + a) * g.gB.G + lcB + b, (double)py[a] * px[b] * (double)y);
    }
  };
  const int64_t nblk = (end - beg + blockDim.x - 1) / blockDim.x;  // the same count in every warp and tile CTA
  __shared__ int s_off;
  if (threadIdx.x == 0) s_off = 0;
  for (int64_t blk = 0; blk < nblk; ++blk) {
    if (g.gsync && blk > 0 && blk % kSyncEvery == 0) group_lockstep(g.gsync, chunk, g.T, blk / kSyncEvery, &s_off);
    const int64_t j = beg + blk * blockDim.x + (int64_t)warp * 32 + lane;
    bool ownA = false, ownB = false;
    float x0 = 0.f, x1 = 0.f, y = 0.f;
    if (j < end) {
      if (g.aos2) {  // interleaved (x0, x1) pairs, 8-byte aligned: one 64-bit load per sample
        // one tile: stream (evict-first); T tiles: the other T - 1 CTAs re-read the block from L2
        // (lockstep), so it must not be marked for early eviction
        const float2 v = g.T > 1 ? __ldg(reinterpret_cast<const float2*>(X) + j) : __ldcs(reinterpret_cast<const float2*>(X) + j);
        x0 = v.x;
        x1 = v.y;
      } else {
        x0 = X[j * g.sn];
        x1 = X[j * g.sn + g.sd];
      }
      const P1 q0 = place_f32<EXACT>(x0, g.a_hi, g.a_lo);
      const P1 q1 = place_f32<EXACT>(x1, g.a_hi, g.a_lo);
      // range check on the moment grid (both coordinates): |X| <= L
      const int lrA = q0.P + g.KA + first_tap(q0.f, W), lcA = q1.P + g.KA + first_tap(q1.f, W);
      if ((unsigned)lrA > (unsigned)(g.gA.G - W) || (unsigned)lcA > (unsigned)(g.gA.G - W) || x0 != x0 || x1 != x1) {
        if (tile == 0) bad = true;
      } else {
        ownA = MU && lrA >= rA0 && lrA < rA0 + g.gA.R;
        if (R) {
          const P1 h0 = halve(q0, 0.f);
          const int lrB = h0.P + g.KB + first_tap(h0.f, W);
          ownB = lrB >= rB0 && lrB < rB0 + g.gB.R;
          if (ownB) y = Y[j];
        }
      }
    }
    if (MU) {
      const unsigned msk = __ballot_sync(0xffffffffu, ownA);
      if (ownA) qa[cA + __popc(msk & lt)] = make_float2(x0, x1);
      cA += __popc(msk);
      if (cA >= 32) {
        __syncwarp();
        const float2 v = qa[cA - 32 + lane];
        cA -= 32;
        __syncwarp();
        spreadA(v.x, v.y);
      }
    }
    if (R) {
      const unsigned msk = __ballot_sync(0xffffffffu, ownB);
      if (ownB) {
        const int at = cB + __popc(msk & lt);
        qb[at] = make_float2(x0, x1);
        qy[at] = y;
      }
      cB += __popc(msk);
      if (cB >= 32) {
        __syncwarp();
        const float2 v = qb[cB - 32 + lane];
        const float vy = qy[cB - 32 + lane];
        cB -= 32;
        __syncwarp();
        spreadB(v.x, v.y, vy);
      }
    }
  }
  __syncwarp();
  if (MU && lane < cA) {
    const float2 v = qa[lane];
    spreadA(v.x, v.y);
  }
  if (R && lane < cB) {
    const float2 v = qb[lane];
    spreadB(v.x, v.y, qy[lane]);
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  if (MU) {
    int* dst = (int*)g.partA + (int64_t)blockIdx.x * g.gA.rows * g.gA.G;
    for (int i = threadIdx.x; i < g.gA.rows * g.gA.G; i += blockDim.x) dst[i] = A[i];
  }
  if (R) {
    int* dst = (int*)g.partB + (int64_t)blockIdx.x * g.gB.rows * g.gB.G;
    for (int i = threadIdx.x; i < g.gB.rows * g.gB.G; i += blockDim.x) dst[i] = B[i];
  }
}

// fp64 path (any input dtype): fp64 window, 64-bit fixed point (pair_add; weights x 2^40, rhs with
// a per-CTA power-of-two scale of Y, |Y| outliers exact in fp64 into the carry grid), 1024 threads
template <int W, typename XT>
__global__ void __launch_bounds__(1024, 1) k_spread2d_f64(const XT* __restrict__ X, const XT* __restrict__ Y, Args2 g, bool MU, bool R) {
  extern __shared__ unsigned smp2[];
  const int cellsA = MU ? g.gA.rows * g.gA.G : 0, cellsB = R ? g.gB.rows * g.gB.G : 0;
  unsigned* Alo = smp2;
  int* Ahi = (int*)(Alo + cellsA);
  unsigned* Blo = smp2 + 2 * cellsA;
  int* Bhi = (int*)(Blo + cellsB);
  const int tile = blockIdx.x % g.T;
  const int chunk = blockIdx.x / g.T;
  for (int i = threadIdx.x; i < 2 * (cellsA + cellsB); i += blockDim.x) smp2[i] = 0u;
  const int64_t beg = (int64_t)chunk * g.per;
  const int64_t end = min(g.n, beg + g.per);
  int E = 0;
  if (R) {  // rhs scale 2^E with max |Y| 2^E in [2^19, 2^20) over the chunk's first samples
    __shared__ double red[32];
    __shared__ int sE;
    double mx = 0.0;
    const int64_t cnt = max((int64_t)0, min(end - beg, (int64_t)4096));
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double v = fabs((double)Y[beg + i]);
      if (v == v) mx = fmax(mx, v);
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
  const double sy = R ? ldexp(1.0, E) : 0.0;
  const double unitA = 4294967296.0 / kSX, unitB = R ? ldexp(4294967296.0, -(E + 20)) : 0.0;
  const int rA0 = tile * g.gA.R, rB0 = tile * g.gB.R;
  double* carA = g.carryA ? g.carryA + (int64_t)rA0 * g.gA.G : nullptr;  // local cell index -> global carry
  double* carB = g.carryB ? g.carryB + (int64_t)rB0 * g.gB.G : nullptr;
  bool bad = false;
  double px[W], py[W];
  for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
    const double x0 = (double)X[j * g.sn], x1 = (double)X[j * g.sn + g.sd];
    const double p0 = x0 * g.a_d, p1 = x1 * g.a_d;
    const double P0 = floor(p0), P1_ = floor(p1);
    const double f0 = p0 - P0, f1 = p1 - P1_;
    if (!(fabs(p0) < 1e8 && fabs(p1) < 1e8)) {
      if (tile == 0) bad = true;
      continue;
    }
    const int d00 = first_tap_d(f0, W);
    const int d01 = first_tap_d(f1, W);
    const int lrA = (int)P0 + g.KA + d00, lcA = (int)P1_ + g.KA + d01;
    if ((unsigned)lrA > (unsigned)(g.gA.G - W) || (unsigned)lcA > (unsigned)(g.gA.G - W)) {
      if (tile == 0) bad = true;
      continue;
    }
    if (MU && lrA >= rA0 && lrA < rA0 + g.gA.R) {
      es_taps2_horner<W>(f0, d00, f1, d01, py, px);
#pragma unroll 1
      for (int a = 0; a < W; ++a) pair_add_row<W>(Alo, Ahi, (lrA - rA0 + a) * g.gA.G + lcA, py[a] * kSX, px, carA, unitA);
    }
    if (R) {
      const double h0 = 0.5 * p0, h1 = 0.5 * p1;
      const double H0 = floor(h0), H1 = floor(h1);
      const double g0 = h0 - H0, g1 = h1 - H1;
      const int e0 = first_tap_d(g0, W);
      const int e1 = first_tap_d(g1, W);
      const int lrB = (int)H0 + g.KB + e0, lcB = (int)H1 + g.KB + e1;
      if (lrB >= rB0 && lrB < rB0 + g.gB.R) {
        es_taps2_horner<W>(g0, e0, g1, e1, py, px);
        const double y = (double)Y[j];
        const double ys = y * sy;
        if (fabs(ys) < 2097152.0) {
#pragma unroll 1
          for (int a = 0; a < W; ++a) pair_add_row<W>(Blo, Bhi, (lrB - rB0 + a) * g.gB.G + lcB, py[a] * ys * 1048576.0, px, carB, unitB);
        } else {  // |Y| outlier or NaN: exact fp64 into the carry grid
          for (int a = 0; a < W; ++a)
            for (int b = 0; b < W; ++b) atomicAdd(carB + (lrB - rB0 + a) * g.gB.G + lcB + b, y * py[a] * px[b]);
        }
      }
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  if (MU) {
    double* dst = (double*)g.partA + (int64_t)blockIdx.x * cellsA;
    for (int i = threadIdx.x; i < cellsA; i += blockDim.x) dst[i] = ((double)Ahi[i] * 4294967296.0 + (double)Alo[i]) / kSX;
  }
  if (R) {
    double* dst = (double*)g.partB + (int64_t)blockIdx.x * cellsB;
    const double sc = ldexp(1.0, -(E + 20));
    for (int i = threadIdx.x; i < cellsB; i += blockDim.x) dst[i] = ((double)Bhi[i] * 4294967296.0 + (double)Blo[i]) * sc;
  }
}

// Cross moments: grid per pair, points (X_l1, -X_l2), unit weight; CTA = (chunk, pair group).
constexpr int kMaxXCtas = 148 * 4;
struct ArgsX {
  int64_t n, sn, sd, per;
  int w;
  float beta_f;
  double beta_d;
  float a_hi, a_lo;
  double a_d;
  int K;       // centre offset
  int G;       // occupied cells per dim
  int npairs, per_cta, ngroups;
  int pl1[528], pl2[528];
  void* part;
  double* carry;  // npairs x G x G
  int* d_status;
  // balanced split (one pair per CTA): CTA c spreads the sample-pair units [ubeg[c], ubeg[c+1]) of
  // the npairs x n sequence -- at most a few pair segments -- into partial slots slot0[c], ...;
  // pair p owns slots [pslot[p], pslot[p+1]) (consecutive, in CTA order)
  int balanced, nctas;
  int64_t ubeg[kMaxXCtas + 1];
  int slot0[kMaxXCtas + 1];
  int pslot[529];
};

// balanced split: CTA blockIdx.x walks its units pair segment by pair segment (one pair grid in
// shared memory at a time), writing one partial slot per segment
template <int W, bool EXACT>
__device__ void cross_balanced(const float* __restrict__ X, const ArgsX& g, int* smx) {
  const int cells = g.G * g.G;
  const int64_t u0 = g.ubeg[blockIdx.x], u1 = g.ubeg[blockIdx.x + 1];
  int slot = g.slot0[blockIdx.x];
  Tile t{g.G, g.K, g.G, g.G};
  bool bad = false;
  float px[W], py[W];
  for (int64_t u = u0; u < u1;) {
    const int p = (int)(u / g.n);
    const int64_t beg = u - (int64_t)p * g.n, end = min(g.n, u1 - (int64_t)p * g.n);
    for (int i = threadIdx.x; i < cells; i += blockDim.x) smx[i] = 0;
    __syncthreads();
    const int l1 = g.pl1[p], l2 = g.pl2[p];
    double* carry = g.carry + (int64_t)p * cells;
    for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
      const float x0 = X[j * g.sn + l1 * g.sd];
      const float x1 = -X[j * g.sn + l2 * g.sd];
      const P1 q0 = place_f32<EXACT>(x0, g.a_hi, g.a_lo);
      const P1 q1 = place_f32<EXACT>(x1, g.a_hi, g.a_lo);
      const int d00 = first_tap(q0.f, W), d01 = first_tap(q1.f, W);
      const int lr = q0.P + g.K + d00, lc = q1.P + g.K + d01;
      if ((unsigned)lr > (unsigned)(g.G - W) || (unsigned)lc > (unsigned)(g.G - W) || x0 != x0 || x1 != x1) {
        bad = true;
        continue;
      }
      es_taps_f32<W>(q0.f, d00, g.beta_f, py);
      es_taps_f32<W>(q1.f, d01, g.beta_f, px);
      spread_fixed<false, W>(smx, t, lr, lc, py, px, kS2, carry, 0, kInvS2);
    }
    __syncthreads();
    int* dst = (int*)g.part + (int64_t)slot * cells;
    for (int i = threadIdx.x; i < cells; i += blockDim.x) dst[i] = smx[i];
    ++slot;
    u = (int64_t)(p + 1) * g.n;
    __syncthreads();
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
}

template <int W, bool EXACT>
__global__ void __launch_bounds__(1024) k_cross2d_fixed(const float* __restrict__ X, const ArgsX* __restrict__ gp) {
  extern __shared__ int smx[];
  const ArgsX& g = *gp;
  if (g.balanced) {
    cross_balanced<W, EXACT>(X, g, smx);
    return;
  }
  const int grp = blockIdx.x % g.ngroups;
  const int chunk = blockIdx.x / g.ngroups;
  const int p0 = grp * g.per_cta;
  const int np = min(g.per_cta, g.npairs - p0);
  const int cells = g.G * g.G;
  for (int i = threadIdx.x; i < np * cells; i += blockDim.x) smx[i] = 0;
  __syncthreads();
  const int64_t beg = (int64_t)chunk * g.per;
  const int64_t end = min(g.n, beg + g.per);
  Tile t{g.G, g.K, g.G, g.G};
  bool bad = false;
  float px[W], py[W];
  for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
    for (int q = 0; q < np; ++q) {
      const int l1 = g.pl1[p0 + q], l2 = g.pl2[p0 + q];
      const float x0 = X[j * g.sn + l1 * g.sd];
      const float x1 = -X[j * g.sn + l2 * g.sd];
      const P1 q0 = place_f32<EXACT>(x0, g.a_hi, g.a_lo);
      const P1 q1 = place_f32<EXACT>(x1, g.a_hi, g.a_lo);
      const int d00 = first_tap(q0.f, W), d01 = first_tap(q1.f, W);
      const int lr = q0.P + g.K + d00, lc = q1.P + g.K + d01;
      if ((unsigned)lr > (unsigned)(g.G - W) || (unsigned)lc > (unsigned)(g.G - W) || x0 != x0 || x1 != x1) {
        bad = true;
        continue;
      }
      es_taps_f32<W>(q0.f, d00, g.beta_f, py);
      es_taps_f32<W>(q1.f, d01, g.beta_f, px);
      spread_fixed<false, W>(smx + q * cells, t, lr, lc, py, px, kS2, g.carry + (int64_t)(p0 + q) * cells, 0, kInvS2);
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  int* dst = (int*)g.part + ((int64_t)chunk * g.npairs + p0) * cells;
  for (int i = threadIdx.x; i < np * cells; i += blockDim.x) dst[i] = smx[i];
}

// fp64-accuracy cross moments: unit weights, 64-bit fixed point (pair_add) in shared memory,
// 1024-thread CTAs (a pair grid of 124^2 cells x 8 B leaves room for one CTA per SM)
template <int W, typename XT>
__global__ void __launch_bounds__(1024, 1) k_cross2d_f64(const XT* __restrict__ X, const ArgsX* __restrict__ gp) {
  extern __shared__ unsigned smxp[];
  const ArgsX& g = *gp;
  const int grp = blockIdx.x % g.ngroups;
  const int chunk = blockIdx.x / g.ngroups;
  const int p0 = grp * g.per_cta;
  const int np = min(g.per_cta, g.npairs - p0);
  const int cells = g.G * g.G;
  for (int i = threadIdx.x; i < 2 * np * cells; i += blockDim.x) smxp[i] = 0u;
  __syncthreads();
  const int64_t beg = (int64_t)chunk * g.per;
  const int64_t end = min(g.n, beg + g.per);
  const double unit = 4294967296.0 / kSX;
  bool bad = false;
  double px[W], py[W];
  for (int64_t j = beg + threadIdx.x; j < end; j += blockDim.x) {
    for (int q = 0; q < np; ++q) {
      const int l1 = g.pl1[p0 + q], l2 = g.pl2[p0 + q];
      const double pa = (double)X[j * g.sn + l1 * g.sd] * g.a_d, pb = -(double)X[j * g.sn + l2 * g.sd] * g.a_d;
      if (!(fabs(pa) < 1e8 && fabs(pb) < 1e8)) {
        bad = true;
        continue;
      }
      const double Pa = floor(pa), Pb = floor(pb), fa = pa - Pa, fb = pb - Pb;
      const int d00 = first_tap_d(fa, W);
      const int d01 = first_tap_d(fb, W);
      const int lr = (int)Pa + g.K + d00, lc = (int)Pb + g.K + d01;
      if ((unsigned)lr > (unsigned)(g.G - W) || (unsigned)lc > (unsigned)(g.G - W)) {
        bad = true;
        continue;
      }
      es_taps2_horner<W>(fa, d00, fb, d01, py, px);
      unsigned* lo = smxp + 2 * q * cells;
      int* hi = (int*)(lo + cells);
      double* carry = g.carry + (int64_t)(p0 + q) * cells;
#pragma unroll 1
      for (int a = 0; a < W; ++a) pair_add_row<W>(lo, hi, (lr + a) * g.G + lc, py[a] * kSX, px, carry, unit);
    }
  }
  if (bad && g.d_status) atomicOr(g.d_status, (int)FK_E_RANGE);
  __syncthreads();
  double* dst = (double*)g.part + ((int64_t)chunk * g.npairs + p0) * cells;
  for (int i = threadIdx.x; i < np * cells; i += blockDim.x) {
    const int q = i / cells, c = i % cells;
    const unsigned* lo = smxp + 2 * q * cells;
    const int* hi = (const int*)(lo + cells);
    dst[i] = ((double)hi[c] * 4294967296.0 + (double)lo[c]) / kSX;
  }
}

// ------------------------------------------------------------------------------------------
// partial tiles -> full-period fp64 grid (fixed order), per batch item
// ------------------------------------------------------------------------------------------
// tiles: cta = chunk*T + t holds rows [t R, t R + rows) of the G x G occupied block
__global__ void k_reduce2d(const void* __restrict__ part, int is_fixed, const int* __restrict__ escale, int nchunks, int T, int R,
                           int rows, int G, int off, int nf, double uniform_inv, const double* __restrict__ carry,
                           double* __restrict__ fine, int batch, int64_t part_batch_stride, int64_t part_cta_stride) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nf * nf;
  if (t >= per * batch) return;
  const int bi = (int)(t / per);
  const int64_t c = t % per;
  const int r = (int)(c / nf) - off, col = (int)(c % nf) - off;
  double s = 0.0;
  if (r >= 0 && r < G && col >= 0 && col < G) {
    for (int tt = 0; tt < T; ++tt) {
      const int lr = r - tt * R;
      if (lr < 0 || lr >= rows) continue;
      for (int ch = 0; ch < nchunks; ++ch) {
        const int64_t cta = (int64_t)ch * T + tt;
        const int64_t idx = bi * part_batch_stride + cta * part_cta_stride + (int64_t)lr * G + col;
        if (is_fixed) {
          const double v = (double)((const int*)part)[idx];
          s += escale ? v * pow2(-escale[cta]) : v * uniform_inv;
        } else {
          s += ((const double*)part)[idx];
        }
      }
    }
    if (carry) s += carry[(int64_t)bi * G * G + (int64_t)r * G + col];
  }
  fine[t] = s;
}

// balanced cross moments: pair bi sums its slots [pslot[bi], pslot[bi+1]) in slot order
__global__ void k_reduce_slots(const int* __restrict__ part, const ArgsX* __restrict__ gp, int off, int nf, double inv,
                               const double* __restrict__ carry, double* __restrict__ fine) {
  const ArgsX& g = *gp;
  const int G = g.G;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)nf * nf;
  if (t >= per * g.npairs) return;
  const int bi = (int)(t / per);
  const int64_t c = t % per;
  const int r = (int)(c / nf) - off, col = (int)(c % nf) - off;
  double s = 0.0;
  if (r >= 0 && r < G && col >= 0 && col < G) {
    const int64_t cell = (int64_t)r * G + col;
    for (int sl = g.pslot[bi]; sl < g.pslot[bi + 1]; ++sl) s += (double)part[(int64_t)sl * G * G + cell] * inv;
    s += carry[(int64_t)bi * G * G + cell];
  }
  fine[t] = s;
}


}  // namespace

// ------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------
// the tap count dispatch_w64 instantiates for w (its Horner table must match)
static int w64_of(int w) { return (w >= 9 && w <= 15) ? w : 16; }

template <typename F>
static void dispatch_w64(int w, F&& f) {
  switch (w) {
    case 9: f(std::integral_constant<int, 9>{}); break;
    case 10: f(std::integral_constant<int, 10>{}); break;
    case 11: f(std::integral_constant<int, 11>{}); break;
    case 12: f(std::integral_constant<int, 12>{}); break;
    case 13: f(std::integral_constant<int, 13>{}); break;
    case 14: f(std::integral_constant<int, 14>{}); break;
    case 15: f(std::integral_constant<int, 15>{}); break;
    default: f(std::integral_constant<int, 16>{}); break;
  }
}

struct Plan2 {
  int m, w;
  double beta;
  bool fp64;
  int nfA, nfB;
  Tile gA, gB;
  int offA, offB, KA, KB;
  int T, chunks, threads;
  size_t smem;
};

static int max_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v > 0 ? v : 232448;
}

// taps per dimension: fp32 fixed-point path 5..8 (eps >= 1e-7), fp64 path 9..16
static int es_width(double eps, bool fp64acc) {
  if (!fp64acc) return std::min(8, std::max(5, (int)std::ceil(std::log10(1.0 / eps)) + 1));
  if (eps >= 1e-7) return 9;
  return std::min(kW, std::max(9, (int)std::ceil(std::log10(1.0 / eps)) + 2));
}

// Geometry of one ES grid: local index = global - off, centre nf/2 at local K, occupied G cells.
static void es_geo(int nf, int w, int* off, int* K, int* G) {
  *off = nf / 4 - w / 2 - 2;
  *K = nf / 2 - *off;
  *G = nf / 2 + w + 4;
}

// fp64 = 64-bit fixed-point accumulation (and fp64 window taps): eps < 1e-7 or fp64 input coordinates
static fk_status make_plan2(int m, double eps, bool mu, bool r, int dtype, Plan2* p) {
  Plan2 q{};
  q.m = m;
  q.fp64 = eps < 1e-7 || dtype == FK_F64;
  q.w = es_width(eps, q.fp64);
  q.beta = 2.30 * q.w;
  // sigma = 2.  sigma = 4 (as the cross moments) saves a tap per dimension (w = 6 at eps = 1e-6:
  // 2 x 36 instead of 2 x 49 atomics per sample) but quadruples the grid, so more row tiles each
  // re-scan the chunk: measured C3 82.3 vs 54.8 ms, C4 5.91 vs 5.95 ms per fit -- not the default.
  // FK_SPREAD2D_SIGMA=4 selects it (fp32 path; measurement).
  int sigma = 2;
  if (const char* e = getenv("FK_SPREAD2D_SIGMA")) sigma = (atoi(e) == 4 && !q.fp64) ? 4 : 2;
  if (sigma == 4) {
    q.w = std::max(5, q.w - 1);
    q.beta = 0.97 * 3.14159265358979 * (1.0 - 1.0 / (2.0 * sigma)) * q.w;
  }
  // tiles (nf/2 + w + 4 cells from nf/4 - w/2 - 2) must not wrap: nfB = nfA/2 >= 2w + 8
  q.nfA = fft_friendly(std::max(sigma * (4 * m + 1), 4 * q.w + 16));
  q.nfB = q.nfA / 2;
  int GA, GB;
  es_geo(q.nfA, q.w, &q.offA, &q.KA, &GA);
  es_geo(q.nfB, q.w, &q.offB, &q.KB, &GB);
  const size_t esz = q.fp64 ? 8 : 4;
  const size_t cap = (size_t)max_optin() - 2048;
  // fp32 path: + per-warp compaction queues (16 warps x 64 x (float2 + float2 + float)), 16-byte aligned
  const size_t queues = q.fp64 ? 0 : (size_t)32 * 64 * 20 + 16;  // 32 warps
  for (int T = 1; T <= 64; ++T) {
    const int RA = (GA + T - 1) / T, RB = (GB + T - 1) / T;
    size_t bytes = ((mu ? (size_t)(RA + q.w - 1) * GA : 0) + (r ? (size_t)(RB + q.w - 1) * GB : 0)) * esz;
    bytes = ((bytes + 15) & ~(size_t)15) + queues;
    if (bytes <= cap) {
      q.T = T;
      q.gA = {GA, q.KA, RA, RA + q.w - 1};
      q.gB = {GB, q.KB, RB, RB + q.w - 1};
      q.smem = bytes;
      break;
    }
  }
  if (q.T == 0) return fail(FK_E_UNSUPPORTED, "d=2 grid too large for 64 row tiles");
  q.threads = 1024;
  const int sms = device_sm_count();
  const int per_sm = std::max(1, std::min(4, (int)(cap / (q.smem + 1024))));
  q.chunks = std::max(1, (sms * per_sm) / q.T);
  *p = q;
  return FK_OK;
}

struct Ws2 {
  void* partA = nullptr;
  void* partB = nullptr;
  int* escale = nullptr;
  double* carryA = nullptr;
  double* carryB = nullptr;
  double* fineA = nullptr;
  double* fineB = nullptr;
  double* tabA = nullptr;
  double* tabB = nullptr;
  void* work = nullptr;
  size_t work_bytes = 0;
  int* gsync = nullptr;
};

static fk_status layout2(const Plan2& p, bool mu, bool r, Bump& b, Ws2& w) {
  const size_t esz = p.fp64 ? 8 : 4;
  const int ctas = p.chunks * p.T;
  size_t fw = 0;
  if (mu) {
    fw = std::max(fw, dft2d_ws_bytes(p.nfA, p.gA.G, 2 * p.m, 1));
    w.partA = b.take((size_t)ctas * p.gA.rows * p.gA.G * esz);
    w.fineA = (double*)b.take((size_t)p.nfA * p.nfA * 8);
    w.tabA = (double*)b.take((size_t)(2 * p.m + 1) * 8);
    w.carryA = (double*)b.take((size_t)p.gA.G * p.gA.G * 8);  // fixed point: drained cells (both paths)
  }
  if (r) {
    fw = std::max(fw, dft2d_ws_bytes(p.nfB, p.gB.G, p.m, 1));
    w.partB = b.take((size_t)ctas * p.gB.rows * p.gB.G * esz);
    w.fineB = (double*)b.take((size_t)p.nfB * p.nfB * 8);
    w.tabB = (double*)b.take((size_t)(p.m + 1) * 8);
    w.carryB = (double*)b.take((size_t)p.gB.G * p.gB.G * 8);
    if (!p.fp64) w.escale = (int*)b.take((size_t)ctas * 4);
  }
  w.work = b.take(std::max<size_t>(fw, 256));  // the hand-written DFT's scratch (dft2d.cu)
  w.work_bytes = std::max<size_t>(fw, 256);
  w.gsync = (int*)b.take((size_t)p.chunks * 4 + 16);
  return FK_OK;
}

size_t type1_2d_ws_bytes(int m, double eps, bool mu, bool r, int dtype) {
  Plan2 p;
  if (make_plan2(m, eps, mu, r, dtype, &p) != FK_OK) return 0;
  Bump b(nullptr, 0);
  Ws2 w;
  if (layout2(p, mu, r, b, w) != FK_OK) return 0;
  return b.used + 256;
}

fk_status type1_2d_run(int m, double eps, const fk_points& X, const void* Y, double L, double* mu_out, double* r_out, bool acc, void* ws,
                       size_t ws_bytes, int* d_status, cudaStream_t s) {
  const bool mu = mu_out != nullptr, r = r_out != nullptr;
  Plan2 p;
  FK_TRY(make_plan2(m, eps, mu, r, X.dtype, &p));
  Bump b(ws, ws_bytes);
  Ws2 w;
  FK_TRY(layout2(p, mu, r, b, w));
  if (!b.ok()) return fail(FK_E_WORKSPACE, "workspace too small");
  const int ctas = p.chunks * p.T;
  const size_t esz = p.fp64 ? 8 : 4;
  if (mu && w.carryA) FK_CUDA_TRY(cudaMemsetAsync(w.carryA, 0, (size_t)p.gA.G * p.gA.G * 8, s));
  if (r && w.carryB) FK_CUDA_TRY(cudaMemsetAsync(w.carryB, 0, (size_t)p.gB.G * p.gB.G * 8, s));
  Args2 a{};
  a.n = X.n;
  a.sn = X.stride_n;
  a.sd = X.stride_d;
  a.aos2 = X.dtype == FK_F32 && X.stride_n == 2 && X.stride_d == 1 && ((uintptr_t)X.ptr & 7) == 0;
  a.per = (X.n + p.chunks - 1) / p.chunks;
  a.w = p.w;
  a.beta_f = (float)(p.beta * 1.4426950408889634);  // beta log2(e) for the ex2-based taps
  a.beta_d = p.beta;
  const double ad = (double)p.nfA / (4.0 * L);
  a.a_d = ad;
  a.a_hi = (float)ad;
  a.a_lo = (float)(ad - (double)a.a_hi);
  int ex = 0;
  const bool exact = std::frexp(ad, &ex) == 0.5;
  a.T = p.T;
  a.gA = p.gA;
  a.gB = p.gB;
  a.KA = p.KA;
  a.KB = p.KB;
  a.partA = w.partA;
  a.partB = w.partB;
  a.escale = w.escale;
  a.carryA = w.carryA;
  a.carryB = w.carryB;
  a.d_status = d_status;
  if (p.T > 1 && !p.fp64) {
    FK_CUDA_TRY(cudaMemsetAsync(w.gsync, 0, (size_t)p.chunks * 4, s));
    a.gsync = w.gsync;
  }
  if (X.n > 0) {
    if (!p.fp64) {
      const float* Xf = (const float*)X.ptr;
      const float* Yf = (const float*)Y;
      auto go = [&](auto k) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        prof_spread_begin(s);
        k<<<ctas, p.threads, p.smem, s>>>(Xf, Yf, a);
        prof_spread_end(s);
      };
      auto byw = [&](auto wtag) {
        constexpr int WW = decltype(wtag)::value;
        if (mu && r) exact ? go(k_spread2d_fixed<WW, true, true, true>) : go(k_spread2d_fixed<WW, true, true, false>);
        else if (mu) exact ? go(k_spread2d_fixed<WW, true, false, true>) : go(k_spread2d_fixed<WW, true, false, false>);
        else exact ? go(k_spread2d_fixed<WW, false, true, true>) : go(k_spread2d_fixed<WW, false, true, false>);
      };
      switch (p.w) {
        case 5: byw(std::integral_constant<int, 5>{}); break;
        case 6: byw(std::integral_constant<int, 6>{}); break;
        case 7: byw(std::integral_constant<int, 7>{}); break;
        default: byw(std::integral_constant<int, 8>{}); break;
      }
    } else {
      auto go = [&](auto k, auto* Xp, auto* Yp) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        prof_spread_begin(s);
        k<<<ctas, p.threads, p.smem, s>>>(Xp, Yp, a, mu, r);
        prof_spread_end(s);
      };
      auto byw = [&](auto wtag) {
        constexpr int WW = decltype(wtag)::value;
        if (X.dtype == FK_F32) go(k_spread2d_f64<WW, float>, (const float*)X.ptr, (const float*)Y);
        else go(k_spread2d_f64<WW, double>, (const double*)X.ptr, (const double*)Y);
      };
      FK_TRY(upload_es2_table(w64_of(p.w), p.beta, s));
      dispatch_w64(p.w, byw);
    }
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
  } else {
    if (mu) FK_CUDA_TRY(cudaMemsetAsync(w.partA, 0, (size_t)ctas * p.gA.rows * p.gA.G * esz, s));
    if (r) FK_CUDA_TRY(cudaMemsetAsync(w.partB, 0, (size_t)ctas * p.gB.rows * p.gB.G * esz, s));
    if (r && w.escale) FK_CUDA_TRY(cudaMemsetAsync(w.escale, 0, (size_t)ctas * 4, s));
  }
  // the fp64 kernel is also used for fp32 inputs when the fp64 path is selected, and for fp64
  // inputs on the fp32 path (its partials are then doubles)
  const bool fixed = !p.fp64;
  EsParams es{p.w, p.beta};
  const int TB = 256;
  auto finish = [&](void* part, int* esc, const Tile& g, int off, int nf, double* carry, double* fine, double* tab,
                    int K, double* out) -> fk_status {
    const int64_t tot = (int64_t)nf * nf;
    k_reduce2d<<<(unsigned)((tot + TB - 1) / TB), TB, 0, s>>>(part, fixed ? 1 : 0, esc, p.chunks, p.T, g.R, g.rows, g.G, off, nf,
                                                             kInvS2, carry, fine, 1, 0,
                                                             (int64_t)g.rows * g.G);
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
    FK_TRY(es_phihat_table(es, nf, K, tab, s));
    return dft2d_run(fine, nf, off, g.G, K, 1, tab, out, acc ? 1 : 0, w.work, w.work_bytes, s);
  };
  if (mu) FK_TRY(finish(w.partA, nullptr, p.gA, p.offA, p.nfA, w.carryA, w.fineA, w.tabA, 2 * m, mu_out));
  if (r) FK_TRY(finish(w.partB, w.escale, p.gB, p.offB, p.nfB, w.carryB, w.fineB, w.tabB, m, r_out));
  return FK_OK;
}

// ------------------------------------------------------------------------------------------
// additive cross moments
// ------------------------------------------------------------------------------------------
struct PlanX {
  int m, w, nf, off, K, G, npairs, per_cta, ngroups, chunks, threads;
  double beta;
  bool fp64;
  bool by_pair;   // one pair grid does not fit a CTA: per-pair 2-D moment passes (cross_by_pair)
  bool balanced;  // one pair per CTA: units split evenly over all resident CTAs (cross_balanced)
  int nctas;
  size_t smem;
};

static fk_status make_planx(int d, int m, double eps, int dtype, PlanX* p) {
  PlanX q{};
  q.m = m;
  q.fp64 = eps < 1e-7 || dtype == FK_F64;
  q.w = es_width(eps, q.fp64);
  q.beta = 2.30 * q.w;
  // fp32 path: sigma = 4 with one tap fewer per dimension (w = 6 at eps = 1e-6, 2.2e-7 in SURVEY
  // V3) when one pair grid still fits a CTA: 36 instead of 49 atomics per sample and pair
  // (C5: 1040 -> 820 ms per fit); sigma = 2 otherwise.  FK_CROSS_SIGMA=2|4 overrides (experiments).
  int sigma = 2;
  if (!q.fp64) {
    const int w4 = std::max(5, q.w - 1);
    const int nf4 = fft_friendly(std::max(4 * (2 * m + 1), 2 * w4 + 8));
    const size_t g4 = (size_t)(nf4 / 2 + w4 + 4);
    if (g4 * g4 * 4 <= (size_t)max_optin() - 2048) sigma = 4;
  }
  if (const char* e = getenv("FK_CROSS_SIGMA")) sigma = atoi(e) == 4 ? 4 : 2;
  if (sigma == 4 && !q.fp64) {
    q.w = std::max(5, q.w - 1);
    q.beta = 0.97 * 3.14159265358979 * (1.0 - 1.0 / (2.0 * sigma)) * q.w;
  }
  q.nf = fft_friendly(std::max(sigma * (2 * m + 1), 2 * q.w + 8));  // tile must not wrap (small m)
  es_geo(q.nf, q.w, &q.off, &q.K, &q.G);
  q.npairs = d * (d - 1) / 2;
  const size_t esz = q.fp64 ? 8 : 4;
  const size_t cap = (size_t)max_optin() - 2048;
  const size_t per = (size_t)q.G * q.G * esz;
  if (per > cap) {  // large m: the tiled 2-D moment pass, one pair at a time
    q.by_pair = true;
    *p = q;
    return FK_OK;
  }
  q.per_cta = (int)std::min<size_t>(q.npairs, cap / per);
  q.ngroups = (q.npairs + q.per_cta - 1) / q.per_cta;
  q.smem = (size_t)q.per_cta * per;
  q.threads = q.fp64 ? 256 : 1024;
  const int sms = device_sm_count();
  const int per_sm = std::max(1, std::min(4, (int)(cap / (q.smem + 1024))));
  // one wave: chunks x groups <= resident CTAs (rounding up left a second wave of a few CTAs
  // that doubled the kernel time)
  q.chunks = std::max(1, (sms * per_sm) / q.ngroups);
  // one pair per CTA (C5: 45 pairs, 1 CTA per SM): chunks x groups = 135 of 148 SMs; the balanced
  // split gives every resident CTA the same number of sample-pair units instead
  q.balanced = !q.fp64 && q.per_cta == 1 && !getenv("FK_CROSS_CHUNKED");
  q.nctas = std::min(kMaxXCtas, sms * per_sm);
  *p = q;
  return FK_OK;
}

static fk_status layoutx(const PlanX& p, Bump& b, void** part, double** carry, double** fine, double2** spec, double** tab, void** work,
                         ArgsX** args) {
  const size_t esz = p.fp64 ? 8 : 4;
  *part = b.take((size_t)std::max(p.chunks * p.npairs, p.nctas + p.npairs) * p.G * p.G * esz);
  *carry = (double*)b.take((size_t)p.npairs * p.G * p.G * 8);
  *fine = (double*)b.take((size_t)p.npairs * p.nf * p.nf * 8);
  *spec = nullptr;
  *tab = (double*)b.take((size_t)(p.m + 1) * 8);
  *args = (ArgsX*)b.take(sizeof(ArgsX));
  *work = b.take(dft2d_ws_bytes(p.nf, p.G, p.m, p.npairs));  // the hand-written DFT's scratch (dft2d.cu)
  return FK_OK;
}

// Large-m cross moments (a pair grid exceeds one CTA's shared memory).  The pair (l1, l2) moments
// are the 2-D unit-weight moments of the points (X_l1, X_l2) read at q = (a, -b):
//   G_{a,b} = sum_j exp(-i (a t_{j,l1} - b t_{j,l2})) = mu_{(a,-b)},  |a|, |b| <= m,
// so each pair is one tiled type-1 pass (type1_2d_run, moments only) at m2 = ceil(m/2), whose
// mode box {-2 m2..2 m2}^2 covers {-m..m}^2, followed by a crop/reflect into G[p].
__global__ void k_cross_from_mu(const double2* __restrict__ mu2, int m2, int m, double2* __restrict__ Gp, int acc) {
  const int K2 = 4 * m2 + 1, D = 2 * m + 1;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)D * D) return;
  const int a = (int)(t / D) - m, b = (int)(t % D) - m;
  const double2 v = mu2[(int64_t)(a + 2 * m2) * K2 + (-b + 2 * m2)];
  if (acc) {
    Gp[t].x += v.x;
    Gp[t].y += v.y;
  } else {
    Gp[t] = v;
  }
}

static size_t cross_by_pair_ws(int m, double eps, int dtype) {
  const int m2 = (m + 1) / 2;
  const size_t inner = type1_2d_ws_bytes(m2, eps, true, false, dtype);
  if (inner == 0) return 0;
  return (((size_t)(4 * m2 + 1) * (4 * m2 + 1) * 16 + 255) & ~(size_t)255) + inner;
}

static fk_status cross_by_pair(const fk_points& X, double L, int m, double eps, double* G, bool accumulate, void* ws, size_t ws_bytes,
                               int* d_status, cudaStream_t s) {
  const int m2 = (m + 1) / 2;
  const size_t need = cross_by_pair_ws(m, eps, X.dtype);
  if (need == 0) return fail(FK_E_UNSUPPORTED, "fk_additive_cross_moments: no 2-D plan for this m");
  if (ws_bytes < need) return fail(FK_E_WORKSPACE, "workspace too small");
  const size_t mub = ((size_t)(4 * m2 + 1) * (4 * m2 + 1) * 16 + 255) & ~(size_t)255;
  double* mu2 = (double*)ws;
  void* inner = (char*)ws + mub;
  const size_t esz = X.dtype == FK_F64 ? 8 : 4;
  const int D = 2 * m + 1;
  int p = 0;
  for (int l1 = 0; l1 < X.d; ++l1)
    for (int l2 = l1 + 1; l2 < X.d; ++l2, ++p) {
      fk_points Xp = X;
      Xp.ptr = (const char*)X.ptr + (size_t)l1 * X.stride_d * esz;
      Xp.d = 2;
      Xp.stride_d = (int64_t)(l2 - l1) * X.stride_d;
      FK_TRY(type1_2d_run(m2, eps, Xp, nullptr, L, mu2, nullptr, false, inner, ws_bytes - mub, d_status, s));
      k_cross_from_mu<<<(D * D + 255) / 256, 256, 0, s>>>((const double2*)mu2, m2, m, (double2*)G + (int64_t)p * D * D,
                                                          accumulate ? 1 : 0);
      FK_CUDA_TRY(cudaGetLastError());
      count_launch();
    }
  return FK_OK;
}

size_t cross_ws_bytes(int d, int m, double eps, int64_t n, int dtype) {
  (void)n;
  if (d < 2) return 0;
  PlanX p;
  if (make_planx(d, m, eps, dtype, &p) != FK_OK) return 0;
  if (p.by_pair) return cross_by_pair_ws(m, eps, dtype);
  Bump b(nullptr, 0);
  void *part, *work;
  double *carry, *fine, *tab;
  double2* spec;
  ArgsX* args;
  if (layoutx(p, b, &part, &carry, &fine, &spec, &tab, &work, &args) != FK_OK) return 0;
  return b.used + 256;
}

fk_status cross_run(const fk_points& X, double L, int m, double eps, double* G, bool accumulate, void* ws, size_t ws_bytes,
                    int* d_status, cudaStream_t s) {
  PlanX p;
  FK_TRY(make_planx(X.d, m, eps, X.dtype, &p));
  if (p.by_pair) return cross_by_pair(X, L, m, eps, G, accumulate, ws, ws_bytes, d_status, s);
  if (p.npairs > 528) return fail(FK_E_UNSUPPORTED, "fk_additive_cross_moments: at most 528 pairs");
  Bump b(ws, ws_bytes);
  void *part, *work;
  double *carry, *fine, *tab;
  double2* spec;
  ArgsX* dargs;
  FK_TRY(layoutx(p, b, &part, &carry, &fine, &spec, &tab, &work, &dargs));
  if (!b.ok()) return fail(FK_E_WORKSPACE, "workspace too small");
  const bool fixed = !p.fp64;
  static thread_local ArgsX a;  // host staging for the argument block (copied to the workspace)
  a = ArgsX{};
  a.n = X.n;
  a.sn = X.stride_n;
  a.sd = X.stride_d;
  a.per = (X.n + p.chunks - 1) / p.chunks;
  a.w = p.w;
  a.beta_f = (float)(p.beta * 1.4426950408889634);  // beta log2(e) for the ex2-based taps
  a.beta_d = p.beta;
  const double ad = (double)p.nf / (4.0 * L);
  a.a_d = ad;
  a.a_hi = (float)ad;
  a.a_lo = (float)(ad - (double)a.a_hi);
  int ex = 0;
  const bool exact = std::frexp(ad, &ex) == 0.5;
  a.K = p.K;
  a.G = p.G;
  a.npairs = p.npairs;
  a.per_cta = p.per_cta;
  a.ngroups = p.ngroups;
  int q = 0;
  for (int l1 = 0; l1 < X.d; ++l1)
    for (int l2 = l1 + 1; l2 < X.d; ++l2) {
      a.pl1[q] = l1;
      a.pl2[q] = l2;
      ++q;
    }
  a.part = part;
  a.carry = carry;
  a.d_status = d_status;
  a.balanced = p.balanced ? 1 : 0;
  a.nctas = p.nctas;
  if (p.balanced) {
    const int64_t U = (int64_t)p.npairs * X.n;
    int slot = 0, pnext = 0;
    for (int c = 0; c < p.nctas; ++c) {
      const int64_t u0 = (int64_t)((__int128)U * c / p.nctas), u1 = (int64_t)((__int128)U * (c + 1) / p.nctas);
      a.ubeg[c] = u0;
      a.slot0[c] = slot;
      if (u1 > u0) {
        for (int64_t pp = u0 / X.n; pp <= (u1 - 1) / X.n; ++pp, ++slot)
          while (pnext <= pp) a.pslot[pnext++] = slot;  // first slot of pair pp
      }
    }
    a.ubeg[p.nctas] = U;
    a.slot0[p.nctas] = slot;
    while (pnext <= p.npairs) a.pslot[pnext++] = slot;
  }
  FK_CUDA_TRY(cudaMemsetAsync(carry, 0, (size_t)p.npairs * p.G * p.G * 8, s));
  FK_CUDA_TRY(cudaMemcpyAsync(dargs, &a, sizeof(ArgsX), cudaMemcpyHostToDevice, s));
  const int ctas = p.balanced ? p.nctas : p.chunks * p.ngroups;
  const size_t esz = p.fp64 ? 8 : 4;
  if (X.n > 0) {
    auto go = [&](auto k, auto* Xp, int threads) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
      prof_spread_begin(s);
      k<<<ctas, threads, p.smem, s>>>(Xp, dargs);
      prof_spread_end(s);
    };
    if (fixed) {
      auto byw = [&](auto wtag) {
        constexpr int WW = decltype(wtag)::value;
        if (exact) go(k_cross2d_fixed<WW, true>, (const float*)X.ptr, 1024);
        else go(k_cross2d_fixed<WW, false>, (const float*)X.ptr, 1024);
      };
      switch (p.w) {
        case 5: byw(std::integral_constant<int, 5>{}); break;
        case 6: byw(std::integral_constant<int, 6>{}); break;
        case 7: byw(std::integral_constant<int, 7>{}); break;
        default: byw(std::integral_constant<int, 8>{}); break;
      }
    } else {
      auto byw = [&](auto wtag) {
        constexpr int WW = decltype(wtag)::value;
        if (X.dtype == FK_F32) go(k_cross2d_f64<WW, float>, (const float*)X.ptr, 1024);  // fp32 points, fp64 accuracy
        else go(k_cross2d_f64<WW, double>, (const double*)X.ptr, 1024);
      };
      FK_TRY(upload_es2_table(w64_of(p.w), p.beta, s));
      dispatch_w64(p.w, byw);
    }
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
  } else {
    FK_CUDA_TRY(cudaMemsetAsync(part, 0, (size_t)p.chunks * p.npairs * p.G * p.G * esz, s));
  }
  const int TB = 256;
  const int64_t tot = (int64_t)p.npairs * p.nf * p.nf;
  // part layout: [chunk][pair][G][G] -> batch stride G*G, "cta" stride npairs*G*G, T = 1
  if (p.balanced && X.n > 0)
    k_reduce_slots<<<(unsigned)((tot + TB - 1) / TB), TB, 0, s>>>((const int*)part, dargs, p.off, p.nf, kInvS2, carry, fine);
  else
    k_reduce2d<<<(unsigned)((tot + TB - 1) / TB), TB, 0, s>>>(part, fixed ? 1 : 0, nullptr, p.chunks, 1, p.G, p.G, p.G, p.off, p.nf,
                                                             kInvS2, carry, fine, p.npairs, (int64_t)p.G * p.G,
                                                             (int64_t)p.npairs * p.G * p.G);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  (void)spec;
  EsParams es{p.w, p.beta};
  FK_TRY(es_phihat_table(es, p.nf, m, tab, s));
  return dft2d_run(fine, p.nf, p.off, p.G, m, p.npairs, tab, G, accumulate ? 1 : 0, work, dft2d_ws_bytes(p.nf, p.G, m, p.npairs), s);
}

}  // namespace fk
