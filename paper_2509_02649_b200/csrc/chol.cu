// chol.cu -- dense fp64 Cholesky of the (augmented) real fit system, A = L L^T, in ONE persistent
// dataflow kernel (the factorisation step of A11; DESIGN.md §5 "Solve").
//
// Why not cuSOLVER potrf at the fit sizes: for N ~ 2000-3500 its factorisation is latency bound
// (~0.45 us per column, 0.83 ms at N = 2002).  Here the matrix is cut into 32 x 32 tiles and every
// task is owned by one 128-thread CTA:
//   * an off-diagonal tile (i, j), i >= j + 2, loads A_ij into fp64 tensor-core accumulators
//     (mma.m8n8k4.f64, a 16 x 16 quadrant per warp), applies A_ij -= L_ik L_jk^T for k < j as soon
//     as both operand tiles are published (flags), then solves X L_jj^T = A_ij (TRSM, a row per
//     lane, 1/L_cc from the diagonal task);
//   * the diagonal task D_j owns the diagonal tile (j, j) AND the sub-diagonal tile (j+1, j): it
//     accumulates both (updates k < j-1), applies the last update of the diagonal tile with
//     L_{j,j-1} (published by D_{j-1} as data), then runs the 32 x 32 POTRF (warp 0, a row per lane,
//     rsqrt per pivot, column broadcast through shared memory) while warp 1 solves
//     L_{j+1,j} = A_{j+1,j} L_jj^{-T} a quarter of the columns at a time as warp 0 releases them
//     (named barriers, bar.arrive on warp 0's side: it never waits).  Warps 2-3 first subtract the
//     sub-diagonal tile's last update P_j = L_{j+1,j-1} L_{j,j-1}^T, which the off-diagonal task
//     (j+1, j-1) forms right after its own TRSM.  So the TRSM runs beside the POTRF instead of
//     after it on the chain (warp 0 also publishes 1/L_CC per column, so warp 1 has no rsqrt on its
//     own chain).  L_jj, 1/diag(L_jj), L_{j+1,j} and P_j live in a sentinel-filled side buffer that
//     consumers poll as data.  (Round 2: round 1 ran the TRSM of (j, j-1) inside D_j before its
//     POTRF; N = 2002 0.45 -> 0.405 ms, 2600 0.70 -> 0.60, 4226 1.48 -> 1.40 ms.  What remains on the chain
//     per 32 columns: the POTRF, ~3.3 us of fp64 latency, warp 1's lag behind it (the SM is shared
//     with update tasks) and one L2 round trip to the next diagonal task.)
// Tasks are handed out by an atomic ticket counter in dependency order, so a CTA only ever waits
// on tasks with smaller tickets -- held by CTAs that are already running and never wait on larger
// tickets: deadlock free for any grid size, no co-residency assumption.  Tiles are read with
// ld.global.cg (L2) because the same addresses held A before they hold L.
// Padding rows/columns beyond N behave as the identity.  info: first failing pivot + 1 (0 = SPD).
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <vector>
#include <mutex>
#include <map>

#include "fk_internal.cuh"

namespace fk {
namespace {

constexpr int TS = 32;    // tile size
constexpr int LDS = 36;   // smem leading dimension of staged tiles [p][r]: conflict-free stores and fragment loads
constexpr int CT = 128;   // threads per CTA

// Flags are polled with relaxed loads: ld.acquire would invalidate the whole L1 (CCTL.IVALL) on every
// poll; the tile data is read with ld.global.cg (L2, coherent), so no L1 invalidation is needed.
// Ordering (PTX memory model): the producer publishes with st.release; the consumer, once its
// relaxed poll has observed the flag, executes ONE fence.acq_rel.gpu (acquire_fence) before the
// CTA barrier that releases the tile reads, which makes the pattern release -> observe -> acquire
// fence a synchronisation, so the tile loads cannot be satisfied by stale data.
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void acquire_fence() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void st_release(int* p, int v) { asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double elem(const double* __restrict__ M, int64_t ld, int N, int r, int c) {
  if (r < N && c < N) return __ldcg(M + r + (int64_t)c * ld);
  return r == c ? 1.0 : 0.0;
}

// tile (ti, tj) into smem T[p][r] = tile(r, p) (column p of the tile is row p of T)
__device__ __forceinline__ void stage(double (*T)[LDS], const double* __restrict__ M, int64_t ld, int N, int ti, int tj) {
  const int r = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < TS * TS / CT; ++q) {
    const int p = (threadIdx.x >> 5) + 4 * q;
    T[p][r] = elem(M, ld, N, ti * TS + r, tj * TS + p);
  }
}

// Watchdog for every spin-wait: a dependency that is not published within 5 s (it never happens
// in a correct schedule -- the longest legitimate wait is a few ms) ends the wait instead of
// hanging the GPU, and records -1 in *info (unless a pivot failure was recorded first), which
// fk_solve turns into FK_DSTATUS_WATCHDOG / FK_E_SOLVE: the factor is then reported invalid.
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr unsigned long long kSpinLimitNs = 5000000000ULL;

// wait until both flags are set (thread 0 polls fa, thread 32 polls fb; fb may be null)
__device__ __forceinline__ void watchdog_expired(int* info) { atomicCAS(info, 0, -1); }

__device__ __forceinline__ void wait_flags(const int* fa, const int* fb, int* info) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtime();
    while (ld_relaxed(fa) == 0) {
      if (gtime() - t0 >= kSpinLimitNs) {
        watchdog_expired(info);
        break;
      }
    }
    acquire_fence();
  }
  if (threadIdx.x == 32 && fb) {
    const unsigned long long t0 = gtime();
    while (ld_relaxed(fb) == 0) {
      if (gtime() - t0 >= kSpinLimitNs) {
        watchdog_expired(info);
        break;
      }
    }
    acquire_fence();
  }
  __syncthreads();
}

// Diagonal factors are also published to a side buffer Ld[j] = {L_jj as [p][r], 1/diag, L_{j+1,j} as
// [p][r], P_j} that is pre-filled with all-ones bytes (a NaN pattern no arithmetic produces):
// consumers poll the data itself (one L2 round trip) instead of a flag followed by the loads.
// P_j, the last update of D_j's sub-diagonal tile, is formed by the off-diagonal task (j+1, j-1)
// right after its own TRSM, so that D_j's trailing TRSM only has to subtract it.
constexpr int LDW = 3 * TS * TS + TS;     // doubles per side-buffer entry
constexpr int LDW_SUB = TS * TS + TS;     // offset of L_{j+1,j} in an entry
constexpr int LDW_P = 2 * TS * TS + TS;   // offset of P_j = L_{j+1,j-1} L_{j,j-1}^T (row-major), for D_j
constexpr unsigned long long kUnset = ~0ULL;

__device__ __forceinline__ double ld_cg_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}

// Ta[p][r] = L_jj(r, p), dv[c] = 1 / L_jj(c, c) from the side buffer, waiting until published
// (the polled words ARE the data, each an 8-byte value written once, so no fence is needed here)
__device__ __forceinline__ void stage_diag(double (*T)[LDS], double* dv, const double* __restrict__ Ld, int* info) {
  constexpr int PER = TS * TS / CT;
  double v[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) v[q] = ld_cg_volatile(Ld + threadIdx.x + CT * q);
  double d = (threadIdx.x < TS) ? ld_cg_volatile(Ld + TS * TS + threadIdx.x) : 0.0;
  const unsigned long long t0 = gtime();
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (__double_as_longlong(v[q]) == (long long)kUnset) {
        v[q] = ld_cg_volatile(Ld + threadIdx.x + CT * q);
        ok = false;
      }
    if (threadIdx.x < TS && __double_as_longlong(d) == (long long)kUnset) {
      d = ld_cg_volatile(Ld + TS * TS + threadIdx.x);
      ok = false;
    }
    if (ok) break;
    if (gtime() - t0 > kSpinLimitNs) {
      watchdog_expired(info);
      break;
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = threadIdx.x + CT * q;
    T[e / TS][e % TS] = v[q];
  }
  if (threadIdx.x < TS) dv[threadIdx.x] = d;
}

__device__ __forceinline__ bool unset(double v) { return __double_as_longlong(v) == (long long)kUnset; }

// T[p][r] = tile(r, p) from a [p][r] side-buffer block, waiting until published (all threads)
__device__ __forceinline__ void stage_side(double (*T)[LDS], const double* __restrict__ src, int* info) {
  constexpr int PER = TS * TS / CT;
  double v[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) v[q] = ld_cg_volatile(src + threadIdx.x + CT * q);
  const unsigned long long t0 = gtime();
  for (;;) {
    bool ok = true;
#pragma unroll
    for (int q = 0; q < PER; ++q)
      if (unset(v[q])) {
        v[q] = ld_cg_volatile(src + threadIdx.x + CT * q);
        ok = false;
      }
    if (ok) break;
    if (gtime() - t0 > kSpinLimitNs) {
      watchdog_expired(info);
      break;
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int e = threadIdx.x + CT * q;
    T[e / TS][e % TS] = v[q];
  }
}

__device__ __forceinline__ void bar_named(int id, int count) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory"); }

// ticket -> task when there are no U tasks (computed: no table load on the chain): column j holds
// D_j, then the tiles (i, j), i >= j + 2.  Returns (type, i, j, 0).
__device__ __forceinline__ int4 task_of(int t, int nt) {
  int c = 0, start = 0;
  for (;;) {
    const int cnt = 1 + max(0, nt - c - 2);
    if (t < start + cnt) break;
    start += cnt;
    ++c;
  }
  return t == start ? make_int4(0, c, c, 0) : make_int4(1, c + 1 + (t - start), c, 0);
}

__device__ __forceinline__ int tile_id(int i, int j, int nt) { return j * nt - j * (j - 1) / 2 + (i - j); }

// Operand readiness for a run of updates k = k0 .. kend-1 that need tiles (ia, k) and (ib, k):
// one parallel scan of both flag columns finds the first k not yet published (smem min), so the
// ready prefix is consumed without a flag round trip per update; at a not-ready k the CTA waits on
// that k alone and scans again afterwards.  Returns the first k that is NOT known ready (> k0).
__device__ __forceinline__ int ready_prefix(const int* __restrict__ flags, int nt, int ia, int ib, int k0, int kend, int* s_min,
                                            int* info) {
  if (threadIdx.x == 0) *s_min = kend;
  __syncthreads();
  for (int k = k0 + threadIdx.x; k < kend; k += blockDim.x)
    if (!ld_relaxed(flags + tile_id(ia, k, nt)) || !ld_relaxed(flags + tile_id(ib, k, nt))) atomicMin(s_min, k);
  acquire_fence();  // every thread that observed a flag orders the later tile loads after it
  __syncthreads();
  int first = *s_min;
  __syncthreads();
  if (first == k0) {  // nothing ready yet: wait for k0 itself
    wait_flags(flags + tile_id(ia, k0, nt), flags + tile_id(ib, k0, nt), info);
    first = k0 + 1;
  }
  return first;
}

// 32 x 32 POTRF step J on a register-resident row (lane r holds row r, one warp), fully unrolled
// by recursion.  dj = pivot J, inv = rsqrt(dj) (MUFU + Newton, no IEEE sqrt/div).  Lane J+1 forms
// the next pivot from its own l_{J+1,J} and publishes it through shared memory before the general
// update, so the dependency chain per column is mul -> fma -> sts/lds -> rsqrt.  The general update
// reads column J of L from shared memory (broadcast loads) instead of 31 shuffles.  1/L_JJ goes to
// my_dinv (lane J), bad = first non-positive pivot (or -1).
__device__ __forceinline__ void bar_arrive(int id, int count) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory"); }

template <int J>
__device__ __forceinline__ void potrf_step(double (&x)[TS], double (*colL)[LDS], double* piv, double* dinv, int lane, double& my_dinv,
                                           int& bad, double dj, double inv, bool trail) {
  if (!(dj > 0.0) && bad < 0) bad = J;
  const double lj = x[J] * inv;
  x[J] = (lane == J) ? dj * inv : lj;
  if (lane == J) {
    my_dinv = inv;
    dinv[J] = inv;
  }
  colL[J][lane] = lj;
  if constexpr (J + 1 < TS) {
    if (lane == J + 1) piv[J + 1] = fma(-lj, lj, x[J + 1]);
  }
  __syncwarp();
  double dn = 0.0, invn = 0.0;
  if constexpr (J + 1 < TS) {
    dn = piv[J + 1];
    invn = rsqrt(dn);
  }
  // lanes r < c update their (unused, later zeroed) upper entries too: no select on the chain
#pragma unroll
  for (int c = J + 1; c < TS; ++c) x[c] = fma(-lj, colL[J][c], x[c]);
  // columns 8q .. 8q+7 and pivots up to 8q+8 are in shared memory: release them to the trailing
  // TRSM warp (bar.arrive does not wait; the matching bar.sync orders the shared-memory writes)
  if constexpr ((J & 7) == 7) {
    if (trail) bar_arrive(3 + J / 8, 64);
  }
  if constexpr (J + 1 < TS) potrf_step<J + 1>(x, colL, piv, dinv, lane, my_dinv, bad, dn, invn, trail);
}


// warp 1 of D_j, lane r: row r of X L^T = A (the sub-diagonal tile), a quarter (8 columns) at a
// time as soon as warp 0's POTRF has released it (named barrier 3 + q: warp 0 arrives without
// waiting after column 8q + 7, warp 1 syncs): colL[C][c2] = L(c2, C), 1 / L_CC = rsqrt(piv[C])
// (bitwise warp 0's value).  Static unrolled code, one barrier per quarter: no polling.
template <int C, int CEND>
__device__ __forceinline__ void trail_step(double (&x)[TS], const double (*colL)[LDS], const double* dinv) {
  x[C] *= dinv[C];
#pragma unroll
  for (int c2 = C + 1; c2 < TS; ++c2) x[c2] = fma(-x[C], colL[C][c2], x[c2]);
  if constexpr (C + 1 < CEND) trail_step<C + 1, CEND>(x, colL, dinv);
}

__device__ __forceinline__ void trail_rows(double (&x)[TS], const double (*colL)[LDS], const double* dinv) {
  bar_named(3, 64);
  trail_step<0, 8>(x, colL, dinv);
  bar_named(4, 64);
  trail_step<8, 16>(x, colL, dinv);
  bar_named(5, 64);
  trail_step<16, 24>(x, colL, dinv);
  bar_named(6, 64);
  trail_step<24, 32>(x, colL, dinv);
}

// row solve x L^T = a, L(c, p) = T[p][c], 1/L(c, c) = dv[c] (forward substitution, right-looking)
template <int C>
__device__ __forceinline__ void trsm_step(double (&x)[TS], const double (*T)[LDS], const double* dv) {
  x[C] *= dv[C];
#pragma unroll
  for (int c2 = C + 1; c2 < TS; ++c2) x[c2] = fma(-x[C], T[C][c2], x[c2]);
  if constexpr (C + 1 < TS) trsm_step<C + 1>(x, T, dv);
}

struct Acc {
  double v[2][2][2];  // v[rb][cb][e] = tile(qr*16 + rb*8 + g, qc*16 + cb*8 + 2tq + e)
};

__device__ __forceinline__ void acc_load(Acc& a, const double* __restrict__ M, int64_t ld, int N, int ti, int tj, int qr, int qc, int g,
                                         int tq) {
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) a.v[rb][cb][e] = elem(M, ld, N, ti * TS + qr * 16 + rb * 8 + g, tj * TS + qc * 16 + cb * 8 + 2 * tq + e);
}

// a -= A B^T (SUB) or a += A B^T with A, B staged as T[p][r] = tile(r, p)
template <bool SUB = true>
__device__ __forceinline__ void acc_update(Acc& a, const double (*A)[LDS], const double (*B)[LDS], int qr, int qc, int g, int tq) {
#pragma unroll
  for (int p0 = 0; p0 < TS; p0 += 4) {
    double fa[2], fb[2];
#pragma unroll
    for (int rb = 0; rb < 2; ++rb) fa[rb] = SUB ? -A[p0 + tq][qr * 16 + rb * 8 + g] : A[p0 + tq][qr * 16 + rb * 8 + g];  // A frag: row g, k tq
#pragma unroll
    for (int cb = 0; cb < 2; ++cb) fb[cb] = B[p0 + tq][qc * 16 + cb * 8 + g];   // B frag: k tq, col g
#pragma unroll
    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) dmma(a.v[rb][cb][0], a.v[rb][cb][1], fa[rb], fb[cb]);
  }
}

__device__ __forceinline__ void acc_gather(const Acc& a, double (*Ct)[TS + 1], int qr, int qc, int g, int tq) {
#pragma unroll
  for (int rb = 0; rb < 2; ++rb)
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int e = 0; e < 2; ++e) Ct[qr * 16 + rb * 8 + g][qc * 16 + cb * 8 + 2 * tq + e] = a.v[rb][cb][e];
}

// write Ct as tile (ti, tj) of M (ends with a CTA barrier)
__device__ __forceinline__ void store_tile(const double (*Ct)[TS + 1], double* __restrict__ M, int64_t ld, int N, int ti, int tj) {
  const int r = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < TS * TS / CT; ++q) {
    const int c = (threadIdx.x >> 5) + 4 * q;
    const int gr = ti * TS + r, gc = tj * TS + c;
    if (gr < N && gc < N) M[gr + (int64_t)gc * ld] = Ct[r][c];
  }
  __syncthreads();
}

// release a tile stored before the last CTA barrier (called by one thread; the fence makes the
// whole CTA's stores visible at GPU scope before the flag)
__device__ __forceinline__ void release(int* flag) {
  __threadfence();
  st_release(flag, 1);
}

__device__ __forceinline__ void publish(const double (*Ct)[TS + 1], double* __restrict__ M, int64_t ld, int N, int ti, int tj, int* flag) {
  store_tile(Ct, M, ld, N, ti, tj);
  if (threadIdx.x == 0) release(flag);
}

// warp 0: Ct <- Ct L^{-T} (TRSM; L staged in Ta, 1/diag in dv)
__device__ __forceinline__ void final_trsm(double (*Ct)[TS + 1], const double (*Ta)[LDS], const double* dv, int lane) {
  double x[TS];
#pragma unroll
  for (int c = 0; c < TS; ++c) x[c] = Ct[lane][c];
  trsm_step<0>(x, Ta, dv);
#pragma unroll
  for (int c = 0; c < TS; ++c) Ct[lane][c] = x[c];
}

// warp 0: Ct <- chol(Ct) (lower, zero upper), also written with 1/diag to the side buffer entry
// Ld_out; first failing pivot to info
__device__ __forceinline__ void final_potrf(double (*Ct)[TS + 1], double (*colL)[LDS], double* piv, double* dinv, double* Ld_out, int col0,
                                            int N, int* info, int lane, bool trail = false) {
  double x[TS];
#pragma unroll
  for (int c = 0; c < TS; ++c) x[c] = Ct[lane][c];
  double my_dinv = 1.0;
  int bad = -1;
  // (2 x 2 pivot blocks in this one-warp loop -- two independent rsqrt per two columns -- measured
  // 11.3k vs 6.5k cycles per tile: tools/microbench/mb_potrf.cu, profiles/r02_solve_study.md)
  if (lane == 0) piv[0] = x[0];
  __syncwarp();
  const double d0 = piv[0];
  potrf_step<0>(x, colL, piv, dinv, lane, my_dinv, bad, d0, rsqrt(d0), trail);
  if (bad >= 0 && lane == 0 && col0 + bad < N) atomicCAS(info, 0, col0 + bad + 1);
#pragma unroll
  for (int c = 0; c < TS; ++c) {
    x[c] = (c > lane) ? 0.0 : x[c];
    Ct[lane][c] = x[c];
    Ld_out[c * TS + lane] = x[c];  // [p][r] order, coalesced
  }
  Ld_out[TS * TS + lane] = my_dinv;
}

// Partial accumulation tasks U(j, c): the updates k in [cB, cB + B) of D_j's two tiles, summed into
// a scratch buffer (fragment layout) that D_j adds in fixed order c = 0, 1, ... -- so the diagonal
// task, which starts late in ticket order, only has the last < B + 2 updates left on the chain.
constexpr int UB = 16;

template <bool USE_U>
__global__ void __launch_bounds__(CT) k_chol_tiles(double* __restrict__ M, int64_t ld, int N, int nt, int* __restrict__ flags,
                                                   int* __restrict__ ticket, int* __restrict__ info, double* __restrict__ Ld,
                                                   const int4* __restrict__ tasks, int ntasks, double* __restrict__ part,
                                                   int* __restrict__ uflags, int maxc, unsigned long long* __restrict__ trace) {
  __shared__ double Ta[TS][LDS], Tb[TS][LDS];
  __shared__ double Ct[TS][TS + 1], Cs[TS][TS + 1];
  __shared__ double dv[TS], piv[TS], dinv_s[TS];
  __shared__ unsigned long long s_tx, s_tw, s_tw2;  // trace: external flag seen, warp 1 start (diagonal tasks)
  __shared__ int s_t;
  __shared__ int s_min;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int qr = w >> 1, qc = w & 1;  // quadrant of a tile held by this warp
  const int g = lane >> 2, tq = lane & 3;
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(ticket, 1);
    __syncthreads();
    const int t = s_t;
    __syncthreads();
    if (t >= ntasks) return;
    const int4 tk = USE_U ? tasks[t] : task_of(t, nt);
    const int i = tk.y, j = tk.z;
    unsigned long long t0 = 0, t1 = 0, t1b = 0, t1c = 0;
    if (trace && threadIdx.x == 0) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      s_tx = 0;
      s_tw = 0;
      s_tw2 = 0;
    }
    if (USE_U && tk.x == 2) {
      // ---- U(j, c): partial sums of D_j's updates over k in [cB, cB + B) ----
      const int c = tk.w;
      Acc ps, pd;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        (&ps.v[0][0][0])[e] = 0.0;
        (&pd.v[0][0][0])[e] = 0.0;
      }
      int rdy = c * UB;
      const int jb = j + 1 < nt ? j + 1 : j;  // the sub-diagonal tile (j+1, j), if any
      for (int k = c * UB; k < (c + 1) * UB; ++k) {
        if (k >= rdy) rdy = ready_prefix(flags, nt, j, jb, k, (c + 1) * UB, &s_min, info);
        stage(Ta, M, ld, N, j, k);
        stage(Tb, M, ld, N, j + 1, k);
        __syncthreads();
        acc_update(ps, Tb, Ta, qr, qc, g, tq);
        acc_update(pd, Ta, Ta, qr, qc, g, tq);
        __syncthreads();
      }
      double* base = part + ((int64_t)j * maxc + c) * 2 * TS * TS;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        base[e * CT + threadIdx.x] = (&ps.v[0][0][0])[e];
        base[TS * TS + e * CT + threadIdx.x] = (&pd.v[0][0][0])[e];
      }
      __syncthreads();
      if (threadIdx.x == 0) release(uflags + j * maxc + c);
    } else if (i != j) {
      // ---- off-diagonal tile (i, j), i >= j + 2: updates k < j, then TRSM with L_jj ----
      Acc a;
      acc_load(a, M, ld, N, i, j, qr, qc, g, tq);
      int rdy = 0;
      for (int k = 0; k < j; ++k) {
        if (k >= rdy) rdy = ready_prefix(flags, nt, i, j, k, j, &s_min, info);
        stage(Ta, M, ld, N, i, k);
        stage(Tb, M, ld, N, j, k);
        __syncthreads();
        acc_update(a, Ta, Tb, qr, qc, g, tq);
        __syncthreads();
      }
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      acc_gather(a, Ct, qr, qc, g, tq);
      stage_diag(Ta, dv, Ld + (int64_t)j * LDW, info);  // Ta[p][r] = L_jj(r, p)
      __syncthreads();
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1b));
      if (w == 0) final_trsm(Ct, Ta, dv, lane);
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1c));
      __syncthreads();
      if (i == j + 2) {
        // P_{j+1} = L_{j+2,j} L_{j+1,j}^T, the last update of D_{j+1}'s sub-diagonal tile (j+2, j+1)
        stage_side(Ta, Ld + (int64_t)j * LDW + LDW_SUB, info);  // Ta[p][r] = L_{j+1,j}(r, p)
#pragma unroll
        for (int q = 0; q < TS * TS / CT; ++q) {
          const int p = (threadIdx.x >> 5) + 4 * q;
          Tb[p][lane] = Ct[lane][p];  // Tb[p][r] = L_{j+2,j}(r, p)
        }
        __syncthreads();
        Acc pp;
#pragma unroll
        for (int e = 0; e < 8; ++e) (&pp.v[0][0][0])[e] = 0.0;
        acc_update<false>(pp, Tb, Ta, qr, qc, g, tq);
        double* P = Ld + (int64_t)(j + 1) * LDW + LDW_P;
#pragma unroll
        for (int rb = 0; rb < 2; ++rb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb)
#pragma unroll
            for (int e = 0; e < 2; ++e) P[(qr * 16 + rb * 8 + g) * TS + qc * 16 + cb * 8 + 2 * tq + e] = pp.v[rb][cb][e];
      }
      publish(Ct, M, ld, N, i, j, flags + tile_id(i, j, nt));
    } else {
      // ---- diagonal task D_j: diagonal tile (j, j) and sub-diagonal tile (j+1, j) ----
      const bool has_sb = j + 1 < nt;
      Acc d;   // A_jj
      Acc sb;  // A_{j+1, j}
      acc_load(d, M, ld, N, j, j, qr, qc, g, tq);
      acc_load(sb, M, ld, N, j + 1, j, qr, qc, g, tq);  // rows past N read as zero (never published)
      const int nc = USE_U ? max(0, (j - 2) / UB) : 0;  // chunks summed by the U tasks (they end before k = j - 2)
      for (int c = 0; c < nc; ++c) {
        wait_flags(uflags + j * maxc + c, nullptr, info);
        const double* base = part + ((int64_t)j * maxc + c) * 2 * TS * TS;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          (&sb.v[0][0][0])[e] += __ldcg(base + e * CT + threadIdx.x);
          (&d.v[0][0][0])[e] += __ldcg(base + TS * TS + e * CT + threadIdx.x);
        }
      }
      int rdy = nc * UB;
      for (int k = nc * UB; k < j - 1; ++k) {
        if (k >= rdy) rdy = ready_prefix(flags, nt, j, has_sb ? j + 1 : j, k, j - 1, &s_min, info);
        stage(Ta, M, ld, N, j, k);
        stage(Tb, M, ld, N, j + 1, k);
        __syncthreads();
        acc_update(d, Ta, Ta, qr, qc, g, tq);
        acc_update(sb, Tb, Ta, qr, qc, g, tq);
        __syncthreads();
      }
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (j > 0) {  // A_jj -= L_{j,j-1} L_{j,j-1}^T with L_{j,j-1} from D_{j-1} (side buffer, polled as data)
        stage_side(Ta, Ld + (int64_t)(j - 1) * LDW + LDW_SUB, info);
        __syncthreads();
        acc_update(d, Ta, Ta, qr, qc, g, tq);
      }
      if (trace && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1b));
      acc_gather(d, Ct, qr, qc, g, tq);
      acc_gather(sb, Cs, qr, qc, g, tq);
      __syncthreads();
      if (w == 0) {
        // POTRF of the diagonal tile: L_jj and 1/diag to the side buffer, then the tile to M
        final_potrf(Ct, Tb, piv, dinv_s, Ld + (int64_t)j * LDW, j * TS, N, info, lane, has_sb);
        if (trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1c));
#pragma unroll 4
        for (int c = 0; c < TS; ++c) {
          const int gr = j * TS + lane, gc = j * TS + c;
          if (gr < N && gc < N) M[gr + (int64_t)gc * ld] = Ct[lane][c];
        }
      } else if (has_sb) {
        if (w >= 2 && j > 0) {
          // the sub-diagonal tile's last update, A_{j+1,j} -= P_j (formed by the off-diagonal task
          // (j+1, j-1), polled as data)
          const int t2 = threadIdx.x - 64;
          const double* P = Ld + (int64_t)j * LDW + LDW_P;
          double v[TS * TS / 64];
#pragma unroll
          for (int q = 0; q < TS * TS / 64; ++q) v[q] = ld_cg_volatile(P + t2 + 64 * q);
          const unsigned long long tw = gtime();
          for (;;) {
            bool ok = true;
#pragma unroll
            for (int q = 0; q < TS * TS / 64; ++q)
              if (unset(v[q])) {
                v[q] = ld_cg_volatile(P + t2 + 64 * q);
                ok = false;
              }
            if (ok) break;
            if (gtime() - tw > kSpinLimitNs) {
              watchdog_expired(info);
              break;
            }
          }
          if (trace && t2 == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_tx));
#pragma unroll
          for (int q = 0; q < TS * TS / 64; ++q) {
            const int e = t2 + 64 * q;
            Cs[e / TS][e % TS] -= v[q];
          }
        }
        bar_named(2, 96);
        if (w == 1) {
          // L_{j+1,j} = A_{j+1,j} L_jj^{-T}, a quarter of the columns at a time as warp 0 releases them
          if (trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_tw));
          double x[TS];
#pragma unroll
          for (int c = 0; c < TS; ++c) x[c] = Cs[lane][c];
          trail_rows(x, Tb, dinv_s);
          if (trace && lane == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(s_tw2));
          double* sub = Ld + (int64_t)j * LDW + LDW_SUB;
          const int gr = (j + 1) * TS + lane;
#pragma unroll
          for (int c = 0; c < TS; ++c) sub[c * TS + lane] = x[c];  // [p][r] order, coalesced: D_{j+1} polls these first
#pragma unroll
          for (int c = 0; c < TS; ++c)
            if (gr < N && j * TS + c < N) M[gr + (int64_t)(j * TS + c) * ld] = x[c];
          __syncwarp();
          if (lane == 0) release(flags + tile_id(j + 1, j, nt));
        }
      }
      __syncthreads();
    }
    if (trace && threadIdx.x == 0) {
      unsigned long long t2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      trace[6 * t] = t0;
      trace[6 * t + 1] = t1;
      trace[6 * t + 2] = t1b;
      trace[6 * t + 3] = t1c;
      trace[6 * t + 4] = t2;
      trace[6 * t + 5] = (tk.x == 0 && i == j) ? s_tw : sm;  // diagonal tasks: warp 1's start
      if (tk.x == 0 && i == j) {
        trace[6 * ntasks + j] = s_tx;
        trace[6 * ntasks + nt + j] = s_tw2;
      }
    }
  }
}

}  // namespace

static size_t flags_bytes(int nt) { return ((size_t)(nt * (nt + 1) / 2 + 8) * sizeof(int) + 255) & ~(size_t)255; }
static int max_chunks(int nt) { return nt / UB + 1; }
static size_t uflags_bytes(int nt) { return ((size_t)nt * max_chunks(nt) * sizeof(int) + 255) & ~(size_t)255; }
static size_t part_bytes(int nt) { return (size_t)nt * max_chunks(nt) * 2 * TS * TS * sizeof(double); }

size_t chol_ws_bytes(int N) {
  const int nt = (N + TS - 1) / TS;
  return flags_bytes(nt) + (size_t)nt * LDW * sizeof(double) + uflags_bytes(nt) + part_bytes(nt);
}

// Task table in ticket order (built once per tile count, device memory): per column col,
// D_col, the off-diagonal tiles (i >= col + 2, col), and after every B-th column the U(j, c) tasks
// whose chunk it completes.  Every task only depends on tasks listed before it.
static std::mutex g_task_mu;
static std::map<std::pair<int, int>, std::pair<int4*, int>> g_tasks;

// U tasks pay off once the diagonal tasks' own update chains dominate (measured with chunks of 16:
// N = 4226 1.83 -> 1.53 ms, 3201 1.03 -> 0.92; at 63 tile columns they cost 5 %), so they are
// generated for nt >= kUMinTiles only.
constexpr int kUMinTiles = 80;

static fk_status task_table(int nt, int4** d_tasks, int* ntasks) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_task_mu);
  auto key = std::make_pair(dev, nt);
  const bool use_u = nt >= kUMinTiles;
  auto it = g_tasks.find(key);
  if (it == g_tasks.end()) {
    std::vector<int4> t;
    for (int col = 0; col < nt; ++col) {
      t.push_back(make_int4(0, col, col, 0));
      for (int i = col + 2; i < nt; ++i) t.push_back(make_int4(1, i, col, 0));
      if (use_u && (col + 1) % UB == 0) {
        const int c = (col + 1) / UB - 1;
        for (int j = (c + 1) * UB + 2; j < nt; ++j) t.push_back(make_int4(2, j, j, c));
      }
    }
    int4* d = nullptr;
    FK_CUDA_TRY(cudaMalloc(&d, t.size() * sizeof(int4)));
    FK_CUDA_TRY(cudaMemcpy(d, t.data(), t.size() * sizeof(int4), cudaMemcpyHostToDevice));
    it = g_tasks.emplace(key, std::make_pair(d, (int)t.size())).first;
  }
  *d_tasks = it->second.first;
  *ntasks = it->second.second;
  return FK_OK;
}

// Factor the N x N SPD matrix M (column-major, leading dimension ld, lower triangle read and
// overwritten with L).  ws: chol_ws_bytes(N) bytes; info: device int, set to 0 here.
// workspace layout: flags (+ ticket) | side buffer Ld | uflags | partial sums
CholReset chol_reset_args(int N, void* ws, int* info) {
  const int nt = (N + TS - 1) / TS;
  CholReset c;
  c.ld = (unsigned long long*)((char*)ws + flags_bytes(nt));
  c.n_ld = (int64_t)nt * LDW;
  c.zero = (int*)ws;  // flags, ticket: flags_bytes(nt); uflags follow the side buffer
  c.n_zero = (int64_t)flags_bytes(nt) / (int64_t)sizeof(int);
  c.info = info;
  return c;
}

// trace (measurement only, tools/microbench/mb_chol_tiles.cu): 6 words per ticket, then 2 per tile
// column (diagonal tasks: the time P_j was seen, the time warp 1's TRSM ended), or null.
fk_status chol_tiles(double* M, int64_t ld, int N, int* info, void* ws, cudaStream_t s, unsigned long long* trace, bool preset) {
  const int nt = (N + TS - 1) / TS;
  const int ntiles = nt * (nt + 1) / 2;
  int4* tasks = nullptr;
  int ntasks = 0;
  FK_TRY(task_table(nt, &tasks, &ntasks));
  int* flags = (int*)ws;
  int* ticket = flags + ntiles;
  double* Ld = (double*)((char*)ws + flags_bytes(nt));
  int* uflags = (int*)((char*)Ld + (size_t)nt * LDW * sizeof(double));
  double* part = (double*)((char*)uflags + uflags_bytes(nt));
  if (!preset) {
    FK_CUDA_TRY(cudaMemsetAsync(Ld, 0xff, (size_t)nt * LDW * sizeof(double), s));
    FK_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)(ntiles + 8) * sizeof(int), s));
    FK_CUDA_TRY(cudaMemsetAsync(info, 0, sizeof(int), s));
  }
  if (nt >= kUMinTiles) FK_CUDA_TRY(cudaMemsetAsync(uflags, 0, uflags_bytes(nt), s));
  const bool use_u = nt >= kUMinTiles;
  auto kern = use_u ? k_chol_tiles<true> : k_chol_tiles<false>;
  static int per_sm = 0;
  if (per_sm == 0) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_chol_tiles<true>, CT, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  }
  // fewer co-resident CTAs shorten the latency-bound critical path at small N; the update throughput
  // needs more at larger N (measured on B200: N = 2002 best at 2/SM, N >= 3000 at 8/SM)
  int ps = std::min(per_sm, N <= 2500 ? 2 : 8);
  if (const char* e = getenv("FK_CHOL_PER_SM")) ps = std::max(1, std::min(per_sm, atoi(e)));  // experiments
  const int grid = std::min(ntasks, ps * device_sm_count());
  kern<<<grid, CT, 0, s>>>(M, ld, N, nt, flags, ticket, info, Ld, tasks, ntasks, part, uflags, max_chunks(nt), trace);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  return FK_OK;
}

}  // namespace fk
