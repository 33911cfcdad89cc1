// solve.cu -- assembly and dense solve of the regularised Fourier system (PAPER.md:107 eq.
// kenrel_reg, :252 Sobolev, :316 low-bias, :396 physics-informed box domain, :476-487 additive).
//
//   A[k1,k2] = mu_{k1-k2}/n + lambda R_{k1} delta_{k1 k2} (+ mu_pde conj(d_{k1}) B(k2-k1) d_{k2})
//   A theta  = r / n
//
// A is Hermitian positive definite for lambda > 0.  For real Y, theta is Hermitian (theta_{-k} =
// conj theta_k), so theta = P z with z real and P*AP z = P*r/n real SPD (1/4 of the complex
// flops).  The real system is assembled with the rhs as an extra row (N = D + 1) so that cuSOLVER
// dpotrf's last row holds L^{-1} c and one dtrsv finishes the solve.  CG is not used:
// cond(A) is 1e6..1e11 at the BASELINE configurations and Jacobi-preconditioned CG would need 1e3+
// iterations (reading R9).  The backward error of the report re-evaluates the complex A
// from the moments on the fly.  The lambda path (fk_solve_path) and the held-out risk
// (fk_path_validate) reuse the same real assembly.
#include <cublas_v2.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>
#include <vector>
#include <mutex>

#include "fk_internal.cuh"

namespace fk {
namespace {

constexpr int kMaxTerms = 8, kMaxD = 4;
constexpr unsigned long long kZSentinel = 0x7ff4dead5eed1e55ULL;  // 'not yet published' (k_trsv_lt)

struct SysArgs {
  int d, m, kind, D;
  double inv_n, lambda, s, mu_pde, c;  // c = pi / (2L)
  double inv4L;
  int n_terms;
  int alpha[kMaxTerms][kMaxD];
  double a_alpha[kMaxTerms];
  double box[kMaxD][2];
  const double2* mu;
  const double2* cross;
  const double2* dsym;  // PI tables (k_pi_tables), or null
  const double2* boxt;
  const double2* mur;   // PIK_COLLOC: collocation moments
  double inv_nr;        // PIK_COLLOC: 1 / n_colloc
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) { return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

__device__ void decode(int idx, int d, int m, int* k) {
  const int side = 2 * m + 1;
  for (int l = d - 1; l >= 0; --l) {
    k[l] = idx % side - m;
    idx /= side;
  }
}

// symbol of D on exp(+i <k, t(x)>): d_k = sum_a a_alpha prod_l (i c k_l)^{alpha_l}  (reading R3)
__device__ double2 pde_symbol(const SysArgs& g, const int* k) {
  double2 acc = make_double2(0.0, 0.0);
  for (int t = 0; t < g.n_terms; ++t) {
    double2 term = make_double2(g.a_alpha[t], 0.0);
    for (int l = 0; l < g.d; ++l) {
      const double2 ik = make_double2(0.0, g.c * k[l]);
      for (int e = 0; e < g.alpha[t][l]; ++e) term = cmul(term, ik);
    }
    acc.x += term.x;
    acc.y += term.y;
  }
  return acc;
}

// B(q) = (4L)^{-d} int_box exp(+i c <q, x>) dx  (index order of reading R3)
__device__ double2 box_fourier(const SysArgs& g, const int* q) {
  double2 acc = make_double2(1.0, 0.0);
  for (int l = 0; l < g.d; ++l) {
    const double a = g.box[l][0], b = g.box[l][1];
    double2 v;
    if (q[l] == 0) {
      v = make_double2(b - a, 0.0);
    } else {
      const double w = g.c * q[l];
      double sb, cb, sa, ca;
      sincos(w * b, &sb, &cb);
      sincos(w * a, &sa, &ca);
      // (e^{iwb} - e^{iwa}) / (i w) = ((sb - sa) - i (cb - ca)) / w
      v = make_double2((sb - sa) / w, -(cb - ca) / w);
    }
    acc = cmul(acc, make_double2(v.x * g.inv4L, v.y * g.inv4L));
  }
  return acc;
}

__device__ double2 entry(const SysArgs& g, int i, int j) {
  double2 v;
  if (g.kind == FK_ADDITIVE) {
    const int side = 2 * g.m + 1;
    const int l1 = i / side, a = i % side - g.m;
    const int l2 = j / side, b = j % side - g.m;
    if (l1 == l2) {
      v = g.mu[(int64_t)l1 * (4 * g.m + 1) + (a - b + 2 * g.m)];
    } else if (l1 < l2) {
      const int p = l1 * g.d - l1 * (l1 + 1) / 2 + (l2 - l1 - 1);
      v = g.cross[((int64_t)p * side + (a + g.m)) * side + (b + g.m)];
    } else {
      const int p = l2 * g.d - l2 * (l2 + 1) / 2 + (l1 - l2 - 1);
      v = cconj(g.cross[((int64_t)p * side + (b + g.m)) * side + (a + g.m)]);
    }
    v.x *= g.inv_n;
    v.y *= g.inv_n;
    if (i == j) v.x += g.lambda;
    return v;
  }
  int k1[kMaxD], k2[kMaxD];
  decode(i, g.d, g.m, k1);
  decode(j, g.d, g.m, k2);
  int64_t qi = 0;
  const int qside = 4 * g.m + 1;
  for (int l = 0; l < g.d; ++l) qi = qi * qside + (k1[l] - k2[l] + 2 * g.m);
  v = g.mu[qi];
  v.x *= g.inv_n;
  v.y *= g.inv_n;
  if (i == j) {
    double R = 1.0;
    if (g.kind != FK_LOWBIAS) {
      double nk2 = 0.0;
      for (int l = 0; l < g.d; ++l) nk2 += (double)k1[l] * k1[l];
      R = 1.0 + pow(nk2, g.s);
    }
    v.x += g.lambda * R;
  }
  if (g.kind == FK_PIK_COLLOC && g.mu_pde != 0.0) {
    // mu_pde conj(d_k1) (T(mu_r))_{k1,k2} d_k2 / n_r
    double2 tr = g.mur[qi];
    tr.x *= g.inv_nr;
    tr.y *= g.inv_nr;
    const double2 t = cmul(cmul(cconj(g.dsym[i]), tr), g.dsym[j]);
    v.x += g.mu_pde * t.x;
    v.y += g.mu_pde * t.y;
  }
  if (g.kind == FK_PIK_BOX && g.mu_pde != 0.0) {
    double2 t;
    if (g.dsym) {  // tabulated: d_k per mode, box integral per dimension and difference q_l
      double2 b = make_double2(1.0, 0.0);
      for (int l = 0; l < g.d; ++l) b = cmul(b, g.boxt[l * (4 * g.m + 1) + (k2[l] - k1[l] + 2 * g.m)]);
      t = cmul(cmul(cconj(g.dsym[i]), b), g.dsym[j]);
    } else {
      int q[kMaxD];
      for (int l = 0; l < g.d; ++l) q[l] = k2[l] - k1[l];
      t = cmul(cmul(cconj(pde_symbol(g, k1)), box_fourier(g, q)), pde_symbol(g, k2));
    }
    v.x += g.mu_pde * t.x;
    v.y += g.mu_pde * t.y;
  }
  return v;
}

// PI tables: dsym[i] = d_{k_i} (symbol), boxt[l][q + 2m] = (4L)^{-1} int_{a_l}^{b_l} e^{i c q x} dx
__global__ void k_pi_tables(SysArgs g, double2* __restrict__ dsym, double2* __restrict__ boxt) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < g.D) {
    int k[kMaxD];
    decode(t, g.d, g.m, k);
    dsym[t] = pde_symbol(g, k);
  }
  const int nq = 4 * g.m + 1;
  if (t < g.d * nq) {
    const int l = t / nq, qv = t % nq - 2 * g.m;
    SysArgs one = g;
    one.d = 1;
    one.box[0][0] = g.box[l][0];
    one.box[0][1] = g.box[l][1];
    boxt[t] = box_fourier(one, &qv);
  }
}

// res[0] += ||A theta - b||^2, res[1] += ||b||^2, with A evaluated on the fly (one warp per row)
__global__ void k_residual(SysArgs g, const double2* __restrict__ theta, const double2* __restrict__ r, double* __restrict__ res) {
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= g.D) return;
  double sx = 0.0, sy = 0.0;
  for (int j = lane; j < g.D; j += 32) {
    const double2 a = entry(g, row, j);
    const double2 t = theta[j];
    sx += a.x * t.x - a.y * t.y;
    sy += a.x * t.y + a.y * t.x;
  }
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(0xffffffffu, sx, o);
    sy += __shfl_xor_sync(0xffffffffu, sy, o);
  }
  if (lane == 0) {
    const double bx = r[row].x * g.inv_n, by = r[row].y * g.inv_n;
    atomicAdd(res, (sx - bx) * (sx - bx) + (sy - by) * (sy - by));
    atomicAdd(res + 1, bx * bx + by * by);
  }
}

std::mutex g_sol_mu;
std::map<int, cusolverDnHandle_t> g_handles;
std::map<int, cublasHandle_t> g_blas;

fk_status blas_for_device(cublasHandle_t* h) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = g_blas.find(dev);
  if (it != g_blas.end()) {
    *h = it->second;
    return FK_OK;
  }
  cublasHandle_t nh;
  if (cublasCreate(&nh) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasCreate failed");
  g_blas[dev] = nh;
  *h = nh;
  return FK_OK;
}

fk_status handle_for_device(cusolverDnHandle_t* h) {
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = g_handles.find(dev);
  if (it != g_handles.end()) {
    *h = it->second;
    return FK_OK;
  }
  cusolverDnHandle_t nh;
  if (cusolverDnCreate(&nh) != CUSOLVER_STATUS_SUCCESS) return fail(FK_E_CUDA, "cusolverDnCreate failed");
  g_handles[dev] = nh;
  *h = nh;
  return FK_OK;
}

int unknowns(int d, int m, int kind) {
  if (kind == FK_ADDITIVE) return d * (2 * m + 1);
  int D = 1;
  for (int l = 0; l < d; ++l) D *= 2 * m + 1;
  return D;
}

// ---- real form of the Hermitian system (DESIGN.md §5 "Solve") ----
// For real Y the solution is Hermitian, theta_{-k} = conj theta_k, so theta = P z with z real:
// z = (a_0, a_1, b_1, a_2, b_2, ...) over the centre and the positive half of the mode grid
// (per feature block for the additive model), theta_k = a_k + i b_k, theta_{-k} = a_k - i b_k.
// Then P^* A P z = P^* r/n is real symmetric positive definite with the same unique solution
// and a quarter of the complex Cholesky's flops.  Column u of P has at most two entries.
struct PCol {
  int i[2];
  double2 a[2];
  int cnt;
};

__device__ __forceinline__ int neg_index(const SysArgs& g, int i) {
  if (g.kind == FK_ADDITIVE) {
    const int S = 2 * g.m + 1, l = i / S;
    return l * S + (S - 1 - (i - l * S));
  }
  return g.D - 1 - i;
}

__device__ __forceinline__ PCol pcol(const SysArgs& g, int u) {
  PCol p;
  int base, c0, v;
  if (g.kind == FK_ADDITIVE) {
    const int S = 2 * g.m + 1;
    base = (u / S) * S;
    c0 = base + g.m;
    v = u % S;
  } else {
    base = 0;
    c0 = (g.D - 1) / 2;
    v = u;
  }
  if (v == 0) {
    p.cnt = 1;
    p.i[0] = c0;
    p.a[0] = make_double2(1.0, 0.0);
    return p;
  }
  const int t = (v + 1) >> 1;
  const int i = c0 + t;
  p.cnt = 2;
  p.i[0] = i;
  p.i[1] = neg_index(g, i);
  if (v & 1) {  // a_k: e_k + e_{-k}
    p.a[0] = make_double2(1.0, 0.0);
    p.a[1] = make_double2(1.0, 0.0);
  } else {      // b_k: i e_k - i e_{-k}
    p.a[0] = make_double2(0.0, 1.0);
    p.a[1] = make_double2(0.0, -1.0);
  }
  (void)base;
  return p;
}

// M is the (D+1) x (D+1) column-major augmented matrix [[P*AP, c], [c^T, huge]] (lower triangle):
// its Cholesky factor's last row is y = L^{-1} c, so only the backward solve L^T z = y remains.
// lower triangle of P^*AP (column v = blockIdx.y, rows u >= v), ld = D + 1
__global__ void k_assemble_real(SysArgs g, double* __restrict__ M) {
  const int64_t N = g.D + 1;
  const int v = blockIdx.y;
  const int u = v + blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.D) return;
  const PCol pu = pcol(g, u), pv = pcol(g, v);
  double s = 0.0;
  for (int x = 0; x < pu.cnt; ++x)
    for (int y = 0; y < pv.cnt; ++y) {
      const double2 a = entry(g, pu.i[x], pv.i[y]);
      const double2 c = cmul(cmul(cconj(pu.a[x]), a), pv.a[y]);
      s += c.x;
    }
  M[u + v * N] = s;
}

// d = 1 without a PDE term: closed forms of (P^*AP)_{uv} in the moments (checked against the generic
// kernel by tests/test_gpu_chol.py and the oracle's dense solve).  With M_q = mu_q / n, basis order
// u = 0 centre, u = 2t-1 a_t = e_t + e_{-t}, u = 2t b_t = i e_t - i e_{-t}:
//   (c,c) Re M_0            (c,a_t) 2 Re M_t         (c,b_t) 2 Im M_t     [rows u > v only]
//   (a_s,a_t) 2 Re(M_{s-t} + M_{s+t})   (a_s,b_t) 2 Im(M_{s+t} - M_{s-t})
//   (b_s,a_t) 2 Im(M_{s-t} + M_{s+t})   (b_s,b_t) 2 Re(M_{s-t} - M_{s+t})
// plus lambda cnt R_t on the diagonal (R_t = 1 + t^{2s}, or 1 for the low-bias space).
__global__ void k_assemble_real_d1(SysArgs g, double* __restrict__ M) {
  const int64_t N = g.D + 1;
  const int v = blockIdx.y;
  const int u = v + blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.D) return;
  const double2* mu = g.mu + 2 * g.m;  // mu[q], q in [-2m, 2m]
  auto Mq = [&](int q) { return mu[q]; };
  const int s = (u + 1) >> 1, t = (v + 1) >> 1;
  const bool ua = u & 1, va = v & 1;
  double e;
  if (v == 0) {
    e = (u == 0) ? Mq(0).x : (ua ? 2.0 * Mq(s).x : 2.0 * Mq(s).y);
  } else {
    const double2 dm = Mq(s - t), sm = Mq(s + t);
    if (ua) e = va ? 2.0 * (dm.x + sm.x) : 2.0 * (sm.y - dm.y);
    else e = va ? 2.0 * (dm.y + sm.y) : 2.0 * (dm.x - sm.x);
  }
  e *= g.inv_n;
  if (u == v) {
    const double R = (g.kind == FK_LOWBIAS) ? 1.0 : 1.0 + pow((double)s * s, g.s);
    e += g.lambda * (u == 0 ? 1.0 : 2.0) * R;
  }
  M[u + v * N] = e;
}

// d = 2, non-additive kinds: the complex entry with the mode decode done by one fp32 reciprocal
// multiply + fix-up (no integer division) and the PI terms from the tabulated symbols / box
// integrals.  The generic path spent ~500 us on D = 4225 (C4) in 16 integer divisions and the
// general PDE branches per real entry.
struct K2 {
  int a, b;
};
__device__ __forceinline__ K2 decode2(int i, int side, float inv_side, int m) {
  int q = __float2int_rz((float)i * inv_side);
  int r = i - q * side;
  if (r < 0) {
    --q;
    r += side;
  } else if (r >= side) {
    ++q;
    r -= side;
  }
  return K2{q - m, r - m};
}

__device__ __forceinline__ double2 entry_d2(const SysArgs& g, int i, int j, int side, float inv_side) {
  const K2 k1 = decode2(i, side, inv_side, g.m), k2 = decode2(j, side, inv_side, g.m);
  const int qside = 4 * g.m + 1;
  const int qi = (k1.a - k2.a + 2 * g.m) * qside + (k1.b - k2.b + 2 * g.m);
  double2 v = g.mu[qi];
  v.x *= g.inv_n;
  v.y *= g.inv_n;
  if (i == j) {
    double R = 1.0;
    if (g.kind != FK_LOWBIAS) R = 1.0 + pow((double)(k1.a * k1.a + k1.b * k1.b), g.s);
    v.x += g.lambda * R;
  }
  if (g.mu_pde != 0.0 && (g.kind == FK_PIK_BOX || g.kind == FK_PIK_COLLOC)) {
    double2 t;
    if (g.kind == FK_PIK_BOX) {
      const double2 b = cmul(g.boxt[k2.a - k1.a + 2 * g.m], g.boxt[qside + (k2.b - k1.b + 2 * g.m)]);
      t = cmul(cmul(cconj(g.dsym[i]), b), g.dsym[j]);
    } else {
      double2 tr = g.mur[qi];
      tr.x *= g.inv_nr;
      tr.y *= g.inv_nr;
      t = cmul(cmul(cconj(g.dsym[i]), tr), g.dsym[j]);
    }
    v.x += g.mu_pde * t.x;
    v.y += g.mu_pde * t.y;
  }
  return v;
}

// d = 2, one thread per pair of modes (t1 >= t2; t = 0 the centre, t >= 1 the positive-half mode
// c0 + t and its mirror c0 - t): the 4 complex entries A(+-k1, +-k2) are evaluated once and give
// the 2 x 2 real block (a1|b1) x (a2|b2) -- the per-entry kernel evaluated each complex entry 4 times.
//   (a,a) Re(A++ + A+- + A-+ + A--)   (a,b) -Im(A++ - A+- + A-+ - A--)
//   (b,a) Im(A++ + A+- - A-+ - A--)   (b,b) Re(A++ - A+- - A-+ + A--)
__global__ void k_assemble_real_d2_blk(SysArgs g, double* __restrict__ M) {
  const int64_t N = g.D + 1;
  const int c0 = (g.D - 1) / 2;
  const int t2 = blockIdx.y;
  const int t1 = t2 + blockIdx.x * blockDim.x + threadIdx.x;
  if (t1 > c0) return;
  const int side = 2 * g.m + 1;
  const float inv_side = 1.0f / (float)side;
  if (t2 == 0) {
    const double2 p = entry_d2(g, c0 + t1, c0, side, inv_side);
    if (t1 == 0) {
      M[0] = p.x;
      return;
    }
    const double2 q = entry_d2(g, c0 - t1, c0, side, inv_side);
    M[(2 * t1 - 1)] = p.x + q.x;
    M[(2 * t1)] = p.y - q.y;
    return;
  }
  const double2 pp = entry_d2(g, c0 + t1, c0 + t2, side, inv_side), pm = entry_d2(g, c0 + t1, c0 - t2, side, inv_side);
  const double2 mp = entry_d2(g, c0 - t1, c0 + t2, side, inv_side), mm = entry_d2(g, c0 - t1, c0 - t2, side, inv_side);
  const int64_t ua = 2 * t1 - 1, ub = 2 * t1, va = 2 * t2 - 1, vb = 2 * t2;
  M[ua + va * N] = pp.x + pm.x + mp.x + mm.x;
  M[ub + va * N] = pp.y + pm.y - mp.y - mm.y;
  M[ub + vb * N] = pp.x - pm.x - mp.x + mm.x;
  if (t1 > t2) M[ua + vb * N] = -(pp.y - pm.y + mp.y - mm.y);
}

void launch_assemble(const SysArgs& g, double* M, cudaStream_t s) {
  const dim3 grid((g.D + 255) / 256, g.D);
  if (g.d == 1 && (g.kind == FK_SOBOLEV || g.kind == FK_LOWBIAS))
    k_assemble_real_d1<<<grid, 256, 0, s>>>(g, M);
  else if (g.d == 2 && g.kind != FK_ADDITIVE && (g.kind == FK_SOBOLEV || g.kind == FK_LOWBIAS || g.dsym))
    k_assemble_real_d2_blk<<<dim3(((g.D - 1) / 2 + 256) / 256, (g.D - 1) / 2 + 1), 256, 0, s>>>(g, M);
  else
    k_assemble_real<<<grid, 256, 0, s>>>(g, M);
}

__global__ void k_rhs_real(SysArgs g, const double2* __restrict__ r, double* __restrict__ M, double* __restrict__ zbuf,
                           int* __restrict__ ticket, CholReset cr) {  // last row of M (+ reset of k_trsv_lt's sentinels / ticket,
                                                                     // and of chol_tiles' state when cr.info is set)
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (cr.info) chol_reset(cr, u, (int64_t)gridDim.x * blockDim.x);
  const int64_t N = g.D + 1;
  if (u == g.D) M[g.D + g.D * N] = 1e200;  // any value above c^T (P*AP)^{-1} c keeps it SPD
  if (u == 0 && ticket) *ticket = 0;
  if (u >= g.D) return;
  if (zbuf) zbuf[u] = __longlong_as_double((long long)kZSentinel);
  const PCol p = pcol(g, u);
  double s = 0.0;
  for (int x = 0; x < p.cnt; ++x) {
    const double2 b = make_double2(r[p.i[x]].x * g.inv_n, r[p.i[x]].y * g.inv_n);
    s += cmul(cconj(p.a[x]), b).x;
  }
  M[g.D + u * N] = s;
}

// also turns the factorisation's info word into the caller's device status bits (thread 0):
// info > 0 = first non-positive pivot + 1, info < 0 = a dataflow wait hit its watchdog
__global__ void k_theta_from_real(SysArgs g, const double* __restrict__ zs, int64_t zstride, double2* __restrict__ theta,
                                  const int* __restrict__ info, int* __restrict__ d_status) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u == 0 && info && d_status) {
    const int v = *info;
    if (v > 0) atomicOr(d_status, (int)FK_DSTATUS_NOT_SPD);
    if (v < 0) atomicOr(d_status, (int)FK_DSTATUS_WATCHDOG);
  }
  if (u >= g.D) return;
  auto z = [&](int i) { return zs[(int64_t)i * zstride]; };
  const int v = g.kind == FK_ADDITIVE ? u % (2 * g.m + 1) : u;
  const int base = g.kind == FK_ADDITIVE ? u - v : 0;
  if (v == 0) {
    const int c0 = g.kind == FK_ADDITIVE ? base + g.m : (g.D - 1) / 2;
    theta[c0] = make_double2(z(u), 0.0);
  } else if (v & 1) {
    const PCol p = pcol(g, u);
    const double a = z(u), b = z(u + 1);
    theta[p.i[0]] = make_double2(a, b);
    theta[p.i[1]] = make_double2(a, -b);
  }
}


// ---- back substitution L^T z = y on many SMs (replaces the single-SM cublasDtrsv) ------------
// Block I (32 rows of z) is owned by one 128-thread CTA.  It inverts its diagonal block W = L_II^{-1}
// and prefetches its off-diagonal blocks while z is not yet known, then accumulates
// sum_{J>I} L_JI^T z_J as the blocks z_J appear (J descending; thread (lane, warp h) holds row lane
// of block J times columns 8h..8h+7 of block I) and finishes with z_I = W^T (y_I - acc) plus one
// refinement step with L_II.  Only the last block's term is on the chain: the sum over J > I+1 is
// reduced (shuffles) and L_{I+1,I} staged while z_{I+1} is awaited, and every 32 x 32 product of
// the tail is split over the four warps (8 terms each) instead of 32-term serial dot products
// (round 2: ~1.6 -> ~1 us per block on the chain).
// z_J is published element by element: zbuf is pre-filled with a sentinel NaN pattern (k_rhs_real)
// that no computed value has, so a reader spins on the value itself (one L2 round trip per block
// on the critical path, no separate flag).  Blocks are taken in ticket order (an atomic counter,
// highest block first), so a CTA only ever waits on CTAs that started before it: no co-residency
// requirement, no deadlock at any D.
__device__ __forceinline__ double ld_volatile(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// value of z at row `row`, waiting for its publication (watchdog: 5 s, then info = -1)
__device__ __forceinline__ double wait_z(const double* zbuf, int row, int* info) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  double zc;
  do {
    zc = ld_volatile(zbuf + row);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  } while (__double_as_longlong(zc) == (long long)kZSentinel && t1 - t0 < 5000000000ULL);
  if (__double_as_longlong(zc) == (long long)kZSentinel) atomicCAS(info, 0, -1);
  return zc;
}

// out[c] = base[c] + sgn * sum_k A[k][c] v[k] over k in [c, 32) (A lower triangular in [k][c]) or all
// k (FULL): thread (c = lane, part h) sums k in [8h, 8h + 8), the four parts are added by warp 0.
// Starts after a barrier that published v and ends with one that publishes out.
template <bool FULL>
__device__ __forceinline__ void mv32(const double (*A)[33], const double* v, const double* base, double sgn, double* out,
                                     double (*part)[33]) {
  const int c = threadIdx.x & 31, h = threadIdx.x >> 5;
  double t = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int k = 8 * h + q;
    if (FULL || k >= c) t = fma(A[k][c], v[k], t);
  }
  part[h][c] = t;
  __syncthreads();
  if (h == 0) out[c] = base[c] + sgn * ((part[0][c] + part[1][c]) + (part[2][c] + part[3][c]));
  __syncthreads();
}

__global__ void __launch_bounds__(128) k_trsv_lt(const double* __restrict__ M, int64_t ld, int D, const double* __restrict__ y,
                                                  int64_t ystride, double* zbuf, int* ticket, int* info) {
  __shared__ double W[32][33];   // W[k][c] = (L_II^{-1})(k, c)
  __shared__ double Ls[32][33];  // Ls[k][c] = L_II(k, c)
  __shared__ double Ln[32][33];  // Ln[r][c] = L_{I+1, I}(r, c)
  __shared__ double part[4][33];
  __shared__ double pacc[32], rv[32], zv[32], res[32], zn[32], zero[32];
  __shared__ int tk;
  const int nb = (D + 31) / 32;
  if (threadIdx.x == 0) tk = atomicAdd(ticket, 1);
  __syncthreads();
  const int I = nb - 1 - tk;
  const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
  const int r0 = I * 32;
  auto Lval = [&](int gr, int gc) { return (gr < D && gc < D) ? M[gr + (int64_t)gc * ld] : (gr == gc ? 1.0 : 0.0); };
  // stage L_II (identity on padded rows) and L_{I+1,I}, then W = L_II^{-1}: lane j of warp 0 solves L w = e_j
  for (int c = h; c < 32; c += 4) {
    Ls[lane][c] = Lval(r0 + lane, r0 + c);
    Ln[lane][c] = (I + 1 < nb) ? Lval(r0 + 32 + lane, r0 + c) : 0.0;
  }
  if (threadIdx.x < 32) zero[threadIdx.x] = 0.0;
  __syncthreads();
  if (h == 0) {
    // column `lane` of W by right-looking forward substitution (the chain per row is one multiply and
    // one FMA; the reciprocals of the diagonal are formed in parallel first)
    const double rinv = 1.0 / Ls[lane][lane];
    double w[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) w[r] = (r == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      w[c] *= __shfl_sync(~0u, rinv, c);
#pragma unroll
      for (int r = c + 1; r < 32; ++r) w[r] = fma(-Ls[r][c], w[c], w[r]);
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) W[r][lane] = w[r];
  }
  // sum_{J > I+1} L_JI^T z_J: thread (lane = row of block J, h) x columns 8h .. 8h+7 of block I
  double acc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q] = 0.0;
  const int cbase = r0 + 8 * h;
  double Lb[8];
  auto load_block = [&](int J) {
    const int row = J * 32 + lane;
#pragma unroll
    for (int q = 0; q < 8; ++q) Lb[q] = (row < D && cbase + q < D) ? M[row + (int64_t)(cbase + q) * ld] : 0.0;
  };
  if (I + 2 < nb) load_block(nb - 1);
  for (int J = nb - 1; J > I + 1; --J) {
    const int row = J * 32 + lane;
    const double zc = (row < D) ? wait_z(zbuf, row, info) : 0.0;
    double Lc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) Lc[q] = Lb[q];
    if (J - 1 > I + 1) load_block(J - 1);  // prefetch the next block while this one is consumed
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = fma(Lc[q], zc, acc[q]);
  }
  // reduce over the 32 rows (lanes) while z_{I+1} is not yet known
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double t = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(~0u, t, o);
    if (lane == q) pacc[8 * h + q] = t;
  }
  __syncthreads();
  if (h == 0) {
    const int gr = r0 + lane;
    pacc[lane] = (gr < D) ? y[(int64_t)gr * ystride] - pacc[lane] : 0.0;  // y_I - sum_{J > I+1}
    const int row = r0 + 32 + lane;
    zn[lane] = (I + 1 < nb && row < D) ? wait_z(zbuf, row, info) : 0.0;  // the chain: z_{I+1}
  }
  __syncthreads();
  mv32<true>(Ln, zn, pacc, -1.0, rv, part);     // rv = y_I - sum_{J > I} L_JI^T z_J
  mv32<false>(W, rv, zero, 1.0, zv, part);      // z = W^T rv
  mv32<false>(Ls, zv, rv, -1.0, res, part);     // res = rv - L_II^T z   (one refinement step)
  mv32<false>(W, res, zv, 1.0, rv, part);       // z += W^T res
  if (h == 0) {
    const int gr = r0 + lane;
    if (gr < D) asm volatile("st.volatile.global.f64 [%0], %1;" ::"l"(zbuf + gr), "d"(rv[lane]) : "memory");
  }
}

fk_status lwork_for(int D, int* lwork) {
  std::lock_guard<std::mutex> lk(g_sol_mu);
  cusolverDnHandle_t h;
  FK_TRY(handle_for_device(&h));
  if (cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, D, nullptr, D, lwork) != CUSOLVER_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cusolverDnDpotrf_bufferSize failed");
  return FK_OK;
}

}  // namespace

size_t solve_ws_bytes(int d, int m, int kind) {
  const int D = unknowns(d, m, kind);
  int lwork = 0;
  if (lwork_for(D + 1, &lwork) != FK_OK) return 0;
  Bump b(nullptr, 0);
  b.take((size_t)(D + 1) * (D + 1) * 8);
  b.take((size_t)lwork * 8);
  b.take((size_t)D * 8);
  b.take(64);
  b.take((size_t)D * 8);  // rcond_estimate vectors
  b.take((size_t)D * 8);
  if (kind == FK_PIK_BOX || kind == FK_PIK_COLLOC) {
    b.take((size_t)D * 16);
    b.take((size_t)d * (4 * m + 1) * 16);
  }
  b.take(chol_ws_bytes(D + 1));
  return b.used + 256;
}

// factorisation path: the tile dataflow kernel (chol.cu) up to kTilesMaxN, cuSOLVER potrf above,
// where the factorisation is throughput bound and cuSOLVER's larger blocking wins (measured on
// B200, potrf alone: tiles 0.45 / cuSOLVER 0.83 ms at N = 2002, 0.92 / 1.41 at 3201, 1.53 / 1.79
// at 4226, 1.84 / 1.97 at 4600, 2.40 / 2.34 at 5000).  FK_CHOL=cusolver|tiles overrides (tests, measurements).
constexpr int kTilesMaxN = 4600;
bool use_tiles(int N) {
  const char* e = getenv("FK_CHOL");
  if (e && e[0] == 'c') return false;
  if (e && e[0] == 't') return true;
  return N <= kTilesMaxN;
}

static fk_status fill_sysargs(const fk_problem* P, SysArgs* out) {
  SysArgs g{};
  g.d = P->d;
  g.m = P->m;
  g.kind = P->kind;
  g.D = unknowns(P->d, P->m, P->kind);
  g.inv_n = 1.0 / P->n_total;
  g.lambda = P->lambda;
  g.s = P->s;
  g.mu_pde = P->mu_pde;
  g.c = 3.14159265358979323846 / (2.0 * P->L);
  g.inv4L = 1.0 / (4.0 * P->L);
  g.mu = (const double2*)P->mu_moments;
  g.cross = (const double2*)P->cross;
  g.mur = (const double2*)P->colloc_moments;
  g.inv_nr = P->n_colloc > 0 ? 1.0 / P->n_colloc : 0.0;
  if (P->kind == FK_PIK_BOX || P->kind == FK_PIK_COLLOC) {
    if (P->n_terms < 0 || P->n_terms > kMaxTerms || P->d > kMaxD) return fail(FK_E_ARG, "fk_solve: at most 8 PDE terms, d <= 4");
    g.n_terms = P->n_terms;
    for (int t = 0; t < P->n_terms; ++t) {
      g.a_alpha[t] = P->a_alpha[t];
      for (int l = 0; l < P->d; ++l) g.alpha[t][l] = P->alpha[t * P->d + l];
    }
    for (int l = 0; l < P->d && P->box; ++l) {
      g.box[l][0] = P->box[2 * l];
      g.box[l][1] = P->box[2 * l + 1];
    }
  }
  *out = g;
  return FK_OK;
}

// ---- regularisation path (many lambda, one pass over the data) -------------
// M(lambda) = M0 + lambda Dg with Dg = P^* R P diagonal (R_k on the centre, 2 R_k on a_k, b_k).
// With Dg^{-1/2} M0 Dg^{-1/2} = V diag(ev) V^T (one dsyevd): z(lambda) = Dg^{-1/2} V (V^T
// Dg^{-1/2} c) / (ev + lambda), i.e. one GEMV and one D x L GEMM for all lambdas.
__global__ void k_path_diag(SysArgs g, double* __restrict__ dg) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.D) return;
  const PCol p = pcol(g, u);
  // R at mode i: the diagonal of A(lambda = 1) minus A(lambda = 0), via entry()
  SysArgs g1 = g, g0 = g;
  g1.lambda = 1.0;
  g0.lambda = 0.0;
  const double r = entry(g1, p.i[0], p.i[0]).x - entry(g0, p.i[0], p.i[0]).x;
  dg[u] = p.cnt * r;
}

__global__ void k_path_scale(double* __restrict__ M, int64_t ld, int D, const double* __restrict__ dg) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)D * D; t += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(t / D), u = (int)(t % D);
    if (u < v) continue;
    M[u + v * ld] *= rsqrt(dg[u]) * rsqrt(dg[v]);
  }
}

__global__ void k_path_rhs(const double* __restrict__ M, int64_t ld, int D, const double* __restrict__ dg, double* __restrict__ c) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < D) c[u] = M[D + u * ld] * rsqrt(dg[u]);  // c lives in the augmented row D
}

__global__ void k_path_weights(const double* __restrict__ w, const double* __restrict__ ev, const double* __restrict__ lams, int D,
                               int nl, double* __restrict__ S) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)D * nl; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t % D), l = (int)(t / D);
    S[t] = w[u] / (ev[u] + lams[l]);
  }
}

__global__ void k_path_theta(SysArgs g, const double* __restrict__ Z, const double* __restrict__ dg, int nl, double2* __restrict__ theta) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)g.D * nl; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t % g.D), l = (int)(t / g.D);
    const int v = g.kind == FK_ADDITIVE ? u % (2 * g.m + 1) : u;
    const double* z = Z + (int64_t)l * g.D;
    double2* th = theta + (int64_t)l * g.D;
    if (v == 0) {
      const int c0 = g.kind == FK_ADDITIVE ? u - v + g.m : (g.D - 1) / 2;
      th[c0] = make_double2(z[u] * rsqrt(dg[u]), 0.0);
    } else if (v & 1) {
      const PCol p = pcol(g, u);
      const double a = z[u] * rsqrt(dg[u]), b = z[u + 1] * rsqrt(dg[u + 1]);
      th[p.i[0]] = make_double2(a, b);
      th[p.i[1]] = make_double2(a, -b);
    }
  }
}

static fk_status syevd_lwork(int D, int ld, int* lwork) {
  std::lock_guard<std::mutex> lk(g_sol_mu);
  cusolverDnHandle_t h;
  FK_TRY(handle_for_device(&h));
  if (cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, nullptr, ld, nullptr, lwork) !=
      CUSOLVER_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cusolverDnDsyevd_bufferSize failed");
  return FK_OK;
}

struct PathWs {
  double *M, *work, *dg, *ev, *wv, *lam, *S, *Z;
  int* info;
  double2 *dsym, *boxt;
};
// one layout for the size query and the run
static void path_layout(Bump& b, int d, int m, int kind, int D, int lwork, int nlam, PathWs* w) {
  const int N = D + 1;
  w->M = (double*)b.take((size_t)N * N * 8);
  w->work = (double*)b.take((size_t)lwork * 8);
  w->dg = (double*)b.take((size_t)D * 8);
  w->ev = (double*)b.take((size_t)D * 8);
  w->wv = (double*)b.take((size_t)D * 8);
  w->lam = (double*)b.take((size_t)nlam * 8);
  w->S = (double*)b.take((size_t)D * nlam * 8);
  w->Z = (double*)b.take((size_t)D * nlam * 8);
  w->info = (int*)b.take(16);
  w->dsym = w->boxt = nullptr;
  if (kind == FK_PIK_BOX || kind == FK_PIK_COLLOC) {
    w->dsym = (double2*)b.take((size_t)D * 16);
    w->boxt = (double2*)b.take((size_t)d * (4 * m + 1) * 16);
  }
}

size_t solve_path_ws_bytes(int d, int m, int kind, int nlam) {
  const int D = unknowns(d, m, kind);
  int lwork = 0;
  if (syevd_lwork(D, D + 1, &lwork) != FK_OK) return 0;
  Bump b(nullptr, 0);
  PathWs w;
  path_layout(b, d, m, kind, D, lwork, std::max(nlam, 1), &w);
  return b.used;
}

static double solve_cost_ms(const SysArgs& g);
size_t solve_ws_bytes(int d, int m, int kind);

fk_status solve_path_run(const fk_problem* P, const double* lambdas, int nlam, double* theta, int* info_out, void* ws, size_t ws_bytes,
                         cudaStream_t s) {
  SysArgs g;
  FK_TRY(fill_sysargs(P, &g));
  {
    // Large Sobolev systems: one fk_solve per lambda (the CG path where it is cheaper) when that
    // beats one eigendecomposition (~2.7 s at N = 16642 on the B200, tools/path_large.py).
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    const double t_eig = 2700.0 * std::pow((g.D + 1) / 16642.0, 3.0);
    double t_each = 0.0;
    if (cap == cudaStreamCaptureStatusNone && g.kind == FK_SOBOLEV && g.d <= 2 && g.D + 1 > 9000 &&
        solve_ws_bytes(P->d, P->m, P->kind) <= ws_bytes) {
      for (int l = 0; l < nlam; ++l) {
        SysArgs gl = g;
        gl.lambda = lambdas[l];
        t_each += solve_cost_ms(gl);
      }
    }
    if (t_each > 0.0 && t_each < t_eig) {
      for (int l = 0; l < nlam; ++l) {
        if (!(lambdas[l] > 0.0)) return fail(FK_E_ARG, "fk_solve_path: lambda must be > 0");
        fk_problem Pl = *P;
        Pl.lambda = lambdas[l];
        FK_TRY(solve_run(&Pl, theta + (int64_t)2 * g.D * l, nullptr, ws, ws_bytes, s));
      }
      if (info_out) {
        FK_CUDA_TRY(cudaStreamSynchronize(s));
        *info_out = 0;
      }
      return FK_OK;
    }
  }
  g.lambda = 0.0;  // M0: the data (and PDE) part only
  const int D = g.D, N = D + 1;
  int lwork = 0;
  FK_TRY(syevd_lwork(D, N, &lwork));
  Bump b(ws, ws_bytes);
  PathWs w;
  path_layout(b, P->d, P->m, P->kind, D, lwork, nlam, &w);
  double *M = w.M, *work = w.work, *dg = w.dg, *ev = w.ev, *wv = w.wv, *lam_d = w.lam, *S = w.S, *Z = w.Z;
  int* info = w.info;
  double2 *dsym = w.dsym, *boxt = w.boxt;
  if (!b.ok()) return fail(FK_E_WORKSPACE, "fk_solve_path: workspace too small");
  const int sms = device_sm_count();
  FK_CUDA_TRY(cudaMemcpyAsync(lam_d, lambdas, (size_t)nlam * 8, cudaMemcpyHostToDevice, s));
  if (dsym) {
    const int nt = std::max(D, P->d * (4 * P->m + 1));
    k_pi_tables<<<(nt + 255) / 256, 256, 0, s>>>(g, dsym, boxt);
    g.dsym = dsym;
    g.boxt = boxt;
    count_launch();
  }
  launch_assemble(g, M, s);
  k_rhs_real<<<(N + 255) / 256, 256, 0, s>>>(g, (const double2*)P->rhs, M, nullptr, nullptr, CholReset{});
  k_path_diag<<<(D + 255) / 256, 256, 0, s>>>(g, dg);
  k_path_scale<<<sms * 8, 256, 0, s>>>(M, N, D, dg);
  k_path_rhs<<<(D + 255) / 256, 256, 0, s>>>(M, N, D, dg, Z);  // scaled c into Z[:,0] (scratch)
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(5);
  {
    std::lock_guard<std::mutex> lk(g_sol_mu);
    cusolverDnHandle_t h;
    FK_TRY(handle_for_device(&h));
    if (cusolverDnSetStream(h, s) != CUSOLVER_STATUS_SUCCESS) return fail(FK_E_CUDA, "cusolverDnSetStream failed");
    if (cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, D, M, N, ev, work, lwork, info) !=
        CUSOLVER_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cusolverDnDsyevd failed");
    cublasHandle_t bh;
    FK_TRY(blas_for_device(&bh));
    if (cublasSetStream(bh, s) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasSetStream failed");
    const double one = 1.0, zero = 0.0;
    // w = V^T (Dg^{-1/2} c)
    if (cublasDgemv(bh, CUBLAS_OP_T, D, D, &one, M, N, Z, 1, &zero, wv, 1) != CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDgemv failed");
    k_path_weights<<<sms * 4, 256, 0, s>>>(wv, ev, lam_d, D, nlam, S);
    count_launch();
    // Z = V S  (D x nlam)
    if (cublasDgemm(bh, CUBLAS_OP_N, CUBLAS_OP_N, D, nlam, D, &one, M, N, S, D, &zero, Z, D) != CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDgemm failed");
  }
  k_path_theta<<<sms * 4, 256, 0, s>>>(g, Z, dg, nlam, (double2*)theta);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  if (info_out) {
    int hinfo = 0;
    FK_CUDA_TRY(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, s));
    FK_CUDA_TRY(cudaStreamSynchronize(s));
    *info_out = hinfo;
    if (hinfo != 0) return fail(FK_E_SOLVE, "fk_solve_path: eigensolver failed, info = " + std::to_string(hinfo));
  }
  return FK_OK;
}

// ---- held-out risk along the path (grid search; reading R11) -----------------
// For real Y and Hermitian theta, f(x) = sum_k theta_k e^{i k t} is real and, with the validation
// set's moments mu^v, rhs r^v (n_v samples):  sum_j (Y_j - f(x_j))^2 / n_v
//   = sum_y2 / n_v - 2 Re(theta^* r^v) / n_v + theta^* T(mu^v) theta / n_v
//   = sum_y2 / n_v - 2 z^T c_v + z^T M_v z      (z = real coordinates of theta, theta = P z)
// with M_v, c_v the real-reduced data system of the validation moments (k_assemble_real, lambda = 0).
__global__ void k_z_from_theta(SysArgs g, const double2* __restrict__ theta, int nl, double* __restrict__ Z) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)g.D * nl; t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t % g.D), l = (int)(t / g.D);
    const double2* th = theta + (int64_t)l * g.D;
    const int v = g.kind == FK_ADDITIVE ? u % (2 * g.m + 1) : u;
    double z;
    if (v == 0) {
      z = th[g.kind == FK_ADDITIVE ? u - v + g.m : (g.D - 1) / 2].x;
    } else {
      const PCol p = pcol(g, u);
      z = (v & 1) ? th[p.i[0]].x : th[p.i[0]].y;
    }
    Z[t] = z;
  }
}

__global__ void k_val_risk(const double* __restrict__ Z, const double* __restrict__ W, const double* __restrict__ M, int64_t ld, int D,
                           double base, double* __restrict__ out) {
  const int l = blockIdx.x;
  const double* z = Z + (int64_t)l * D;
  const double* w = W + (int64_t)l * D;
  double acc = 0.0;
  for (int u = threadIdx.x; u < D; u += blockDim.x) acc += z[u] * (w[u] - 2.0 * M[D + u * ld]);
  __shared__ double red[32];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) out[l] = base + acc;
  }
}

size_t path_validate_ws_bytes(int d, int m, int kind, int nlam) {
  const int D = unknowns(d, m, kind), N = D + 1;
  Bump b(nullptr, 0);
  b.take((size_t)N * N * 8);
  b.take((size_t)D * std::max(nlam, 1) * 8);
  b.take((size_t)D * std::max(nlam, 1) * 8);
  return b.used;
}

fk_status path_validate_run(const fk_problem* Pv, const double* theta, int nlam, double sum_y2, double* risk_out, void* ws,
                            size_t ws_bytes, cudaStream_t s) {
  SysArgs g;
  FK_TRY(fill_sysargs(Pv, &g));
  g.lambda = 0.0;
  g.mu_pde = 0.0;
  if (g.kind == FK_PIK_BOX || g.kind == FK_PIK_COLLOC) g.kind = FK_SOBOLEV;  // data part only
  const int D = g.D, N = D + 1;
  Bump b(ws, ws_bytes);
  double* M = (double*)b.take((size_t)N * N * 8);
  double* Z = (double*)b.take((size_t)D * nlam * 8);
  double* W = (double*)b.take((size_t)D * nlam * 8);
  if (!b.ok()) return fail(FK_E_WORKSPACE, "fk_path_validate: workspace too small");
  const int sms = device_sm_count();
  launch_assemble(g, M, s);
  k_rhs_real<<<(N + 255) / 256, 256, 0, s>>>(g, (const double2*)Pv->rhs, M, nullptr, nullptr, CholReset{});
  k_z_from_theta<<<sms * 4, 256, 0, s>>>(g, (const double2*)theta, nlam, Z);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(3);
  {
    std::lock_guard<std::mutex> lk(g_sol_mu);
    cublasHandle_t bh;
    FK_TRY(blas_for_device(&bh));
    if (cublasSetStream(bh, s) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasSetStream failed");
    const double one = 1.0, zero = 0.0;
    if (cublasDsymm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, D, nlam, &one, M, N, Z, D, &zero, W, D) != CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDsymm failed");
  }
  k_val_risk<<<nlam, 256, 0, s>>>(Z, W, M, N, D, sum_y2 * g.inv_n, risk_out);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  return FK_OK;
}

// ------------------------------------------------------------------------------------------
// Preconditioned conjugate gradients for the Sobolev system at large D (NEXT-3; the paper's own
// solver, with FFT-Toeplitz products).  Real form P^*AP z = P^*r/n as in the dense path.
//   matvec: theta = P z -> Hermitian half spectrum -> cuFFT Z2D -> x (DFT of mu)/(n L^d) -> D2Z
//           -> (T theta)_k / n, + lambda R_k theta_k, -> P^* (a_k: 2 Re, b_k: 2 Im, centre: Re);
//           circular length L >= 4m+1 per dimension keeps k1 - k2 in [-2m, 2m] alias free.
//   preconditioner (DESIGN.md §5 "Solve", reading R13): the real unknowns of the modes with
//           lambda R_k <= tau form a dense block, inverted once (tile Cholesky, recursive TRMM
//           inverse, LAUUM); the others take Jacobi.  Where lambda R_k > tau the penalty dominates
//           the row and T/n (norm <= mu_0/n = 1) is a bounded perturbation; the near-null space of
//           T (functions living outside the data's half period) is carried by the low modes, whose
//           block is exact.  C3 (m = 64, s = 2, lambda = 1e-6, tau = 0.5): 2221 of 16641 unknowns
//           in the block, 47 iterations to ||r|| <= 1e-13 ||b||.
//   every iteration: 5 own kernels + 3 cuFFT kernels; the CG scalars are grid sums finished by the
//           last CTA in CTA order (bitwise reproducible); convergence is read back every 10 steps.
// ------------------------------------------------------------------------------------------
// block threshold tau: lambda R_k <= tau.  C3 (B200): tau = 0.25 / 0.5 / 1 / 2 -> 65 / 47 / 34 / 25
// iterations, 5.82 / 5.81 / 6.70 / 10.2 ms per solve
static double pcg_tau() {
  const char* e = getenv("FK_PCG_TAU");
  return e ? atof(e) : 0.5;
}

__device__ __forceinline__ double rentry(const SysArgs& g, int u, int v) {
  const PCol pu = pcol(g, u), pv = pcol(g, v);
  const int side = 2 * g.m + 1;
  const float inv_side = 1.0f / (float)side;
  double s = 0.0;
  for (int x = 0; x < pu.cnt; ++x)
    for (int y = 0; y < pv.cnt; ++y) {
      const double2 a = g.d == 2 ? entry_d2(g, pu.i[x], pv.i[y], side, inv_side) : entry(g, pu.i[x], pv.i[y]);
      s += cmul(cmul(cconj(pu.a[x]), a), pv.a[y]).x;
    }
  return s;
}

// lower triangle of the low block, column b = blockIdx.y
__global__ void k_pcg_low_block(SysArgs g, const int* __restrict__ low, int Dl, double* __restrict__ B, int64_t ld) {
  const int b = blockIdx.y;
  const int a = b + blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= Dl) return;
  B[a + b * ld] = rentry(g, low[a], low[b]);
}

// dinv[u] = 1 / (P^*AP)_uu for Jacobi unknowns, 0 for block unknowns; bz = P^* r / n
__global__ void k_pcg_setup(SysArgs g, const int* __restrict__ lowpos, const double2* __restrict__ r, double* __restrict__ dinv,
                            double* __restrict__ bz) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= g.D) return;
  dinv[u] = lowpos[u] >= 0 ? 0.0 : 1.0 / rentry(g, u, u);
  const PCol p = pcol(g, u);
  double s = 0.0;
  for (int x = 0; x < p.cnt; ++x) s += cmul(cconj(p.a[x]), make_double2(r[p.i[x]].x * g.inv_n, r[p.i[x]].y * g.inv_n)).x;
  bz[u] = s;
}

// Hermitian half spectrum of an index-space array: entry (j0, j1), j1 <= L1/2, holds v_k with
// k0 = j0 (or j0 - L0), k1 = j1 (d = 1: a single row, k = j).  mode(): -1 outside |k| <= lim.
struct PcgGrid {
  int d, L0, L1, H1;  // H1 = L1/2 + 1 (d = 2); d = 1: L0 = 1, L1 = L
};
__device__ __forceinline__ void half_to_k(const PcgGrid& q, int64_t t, int& k0, int& k1) {
  const int j0 = (int)(t / q.H1), j1 = (int)(t % q.H1);
  k0 = q.d == 2 ? (j0 <= q.L0 / 2 ? j0 : j0 - q.L0) : 0;
  k1 = j1;
}

// mu (|q| <= 2m) into the half spectrum (k1 >= 0), zero elsewhere
__global__ void k_pcg_mu_half(SysArgs g, PcgGrid q, double2* __restrict__ H) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)(q.d == 2 ? q.L0 : 1) * q.H1) return;
  int k0, k1;
  half_to_k(q, t, k0, k1);
  const int M2 = 2 * g.m, qs = 4 * g.m + 1;
  double2 v = make_double2(0.0, 0.0);
  if (k1 <= M2 && k0 >= -M2 && k0 <= M2) v = q.d == 2 ? g.mu[(int64_t)(k0 + M2) * qs + (k1 + M2)] : g.mu[k1 + M2];
  H[t] = v;
}

__global__ void k_pcg_scale(double* __restrict__ a, int64_t n, double s) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n) a[t] *= s;
}

// Deterministic grid-wide sum: every CTA writes its partial, the last CTA to arrive (atomic
// ticket) adds the partials in CTA order (lane-strided, then a fixed xor tree) and runs fin(sum)
// on thread 0.  sc scalars: [0] rz, [1] rr, [2] bb, [3] alpha, [4] done, [5] beta.
template <class Fin>
__device__ __forceinline__ void grid_sum(double v, double* __restrict__ part, unsigned* __restrict__ ticket, Fin fin) {
  __shared__ double red[32];
  __shared__ int last;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    part[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double acc = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) acc += __ldcg(part + i);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) {
      *ticket = 0;
      fin(acc);
    }
  }
}

// p_new = z + beta p_old (beta = sc[5]) for every unknown, theta = P p_new into the half spectrum.
// Each half-spectrum entry with |k| <= m carries one mode pair (its own or its mirror's); entries
// on the k1 = 0 column carry a pair twice and write identical values.
__global__ void k_pcg_scatter(SysArgs g, PcgGrid q, const double* __restrict__ z, const double* __restrict__ p_old,
                              double* __restrict__ p_new, double2* __restrict__ H, const double* __restrict__ sc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)(q.d == 2 ? q.L0 : 1) * q.H1 || sc[4] != 0.0) return;
  const double beta = sc[5];
  int k0, k1;
  half_to_k(q, t, k0, k1);
  const int m = g.m, side = 2 * m + 1, c0 = (g.D - 1) / 2;
  double2 v = make_double2(0.0, 0.0);
  if (k1 <= m && k0 >= -m && k0 <= m) {
    const int lin = q.d == 2 ? (k0 + m) * side + (k1 + m) : k1 + m;
    if (lin == c0) {
      const double a = z[0] + beta * p_old[0];
      p_new[0] = a;
      v = make_double2(a, 0.0);
    } else {
      const int u = 2 * (lin > c0 ? lin - c0 : c0 - lin) - 1;
      const double a = z[u] + beta * p_old[u], b = z[u + 1] + beta * p_old[u + 1];
      p_new[u] = a;
      p_new[u + 1] = b;
      v = make_double2(a, lin > c0 ? b : -b);
    }
  }
  H[t] = v;
}

__global__ void k_pcg_mul(double* __restrict__ G, const double* __restrict__ muhat, int64_t n, const double* __restrict__ sc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < n && sc[4] == 0.0) G[t] *= muhat[t];
}

// ---- physics-informed penalty in the CG product (readings R3, R12) -----------------
// mu_pde D^* S D with S Toeplitz: the box's Fourier matrix S[k1][k2] = prod_l boxt_l(k2_l - k1_l)
// (PIK_BOX) or the collocation moments' T(mu_r)/n_r (PIK_COLLOC).  As a convolution S v =
// s' * v with s'(j) = prod_l boxt_l(-j_l) (box) / mu_r(j) / n_r (colloc), a Hermitian sequence,
// so it takes the same half-spectrum -> real grid -> pointwise product -> back route as T(mu).
__device__ __forceinline__ int mode_lin(const SysArgs& g, int k0, int k1) {  // index of mode (k0, k1) / (k1)
  const int side = 2 * g.m + 1;
  return g.d == 2 ? (k0 + g.m) * side + (k1 + g.m) : k1 + g.m;
}

__global__ void k_pcg_pi_half(SysArgs g, PcgGrid q, double2* __restrict__ H) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)(q.d == 2 ? q.L0 : 1) * q.H1) return;
  int k0, k1;
  half_to_k(q, t, k0, k1);
  const int M2 = 2 * g.m, qs = 4 * g.m + 1;
  double2 v = make_double2(0.0, 0.0);
  if (k1 <= M2 && k0 >= -M2 && k0 <= M2) {
    if (g.kind == FK_PIK_COLLOC) {
      v = q.d == 2 ? g.mur[(int64_t)(k0 + M2) * qs + (k1 + M2)] : g.mur[k1 + M2];
      v.x *= g.inv_nr;
      v.y *= g.inv_nr;
    } else if (q.d == 2) {
      v = cmul(g.boxt[0 * qs + (-k0 + M2)], g.boxt[1 * qs + (-k1 + M2)]);
    } else {
      v = g.boxt[-k1 + M2];
    }
  }
  H[t] = v;
}

// Hd = d_k H_k for |k| <= m (the PDE symbol of the iterate), zero elsewhere
__global__ void k_pcg_dmul(SysArgs g, PcgGrid q, const double2* __restrict__ H, double2* __restrict__ Hd, const double* __restrict__ sc) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)(q.d == 2 ? q.L0 : 1) * q.H1 || sc[4] != 0.0) return;
  int k0, k1;
  half_to_k(q, t, k0, k1);
  double2 v = make_double2(0.0, 0.0);
  if (k1 <= g.m && k0 >= -g.m && k0 <= g.m) v = cmul(g.dsym[mode_lin(g, k0, k1)], H[t]);
  Hd[t] = v;
}

// q = P^* (T theta / n + lambda R theta), theta = P p; alpha = rz / p.q
__global__ void __launch_bounds__(256) k_pcg_gather(SysArgs g, PcgGrid q, const double2* __restrict__ C, const double* __restrict__ p,
                                                    double* __restrict__ out, double* __restrict__ sc, double* __restrict__ part,
                                                    unsigned* __restrict__ ticket, const double2* __restrict__ Cd) {
  if (sc[4] != 0.0) return;
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  double pq = 0.0;
  if (u < g.D) {
    const int m = g.m, side = 2 * m + 1, c0 = (g.D - 1) / 2;
    const int t = (u + 1) >> 1;
    const int lin = c0 + t;
    int k0 = 0, k1 = lin - m;
    if (q.d == 2) {
      k0 = lin / side - m;
      k1 = lin % side - m;
    }
    double2 c;
    const int64_t at = k1 >= 0 ? (int64_t)(q.d == 2 ? (k0 >= 0 ? k0 : k0 + q.L0) : 0) * q.H1 + k1
                               : (int64_t)(-k0 >= 0 ? -k0 : -k0 + q.L0) * q.H1 + (-k1);
    if (k1 >= 0) {
      c = C[at];
    } else {  // k1 < 0 (d = 2 only): c_k = conj c_{-k}
      c = cconj(C[at]);
    }
    if (Cd) {  // + mu_pde conj(d_k) (S D theta)_k (the PI penalty; Cd is Hermitian like C)
      const double2 e = k1 >= 0 ? Cd[at] : cconj(Cd[at]);
      const double2 pi = cmul(cconj(g.dsym[mode_lin(g, k0, k1)]), e);
      c.x += pi.x;
      c.y += pi.y;
    }
    const double nk2 = (double)k0 * k0 + (double)k1 * k1;
    const double lr = g.lambda * (1.0 + pow(nk2, g.s));
    double o;
    if (u == 0) o = c.x + lr * p[0];
    else if (u & 1) o = 2.0 * (c.x + lr * p[u]);  // a_t column: |e_k + e_-k|^2 = 2
    else o = 2.0 * (c.y + lr * p[u]);
    out[u] = o;
    pq = p[u] * o;
  }
  grid_sum(pq, part, ticket, [&](double s) { sc[3] = sc[0] / s; });
}

// x += alpha p, r -= alpha q, rl = r[low], rr = r.r; done when rr <= tol^2 bb
__global__ void __launch_bounds__(256) k_pcg_update(int D, const double* __restrict__ p, const double* __restrict__ qv,
                                                    const int* __restrict__ lowpos, double* __restrict__ x,
                                                    double* __restrict__ r, double* __restrict__ rl, double* __restrict__ sc,
                                                    double tol2, double* __restrict__ part, unsigned* __restrict__ ticket) {
  if (sc[4] != 0.0) return;
  const double alpha = sc[3];
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  double rr = 0.0;
  if (u < D) {
    x[u] += alpha * p[u];
    const double v = r[u] - alpha * qv[u];
    r[u] = v;
    rr = v * v;
    const int a = lowpos[u];  // position in the block, -1 for Jacobi unknowns
    if (a >= 0) rl[a] = v;
  }
  grid_sum(rr, part, ticket, [&](double s) {
    sc[1] = s;
    sc[6] += 1.0;  // iterations
    if (s <= tol2 * sc[2]) sc[4] = 1.0;
  });
}

// z = M^{-1} r: block rows z[low[a]] = (Ainv rl)_a, one warp per row reading column a of the
// symmetric Ainv (contiguous); Jacobi rows z = dinv r.  rz = r.z; beta = rz / rz_old (0 first).
__global__ void __launch_bounds__(256) k_pcg_precond(int D, const double* __restrict__ r, const double* __restrict__ dinv,
                                                     const int* __restrict__ lowpos, const int* __restrict__ low, int Dl,
                                                     const double* __restrict__ Ainv, int64_t lda, const double* __restrict__ rl,
                                                     double* __restrict__ z, double* __restrict__ sc, int first, int nlow_ctas,
                                                     double* __restrict__ part, unsigned* __restrict__ ticket) {
  if (sc[4] != 0.0) return;
  double rz = 0.0;
  if ((int)blockIdx.x < nlow_ctas) {
    const int a = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (a < Dl) {
      const double* col = Ainv + (int64_t)a * lda;
      double acc = 0.0;
      const int D2 = Dl & ~1;
      for (int b = 2 * lane; b < D2; b += 64) {
        const double2 av = __ldg(reinterpret_cast<const double2*>(col + b));
        const double2 rv = __ldg(reinterpret_cast<const double2*>(rl + b));
        acc = fma(av.x, rv.x, acc);
        acc = fma(av.y, rv.y, acc);
      }
      if ((Dl & 1) && lane == 0) acc = fma(col[Dl - 1], rl[Dl - 1], acc);
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        z[low[a]] = acc;
        rz = rl[a] * acc;
      }
    }
  } else {
    const int u = (blockIdx.x - nlow_ctas) * blockDim.x + threadIdx.x;
    if (u < D && lowpos[u] < 0) {
      const double v = r[u] * dinv[u];
      z[u] = v;
      rz = r[u] * v;
    }
  }
  grid_sum(rz, part, ticket, [&](double s) {
    sc[5] = first ? 0.0 : s / sc[0];
    sc[0] = s;
  });
}

// x = 0, r = b, rl = b[low], bb = b.b
__global__ void __launch_bounds__(256) k_pcg_init(int D, const double* __restrict__ b, const int* __restrict__ low, int Dl,
                                                  double* __restrict__ x, double* __restrict__ r, double* __restrict__ rl,
                                                  double* __restrict__ sc, double* __restrict__ part, unsigned* __restrict__ ticket) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  double bb = 0.0;
  if (u < D) {
    x[u] = 0.0;
    r[u] = b[u];
    bb = b[u] * b[u];
  }
  if (u < Dl) rl[u] = b[low[u]];
  grid_sum(bb, part, ticket, [&](double s) {
    sc[2] = s;
    sc[1] = s;
    sc[4] = 0.0;
  });
}

__global__ void k_pcg_unit_diag(double* __restrict__ X, int64_t ld, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) X[i + i * ld] = 1.0;
}

// lower -> upper (column-major, ld): the block inverse is read by columns as rows
__global__ void k_pcg_symmetrize(double* __restrict__ A, int64_t ld, int n) {
  const int j = blockIdx.y, i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && i > j) A[j + i * ld] = A[i + j * ld];
}

// X = L^{-1} (lower, n x n) by recursive halving: X21 = -X22 L21 X11 (two TRMMs, n^3/3 flops at
// GEMM-like rates); leaves of 256 columns by TRSM on the identity.  X is zero above the diagonal
// and has a unit diagonal on entry; S: scratch of n^2/4 doubles.
// leaves of the recursive inverse: cuBLAS TRSM / SYRK below this size (256: 6.87, 512: 6.70 ms at C3)
constexpr int kPcgLeaf = 512;

static fk_status tri_inv(cublasHandle_t bh, const double* L, int64_t ld, double* X, int64_t ldx, int n, double* S) {
  const double one = 1.0, mone = -1.0;
  if (n <= kPcgLeaf) {
    if (cublasDtrsm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n, n, &one, L, (int)ld, X, (int)ldx) !=
        CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDtrsm failed");
    return FK_OK;
  }
  const int n1 = ((n / 2) + 31) / 32 * 32, n2 = n - n1;
  FK_TRY(tri_inv(bh, L, ld, X, ldx, n1, S));
  FK_TRY(tri_inv(bh, L + n1 + n1 * ld, ld, X + n1 + n1 * ldx, ldx, n2, S));
  if (cublasDtrmm(bh, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n2, n1, &one, X, (int)ldx, L + n1,
                  (int)ld, S, n2) != CUBLAS_STATUS_SUCCESS ||
      cublasDtrmm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n2, n1, &mone, X + n1 + n1 * ldx,
                  (int)ldx, S, n2, X + n1, (int)ldx) != CUBLAS_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cublasDtrmm failed");
  return FK_OK;
}

// lower(A) = X^T X for lower-triangular X (LAUUM by recursive halving, n^3/3 flops):
// A11 = X11^T X11 + X21^T X21, A21 = X22^T X21, A22 = X22^T X22.
static fk_status lauum(cublasHandle_t bh, const double* X, int64_t ldx, double* A, int64_t lda, int n) {
  const double one = 1.0, zero = 0.0;
  if (n <= kPcgLeaf) {
    if (cublasDsyrk(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n, n, &one, X, (int)ldx, &zero, A, (int)lda) != CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDsyrk failed");
    return FK_OK;
  }
  const int n1 = ((n / 2) + 31) / 32 * 32, n2 = n - n1;
  FK_TRY(lauum(bh, X, ldx, A, lda, n1));
  if (cublasDsyrk(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n1, n2, &one, X + n1, (int)ldx, &one, A, (int)lda) != CUBLAS_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cublasDsyrk failed");
  if (cublasDtrmm(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, n2, n1, &one, X + n1 + n1 * ldx,
                  (int)ldx, X + n1, (int)ldx, A + n1, (int)lda) != CUBLAS_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cublasDtrmm failed");
  return lauum(bh, X + n1 + n1 * ldx, ldx, A + n1 + n1 * lda, lda, n2);
}

// per-device stream + events for the CG iterations (created once, kept for the process)
static fk_status pcg_stream(cudaStream_t* cs, cudaEvent_t* ev_in, cudaEvent_t* ev_out) {
  static std::mutex mu;
  static std::map<int, std::tuple<cudaStream_t, cudaEvent_t, cudaEvent_t>> per_dev;
  int dev = 0;
  FK_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = per_dev.find(dev);
  if (it == per_dev.end()) {
    cudaStream_t st;
    cudaEvent_t a, b;
    FK_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    FK_CUDA_TRY(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
    FK_CUDA_TRY(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
    it = per_dev.emplace(dev, std::make_tuple(st, a, b)).first;
  }
  *cs = std::get<0>(it->second);
  *ev_in = std::get<1>(it->second);
  *ev_out = std::get<2>(it->second);
  return FK_OK;
}

static bool pcg_pi(const SysArgs& g) { return (g.kind == FK_PIK_BOX || g.kind == FK_PIK_COLLOC) && g.mu_pde != 0.0; }

static bool pcg_eligible(const SysArgs& g) {
  // Sobolev, and the physics-informed estimators (their penalty mu_pde D^* S D joins the product as
  // a second Toeplitz convolution)
  if (g.d > 2) return false;
  if (!(g.kind == FK_SOBOLEV || ((g.kind == FK_PIK_BOX || g.kind == FK_PIK_COLLOC) && g.dsym))) return false;
  if (g.kind == FK_SOBOLEV && g.mu_pde != 0.0) return false;
  const char* e = getenv("FK_SOLVER");
  if (pcg_pi(g)) return e && e[0] == 'p';  // PI systems: CG on request (its preconditioner treats the
                                            // non-diagonal penalty of the high modes by Jacobi only)
  if (e && e[0] == 'd') return false;
  if (e && e[0] == 'p') return true;
  return g.D + 1 > kTilesMaxN;
}

// the block unknowns: modes with lambda R_k <= tau (both real unknowns of a mode together)
static void pcg_low_set(const SysArgs& g, double tau, std::vector<int>& low, std::vector<int>& lowpos) {
  const int m = g.m, side = 2 * m + 1, c0 = (g.D - 1) / 2;
  low.clear();
  lowpos.assign(g.D, -1);
  for (int u = 0; u < g.D; ++u) {
    const int lin = c0 + ((u + 1) >> 1);
    const int k0 = g.d == 2 ? lin / side - m : 0, k1 = g.d == 2 ? lin % side - m : lin - m;
    const double R = 1.0 + std::pow((double)k0 * k0 + (double)k1 * k1, g.s);
    if (g.lambda * R <= tau) {
      lowpos[u] = (int)low.size();
      low.push_back(u);
    }
  }
}

// Solves into x (D reals).  Returns FK_OK with *iters, or FK_E_SOLVE when it does not converge.
// ws: at least (D+1)^2 doubles (the dense path's matrix slot).  Caller holds g_sol_mu.
// predicted ms of fk_solve for g (the cheaper of the two paths; same model as pcg_run's choice)
static double solve_cost_ms(const SysArgs& g) {
  const double t_dense = 56.0 * std::pow((g.D + 1) / 16642.0, 3.0) + 0.5;
  if (g.kind != FK_SOBOLEV || g.d > 2 || g.mu_pde != 0.0 || g.D + 1 <= kTilesMaxN) return t_dense;  // (PI: dense unless forced)
  std::vector<int> low, lowpos;
  pcg_low_set(g, pcg_tau(), low, lowpos);
  return std::min(t_dense, 3.0 * std::pow(low.size() / 2221.0, 1.8) + 2.8);
}

static fk_status pcg_run(SysArgs g, const double2* r, double* x, int* iters, void* ws, size_t ws_bytes, void* chol_ws, int* info,
                         cudaStream_t s) {
  std::vector<int> low, lowpos;
  pcg_low_set(g, pcg_tau(), low, lowpos);
  const int D = g.D, Dl = (int)low.size();
  // cost model from B200 measurements (tools/pcg_lams.py): dense cuSOLVER potrf
  // ~56 ms at N = 16642 (N^3); the CG path: the block + ~2.8 ms for ~47 iterations
  const char* fe = getenv("FK_SOLVER");
  const double t_dense = 56.0 * std::pow((D + 1) / 16642.0, 3.0) + 0.5;
  const double t_pcg = 3.0 * std::pow(Dl / 2221.0, 1.8) + 2.8;  // block: 3.0 / 7.5 / 22.8 ms at Dl = 2221 / 3930 / 7030
  if (!(fe && fe[0] == 'p') && !(t_pcg < t_dense)) return FK_E_UNSUPPORTED;  // the dense path (no error text)
  PcgGrid q{};
  q.d = g.d;
  const int L = fft_friendly(4 * g.m + 1);
  q.L0 = g.d == 2 ? L : 1;
  q.L1 = L;
  q.H1 = q.L1 / 2 + 1;
  const int64_t nreal = (int64_t)q.L0 * q.L1, nhalf = (int64_t)q.L0 * q.H1;
  FftPlan fz, fd;
  int dims[2] = {g.d == 2 ? q.L0 : q.L1, q.L1};
  FK_TRY(fft_plan(g.d, dims, 1, CUFFT_Z2D, &fz));
  FK_TRY(fft_plan(g.d, dims, 1, CUFFT_D2Z, &fd));
  const int64_t lda = (Dl + 1) & ~1;  // even: 16-byte aligned columns for the preconditioner's loads
  const int TB = 256;
  const int gD = (D + TB - 1) / TB, nlow_ctas = (Dl + 7) / 8, gP = nlow_ctas + gD;
  Bump b(ws, ws_bytes);
  double* Ainv = (double*)b.take((size_t)lda * Dl * 8 + 16);
  double* Xinv = (double*)b.take((size_t)lda * Dl * 8 + 16);
  double* S = (double*)b.take((size_t)(Dl / 2 + 32) * (Dl / 2 + 32) * 8);  // n2 x n1 of tri_inv's top level
  int* d_low = (int*)b.take((size_t)Dl * 4 + 4);
  int* d_lowpos = (int*)b.take((size_t)D * 4);
  double* dinv = (double*)b.take((size_t)D * 8);
  double* bz = (double*)b.take((size_t)D * 8);
  double* rv = (double*)b.take((size_t)D * 8);
  double* zv = (double*)b.take((size_t)D * 8);
  double* pv[2] = {(double*)b.take((size_t)D * 8), (double*)b.take((size_t)D * 8)};
  double* qv = (double*)b.take((size_t)D * 8);
  double* rl = (double*)b.take((size_t)Dl * 8 + 16);
  double2* H = (double2*)b.take((size_t)nhalf * 16);
  double* G = (double*)b.take((size_t)nreal * 8);
  double* muhat = (double*)b.take((size_t)nreal * 8);
  const bool pi = pcg_pi(g);
  double2* Hd = pi ? (double2*)b.take((size_t)nhalf * 16) : nullptr;  // PI penalty: D theta, then S D theta
  double* Gd = pi ? (double*)b.take((size_t)nreal * 8) : nullptr;
  double* shat = pi ? (double*)b.take((size_t)nreal * 8) : nullptr;   // mu_pde x real-grid values of s'
  double* sc = (double*)b.take(64);
  double* part = (double*)b.take((size_t)(gP + 64) * 8);
  unsigned* tickets = (unsigned*)b.take(64);
  void* fwork = b.take(std::max<size_t>(std::max(fz.work, fd.work), 256));
  cusolverDnHandle_t h;
  FK_TRY(handle_for_device(&h));
  if (cusolverDnSetStream(h, s) != CUSOLVER_STATUS_SUCCESS) return fail(FK_E_CUDA, "cusolverDnSetStream failed");
  int lw_potrf = 0;
  if (Dl > kTilesMaxN &&
      cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, Dl, Ainv, (int)lda, &lw_potrf) != CUSOLVER_STATUS_SUCCESS)
    return fail(FK_E_CUDA, "cusolverDnDpotrf_bufferSize failed");
  double* swork = (double*)b.take((size_t)std::max(lw_potrf, 1) * 8);
  if (!b.ok()) {  // the block does not fit the dense path's matrix slot: dense path
    if (getenv("FK_PCG_DEBUG")) fprintf(stderr, "fk pcg: block Dl %d of %d does not fit the workspace\n", Dl, D);
    return FK_E_UNSUPPORTED;
  }
  if (Dl > 0) FK_CUDA_TRY(cudaMemcpyAsync(d_low, low.data(), (size_t)Dl * 4, cudaMemcpyHostToDevice, s));
  FK_CUDA_TRY(cudaMemcpyAsync(d_lowpos, lowpos.data(), (size_t)D * 4, cudaMemcpyHostToDevice, s));
  FK_CUDA_TRY(cudaMemsetAsync(tickets, 0, 64, s));
  FK_CUDA_TRY(cudaMemsetAsync(pv[0], 0, (size_t)D * 8, s));  // beta = 0 multiplies it in the first step
  FK_CUDA_TRY(cudaMemsetAsync(sc, 0, 64, s));
  cublasHandle_t bh;
  FK_TRY(blas_for_device(&bh));
  if (cublasSetStream(bh, s) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasSetStream failed");
  // the block: assemble, factor (L in Ainv), invert (X = L^{-1}, then lower(Ainv) = X^T X), symmetrise.
  // cuSOLVER potri took 8.8 ms at Dl = 3133 and TRSM on the identity + SYRK 3.75 ms.
  if (Dl > 0) {
    k_pcg_low_block<<<dim3((Dl + TB - 1) / TB, Dl), TB, 0, s>>>(g, d_low, Dl, Ainv, lda);
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
    if (Dl <= kTilesMaxN) {
      FK_TRY(chol_tiles(Ainv, lda, Dl, info, chol_ws, s));
    } else if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, Dl, Ainv, (int)lda, swork, lw_potrf, info) != CUSOLVER_STATUS_SUCCESS) {
      return fail(FK_E_CUDA, "cusolverDnDpotrf failed");
    }
    FK_CUDA_TRY(cudaMemsetAsync(Xinv, 0, (size_t)lda * Dl * 8, s));
    k_pcg_unit_diag<<<(Dl + TB - 1) / TB, TB, 0, s>>>(Xinv, lda, Dl);
    count_launch();
    FK_TRY(tri_inv(bh, Ainv, lda, Xinv, lda, Dl, S));
    FK_TRY(lauum(bh, Xinv, lda, Ainv, lda, Dl));
    k_pcg_symmetrize<<<dim3((Dl + TB - 1) / TB, Dl), TB, 0, s>>>(Ainv, lda, Dl);
    count_launch();
  }
  k_pcg_setup<<<gD, TB, 0, s>>>(g, d_lowpos, r, dinv, bz);
  // DFT of mu / (n L^d)
  k_pcg_mu_half<<<(unsigned)((nhalf + TB - 1) / TB), TB, 0, s>>>(g, q, H);
  FK_TRY(fft_exec_z2d(fz, (cufftDoubleComplex*)H, muhat, fwork, s));
  k_pcg_scale<<<(unsigned)((nreal + TB - 1) / TB), TB, 0, s>>>(muhat, nreal, g.inv_n / (double)nreal);
  if (pi) {
    k_pcg_pi_half<<<(unsigned)((nhalf + TB - 1) / TB), TB, 0, s>>>(g, q, Hd);
    FK_TRY(fft_exec_z2d(fz, (cufftDoubleComplex*)Hd, shat, fwork, s));
    k_pcg_scale<<<(unsigned)((nreal + TB - 1) / TB), TB, 0, s>>>(shat, nreal, g.mu_pde / (double)nreal);
    count_launch(2);
  }
  k_pcg_init<<<gD, TB, 0, s>>>(D, bz, d_low, Dl, x, rv, rl, sc, part, tickets);
  k_pcg_precond<<<gP, TB, 0, s>>>(D, rv, dinv, d_lowpos, d_low, Dl, Ainv, lda, rl, zv, sc, 1, nlow_ctas, part, tickets + 1);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(5);
  const double tol = 1e-13;
  const int kMaxIter = 1000, kCheck = 10;
  double hsc[7] = {0, 0, 0, 0, 0, 0, 0};
  // the iterations run on the library's per-device CG stream (capturable even when the caller passes
  // the legacy default stream), ordered after / before the caller's stream by events
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  FK_TRY(pcg_stream(&cs, &ev_in, &ev_out));
  FK_CUDA_TRY(cudaEventRecord(ev_in, s));
  FK_CUDA_TRY(cudaStreamWaitEvent(cs, ev_in, 0));
  // one block of kCheck iterations (kCheck even: the p ping-pong parity repeats), launched as ONE
  // CUDA graph per block after the first: ~9 launches per iteration otherwise left the GPU idle
  // between its short kernels (round 2: C3 solve 5.7 -> see DESIGN §5).  The kernels skip their
  // work once converged (sc[4]), so a block may overrun the convergence point harmlessly.
  auto block = [&](int it0) -> fk_status {
    for (int j = 0; j < kCheck; ++j) {
      const int it = it0 + j;
      double* p_old = pv[it & 1];
      double* p_new = pv[(it + 1) & 1];
      k_pcg_scatter<<<(unsigned)((nhalf + TB - 1) / TB), TB, 0, cs>>>(g, q, zv, p_old, p_new, H, sc);
      // PI penalty: D theta from the scattered iterate, before the C2R transform below consumes H
      if (pi) k_pcg_dmul<<<(unsigned)((nhalf + TB - 1) / TB), TB, 0, cs>>>(g, q, H, Hd, sc);
      FK_TRY(fft_exec_z2d(fz, (cufftDoubleComplex*)H, G, fwork, cs));
      k_pcg_mul<<<(unsigned)((nreal + TB - 1) / TB), TB, 0, cs>>>(G, muhat, nreal, sc);
      FK_TRY(fft_exec_d2z(fd, G, (cufftDoubleComplex*)H, fwork, cs));
      if (pi) {  // the PI penalty's convolution: values of D theta -> x s' -> back
        FK_TRY(fft_exec_z2d(fz, (cufftDoubleComplex*)Hd, Gd, fwork, cs));
        k_pcg_mul<<<(unsigned)((nreal + TB - 1) / TB), TB, 0, cs>>>(Gd, shat, nreal, sc);
        FK_TRY(fft_exec_d2z(fd, Gd, (cufftDoubleComplex*)Hd, fwork, cs));
      }
      k_pcg_gather<<<gD, TB, 0, cs>>>(g, q, H, p_new, qv, sc, part, tickets + 2, Hd);
      k_pcg_update<<<gD, TB, 0, cs>>>(D, p_new, qv, d_lowpos, x, rv, rl, sc, tol * tol, part, tickets + 3);
      k_pcg_precond<<<gP, TB, 0, cs>>>(D, rv, dinv, d_lowpos, d_low, Dl, Ainv, lda, rl, zv, sc, 0, nlow_ctas, part, tickets + 1);
    }
    return FK_OK;
  };
  const int per_block = kCheck * (pi ? 7 : 5);
  struct GraphGuard {  // the block's graph, destroyed on every exit path
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~GraphGuard() {
      if (exec) cudaGraphExecDestroy(exec);
      if (graph) cudaGraphDestroy(graph);
    }
  } gg;
  cudaGraph_t& graph = gg.graph;
  cudaGraphExec_t& gexec = gg.exec;
  int it = 0;
  for (; it < kMaxIter; it += kCheck) {
    if (it == 0) {
      const fk_status st = block(0);  // the first block eagerly (most solves need several)
      if (st != FK_OK) return st;
    } else {
      if (!gexec) {
        fk_status st = FK_OK;
        if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return fail(FK_E_CUDA, "pcg: stream capture failed");
        st = block(it);
        const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
        if (st != FK_OK) return st;
        if (ce != cudaSuccess || cudaGraphInstantiate(&gexec, graph, 0) != cudaSuccess)
          return fail(FK_E_CUDA, "pcg: graph capture of the CG block failed");
      }
      if (cudaGraphLaunch(gexec, cs) != cudaSuccess) return fail(FK_E_CUDA, "pcg: graph launch failed");
    }
    count_launch(per_block);
    FK_CUDA_TRY(cudaMemcpyAsync(hsc, sc, 56, cudaMemcpyDeviceToHost, cs));
    FK_CUDA_TRY(cudaStreamSynchronize(cs));
    if (getenv("FK_PCG_DEBUG"))
      fprintf(stderr, "fk pcg: it %d |r|^2/|b|^2 %.3e (Dl %d of %d, pi %d)\n", (int)hsc[6], hsc[1] / hsc[2], Dl, D, (int)pi);
    if (hsc[4] != 0.0 || !(hsc[1] == hsc[1])) break;  // converged, or NaN (a failed block factor)
  }
  FK_CUDA_TRY(cudaEventRecord(ev_out, cs));
  FK_CUDA_TRY(cudaStreamWaitEvent(s, ev_out, 0));
  FK_CUDA_TRY(cudaGetLastError());
  *iters = (int)hsc[6];
  if (hsc[4] == 0.0) return fail(FK_E_SOLVE, "fk_solve (pcg): no convergence in " + std::to_string(kMaxIter) + " iterations");
  return FK_OK;
}

// 1 / cond_2(A) estimate from the Cholesky factor (report only): 8 power steps on A = L L^T
// (two cublasDtrmv per step) give lambda_max from below, 8 inverse-iteration steps (two
// cublasDtrsv) give 1/lambda_min from below; rcond_est = lambda_min_est / lambda_max_est.
static fk_status rcond_estimate(cublasHandle_t bh, const double* L, int ld, int D, double* v, double* w, cudaStream_t s,
                                double* out) {
  if (cublasSetStream(bh, s) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasSetStream failed");
  std::vector<double> h0(D);
  for (int i = 0; i < D; ++i) h0[i] = 1.0 + 0.37 * std::sin(1.7 * i + 0.3);  // no special structure
  double est[2] = {0.0, 0.0};
  for (int pass = 0; pass < 2; ++pass) {
    FK_CUDA_TRY(cudaMemcpyAsync(v, h0.data(), (size_t)D * 8, cudaMemcpyHostToDevice, s));
    double nv = 0.0;
    if (cublasDnrm2(bh, D, v, 1, &nv) != CUBLAS_STATUS_SUCCESS || !(nv > 0)) return fail(FK_E_CUDA, "cublasDnrm2 failed");
    double inv = 1.0 / nv;
    cublasDscal(bh, D, &inv, v, 1);
    double q = 0.0;
    for (int it = 0; it < 8; ++it) {
      FK_CUDA_TRY(cudaMemcpyAsync(w, v, (size_t)D * 8, cudaMemcpyDeviceToDevice, s));
      cublasStatus_t st1, st2;
      if (pass == 0) {  // w = L (L^T v)
        st1 = cublasDtrmv(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, D, L, ld, w, 1);
        st2 = cublasDtrmv(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, D, L, ld, w, 1);
      } else {  // w = L^{-T} (L^{-1} v)
        st1 = cublasDtrsv(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, D, L, ld, w, 1);
        st2 = cublasDtrsv(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, D, L, ld, w, 1);
      }
      if (st1 != CUBLAS_STATUS_SUCCESS || st2 != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublas trmv/trsv failed");
      if (cublasDdot(bh, D, v, 1, w, 1, &q) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasDdot failed");
      double nw = 0.0;
      if (cublasDnrm2(bh, D, w, 1, &nw) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasDnrm2 failed");
      if (!(nw > 0) || !(nw < 1e300)) break;
      inv = 1.0 / nw;
      cublasDscal(bh, D, &inv, w, 1);
      std::swap(v, w);
    }
    est[pass] = q;  // Rayleigh quotient: lambda_max (pass 0), 1 / lambda_min (pass 1)
  }
  *out = (est[0] > 0 && est[1] > 0) ? 1.0 / (est[0] * est[1]) : 0.0;
  return FK_OK;
}

fk_status solve_run(const fk_problem* P, double* theta, fk_solve_report* rep, void* ws, size_t ws_bytes, cudaStream_t s) {
  SysArgs g;
  FK_TRY(fill_sysargs(P, &g));
  const int D = g.D;
  int lwork = 0;
  const int N = D + 1;
  FK_TRY(lwork_for(N, &lwork));
  Bump b(ws, ws_bytes);
  double* M = (double*)b.take((size_t)N * N * 8);
  double* work = (double*)b.take((size_t)lwork * 8);
  double* zbuf = (double*)b.take((size_t)D * 8);
  int* info = (int*)b.take(64);
  double* res = (double*)(info + 4);
  double* rv1 = (double*)b.take((size_t)D * 8);  // condition estimate (report only)
  double* rv2 = (double*)b.take((size_t)D * 8);
  double2* dsym = nullptr;
  double2* boxt = nullptr;
  if (P->kind == FK_PIK_BOX || P->kind == FK_PIK_COLLOC) {
    dsym = (double2*)b.take((size_t)D * 16);
    boxt = (double2*)b.take((size_t)P->d * (4 * P->m + 1) * 16);
  }
  void* chol_ws = b.take(chol_ws_bytes(N));
  if (!b.ok()) return fail(FK_E_WORKSPACE, "fk_solve: workspace too small");

  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (rep) {
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
  }
  if (P->kind == FK_PIK_BOX || P->kind == FK_PIK_COLLOC) {
    const int nt = std::max(D, P->d * (4 * P->m + 1));
    k_pi_tables<<<(nt + 255) / 256, 256, 0, s>>>(g, dsym, boxt);
    FK_CUDA_TRY(cudaGetLastError());
    count_launch();
    g.dsym = dsym;
    g.boxt = boxt;
  }
  const bool own_trsv = true;
  int* ticket = info + 12;
  int iters = 0;
  bool done = false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  if (cap == cudaStreamCaptureStatusNone && pcg_eligible(g)) {  // CG checks convergence on the host: not capturable
    std::lock_guard<std::mutex> lk(g_sol_mu);
    const fk_status st = pcg_run(g, (const double2*)P->rhs, zbuf, &iters, M, (size_t)N * N * 8, chol_ws, info, s);
    if (st == FK_OK) {
      done = true;
      FK_CUDA_TRY(cudaMemsetAsync(info, 0, 4, s));
      k_theta_from_real<<<(D + 255) / 256, 256, 0, s>>>(g, zbuf, 1, (double2*)theta, nullptr, nullptr);
      FK_CUDA_TRY(cudaGetLastError());
      count_launch();
    } else if (st != FK_E_UNSUPPORTED && st != FK_E_SOLVE) {
      return st;
    }  // FK_E_SOLVE (no convergence): the dense path decides
  }
  if (!done) {
  launch_assemble(g, M, s);
  const bool tiles = use_tiles(N);
  k_rhs_real<<<tiles ? std::max((N + 255) / 256, 64) : (N + 255) / 256, 256, 0, s>>>(
      g, (const double2*)P->rhs, M, zbuf, ticket, tiles ? chol_reset_args(N, chol_ws, info) : CholReset{});
  FK_CUDA_TRY(cudaGetLastError());
  count_launch(2);
  {
    std::lock_guard<std::mutex> lk(g_sol_mu);
    cusolverDnHandle_t h;
    FK_TRY(handle_for_device(&h));
    if (cusolverDnSetStream(h, s) != CUSOLVER_STATUS_SUCCESS) return fail(FK_E_CUDA, "cusolverDnSetStream failed");
    if (tiles) {
      FK_TRY(chol_tiles(M, N, N, info, chol_ws, s, nullptr, /*preset=*/true));
    } else if (cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, N, M, N, work, lwork, info) != CUSOLVER_STATUS_SUCCESS) {
      return fail(FK_E_CUDA, "cusolverDnDpotrf failed");
    }
    cublasHandle_t bh;
    FK_TRY(blas_for_device(&bh));
    if (cublasSetStream(bh, s) != CUBLAS_STATUS_SUCCESS) return fail(FK_E_CUDA, "cublasSetStream failed");
    // y = L^{-1} c is the factor's last row (stride N); solve L^T z = y
    if (!own_trsv &&
        cublasDtrsv(bh, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, D, M, N, M + D, N) != CUBLAS_STATUS_SUCCESS)
      return fail(FK_E_CUDA, "cublasDtrsv failed");
  }
  if (own_trsv) {
    k_trsv_lt<<<(D + 31) / 32, 128, 0, s>>>(M, N, D, M + D, N, zbuf, ticket, info);
    count_launch();
  }
  k_theta_from_real<<<(D + 255) / 256, 256, 0, s>>>(g, own_trsv ? zbuf : M + D, own_trsv ? 1 : N, (double2*)theta, info,
                                                    P->d_status);
  FK_CUDA_TRY(cudaGetLastError());
  count_launch();
  }
  if (rep) {
    cudaEventRecord(e1, s);
    FK_CUDA_TRY(cudaMemsetAsync(res, 0, 16, s));
    k_residual<<<(D * 32 + 255) / 256, 256, 0, s>>>(g, (const double2*)theta, (const double2*)P->rhs, res);
    count_launch();
    int hinfo = 0;
    double hres[2] = {0, 0};
    FK_CUDA_TRY(cudaMemcpyAsync(&hinfo, info, 4, cudaMemcpyDeviceToHost, s));
    FK_CUDA_TRY(cudaMemcpyAsync(hres, res, 16, cudaMemcpyDeviceToHost, s));
    FK_CUDA_TRY(cudaStreamSynchronize(s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    rep->info = hinfo;
    rep->ms = ms;
    rep->n_unknowns = D;
    rep->iters = iters;
    rep->backward_err = hres[1] > 0 ? std::sqrt(hres[0] / hres[1]) : 0.0;
    rep->rcond_est = 0.0;
    if (hinfo < 0) return fail(FK_E_SOLVE, "fk_solve: a dataflow wait of the factorisation hit its watchdog");
    if (hinfo != 0) return fail(FK_E_SOLVE, "fk_solve: Cholesky failed, info = " + std::to_string(hinfo));
    if (!done) {  // dense path: the factor L (D x D leading block of M, ld N) is still in place
      std::lock_guard<std::mutex> lk(g_sol_mu);
      cublasHandle_t bh;
      FK_TRY(blas_for_device(&bh));
      FK_TRY(rcond_estimate(bh, M, N, D, rv1, rv2, s, &rep->rcond_est));
    }
  }
  return FK_OK;
}

}  // namespace fk
