// fk_api.cu -- the extern "C" entry points of libfk (include/fk.h): argument validation on the
// host, then dispatch to the stream-ordered implementations.
#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

#include "fk_internal.cuh"

namespace fk {
const char* last_error_cstr();
int profile_read(double* ms, int64_t* launches, int64_t* kernels);
void profile_enable(int on);
}

using namespace fk;

namespace {

fk_status check_eps(double eps) {
  if (!(eps >= 1e-14 && eps <= 1e-1)) return fail(FK_E_EPS, "eps must lie in [1e-14, 1e-1]");
  return FK_OK;
}

fk_status check_points(const fk_points& X, int dmin, int dmax, const char* who) {
  if (X.n < 0) return fail(FK_E_ARG, std::string(who) + ": n < 0");
  if (X.d < dmin || X.d > dmax) return fail(FK_E_UNSUPPORTED, std::string(who) + ": unsupported dimension d = " + std::to_string(X.d));
  if (X.dtype != FK_F32 && X.dtype != FK_F64) return fail(FK_E_ARG, std::string(who) + ": dtype must be FK_F32 or FK_F64");
  if (X.n > 0 && X.ptr == nullptr) return fail(FK_E_ARG, std::string(who) + ": null points");
  if (X.stride_n < 0 || X.stride_d < 0 || (X.n > 1 && X.stride_n == 0)) return fail(FK_E_ARG, std::string(who) + ": bad strides");
  return FK_OK;
}

fk_status check_common(double L, int m, double eps, const char* who) {
  if (!(L > 0.0) || !std::isfinite(L)) return fail(FK_E_ARG, std::string(who) + ": L must be positive");
  if (m < 1 || m > (1 << 20)) return fail(FK_E_ARG, std::string(who) + ": m must be >= 1");
  return check_eps(eps);
}

fk_status type1_entry(const fk_points& X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags,
                      void* ws, size_t ws_bytes, int* d_status, cudaStream_t s, const char* who) {
  set_error("");
  FK_TRY(check_common(L, m, eps, who));
  FK_TRY(check_points(X, 1, 2, who));
  if (!r_out && !mu_out) return fail(FK_E_ARG, std::string(who) + ": no output requested");
  if (r_out && X.n > 0 && Y == nullptr) return fail(FK_E_ARG, std::string(who) + ": Y is null");
  if (X.d == 2) return type1_2d_run(m, eps, X, Y, L, mu_out, r_out, (flags & FK_ACCUMULATE) != 0, ws, ws_bytes, d_status, s);
  Plan1 p;
  FK_TRY(make_plan1(X.d, m, eps, mu_out != nullptr, r_out != nullptr, &p));
  // small n: no more CTAs than ~8 samples per thread need (fewer partial grids to reduce); the
  // workspace query sized the full count, of which this layout is a prefix
  if (p.smem) p.ctas = (int)std::min<int64_t>(p.ctas, std::max<int64_t>(1, (X.n + 8 * p.threads - 1) / (8 * p.threads)));
  Type1Out out{mu_out, r_out, (flags & FK_ACCUMULATE) != 0};
  return type1_run(p, X, Y, L, out, ws, ws_bytes, d_status, s);
}

// ---- host streaming (fk_rhs_type1_host) ----------------------------------------------------
constexpr int64_t kHostChunk = 1 << 24;

int64_t host_chunk(int64_t c) { return c > 0 ? c : kHostChunk; }

size_t rhs_host_ws_bytes(int d, int m, double eps, int dtype, int64_t chunk) {
  chunk = host_chunk(chunk);
  const size_t esz = dtype == FK_F64 ? 8 : 4;
  size_t t1 = 0;
  if (d == 2) {
    t1 = type1_2d_ws_bytes(m, eps, true, true, dtype);
  } else {
    Plan1 p;
    if (make_plan1(d, m, eps, true, true, &p) != FK_OK) return 0;
    t1 = type1_ws_bytes(p, true, true);
  }
  if (t1 == 0) return 0;
  Bump b(nullptr, 0);
  for (int k = 0; k < 2; ++k) {
    b.take((size_t)chunk * d * esz);  // X staging
    b.take((size_t)chunk * esz);      // Y staging
  }
  b.take(t1);
  return b.used + 256;
}

// one copy stream per device, created on first use; the enqueue loop holds the mutex so two
// concurrent callers' copies cannot interleave their event sequences
struct HostCopy {
  cudaStream_t cs = nullptr;
};
std::mutex g_host_mu;
std::map<int, HostCopy> g_host;

fk_status rhs_host(const fk_points& X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags,
                   int64_t chunk, void* ws, size_t ws_bytes, int* d_status, cudaStream_t s) {
  const char* who = "fk_rhs_type1_host";
  set_error("");
  FK_TRY(check_common(L, m, eps, who));
  FK_TRY(check_points(X, 1, 2, who));
  if (!r_out) return fail(FK_E_ARG, std::string(who) + ": r_out is null");
  if (X.n > 0 && (!Y || !X.ptr)) return fail(FK_E_ARG, std::string(who) + ": null X or Y");
  if (X.n > 1 && (X.stride_n != X.d || (X.d > 1 && X.stride_d != 1)))
    return fail(FK_E_ARG, std::string(who) + ": host X must be contiguous (stride_n = d, stride_d = 1)");
  chunk = host_chunk(chunk);
  const size_t esz = X.dtype == FK_F64 ? 8 : 4;
  const int d = X.d;
  const size_t need = rhs_host_ws_bytes(d, m, eps, X.dtype, chunk);
  if (need == 0) return fail(FK_E_UNSUPPORTED, std::string(who) + ": no plan for this shape");
  if (ws_bytes < need) return fail(FK_E_WORKSPACE, std::string(who) + ": workspace too small: need " + std::to_string(need) + " bytes");
  Bump b(ws, ws_bytes);
  char* xs[2];
  char* ys[2];
  for (int k = 0; k < 2; ++k) {
    xs[k] = (char*)b.take((size_t)chunk * d * esz);
    ys[k] = (char*)b.take((size_t)chunk * esz);
  }
  void* ws1 = b.take(0);
  const size_t ws1_bytes = ws_bytes - (size_t)((char*)ws1 - (char*)ws);
  if (X.n == 0) {
    fk_points Z = X;
    Z.n = 0;
    Z.ptr = xs[0];
    return type1_entry(Z, ys[0], L, m, eps, r_out, mu_out, flags, ws1, ws1_bytes, d_status, s, who);
  }
  int dev = 0;
  FK_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_host_mu);
  HostCopy& hc = g_host[dev];
  if (!hc.cs) FK_CUDA_TRY(cudaStreamCreateWithFlags(&hc.cs, cudaStreamNonBlocking));
  cudaEvent_t copied[2], consumed[2];
  for (int k = 0; k < 2; ++k) {
    FK_CUDA_TRY(cudaEventCreateWithFlags(&copied[k], cudaEventDisableTiming));
    FK_CUDA_TRY(cudaEventCreateWithFlags(&consumed[k], cudaEventDisableTiming));
    FK_CUDA_TRY(cudaEventRecord(consumed[k], s));  // staging k is free once prior work on s is done
  }
  const int64_t nch = (X.n + chunk - 1) / chunk;
  fk_status st = FK_OK;
  for (int64_t i = 0; i < nch && st == FK_OK; ++i) {
    const int k = (int)(i & 1);
    const int64_t lo = i * chunk, c = std::min(chunk, X.n - lo);
    FK_CUDA_TRY(cudaStreamWaitEvent(hc.cs, consumed[k], 0));
    FK_CUDA_TRY(cudaMemcpyAsync(xs[k], (const char*)X.ptr + (size_t)lo * d * esz, (size_t)c * d * esz, cudaMemcpyHostToDevice, hc.cs));
    FK_CUDA_TRY(cudaMemcpyAsync(ys[k], (const char*)Y + (size_t)lo * esz, (size_t)c * esz, cudaMemcpyHostToDevice, hc.cs));
    FK_CUDA_TRY(cudaEventRecord(copied[k], hc.cs));
    FK_CUDA_TRY(cudaStreamWaitEvent(s, copied[k], 0));
    fk_points Xc = X;
    Xc.ptr = xs[k];
    Xc.n = c;
    const int fl = (i == 0) ? flags : (flags | FK_ACCUMULATE);
    st = type1_entry(Xc, ys[k], L, m, eps, r_out, mu_out, fl, ws1, ws1_bytes, d_status, s, who);
    FK_CUDA_TRY(cudaEventRecord(consumed[k], s));
  }
  for (int k = 0; k < 2; ++k) {  // released once the recorded work completes
    cudaEventDestroy(copied[k]);
    cudaEventDestroy(consumed[k]);
  }
  return st;
}

}  // namespace

extern "C" {

fk_status fk_rhs_type1_host(fk_points X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags,
                            int64_t chunk, void* ws, size_t ws_bytes, int* d_status, fk_stream_t stream) {
  return rhs_host(X, Y, L, m, eps, r_out, mu_out, flags, chunk, ws, ws_bytes, d_status, (cudaStream_t)stream);
}

const char* fk_last_error(void) { return last_error_cstr(); }

const char* fk_version(void) { return "fk 0.1 (sm_100a)"; }

void fk_profile_enable(int on) { profile_enable(on); }

int fk_profile_read(double* spread_ms, int64_t* spread_launches, int64_t* kernel_launches) {
  return profile_read(spread_ms, spread_launches, kernel_launches);
}

fk_status fk_moments_type1(fk_points X, double L, int m, double eps, double* mu_out, int flags, void* ws, size_t ws_bytes,
                           int* d_status, fk_stream_t stream) {
  if (!mu_out) return fail(FK_E_ARG, "fk_moments_type1: mu_out is null");
  return type1_entry(X, nullptr, L, m, eps, nullptr, mu_out, flags, ws, ws_bytes, d_status, (cudaStream_t)stream, "fk_moments_type1");
}

fk_status fk_rhs_type1(fk_points X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags, void* ws,
                       size_t ws_bytes, int* d_status, fk_stream_t stream) {
  if (!r_out) return fail(FK_E_ARG, "fk_rhs_type1: r_out is null");
  return type1_entry(X, Y, L, m, eps, r_out, mu_out, flags, ws, ws_bytes, d_status, (cudaStream_t)stream, "fk_rhs_type1");
}

fk_status fk_additive_cross_moments(fk_points X, double L, int m, double eps, double* G_out, int flags, void* ws, size_t ws_bytes,
                                    int* d_status, fk_stream_t stream) {
  set_error("");
  FK_TRY(check_common(L, m, eps, "fk_additive_cross_moments"));
  FK_TRY(check_points(X, 2, 32, "fk_additive_cross_moments"));
  if (!G_out) return fail(FK_E_ARG, "fk_additive_cross_moments: G_out is null");
  return cross_run(X, L, m, eps, G_out, (flags & FK_ACCUMULATE) != 0, ws, ws_bytes, d_status, (cudaStream_t)stream);
}

static fk_status check_problem(const fk_problem* P, bool need_lambda) {
  if (!P) return fail(FK_E_ARG, "fk_solve: null problem");
  if (P->m < 1 || P->d < 1) return fail(FK_E_ARG, "fk_solve: d, m must be >= 1");
  if (need_lambda && !(P->lambda > 0.0)) return fail(FK_E_ARG, "fk_solve: lambda must be > 0");
  if (!(P->n_total > 0.0)) return fail(FK_E_ARG, "fk_solve: n_total must be > 0");
  if (!(P->L > 0.0)) return fail(FK_E_ARG, "fk_solve: L must be > 0");
  if (P->kind < FK_SOBOLEV || P->kind > FK_PIK_COLLOC) return fail(FK_E_ARG, "fk_solve: unknown kind");
  if (!P->mu_moments || !P->rhs) return fail(FK_E_ARG, "fk_solve: null moments or rhs");
  if (P->kind == FK_ADDITIVE && P->d > 1 && !P->cross) return fail(FK_E_ARG, "fk_solve: ADDITIVE needs cross moments");
  if (P->kind != FK_ADDITIVE && P->d > 3) return fail(FK_E_UNSUPPORTED, "fk_solve: d <= 3 for the dense tensor-grid system");
  if ((P->kind == FK_SOBOLEV || P->kind == FK_PIK_BOX || P->kind == FK_PIK_COLLOC) && !(P->s > 0.0))
    return fail(FK_E_ARG, "fk_solve: s must be > 0");
  if (P->kind == FK_PIK_COLLOC) {
    if (P->n_terms < 1 || !P->alpha || !P->a_alpha) return fail(FK_E_ARG, "fk_solve: PIK_COLLOC needs alpha, a_alpha");
    if (!P->colloc_moments || !(P->n_colloc > 0.0)) return fail(FK_E_ARG, "fk_solve: PIK_COLLOC needs colloc_moments and n_colloc > 0");
  }
  if (P->kind == FK_PIK_BOX) {
    if (P->n_terms < 1 || !P->alpha || !P->a_alpha || !P->box) return fail(FK_E_ARG, "fk_solve: PIK_BOX needs alpha, a_alpha, box");
    for (int l = 0; l < P->d; ++l) {
      const double a = P->box[2 * l], b = P->box[2 * l + 1];
      if (!(a < b) || a < -P->L || b > P->L) return fail(FK_E_ARG, "fk_solve: box must satisfy -L <= a < b <= L");
    }
  }
  // dense systems above ~2.5e4 unknowns exceed a sensible workspace
  long D = P->kind == FK_ADDITIVE ? (long)P->d * (2 * P->m + 1) : (long)std::pow(2.0 * P->m + 1, P->d);
  if (D > 40000) return fail(FK_E_UNSUPPORTED, "fk_solve: dense system too large (D = " + std::to_string(D) + ")");
  return FK_OK;
}

fk_status fk_solve(const fk_problem* P, double* theta_out, fk_solve_report* rep, void* ws, size_t ws_bytes, fk_stream_t stream) {
  set_error("");
  if (!theta_out) return fail(FK_E_ARG, "fk_solve: null output");
  FK_TRY(check_problem(P, true));
  return solve_run(P, theta_out, rep, ws, ws_bytes, (cudaStream_t)stream);
}

fk_status fk_solve_path(const fk_problem* P, const double* lambdas, int nlam, double* theta_out, int* info, void* ws,
                        size_t ws_bytes, fk_stream_t stream) {
  set_error("");
  if (!theta_out || !lambdas || nlam < 1) return fail(FK_E_ARG, "fk_solve_path: null output / lambdas or nlam < 1");
  for (int l = 0; l < nlam; ++l)
    if (!(lambdas[l] > 0.0)) return fail(FK_E_ARG, "fk_solve_path: every lambda must be > 0");
  FK_TRY(check_problem(P, false));
  return solve_path_run(P, lambdas, nlam, theta_out, info, ws, ws_bytes, (cudaStream_t)stream);
}

fk_status fk_path_validate(const fk_problem* Pv, const double* theta, int nlam, double sum_y2, double* risk_out, void* ws,
                           size_t ws_bytes, fk_stream_t stream) {
  set_error("");
  if (!theta || !risk_out || nlam < 1) return fail(FK_E_ARG, "fk_path_validate: null theta / risk_out or nlam < 1");
  if (!Pv) return fail(FK_E_ARG, "fk_path_validate: null problem");
  fk_problem q = *Pv;  // data part only: lambda, s and the PI fields are not used
  if (q.kind == FK_PIK_BOX || q.kind == FK_PIK_COLLOC) q.kind = FK_SOBOLEV;
  q.s = 1.0;
  q.n_terms = 0;
  FK_TRY(check_problem(&q, false));
  return path_validate_run(&q, theta, nlam, sum_y2, risk_out, ws, ws_bytes, (cudaStream_t)stream);
}

fk_status fk_predict_type2(const double* theta, int d, int m, double L, int additive, fk_points Xq, double eps, void* out, void* ws,
                           size_t ws_bytes, int* d_status, fk_stream_t stream) {
  set_error("");
  FK_TRY(check_common(L, m, eps, "fk_predict_type2"));
  FK_TRY(check_points(Xq, 1, 32, "fk_predict_type2"));
  if (Xq.d != d) return fail(FK_E_ARG, "fk_predict_type2: Xq.d != d");
  if (!theta || (Xq.n > 0 && !out)) return fail(FK_E_ARG, "fk_predict_type2: null theta or out");
  return predict_run(theta, d, m, L, additive, Xq, eps, out, ws, ws_bytes, d_status, (cudaStream_t)stream);
}

size_t fk_workspace_bytes(int entry, int d, int m, double eps, int dtype, int64_t n, int kind) {
  set_error("");
  if (m < 1 || d < 1 || !(eps >= 1e-14 && eps <= 1e-1)) {
    set_error("fk_workspace_bytes: bad arguments");
    return 0;
  }
  switch (entry) {
    case FK_ENTRY_MOMENTS:
    case FK_ENTRY_RHS: {
      if (d == 2) return type1_2d_ws_bytes(m, eps, true, entry == FK_ENTRY_RHS, dtype);
      Plan1 p;
      const bool mu = true, r = entry == FK_ENTRY_RHS;
      if (make_plan1(d, m, eps, mu, r, &p) != FK_OK) return 0;
      return type1_ws_bytes(p, mu, r);
    }
    case FK_ENTRY_CROSS:
      return cross_ws_bytes(d, m, eps, n, dtype);
    case FK_ENTRY_SOLVE:
      return solve_ws_bytes(d, m, kind);
    case FK_ENTRY_PREDICT:
      return predict_ws_bytes(d, m, eps, kind);
    case FK_ENTRY_PATH_VALIDATE:
      return path_validate_ws_bytes(d, m, kind, (int)std::min<int64_t>(n, 1 << 20));
    case FK_ENTRY_SOLVE_PATH:
      return solve_path_ws_bytes(d, m, kind, (int)std::min<int64_t>(n, 1 << 20));
    case FK_ENTRY_RHS_HOST:
      if (d > 2) return 0;
      return rhs_host_ws_bytes(d, m, eps, dtype, n);
    default:
      set_error("fk_workspace_bytes: unknown entry");
      return 0;
  }
}

}  // extern "C"
