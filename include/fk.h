/*
 * fk.h -- C ABI of the B200-native fast-kernel-regression fit path (arXiv 2509.02649).
 *
 * libfk.so (paper_2509_02649_b200/libfk.so) exports the five calls of the method's data-parallel
 * hot path plus a workspace query and a last-error string.  "P:<line>" cites PAPER.md, DESIGN.md
 * lists the readings R1..R9 taken where the paper is ambiguous.
 *
 * Notation (reading R1):
 *   t(x)     = pi x / (2L)            x in [-L, L]^d  (closed box)
 *   f(x)     = sum_{||k||_inf <= m} theta_k exp(+i <k, t(x)>)
 *   mu_q     = sum_j exp(-i <q, t(X_j)>)        ||q||_inf <= 2m   (first row of n*Sigma-hat)
 *   r_k      = sum_j Y_j exp(-i <k, t(X_j)>)    ||k||_inf <= m    (n*v = Phi^* Y)
 *   A theta  = r / n,  A = T(mu)/n + lambda M^*M (+ mu_pde D^* C D)
 *
 * Conventions shared by every call
 *   - Layout: a mode vector over {-K..K}^d is stored lexicographically with the LAST coordinate
 *     fastest, index of k = sum_l (k_l + K) (2K+1)^(d-1-l); complex values are interleaved
 *     (re, im) doubles (complex128).
 *   - Outputs are UNNORMALISED sums (reading R5): results of disjoint sample shards add, so a
 *     multi-GPU fit all-reduces them (sum) and fk_solve divides by the total n.
 *   - Ownership: every data pointer (points, Y, outputs, workspace, d_status) is caller-owned
 *     DEVICE memory unless marked "host".  The library never allocates device memory on a call
 *     after the first one with the same shape (cuFFT plans and the cuSOLVER handle are created
 *     once and cached); scratch comes from `ws`, sized by fk_workspace_bytes().
 *   - Ordering: every call is asynchronous and stream-ordered on `stream` (a cudaStream_t; NULL
 *     = legacy default stream), except fk_solve with rep != NULL, which synchronises `stream`.
 *   - Errors: argument errors are detected on the host and returned synchronously (no work is
 *     enqueued); the message is available from fk_last_error() (thread-local).  Data errors found
 *     by a kernel (a coordinate outside [-L, L], NaN) are OR-ed into *d_status (device int, bit
 *     FK_E_RANGE) -- the caller zeroes it before and inspects it after synchronising.  Samples
 *     with such a coordinate are skipped (predict: NaN at that query).  The check is made on the
 *     fine grid: a coordinate within the window's halo beyond +-L (at most w/2 + 2 fine cells,
 *     i.e. 4L (w/2 + 2) / nf) is still on the grid and is summed exactly (the sums are
 *     4L-periodic), without a flag.
 *   - Accuracy: eps is the requested relative l2 accuracy of each output vector against the
 *     exact sums (reading R7); valid range [1e-14, 1e-1].  eps >= 1e-7 selects the fp32
 *     spreading path (cubic B-spline window, fixed-point shared-memory accumulation); smaller eps
 *     selects the fp64 mode (d = 1: septic B-spline window; d = 2 / cross moments:
 *     exponential-of-semicircle window at sigma = 2; both accumulate in 64-bit fixed point held
 *     as int32 pairs in shared memory, drained into fp64 carry grids).
 */
#ifndef FK_H
#define FK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fk_stream_t; /* == cudaStream_t */

typedef enum fk_status {
  FK_OK = 0,
  FK_E_ARG = 1,         /* invalid argument (n < 0, m < 1, L <= 0, bad dtype/stride, lambda <= 0, ...) */
  FK_E_RANGE = 2,       /* (d_status bit) a coordinate outside [-L, L] or NaN was skipped */
  FK_E_EPS = 3,         /* eps outside [1e-14, 1e-1] */
  FK_E_CUDA = 4,        /* a CUDA / cuFFT / cuSOLVER call failed */
  FK_E_WORKSPACE = 5,   /* ws_bytes smaller than fk_workspace_bytes() */
  FK_E_SOLVE = 6,       /* the system is not Hermitian positive definite (Cholesky info > 0) */
  FK_E_UNSUPPORTED = 7  /* a shape this build does not handle (see fk_last_error) */
} fk_status;

typedef enum fk_dtype { FK_F32 = 0, FK_F64 = 1 } fk_dtype;

/* Bits a kernel ORs into the caller's device status word (d_status arguments, fk_problem.d_status).
 * FK_E_RANGE (2) doubles as the bit of a skipped out-of-range / NaN coordinate; the solve adds: */
enum {
  FK_DSTATUS_RANGE = FK_E_RANGE, /* a coordinate outside [-L, L] or NaN was skipped */
  FK_DSTATUS_NOT_SPD = 0x10,     /* fk_solve: the Cholesky factorisation met a non-positive pivot */
  FK_DSTATUS_WATCHDOG = 0x20     /* fk_solve: a dataflow wait of the factorisation / back
                                    substitution hit its 5 s watchdog (theta is not valid) */
};

/* n points in d dimensions: coordinate l of sample j is at element ptr[j*stride_n + l*stride_d]
 * (element strides, not bytes).  Row-major n x d: stride_n = d, stride_d = 1; SoA columns:
 * stride_n = 1, stride_d = column pitch.  The fast streaming path needs d = 1 and stride_n = 1. */
typedef struct fk_points {
  const void* ptr;
  int32_t dtype; /* fk_dtype */
  int32_t d;
  int64_t n;
  int64_t stride_n;
  int64_t stride_d;
} fk_points;

enum { FK_ACCUMULATE = 1 }; /* flags: add into the outputs instead of overwriting them */

/* Moments mu_q = sum_j exp(-i pi <q, X_j> / 2L), ||q||_inf <= 2m (the first row of
 * n * Sigma-hat, Sigma-hat_{k1,k2} = mu_{k1-k2}/n).  mu_out: (4m+1)^d complex128.  d in {1, 2}.
 * n = 0 is valid (all moments 0). */
fk_status fk_moments_type1(fk_points X, double L, int m, double eps, double* mu_out, int flags, void* ws, size_t ws_bytes,
                           int* d_status, fk_stream_t stream);

/* Right-hand side r_k = sum_j Y_j exp(-i pi <k, X_j> / 2L), ||k||_inf <= m (n v =
 * Phi^* Y).  r_out: (2m+1)^d complex128.  Y: n values of X.dtype, contiguous.  If mu_out != NULL
 * the moments are produced by the SAME pass over (X, Y) (one read of the data).  d in {1, 2}. */
fk_status fk_rhs_type1(fk_points X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags,
                       void* ws, size_t ws_bytes, int* d_status, fk_stream_t stream);

/* Additive-model cross moments for every feature pair l1 < l2 in lexicographic pair order
 * (P:505-512): G[p][a][b] = sum_j exp(-i pi (a X_{j,l1} - b X_{j,l2}) / 2L), a, b in {-m..m}:
 * the 2-D type-1 sum of unit weights at the points (X_{l1}, -X_{l2}).  G_out: d(d-1)/2 blocks of
 * (2m+1)^2 complex128, b fastest.  2 <= d <= 32.  A coordinate outside [-L, L] (or NaN) flags
 * FK_E_RANGE and drops the sample from the pairs that use that coordinate only (as the per-feature
 * 1-D passes drop it from that feature only).  Any m: when one pair grid exceeds a CTA's shared
 * memory each pair is computed by a tiled 2-D moment pass (one read of its two columns per pair). */
fk_status fk_additive_cross_moments(fk_points X, double L, int m, double eps, double* G_out, int flags, void* ws,
                                    size_t ws_bytes, int* d_status, fk_stream_t stream);

typedef enum fk_kind {
  FK_SOBOLEV = 0,  /* M = S, S_kk^2 = 1 + ||k||_2^{2s} */
  FK_LOWBIAS = 1,  /* M = I */
  FK_PIK_BOX = 2,  /* Sobolev + mu_pde D^* C D, Omega a box in [-L,L]^d          (reading R3) */
  FK_ADDITIVE = 3, /* low-bias additive block system, theta in C^{d(2m+1)} */
  FK_PIK_COLLOC = 4 /* Sobolev + mu_pde n_r^{-1} D^* (Phi^r)^* Phi^r D from collocation points'
                       moments, for domains without a closed-form Fourier matrix */
} fk_kind;

typedef struct fk_problem {
  int32_t d, m, kind, n_terms;
  double n_total; /* total number of samples the moments were summed over (all shards) */
  double L, s, lambda, mu_pde;
  const int32_t* alpha;      /* host, n_terms x d multi-indices of D = sum a_alpha d^alpha (PIK_BOX) */
  const double* a_alpha;     /* host, n_terms coefficients (PIK_BOX) */
  const double* box;         /* host, 2d values [a_0, b_0, a_1, b_1, ...], Omega = prod [a_l, b_l] (PIK_BOX) */
  const double* mu_moments;  /* device: (4m+1)^d complex128; ADDITIVE: d x (4m+1) (per-feature 1-D moments) */
  const double* rhs;         /* device: (2m+1)^d complex128; ADDITIVE: d x (2m+1) (per-feature 1-D rhs) */
  const double* cross;       /* device: ADDITIVE only, d(d-1)/2 x (2m+1)^2 from fk_additive_cross_moments */
  const double* colloc_moments; /* device: PIK_COLLOC only, (4m+1)^d moments of the n_colloc collocation
                                   points (fk_moments_type1 on them); D is given by alpha / a_alpha */
  double n_colloc;              /* PIK_COLLOC: number of collocation points n_r */
  int* d_status;                /* optional device int (may be NULL): fk_solve ORs FK_DSTATUS_NOT_SPD /
                                   FK_DSTATUS_WATCHDOG into it from the device, so a failed
                                   factorisation is reported even on the asynchronous rep == NULL path */
} fk_problem;

typedef struct fk_solve_report {
  double backward_err; /* ||A theta - r/n|| / ||r/n|| with A re-evaluated from the moments (reading R8) */
  double ms;           /* device time of the solve (assembly + factorisation + solves) */
  int32_t info;        /* Cholesky info (0 = success) */
  int32_t n_unknowns;  /* D */
  int32_t iters;       /* conjugate-gradient iterations (0: dense Cholesky) */
  int32_t reserved;
  double rcond_est;    /* estimate of 1 / cond_2(A) of the solved real-symmetric system (dense path:
                          8 power steps on A = L L^T and 8 inverse-iteration steps with the factor;
                          the ratio of the two Rayleigh quotients); 0 on the CG path (not estimated).
                          With it an fp32-mode theta error ~ cond(A) x moment error can be read. */
} fk_solve_report;

/* theta = A^{-1} r / n in fp64 (P:513 for the additive block system).  For real Y theta
 * is Hermitian, so the real-symmetric form P^*AP z = P^*r/n (D unknowns) is solved: by dense
 * Cholesky (reading R9) -- a tile dataflow kernel up to D = 4599, cuSOLVER potrf above -- except
 * for the Sobolev estimator with D >= 4600, d <= 2, where the paper's conjugate gradients
 * run with FFT-Toeplitz products and a block preconditioner (reading R13) to a
 * relative residual of 1e-13 when a cost model predicts it faster; that path reads
 * a convergence flag back every 10 iterations (the stream is synchronised even with rep == NULL)
 * and is skipped while the stream is being captured into a CUDA graph.  theta_out: D complex128,
 * D = (2m+1)^d (d(2m+1) for ADDITIVE).  rep may be NULL (dense path: no synchronisation,
 * CUDA-graph capturable); otherwise the call synchronises `stream` and fills *rep.  Returns FK_E_SOLVE if A is not numerically positive
 * definite when rep != NULL; on every path a non-positive pivot or a watchdog expiry is also ORed
 * into *P->d_status (FK_DSTATUS_NOT_SPD / FK_DSTATUS_WATCHDOG) by the device, when d_status != NULL. */
fk_status fk_solve(const fk_problem* P, double* theta_out, fk_solve_report* rep, void* ws, size_t ws_bytes,
                   fk_stream_t stream);

/* Prediction by the type-2 sum: out_j = Re sum_k theta_k exp(+i pi <k, Xq_j> / 2L);
 * additive != 0: out_j = sum_l Re sum_a theta_{l,a} exp(+i pi a Xq_{j,l} / 2L).
 * out: Xq.n values of Xq.dtype.  d in {1, 2} (any d for additive). */
fk_status fk_predict_type2(const double* theta, int d, int m, double L, int additive, fk_points Xq, double eps, void* out,
                           void* ws, size_t ws_bytes, int* d_status, fk_stream_t stream);

/* Regularisation path (grid search over lambda reusing one pass over the data):
 * theta_l = A(lambda_l)^{-1} r / n for nlam values lambdas[l] (host array), all other fields of *P
 * as for fk_solve (P->lambda is ignored).  A(lambda) = A0 + lambda M^*M with the real-symmetric
 * reduction of fk_solve; one eigendecomposition of Dg^{-1/2} A0 Dg^{-1/2} (Dg = the diagonal of
 * M^*M in the real basis) then costs O(D^2) per lambda.  theta_out: nlam x D complex128 (device,
 * row l = theta(lambda_l)).  If info != NULL the call synchronises `stream` and stores the
 * eigensolver's info (0 = success; FK_E_SOLVE otherwise).  Sobolev systems with D >= 9000, d <= 2:
 * when one fk_solve per lambda (CG where cheaper) is predicted faster than the eigendecomposition,
 * the path runs those solves instead (same result to the solvers' accuracy; not-SPD systems are
 * then not reported) and synchronises `stream` (CG convergence checks). */
fk_status fk_solve_path(const fk_problem* P, const double* lambdas, int nlam, double* theta_out, int* info, void* ws,
                        size_t ws_bytes, fk_stream_t stream);

/* Held-out risk along a path (grid search; reading R11):
 * risk_out[l] = (1/n_v) sum_j (Y_j - f_l(x_j))^2 over a validation set, f_l the predictor of
 * theta[l] (nlam x D complex128, device, Hermitian as produced by fk_solve / fk_solve_path), computed
 * WITHOUT predicting at the validation points: from the validation set's moments and rhs (the same
 * type-1 calls on (X_v, Y_v)), Pv->mu_moments / rhs / cross / n_total = those sums and n_v, Pv->d, m,
 * kind as for the fit (lambda, mu_pde and PI fields ignored).  sum_y2 = sum_j Y_j^2 (host scalar; it
 * only shifts every risk equally).  risk_out: nlam doubles (device).  Asynchronous on `stream`. */
fk_status fk_path_validate(const fk_problem* Pv, const double* theta, int nlam, double sum_y2, double* risk_out, void* ws,
                           size_t ws_bytes, fk_stream_t stream);

/* The same one-pass rhs (+ moments) from HOST memory (the end-to-end path of a fit whose data live
 * on the host): X.ptr and Y point to host arrays (page-locked for overlap; pageable works but the
 * copies then serialise), X contiguous (stride_n = d, stride_d = 1), d in {1, 2}.  The samples are
 * streamed in chunks of `chunk` samples (0 = 2^24) through two device staging buffers taken from
 * `ws`: chunk i+1 is copied host->device on the library's copy stream while `stream` spreads chunk
 * i (FK_ACCUMULATE across chunks), so the PCIe transfer and the spreading overlap.  Outputs, flags,
 * d_status and ordering as fk_rhs_type1 (all work is ordered after prior work on `stream`; the
 * host arrays must stay valid until `stream` has passed the call).  ws: fk_workspace_bytes(
 * FK_ENTRY_RHS_HOST, d, m, eps, dtype, chunk, 0). */
fk_status fk_rhs_type1_host(fk_points X, const void* Y, double L, int m, double eps, double* r_out, double* mu_out, int flags,
                            int64_t chunk, void* ws, size_t ws_bytes, int* d_status, fk_stream_t stream);

typedef enum fk_entry {
  FK_ENTRY_MOMENTS = 0,
  FK_ENTRY_RHS = 1,
  FK_ENTRY_CROSS = 2,
  FK_ENTRY_SOLVE = 3,
  FK_ENTRY_PREDICT = 4,
  FK_ENTRY_SOLVE_PATH = 5, /* n = number of lambdas */
  FK_ENTRY_PATH_VALIDATE = 6, /* n = number of lambdas */
  FK_ENTRY_RHS_HOST = 7        /* n = chunk (samples per staged chunk; 0 = 2^24) */
} fk_entry;

/* Workspace bytes the call `entry` needs for (d, m, eps, dtype, n, kind) on the current device
 * (kind: fk_kind for SOLVE, the additive flag for PREDICT, ignored otherwise).  0 on error. */
size_t fk_workspace_bytes(int entry, int d, int m, double eps, int dtype, int64_t n, int kind);

/* Last error message of the calling thread ("" if none). */
const char* fk_last_error(void);

/* Library version string. */
const char* fk_version(void);

/* Diagnostics (not part of the method; used by bench.py for the roofline line):
 * fk_profile_enable(1) brackets every spreading-kernel launch with CUDA events recorded on the
 * launching stream; fk_profile_read() waits for the recorded events, returns the summed
 * spreading-kernel device time (ms) and launch count since the last read, and the number of
 * kernels libfk itself launched (cuFFT / cuSOLVER internals excluded), then resets all three. */
void fk_profile_enable(int on);
int fk_profile_read(double* spread_ms, int64_t* spread_launches, int64_t* kernel_launches);

#ifdef __cplusplus
}
#endif
#endif /* FK_H */
