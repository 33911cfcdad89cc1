/*
 * oracle/direct.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle of the fit path).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library.  The product path (paper_2509_02649_b200/) never does;
 * the two share no code, headers, tables or constants.
 *
 * Plain fp64 direct summation of the exponential sums of arXiv 2509.02649:
 *   t_j          = pi * X_j / (2L)
 *   type1_k      = sum_j w_j exp(-i <k, t_j>),  ||k||_inf <= K   (sec. 2.3
 *                  "Covariance vector"/"Covariance matrix"; sign per DESIGN.md reading R1:
 *                  Phi* Phi and Phi* Y with phi(x) = exp(-i pi <k,x>/2L))
 *   cross_{a,b}  = sum_j exp(-i (a t_{j,l1} - b t_{j,l2}))       (sec. 5
 *                  "Complexity": the 2-D NUFFT at (X_l1, -X_l2))
 *   type2(x)     = Re sum_k theta_k exp(+i <k, t(x)>)
 *
 * Every term is evaluated with libm cos/sin of the full argument (no recurrences,
 * no blocking); sums over samples use Kahan compensation in the natural sample order,
 * so the result does not depend on the thread count.  OpenMP parallelises over the
 * output modes only (each mode's sum is computed by one thread, start to end).
 *
 * Mode layout: multi-index k in {-K..K}^d, lexicographic, last coordinate fastest
 * (the layout of include/fk.h); complex outputs are interleaved (re, im) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORACLE_PI 3.14159265358979323846

/* decode a flat mode index into the multi-index k (last coordinate fastest) */
static void decode(int64_t idx, int d, int K, int* k) {
  const int64_t side = 2 * (int64_t)K + 1;
  for (int l = d - 1; l >= 0; --l) {
    k[l] = (int)(idx % side) - K;
    idx /= side;
  }
}

/* type1_k = sum_j w_j exp(-i <k, pi X_j / 2L>) for ||k||_inf <= K.
 * X: n x d row-major (sample j, coordinate l at X[j*d + l]); w: n weights or NULL (all ones). */
void oracle_type1(const double* X, const double* w, int64_t n, int d, double L, int K, double* out) {
  const int64_t side = 2 * (int64_t)K + 1;
  int64_t nmodes = 1;
  for (int l = 0; l < d; ++l) nmodes *= side;
  const double scale = ORACLE_PI / (2.0 * L);
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t idx = 0; idx < nmodes; ++idx) {
    int k[16];
    decode(idx, d, K, k);
    double sr = 0.0, cr = 0.0, si = 0.0, ci = 0.0; /* Kahan sums of re and im */
    for (int64_t j = 0; j < n; ++j) {
      double phase = 0.0;
      for (int l = 0; l < d; ++l) phase += (double)k[l] * (scale * X[j * d + l]);
      const double wj = w ? w[j] : 1.0;
      const double tr = wj * cos(phase) - cr;
      const double ur = sr + tr;
      cr = (ur - sr) - tr;
      sr = ur;
      const double ti = -wj * sin(phase) - ci;
      const double ui = si + ti;
      ci = (ui - si) - ti;
      si = ui;
    }
    out[2 * idx] = sr;
    out[2 * idx + 1] = si;
  }
}

/* Cross moments of every feature pair l1 < l2 (lexicographic pair order):
 * G[p][a][b] = sum_j exp(-i (a t_{j,l1} - b t_{j,l2})), a, b in {-m..m}. */
void oracle_cross(const double* X, int64_t n, int d, double L, int m, double* out) {
  const int side = 2 * m + 1;
  const double scale = ORACLE_PI / (2.0 * L);
  int npairs = d * (d - 1) / 2;
  int* P1 = (int*)malloc(sizeof(int) * (npairs > 0 ? npairs : 1));
  int* P2 = (int*)malloc(sizeof(int) * (npairs > 0 ? npairs : 1));
  int p = 0;
  for (int l1 = 0; l1 < d; ++l1)
    for (int l2 = l1 + 1; l2 < d; ++l2) { P1[p] = l1; P2[p] = l2; ++p; }
  const int64_t total = (int64_t)npairs * side * side;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t idx = 0; idx < total; ++idx) {
    const int pp = (int)(idx / ((int64_t)side * side));
    const int a = (int)((idx / side) % side) - m;
    const int b = (int)(idx % side) - m;
    const int l1 = P1[pp], l2 = P2[pp];
    double sr = 0.0, cr = 0.0, si = 0.0, ci = 0.0;
    for (int64_t j = 0; j < n; ++j) {
      const double phase = (double)a * (scale * X[j * d + l1]) - (double)b * (scale * X[j * d + l2]);
      const double tr = cos(phase) - cr;
      const double ur = sr + tr;
      cr = (ur - sr) - tr;
      sr = ur;
      const double ti = -sin(phase) - ci;
      const double ui = si + ti;
      ci = (ui - si) - ti;
      si = ui;
    }
    out[2 * idx] = sr;
    out[2 * idx + 1] = si;
  }
  free(P1);
  free(P2);
}

/* f(x_q) = Re sum_{||k||_inf <= m} theta_k exp(+i <k, pi x_q / 2L>), theta complex interleaved. */
void oracle_type2(const double* theta, int d, int m, double L, const double* Xq, int64_t nq, double* out) {
  const int64_t side = 2 * (int64_t)m + 1;
  int64_t nmodes = 1;
  for (int l = 0; l < d; ++l) nmodes *= side;
  const double scale = ORACLE_PI / (2.0 * L);
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nq; ++q) {
    double s = 0.0, c = 0.0;
    int k[16];
    for (int64_t idx = 0; idx < nmodes; ++idx) {
      decode(idx, d, m, k);
      double phase = 0.0;
      for (int l = 0; l < d; ++l) phase += (double)k[l] * (scale * Xq[q * d + l]);
      /* Re(theta * e^{i phase}) = re*cos - im*sin */
      const double t = theta[2 * idx] * cos(phase) - theta[2 * idx + 1] * sin(phase) - c;
      const double u = s + t;
      c = (u - s) - t;
      s = u;
    }
    out[q] = s;
  }
}

/* Additive model prediction: f(x) = Re sum_l sum_a theta_{l,a} exp(+i a t_l). */
void oracle_type2_additive(const double* theta, int d, int m, double L, const double* Xq, int64_t nq, double* out) {
  const int side = 2 * m + 1;
  const double scale = ORACLE_PI / (2.0 * L);
#pragma omp parallel for schedule(static)
  for (int64_t q = 0; q < nq; ++q) {
    double s = 0.0, c = 0.0;
    for (int l = 0; l < d; ++l) {
      for (int a = -m; a <= m; ++a) {
        const double phase = (double)a * (scale * Xq[q * d + l]);
        const int64_t idx = (int64_t)l * side + (a + m);
        const double t = theta[2 * idx] * cos(phase) - theta[2 * idx + 1] * sin(phase) - c;
        const double u = s + t;
        c = (u - s) - t;
        s = u;
      }
    }
    out[q] = s;
  }
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}
