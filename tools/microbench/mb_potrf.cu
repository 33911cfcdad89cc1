// Latency of the diagonal-tile POTRF and of the tile TRSM of csrc/chol.cu (final_potrf / final_trsm,
// 32 x 32, one warp) in isolation, in SM clocks.  Round-2 solve study.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o mb_potrf mb_potrf.cu -I../../paper_2509_02649_b200/csrc \
//        -I../../include -L../../paper_2509_02649_b200 -lfk -Xlinker -rpath=$PWD/../../paper_2509_02649_b200
#include "../../paper_2509_02649_b200/csrc/chol.cu"
#include <cstdio>

namespace fk {
namespace {
// mode 0: final_potrf (diagonal tile), mode 1: final_trsm (X L^T = A, L from mode 0)
__global__ void __launch_bounds__(CT) k_potrf_lat(const double* A, double* Lout, double* Wout, long long* cyc, int reps, int mode) {
  __shared__ double Tb[TS][LDS];
  __shared__ double Ct[TS][TS + 1];
  __shared__ double dv[TS], piv[TS];
  __shared__ int info;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < TS * TS; e += CT) Ct[e % TS][e / TS] = A[e];
    if (mode == 1)
      for (int e = threadIdx.x; e < TS * TS; e += CT) Tb[e / TS][e % TS] = Lout[(e % TS) + (e / TS) * TS];  // [p][r] = L(r, p)
    if (mode == 1 && threadIdx.x < TS) dv[threadIdx.x] = 1.0 / Lout[threadIdx.x * TS + threadIdx.x];
    if (threadIdx.x == 0) info = 0;
    __syncthreads();
    long long t0 = clock64();
    if (w == 0) {
      if (mode == 0) final_potrf(Ct, Tb, piv, dv, Wout, 0, TS, &info, lane);
      else final_trsm(Ct, Tb, dv, lane);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[r] = t1 - t0;
  }
  if (mode == 0)
    for (int e = threadIdx.x; e < TS * TS; e += CT) Lout[e] = Ct[e % TS][e / TS];  // column-major L
  else
    for (int e = threadIdx.x; e < TS * TS; e += CT) Wout[e] = Ct[e % TS][e / TS];  // column-major X
}
}  // namespace
}  // namespace fk

int main() {
  const int n = 32, reps = 64;
  double hA[n * n];
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) hA[i + j * n] = (i == j ? 40.0 + i : 1.0 / (1.0 + (i > j ? i - j : j - i)));
  double *A, *L, *W;
  long long* cyc;
  cudaMalloc(&A, sizeof hA);
  cudaMalloc(&L, sizeof hA);
  cudaMalloc(&W, 2 * sizeof hA);
  cudaMalloc(&cyc, reps * 8);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
  double hL[n * n], hX[n * n];
  long long hc[reps];
  for (int mode = 0; mode < 2; ++mode) {
    fk::k_potrf_lat<<<1, fk::CT>>>(A, L, W, cyc, reps, mode);
    cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
    long long mn = hc[1];
    for (int r = 1; r < reps; ++r) mn = hc[r] < mn ? hc[r] : mn;
    printf("%s: first %lld, min over %d calls %lld cycles (%.2f us at 1.965 GHz)  %s\n", mode ? "final_trsm" : "final_potrf", hc[0], reps,
           mn, mn / 1965.0, cudaGetErrorString(cudaGetLastError()));
  }
  cudaMemcpy(hL, L, sizeof hL, cudaMemcpyDeviceToHost);
  cudaMemcpy(hX, W, sizeof hX, cudaMemcpyDeviceToHost);
  // checks: L L^T = A; X L^T = A (X the TRSM of A itself, i.e. X = L)
  double e1 = 0, e2 = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0, t = 0;
      for (int k = 0; k < n; ++k) s += hL[i + k * n] * hL[j + k * n];
      for (int k = 0; k < n; ++k) t += hX[i + k * n] * hL[j + k * n];
      e1 = fmax(e1, fabs(s - hA[i + j * n]));
      e2 = fmax(e2, fabs(t - hA[i + j * n]));
    }
  printf("max |L L^T - A| = %.2e   max |X L^T - A| = %.2e\n", e1, e2);
  return 0;
}
