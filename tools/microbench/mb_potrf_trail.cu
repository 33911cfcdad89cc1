// The diagonal task's two warps in isolation (csrc/chol.cu): warp 0 POTRF with quarter releases, warp 1
// the trailing TRSM of the sub-diagonal tile; cycles of both and the residual |X L^T - B|.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o mb_potrf_trail mb_potrf_trail.cu \
//        -I../../paper_2509_02649_b200/csrc -I../../include -L../../paper_2509_02649_b200 -lfk
#include "../../paper_2509_02649_b200/csrc/chol.cu"
#include <cstdio>
namespace fk { namespace {
__global__ void __launch_bounds__(CT) k_conc(const double* A, const double* B, double* Lout, double* Xout, long long* cyc, int reps, int mode) {
  __shared__ double Tb[TS][LDS];
  __shared__ double Ct[TS][TS + 1], Cs[TS][TS + 1];
  __shared__ double piv[TS], dinv[TS];
  __shared__ int info;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int r = 0; r < reps; ++r) {
    for (int e = threadIdx.x; e < TS * TS; e += CT) { Ct[e % TS][e / TS] = A[e]; Cs[e % TS][e / TS] = B[e]; }
    if (threadIdx.x == 0) info = 0;
    __syncthreads();
    long long t0 = clock64(), t1 = 0;
    if (w == 0) { final_potrf(Ct, Tb, piv, dinv, Lout + 2 * TS * TS, 0, TS, &info, lane, mode != 0); t1 = clock64(); }
    else if (w == 1 && mode) {
      double x[TS];
      for (int c = 0; c < TS; ++c) x[c] = Cs[lane][c];
      trail_rows(x, Tb, dinv);
      for (int c = 0; c < TS; ++c) Cs[lane][c] = x[c];
      t1 = clock64();
    }
    __syncthreads();
    if (lane == 0 && w < 2) cyc[r * 2 + w] = t1 - t0;
  }
  for (int e = threadIdx.x; e < TS * TS; e += CT) { Lout[e] = Ct[e % TS][e / TS]; Xout[e] = Cs[e % TS][e / TS]; }
}
}}
int main() {
  const int n = 32, reps = 32;
  double hA[n * n], hB[n * n];
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { hA[i + j * n] = (i == j ? 40.0 + i : 1.0 / (1.0 + (i > j ? i - j : j - i))); hB[i + j * n] = 0.1 * ((i * 7 + j * 3) % 11); }
  double *A, *B, *L, *X; long long* cyc;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&L, 4 * sizeof hA); cudaMalloc(&X, sizeof hA); cudaMalloc(&cyc, reps * 16);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  long long hc[reps * 2];
  for (int mode = 0; mode < 2; ++mode) {
    fk::k_conc<<<1, fk::CT>>>(A, B, L, X, cyc, reps, mode);
    cudaMemcpy(hc, cyc, sizeof hc, cudaMemcpyDeviceToHost);
    printf("mode %d: warp0 POTRF %lld cycles, warp1 TRSM end %lld cycles  %s\n", mode, hc[2 * (reps - 1)], mode ? hc[2 * (reps - 1) + 1] : 0LL, cudaGetErrorString(cudaGetLastError()));
  }
  double hL[n * n], hX[n * n];
  cudaMemcpy(hL, L, sizeof hL, cudaMemcpyDeviceToHost); cudaMemcpy(hX, X, sizeof hX, cudaMemcpyDeviceToHost);
  double e = 0;
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double t = 0; for (int k = 0; k < n; ++k) t += hX[i + k * n] * hL[j + k * n]; e = fmax(e, fabs(t - hB[i + j * n])); }
  printf("max |X L^T - B| = %.2e\n", e);
  return 0;
}
