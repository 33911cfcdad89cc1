// Timing + per-tile trace of the tile dataflow Cholesky (csrc/chol.cu) against cuSOLVER potrf.
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -o mb_chol_tiles mb_chol_tiles.cu \
//     -I../../paper_2509_02649_b200/csrc -L../../paper_2509_02649_b200 -lfk -lcusolver
//   ./mb_chol_tiles N [trace.txt]      trace lines: ticket t_start t_updates_done t_compute_start t_compute_end t_published smid (ns)
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "fk_internal.cuh"

__global__ void fill(double* A, int D) {  // SPD: Toeplitz-like + diagonal
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)D * D; t += (long)gridDim.x * blockDim.x) {
    int i = t % D, j = t / D;
    int q = i > j ? i - j : j - i;
    A[t] = (q == 0 ? 1.0 + 1e-3 * i : 0.5 / (1.0 + q));
  }
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 2002;
  const char* tr = argc > 2 ? argv[2] : nullptr;
  double *A, *A0, *work;
  int* info;
  cudaMalloc(&A, (size_t)N * N * 8);
  cudaMalloc(&A0, (size_t)N * N * 8);
  cudaMalloc(&info, 64);
  fill<<<1024, 256>>>(A0, N);
  void* ws;
  cudaMalloc(&ws, fk::chol_ws_bytes(N));
  const int nt = (N + 31) / 32, ntiles = nt * (nt + 1) / 2;
  unsigned long long* trace;
  // trace layout (chol.cu): 6 words per ticket (U tasks included: < ntiles + nt * (nt / 16 + 1) tickets),
  // then 2 * nt words for the diagonal tasks
  const size_t tr_words = (size_t)6 * (ntiles + (size_t)nt * (nt / 16 + 1)) + 2 * nt + 64;
  cudaMalloc(&trace, tr_words * 8);
  cudaMemset(trace, 0, tr_words * 8);
  cusolverDnHandle_t h;
  cusolverDnCreate(&h);
  int lwork = 0;
  cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, N, A, N, &lwork);
  cudaMalloc(&work, (size_t)lwork * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  std::vector<double> Lt((size_t)N * N), Lc((size_t)N * N);
  for (int rep = 0; rep < 4; ++rep) {
    cudaMemcpy(A, A0, (size_t)N * N * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    fk::chol_tiles(A, N, N, info, ws, 0, rep == 3 ? trace : nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("N=%d tiles %.3f ms (%s)\n", N, ms, cudaGetErrorString(cudaGetLastError()));
    if (rep == 3) cudaMemcpy(Lt.data(), A, (size_t)N * N * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(A, A0, (size_t)N * N * 8, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, N, A, N, work, lwork, info);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("N=%d cusolver %.3f ms\n", N, ms);
    if (rep == 3) cudaMemcpy(Lc.data(), A, (size_t)N * N * 8, cudaMemcpyDeviceToHost);
  }
  double md = 0;
  for (int j = 0; j < N; ++j)
    for (int i = j; i < N; ++i) md = std::max(md, std::fabs(Lt[i + (size_t)j * N] - Lc[i + (size_t)j * N]));
  printf("max |L_tiles - L_cusolver| = %.3e\n", md);
  if (tr) {
    std::vector<unsigned long long> t(tr_words);
    cudaMemcpy(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost);
    FILE* f = fopen(tr, "w");
    unsigned long long base = ~0ULL;
    for (int k = 0; k < ntiles; ++k)
      if (t[6 * k]) base = std::min(base, t[6 * k]);  // slots past the last ticket stay 0
    for (int k = 0; k < ntiles; ++k)
      fprintf(f, "%d %llu %llu %llu %llu %llu %llu\n", k, t[6 * k] - base, t[6 * k + 1] - base, t[6 * k + 2] - base,
              t[6 * k + 3] - base, t[6 * k + 4] - base, t[6 * k + 5]);
    fclose(f);
    // diagonal tasks: the external-flag time (slot 6 * ntasks + j; ntasks <= ntiles), raw
    std::string ex = std::string(tr) + ".ext";
    FILE* g = fopen(ex.c_str(), "w");
    for (size_t k = 0; k < t.size(); ++k) fprintf(g, "%llu\n", t[k]);
    fclose(g);
  }
  return 0;
}
