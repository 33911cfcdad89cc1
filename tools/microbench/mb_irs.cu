// Mixed-precision iterative-refinement solvers of cuSOLVER vs fp64 potrf on a C3-like SPD system.
#include <cstdio>
#include <cmath>
#include <vector>
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>
__global__ void fill(double* A, int m, int D, double lam, double s, const double* c) {
  const int side = 2 * m + 1;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)D * D; t += (long)gridDim.x * blockDim.x) {
    int i = t % D, j = t / D;
    int i0 = i / side - m, i1 = i % side - m, j0 = j / side - m, j1 = j % side - m;
    double v = c[i0 - j0 + 2 * m] * c[i1 - j1 + 2 * m];
    if (i == j) v += lam * (1.0 + pow((double)(i0 * i0 + i1 * i1), s));
    A[t] = v;
  }
}
__global__ void scale(double* A, int D) {  // Jacobi: A_ij / sqrt(A_ii A_jj) (diagonal read from a copy)
}
int main(int argc, char** argv) {
  int m = argc > 1 ? atoi(argv[1]) : 64;
  double lam = 1e-6, s = 2.0;
  int D = (2 * m + 1) * (2 * m + 1);
  std::vector<double> hc(4 * m + 1);
  for (int q = -2 * m; q <= 2 * m; ++q) { double x = q / 2.0; hc[q + 2 * m] = q == 0 ? 1.0 : sin(M_PI * x) / (M_PI * x); }
  double *c, *A0, *A, *b, *x, *x0, *r; cudaMalloc(&c, hc.size() * 8); cudaMemcpy(c, hc.data(), hc.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&A0, (size_t)D * D * 8); cudaMalloc(&A, (size_t)D * D * 8); cudaMalloc(&b, D * 8); cudaMalloc(&x, D * 8); cudaMalloc(&x0, D * 8); cudaMalloc(&r, D * 8);
  fill<<<4096, 256>>>(A0, m, D, lam, s, c);
  std::vector<double> hb(D); for (int i = 0; i < D; ++i) hb[i] = sin(0.37 * i) + 0.1;
  cudaMemcpy(b, hb.data(), D * 8, cudaMemcpyHostToDevice);
  cusolverDnHandle_t h; cusolverDnCreate(&h); cublasHandle_t cb; cublasCreate(&cb);
  int* info; cudaMalloc(&info, 4); int* ipiv; cudaMalloc(&ipiv, D * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  auto resid = [&](const double* xx) {
    const double one = 1.0, mone = -1.0;
    cudaMemcpy(r, b, D * 8, cudaMemcpyDeviceToDevice);
    cublasDgemv(cb, CUBLAS_OP_N, D, D, &mone, A0, D, xx, 1, &one, r, 1);
    double nr, nb; cublasDnrm2(cb, D, r, 1, &nr); cublasDnrm2(cb, D, b, 1, &nb); return nr / nb;
  };
  auto diff = [&](const double* xx) {
    const double mone = -1.0; cudaMemcpy(r, xx, D * 8, cudaMemcpyDeviceToDevice);
    cublasDaxpy(cb, D, &mone, x0, 1, r, 1); double nr, nx; cublasDnrm2(cb, D, r, 1, &nr); cublasDnrm2(cb, D, x0, 1, &nx); return nr / nx;
  };
  // baseline potrf + potrs
  {
    int lw = 0; cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, D, A, D, &lw); double* w; cudaMalloc(&w, (size_t)lw * 8);
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(A, A0, (size_t)D * D * 8, cudaMemcpyDeviceToDevice); cudaMemcpy(x0, b, D * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, D, A, D, w, lw, info);
      cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, D, 1, A, D, x0, D, info);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("D=%d potrf+potrs: %.2f ms  resid %.2e\n", D, ms, resid(x0));
    cudaFree(w);
  }
  typedef cusolverStatus_t (*gesv_t)(cusolverDnHandle_t, int, int, double*, int, int*, double*, int, double*, int, void*, size_t, int*, int*);
  typedef cusolverStatus_t (*gesvbs_t)(cusolverDnHandle_t, int, int, double*, int, int*, double*, int, double*, int, void*, size_t*);
  struct V { const char* name; gesv_t f; gesvbs_t bs; } vs[] = {
    {"DDgesv (fp64 LU)", cusolverDnDDgesv, cusolverDnDDgesv_bufferSize},
    {"DSgesv (fp32 LU + IR)", cusolverDnDSgesv, cusolverDnDSgesv_bufferSize},
    {"DXgesv (tf32 LU + IR)", cusolverDnDXgesv, cusolverDnDXgesv_bufferSize},
    {"DBgesv (bf16 LU + IR)", cusolverDnDBgesv, cusolverDnDBgesv_bufferSize},
    {"DHgesv (fp16 LU + IR)", cusolverDnDHgesv, cusolverDnDHgesv_bufferSize}};
  for (auto& v : vs) {
    size_t lw = 0; v.bs(h, D, 1, A, D, ipiv, b, D, x, D, nullptr, &lw);
    void* w; if (cudaMalloc(&w, lw) != cudaSuccess) { printf("%s: no memory for %zu\n", v.name, lw); continue; }
    int iter = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemcpy(A, A0, (size_t)D * D * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      cusolverStatus_t st = v.f(h, D, 1, A, D, ipiv, b, D, x, D, w, lw, &iter, info);
      cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
      if (st != CUSOLVER_STATUS_SUCCESS) printf("  status %d\n", (int)st);
    }
    int hinfo; cudaMemcpy(&hinfo, info, 4, cudaMemcpyDeviceToHost);
    printf("%s: %.2f ms  iter %d info %d  resid %.2e  vs potrf %.2e\n", v.name, ms, iter, hinfo, resid(x), diff(x));
    cudaFree(w);
  }
  return 0;
}
