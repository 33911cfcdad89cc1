// Timing of dense SPD factor + solve options for the fit system sizes (D = 2001, 4225).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_chol mb_chol.cu -lcusolver -lcublas
#include <cstdio>
#include <vector>
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <cuda_runtime.h>

__global__ void fill(double* A, int D) {  // SPD: Toeplitz-like + diagonal
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < (long)D * D; t += (long)gridDim.x * blockDim.x) {
    int i = t % D, j = t / D;
    int q = i > j ? i - j : j - i;
    A[t] = (q == 0 ? 1.0 + 1e-3 * i : 0.5 / (1.0 + q)) ;
  }
}

int main() {
  cusolverDnHandle_t h; cusolverDnCreate(&h);
  cublasHandle_t cb; cublasCreate(&cb);
  for (int D : {2001, 4225}) {
    double *A, *A0, *b, *work; int* info;
    cudaMalloc(&A, (size_t)D * D * 8); cudaMalloc(&A0, (size_t)D * D * 8); cudaMalloc(&b, D * 8); cudaMalloc(&info, 4);
    fill<<<1024, 256>>>(A0, D);
    int lwork = 0; cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_LOWER, D, A, D, &lwork);
    cudaMalloc(&work, (size_t)lwork * 8);
    // 64-bit API
    cusolverDnParams_t prm; cusolverDnCreateParams(&prm);
    size_t wd = 0, wh = 0;
    cusolverDnXpotrf_bufferSize(h, prm, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, A, D, CUDA_R_64F, &wd, &wh);
    void* xwd; cudaMalloc(&xwd, wd); std::vector<char> xwh(wh + 1);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemcpy(A, A0, (size_t)D * D * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0); cusolverDnDpotrf(h, CUBLAS_FILL_MODE_LOWER, D, A, D, work, lwork, info); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dpotrf %.3f ms\n", D, ms);
      cudaMemcpy(A, A0, (size_t)D * D * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0); cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, D, A, D, work, lwork, info); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dpotrf UPPER %.3f ms\n", D, ms);
      cudaEventRecord(e0); cublasDtrsv(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, D, A, D, b, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dtrsv T %.3f ms\n", D, ms);
      cudaEventRecord(e0); cusolverDnDpotrs(h, CUBLAS_FILL_MODE_LOWER, D, 1, A, D, b, D, info); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dpotrs %.3f ms\n", D, ms);
      cudaEventRecord(e0); cublasDtrsv(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, D, A, D, b, 1); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dtrsv N %.3f ms\n", D, ms);
      cudaEventRecord(e0); cublasDtrsm(cb, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, D, 1, (const double[]){1.0}, A, D, b, D); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dtrsm 1 col %.3f ms\n", D, ms);
      cudaMemcpy(A, A0, (size_t)D * D * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0); cusolverDnXpotrf(h, prm, CUBLAS_FILL_MODE_LOWER, D, CUDA_R_64F, A, D, CUDA_R_64F, xwd, wd, xwh.data(), wh, info); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Xpotrf %.3f ms\n", D, ms);
      // GEMM rate reference: D x D x 64
      double *C; cudaMalloc(&C, (size_t)D * D * 8); const double one = 1.0, mone = -1.0;
      cudaEventRecord(e0); cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, D, 128, &mone, A0, D, &one, C, D); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); printf("D=%d Dsyrk k=128 %.3f ms (%.1f TF)\n", D, ms, (double)D * D * 128 / ms / 1e9);
      cudaFree(C);
    }
    cudaFree(A); cudaFree(A0); cudaFree(b); cudaFree(work); cudaFree(info); cudaFree(xwd);
  }
  printf("done\n");
}
