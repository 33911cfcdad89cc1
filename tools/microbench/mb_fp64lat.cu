// fp64 ALU latency / throughput on the B200 (DFMA, DMUL, MUFU.RSQ64H-based rsqrt, LDS, STS+LDS via
// __syncwarp) in SM clocks: the per-pivot chain of the diagonal-tile POTRF (round-2 solve study).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_fp64lat mb_fp64lat.cu
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a0, double b0) {
  __shared__ double sm[64];
  double a = a0 + threadIdx.x, b = b0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u) a = fma(a, b, 1e-300);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 128; ++i)
#pragma unroll
    for (int u = 0; u < 8; ++u) a = rsqrt(a) + 1.0;
  long long t2 = clock64();
  sm[threadIdx.x] = a;
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    a = sm[((int)a) & 31] + 0.5;  // dependent LDS
  }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    sm[threadIdx.x & 31] = a;
    __syncwarp();
    a = sm[(threadIdx.x + 1) & 31] * 0.999;
    __syncwarp();
  }
  long long t4 = clock64();
  float f = (float)a;
#pragma unroll 1
  for (int i = 0; i < 64; ++i)
#pragma unroll
    for (int u = 0; u < 16; ++u) f = fmaf(f, 0.999f, 1e-30f);
  long long t5 = clock64();
  out[threadIdx.x] = a + f;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
    cyc[3] = t4 - t3;
    cyc[4] = t5 - t4;
  }
}
// one owner step of the 2 x 2 pivot POTRF as a dependent chain: shuffles -> det -> 2 rsqrt -> l
__global__ void owner_chain(double* out, long long* cyc, double x0i, double x1i) {
  const int lane = threadIdx.x & 31;
  double x0 = x0i + lane, x1 = x1i + 0.5 * lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    const int J = (i & 15) * 2;
    const double a = __shfl_sync(~0u, x0, J), b = __shfl_sync(~0u, x0, J + 1), c = __shfl_sync(~0u, x1, J + 1);
    const double det = fma(a, c, -b * b);
    const double ra = rsqrt(a), rd = rsqrt(det);
    const double rard = ra * rd;
    const double l0 = x0 * ra, l1 = rard * fma(a, x1, -b * x0);
    x0 = fma(l0, 1e-3, 40.0 + lane);
    x1 = fma(l1, 1e-3, 1.0);
  }
  long long t1 = clock64();
  double a = x0;
#pragma unroll 1
  for (int i = 0; i < 256; ++i) {
    const double b = __shfl_sync(~0u, a, i & 31);
    a = fma(b, 1e-3, 40.0 + lane);
  }
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 256; ++i) a = rsqrt(a) + 40.0;
  long long t3 = clock64();
  out[threadIdx.x] = x0 + x1 + a;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}

template <int CH>
__global__ void thr(double* out, long long* cyc, double b) {
  double a[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) a[c] = threadIdx.x + c;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 64; ++i)
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c = 0; c < CH; ++c) a[c] = fma(a[c], b, 1e-300);
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 24);
  cudaMalloc(&cyc, 64);
  long long h[8];
  lat<<<1, 32>>>(out, cyc, 1.0, 0.9999);
  lat<<<1, 32>>>(out, cyc, 1.0, 0.9999);
  cudaMemcpy(h, cyc, 40, cudaMemcpyDeviceToHost);
  printf("per op (dependent chain, one warp): DFMA %.1f  rsqrt(double)+DADD %.1f  LDS.64+DADD %.1f  STS+syncwarp+LDS+DMUL+syncwarp %.1f  FFMA %.1f cycles\n",
         h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0, h[3] / 1024.0, h[4] / 1024.0);
  owner_chain<<<1, 32>>>(out, cyc, 40.0, 1.0);
  owner_chain<<<1, 32>>>(out, cyc, 40.0, 1.0);
  cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  printf("owner step chain %.1f cycles; shfl.f64+DFMA %.1f; rsqrt+DADD (rolled) %.1f\n", h[0] / 256.0, h[1] / 256.0, h[2] / 256.0);
  for (int warps : {1, 4, 8, 32}) {
    thr<8><<<1, 32 * warps>>>(out, cyc, 0.9999);
    thr<8><<<1, 32 * warps>>>(out, cyc, 0.9999);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %2d warps x 8 chains: %.2f cycles per warp-instruction per SM (%.1f lanes/clk/SM)\n", warps,
           h[0] / (256.0 * 8 * warps), 32.0 * 256 * 8 * warps / h[0]);
    thr<16><<<1, 32 * warps>>>(out, cyc, 0.9999);
    thr<16><<<1, 32 * warps>>>(out, cyc, 0.9999);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA throughput, %2d warps x 16 chains: %.2f cycles per warp-instruction per SM (%.1f lanes/clk/SM)\n", warps,
           h[0] / (256.0 * 16 * warps), 32.0 * 256 * 16 * warps / h[0]);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
