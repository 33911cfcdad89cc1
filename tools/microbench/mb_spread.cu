// Microbenchmarks that decide the d=1 spreading design (build-plan step 5).
// Not product code: a standalone executable, run once on a B200 via gpurun.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mb_spread mb_spread.cu
// Prints one line per experiment: name, time, and the derived per-SM rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void gen(float* X, float* Y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = hash32((uint32_t)i * 2654435761u + 17u);
    float x = (float)(h >> 8) * (2.0f / 16777216.0f) - 1.0f;
    X[i] = x; Y[i] = __sinf(x) + ((float)(hash32(h) >> 8) * (1.0f / 16777216.0f) - 0.5f);
  }
}

// (A) streaming read of X and Y (float4), the HBM floor for 8 B/sample.
__global__ void stream_read(const float4* __restrict__ X, const float4* __restrict__ Y, int64_t n4, float* out) {
  float acc = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = __ldcs(X + i); float4 b = __ldcs(Y + i);
    acc += a.x + a.y + a.z + a.w + b.x + b.y + b.z + b.w;
  }
  if (acc == 123.456f) out[0] = acc;
}

// (B) int32 smem atomics, random addresses, 4 consecutive cells in grid A and 4 in grid B per "sample".
template <bool RET>
__global__ void atoms_rand(int iters, int* out) {
  extern __shared__ int sm[];
  const int GA = 32772, GB = 16388;
  int* A = sm; int* B = sm + GA;
  for (int i = threadIdx.x; i < GA + GB; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t s = hash32(threadIdx.x + 7919u * blockIdx.x);
  int chk = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    int ca = (s >> 8) % (GA - 4);
    int cb = ca >> 1;
    if (RET) {
      int o0 = atomicAdd(A + ca, 1), o1 = atomicAdd(A + ca + 1, 2), o2 = atomicAdd(A + ca + 2, 3), o3 = atomicAdd(A + ca + 3, 4);
      int p0 = atomicAdd(B + cb, 1), p1 = atomicAdd(B + cb + 1, 2), p2 = atomicAdd(B + cb + 2, 3), p3 = atomicAdd(B + cb + 3, 4);
      chk |= (o0 | o1 | o2 | o3 | p0 | p1 | p2 | p3);
    } else {
      atomicAdd(A + ca, 1); atomicAdd(A + ca + 1, 2); atomicAdd(A + ca + 2, 3); atomicAdd(A + ca + 3, 4);
      atomicAdd(B + cb, 1); atomicAdd(B + cb + 1, 2); atomicAdd(B + cb + 2, 3); atomicAdd(B + cb + 3, 4);
    }
  }
  __syncthreads();
  if (chk == 0x7fffffff) out[0] = chk;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = A[5];
}

// (C) int32 smem atomics, lane-consecutive (conflict-free) addresses.
__global__ void atoms_cfree(int iters, int* out) {
  extern __shared__ int sm[];
  for (int i = threadIdx.x; i < 49160; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    int base = ((it * 37 + w * 101) & 1023) * 32 + lane;
#pragma unroll
    for (int k = 0; k < 8; ++k) atomicAdd(sm + base + k * 32 * 8 % 16384, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x + 1] = sm[5];
}

// (D) fp32 smem atomicAdd (CAS loop on sm_100a), random addresses.
__global__ void atoms_f32(int iters, int* out) {
  extern __shared__ float smf[];
  const int GA = 32772, GB = 16388;
  float* A = smf; float* B = smf + GA;
  for (int i = threadIdx.x; i < GA + GB; i += blockDim.x) smf[i] = 0;
  __syncthreads();
  uint32_t s = hash32(threadIdx.x + 7919u * blockIdx.x);
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    int ca = (s >> 8) % (GA - 4);
    int cb = ca >> 1;
    atomicAdd(A + ca, 1.f); atomicAdd(A + ca + 1, 2.f); atomicAdd(A + ca + 2, 3.f); atomicAdd(A + ca + 3, 4.f);
    atomicAdd(B + cb, 1.f); atomicAdd(B + cb + 1, 2.f); atomicAdd(B + cb + 2, 3.f); atomicAdd(B + cb + 3, 4.f);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x + 1] = (int)A[5];
}

// (E) prototype of the real d=1 spread: cubic B-spline, density grid nf=65536, Y grid nf=32768,
// int32 fixed point, returning atomics + threshold check (slow path = exchange + global fp64 add).
#define MAGIC 12582912.0f
#define MAGIC_BITS 0x4B400000
template <bool CHECK>
__global__ void __launch_bounds__(1024, 1) spread_proto(const float4* __restrict__ X, const float4* __restrict__ Y, int64_t n4,
                                                         double* gcarry, int* gpart) {
  extern __shared__ int sm[];
  const int GA = 32772, GB = 16388;
  int* A = sm; int* B = sm + GA;
  for (int i = threadIdx.x; i < GA + GB; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const float SA = 1048576.f, KA = SA / 6.f;
  const float SY = 131072.f;
  int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  int64_t beg = per * blockIdx.x, end = min(n4, beg + per);
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    float4 xv = __ldcs(X + i), yv = __ldcs(Y + i);
    float xs[4] = {xv.x, xv.y, xv.z, xv.w}, ys[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x = xs[q], y = ys[q];
      // density grid: u = x*16384 + 32768, local cell = floor(u) - (16384-1) -> taps ca-1..ca+2 at local ca..ca+3
      float p = x * 16384.f;
      float fl = floorf(p);
      float f = p - fl;
      int ca = __float_as_int(fl + MAGIC) - MAGIC_BITS + 16384;  // in [0, 32768]
      float g = 1.f - f, f2 = f * f, f3 = f2 * f, g3 = g * g * g;
      int i0 = __float_as_int(fmaf(g3, KA, MAGIC)) - MAGIC_BITS;
      int i3 = __float_as_int(fmaf(f3, KA, MAGIC)) - MAGIC_BITS;
      int i1 = __float_as_int(fmaf(f3, 3.f * KA, fmaf(f2, -6.f * KA, 4.f * KA + MAGIC))) - MAGIC_BITS;
      int i2 = (int)SA - i0 - i1 - i3;
      // Y grid: u = x*8192 + 16384
      float pb = x * 8192.f;
      float flb = floorf(pb);
      float fb = pb - flb;
      int cb = __float_as_int(flb + MAGIC) - MAGIC_BITS + 8192;
      float yk = y * (SY / 6.f);
      float gb = 1.f - fb, fb2 = fb * fb, fb3 = fb2 * fb, gb3 = gb * gb * gb;
      int j0 = __float_as_int(fmaf(gb3, yk, MAGIC)) - MAGIC_BITS;
      int j3 = __float_as_int(fmaf(fb3, yk, MAGIC)) - MAGIC_BITS;
      int j1 = __float_as_int(fmaf(fmaf(fb3, 3.f, fmaf(fb2, -6.f, 4.f)), yk, MAGIC)) - MAGIC_BITS;
      int jS = __float_as_int(fmaf(y, SY, MAGIC)) - MAGIC_BITS;
      int j2 = jS - j0 - j1 - j3;
      if (CHECK) {
        int o0 = atomicAdd(A + ca, i0), o1 = atomicAdd(A + ca + 1, i1), o2 = atomicAdd(A + ca + 2, i2), o3 = atomicAdd(A + ca + 3, i3);
        int p0 = atomicAdd(B + cb, j0), p1 = atomicAdd(B + cb + 1, j1), p2 = atomicAdd(B + cb + 2, j2), p3 = atomicAdd(B + cb + 3, j3);
        const int T = 1 << 30;
        int fa = (o0 | o1 | o2 | o3) & T;
        int fb_ = ((p0 + T) | (p1 + T) | (p2 + T) | (p3 + T)) & (int)0x80000000;
        if (fa | fb_) {
          for (int k = 0; k < 4; ++k) {
            int v = atomicExch(A + ca + k, 0); atomicAdd(gcarry + ca + k, (double)v);
            int w = atomicExch(B + cb + k, 0); atomicAdd(gcarry + GA + cb + k, (double)w);
          }
        }
      } else {
        atomicAdd(A + ca, i0); atomicAdd(A + ca + 1, i1); atomicAdd(A + ca + 2, i2); atomicAdd(A + ca + 3, i3);
        atomicAdd(B + cb, j0); atomicAdd(B + cb + 1, j1); atomicAdd(B + cb + 2, j2); atomicAdd(B + cb + 3, j3);
      }
    }
  }
  __syncthreads();
  int* dst = gpart + (int64_t)blockIdx.x * (GA + GB);
  for (int i = threadIdx.x; i < GA + GB; i += blockDim.x) dst[i] = sm[i];
}

// (F) the same arithmetic without any shared-memory accumulation (issue-rate ceiling of the math).
__global__ void __launch_bounds__(1024, 1) math_only(const float4* __restrict__ X, const float4* __restrict__ Y, int64_t n4, int* out) {
  const float SA = 1048576.f, KA = SA / 6.f, SY = 131072.f;
  int64_t per = (n4 + gridDim.x - 1) / gridDim.x;
  int64_t beg = per * blockIdx.x, end = min(n4, beg + per);
  int acc = 0;
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    float4 xv = __ldcs(X + i), yv = __ldcs(Y + i);
    float xs[4] = {xv.x, xv.y, xv.z, xv.w}, ys[4] = {yv.x, yv.y, yv.z, yv.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float x = xs[q], y = ys[q];
      float p = x * 16384.f; float fl = floorf(p); float f = p - fl;
      int ca = __float_as_int(fl + MAGIC) - MAGIC_BITS + 16384;
      float g = 1.f - f, f2 = f * f, f3 = f2 * f, g3 = g * g * g;
      int i0 = __float_as_int(fmaf(g3, KA, MAGIC)) - MAGIC_BITS;
      int i3 = __float_as_int(fmaf(f3, KA, MAGIC)) - MAGIC_BITS;
      int i1 = __float_as_int(fmaf(f3, 3.f * KA, fmaf(f2, -6.f * KA, 4.f * KA + MAGIC))) - MAGIC_BITS;
      int i2 = (int)SA - i0 - i1 - i3;
      float pb = x * 8192.f; float flb = floorf(pb); float fb = pb - flb;
      int cb = __float_as_int(flb + MAGIC) - MAGIC_BITS + 8192;
      float yk = y * (SY / 6.f);
      float gb = 1.f - fb, fb2 = fb * fb, fb3 = fb2 * fb, gb3 = gb * gb * gb;
      int j0 = __float_as_int(fmaf(gb3, yk, MAGIC)) - MAGIC_BITS;
      int j3 = __float_as_int(fmaf(fb3, yk, MAGIC)) - MAGIC_BITS;
      int j1 = __float_as_int(fmaf(fmaf(fb3, 3.f, fmaf(fb2, -6.f, 4.f)), yk, MAGIC)) - MAGIC_BITS;
      int jS = __float_as_int(fmaf(y, SY, MAGIC)) - MAGIC_BITS;
      int j2 = jS - j0 - j1 - j3;
      acc += (i0 ^ i1 ^ i2 ^ i3 ^ ca) + (j0 ^ j1 ^ j2 ^ j3 ^ cb);
    }
  }
  if (acc == 0x12345) out[0] = acc;
}

int main(int argc, char** argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("device %s sms %d clock_attr %d kHz smem_optin %zu\n", prop.name, sms, clk_khz, prop.sharedMemPerBlockOptin);
  const int64_t n = 1LL << 30;  // 1.07e9 samples = 8.6 GB
  float *X, *Y; double* gcarry; int* gpart; int* out;
  CK(cudaMalloc(&X, n * 4)); CK(cudaMalloc(&Y, n * 4));
  CK(cudaMalloc(&gcarry, 49160 * 8)); CK(cudaMalloc(&gpart, (size_t)sms * 2 * 49160 * 4)); CK(cudaMalloc(&out, 4096 * 4));
  CK(cudaMemset(gcarry, 0, 49160 * 8));
  gen<<<sms * 8, 512>>>(X, Y, n); CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  const size_t SMEM = 49160 * 4;
  CK(cudaFuncSetAttribute(atoms_rand<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  CK(cudaFuncSetAttribute(atoms_rand<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  CK(cudaFuncSetAttribute(atoms_cfree, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  CK(cudaFuncSetAttribute(atoms_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  CK(cudaFuncSetAttribute(spread_proto<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
  CK(cudaFuncSetAttribute(spread_proto<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));

  for (int rep = 0; rep < 2; ++rep) {
    for (int mult : {1, 2, 4, 8}) {
      cudaEventRecord(e0);
      stream_read<<<sms * mult, 1024>>>((const float4*)X, (const float4*)Y, n / 4, (float*)out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      printf("stream_read grid=%d*148: %.3f ms  %.1f GB/s  %.3e samples/s\n", mult, ms, n * 8.0 / ms / 1e6, n / ms * 1e3);
    }
  }
  const int iters = 4096;
  for (int thr : {512, 1024}) {
    double ops = (double)sms * thr * iters * 8;
    cudaEventRecord(e0); atoms_rand<false><<<sms, thr, SMEM>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("atoms_rand_noret thr=%d: %.3f ms  %.3e atom-lanes/s  %.2f lanes/clk/SM@1.9GHz\n", thr, ms, ops / ms * 1e3, ops / ms * 1e3 / sms / 1.9e9);
    cudaEventRecord(e0); atoms_rand<true><<<sms, thr, SMEM>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("atoms_rand_ret   thr=%d: %.3f ms  %.3e atom-lanes/s  %.2f lanes/clk/SM@1.9GHz\n", thr, ms, ops / ms * 1e3, ops / ms * 1e3 / sms / 1.9e9);
    cudaEventRecord(e0); atoms_cfree<<<sms, thr, SMEM>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("atoms_cfree      thr=%d: %.3f ms  %.3e atom-lanes/s  %.2f lanes/clk/SM@1.9GHz\n", thr, ms, ops / ms * 1e3, ops / ms * 1e3 / sms / 1.9e9);
    cudaEventRecord(e0); atoms_f32<<<sms, thr, SMEM>>>(iters, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("atoms_f32_cas    thr=%d: %.3f ms  %.3e atom-lanes/s  %.2f lanes/clk/SM@1.9GHz\n", thr, ms, ops / ms * 1e3, ops / ms * 1e3 / sms / 1.9e9);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); math_only<<<sms, 1024>>>((const float4*)X, (const float4*)Y, n / 4, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("math_only: %.3f ms  %.3e samples/s  %.1f GB/s-equiv\n", ms, n / ms * 1e3, n * 8.0 / ms / 1e6);
    cudaEventRecord(e0); spread_proto<false><<<sms, 1024, SMEM>>>((const float4*)X, (const float4*)Y, n / 4, gcarry, gpart); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("spread_proto_nocheck: %.3f ms  %.3e samples/s  %.1f GB/s-equiv\n", ms, n / ms * 1e3, n * 8.0 / ms / 1e6);
    cudaEventRecord(e0); spread_proto<true><<<sms, 1024, SMEM>>>((const float4*)X, (const float4*)Y, n / 4, gcarry, gpart); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("spread_proto_check: %.3f ms  %.3e samples/s  %.1f GB/s-equiv\n", ms, n / ms * 1e3, n * 8.0 / ms / 1e6);
  }
  CK(cudaGetLastError());
  printf("done\n");
  return 0;
}
