// datagen/gen.cu -- on-device seeded synthetic inputs (libfkgen.so).
//
// Holds none of the method's arithmetic.  Implements exactly the counter-based generator of
// datagen/__init__.py (splitmix64 of (seed, stream, sample id), 24-bit draws, fp32 formulas with
// explicit round-to-nearest operations and no FMA contraction), so a sample is bit-identical
// whether numpy or this kernel produced it.  Used by bench.py and the full-size GPU tests to
// materialise inputs in HBM without a host copy (n = 1e10 samples is 80 GB).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__device__ __forceinline__ void u24pair(uint64_t i, int stream, uint32_t seed, int64_t& a, int64_t& b) {
  const uint64_t key = ((uint64_t)(seed & 0xFFFF) << 48) ^ ((uint64_t)(stream & 0xFF) << 40);
  const uint64_t z = splitmix64(i ^ key);
  a = (int64_t)(z >> 40);
  b = (int64_t)((z >> 16) & 0xFFFFFF);
}

__device__ __forceinline__ float uniform_x(uint64_t i, int stream, uint32_t seed) {
  int64_t u, v;
  u24pair(i, stream, seed, u, v);
  return __fmul_rn((float)(2 * u + 1 - (1LL << 24)), 5.9604644775390625e-08f);
}

__device__ __forceinline__ float unit_x(uint64_t i, int stream, uint32_t seed) {  // [0, 1), exact in fp32
  int64_t u, v;
  u24pair(i, stream, seed, u, v);
  return __fmul_rn((float)u, 5.9604644775390625e-08f);
}

__device__ __forceinline__ float gaussian_x(uint64_t i, int stream, uint32_t seed) {
  int64_t a, b, c, e;
  u24pair(i, stream, seed, a, b);
  u24pair(i, stream + 64, seed, c, e);
  const float s = __fmul_rn((float)(a + b + c + e - (2LL << 24)), 5.9604644775390625e-08f);
  float x = __fmul_rn(s, 0.6928203f);
  return fminf(fmaxf(x, -1.0f), 1.0f);
}

__device__ __forceinline__ float noise(uint64_t i, uint32_t seed) {
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    int64_t a, b;
    u24pair(i, 128 + k, seed, a, b);
    s += a + b;
  }
  return __fmul_rn(__ll2float_rn(s - 6LL * (1LL << 24)), 5.9604644775390625e-08f);
}

__device__ __forceinline__ float fstar_sin(float x) {
  const float x2 = __fmul_rn(x, x);
  float t = __fsub_rn(1.0f, __fmul_rn(x2, 0.05f));
  t = __fmul_rn(__fmul_rn(x2, t), (float)(1.0 / 6.0));
  return __fmul_rn(x, __fsub_rn(1.0f, t));
}

__device__ __forceinline__ float expm1_poly(float z) {
  float p = __fadd_rn(__fmul_rn(z, (float)(1.0 / 24.0)), (float)(1.0 / 6.0));
  p = __fadd_rn(__fmul_rn(z, p), 0.5f);
  p = __fadd_rn(__fmul_rn(z, p), 1.0f);
  return __fmul_rn(z, p);
}

__device__ __forceinline__ float fstar_expcos(float x1, float x2) {
  const float e = __fadd_rn(expm1_poly(x1), 1.0f);
  const float y2 = __fmul_rn(x2, x2);
  const float c = __fsub_rn(1.0f, __fmul_rn(y2, __fsub_rn(0.5f, __fmul_rn(y2, (float)(1.0 / 24.0)))));
  return __fmul_rn(e, c);
}

// xkind: 0 uniform, 1 gaussian, 3 unit (U[0,1)).  ykind: 0 sin, 1 expcos, 2 additive, 4 zero, 5 exp.  X written at
// X[j*stride_n + l*stride_d] (element strides), Y[j] contiguous; sample ids i0 + j.
__global__ void gen_dataset(float* __restrict__ X, float* __restrict__ Y, int64_t n, int d, int64_t stride_n,
                            int64_t stride_d, int64_t i0, int xkind, int ykind, uint32_t seed, float L, int with_noise) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t i = (uint64_t)(i0 + j);
    float x0 = 0.f, x1 = 0.f, yacc = 0.f;
    for (int l = 0; l < d; ++l) {
      const float xu = xkind == 0 ? uniform_x(i, l, seed) : (xkind == 3 ? unit_x(i, l, seed) : gaussian_x(i, l, seed));
      if (l == 0) x0 = xu;
      if (l == 1) x1 = xu;
      if (ykind == 2) yacc = __fadd_rn(yacc, expm1_poly(__fmul_rn(xu, (float)(1.0 / (double)(l + 1)))));
      if (X) X[j * stride_n + l * stride_d] = (L == 1.0f) ? xu : __fmul_rn(xu, L);
    }
    if (Y) {
      float y = 0.f;
      if (ykind == 0) y = fstar_sin(x0);
      else if (ykind == 1) y = fstar_expcos(x0, x1);
      else if (ykind == 2) y = yacc;
      else if (ykind == 5) y = __fadd_rn(expm1_poly(x0), 1.0f);
      if (with_noise) y = __fadd_rn(y, noise(i, seed));
      Y[j] = y;
    }
  }
}

// equispaced-replicated permuted points: v = ((a i + b) mod n_total) mod N, X = (2v+1-N)/N, Y = [v even].
__global__ void gen_equispaced(float* __restrict__ X, float* __restrict__ Y, int64_t count, int64_t i0, uint64_t n_total,
                               uint64_t a, uint64_t b, int log2N) {
  const uint64_t N = 1ULL << log2N;
  const float invN = 1.0f / (float)N;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned __int128 prod = (unsigned __int128)a * (uint64_t)(i0 + j) + b;
    const uint64_t jj = (uint64_t)(prod % n_total);
    const int64_t v = (int64_t)(jj & (N - 1));
    if (X) X[j] = __fmul_rn((float)(2 * v + 1 - (int64_t)N), invN);
    if (Y) Y[j] = (v & 1) ? 0.0f : 1.0f;
  }
}

}  // namespace

extern "C" {

int fkgen_dataset(float* X, float* Y, int64_t n, int d, int64_t stride_n, int64_t stride_d, int64_t i0, int xkind,
                  int ykind, uint32_t seed, float L, int with_noise, cudaStream_t stream) {
  if (n <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gen_dataset<<<sms * 8, 256, 0, stream>>>(X, Y, n, d, stride_n, stride_d, i0, xkind, ykind, seed, L, with_noise);
  return (int)cudaGetLastError();
}

int fkgen_equispaced(float* X, float* Y, int64_t count, int64_t i0, uint64_t n_total, uint64_t a, uint64_t b, int log2N,
                     cudaStream_t stream) {
  if (count <= 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  gen_equispaced<<<sms * 8, 256, 0, stream>>>(X, Y, count, i0, n_total, a, b, log2N);
  return (int)cudaGetLastError();
}

}  // extern "C"
