// Can L2 atomics add accumulation throughput to the d=1 spread?  (round-2 study of verdict r01 #2:
// the shared-memory atomic unit caps k_spread1d_bs3 at ~9.5 random lane-ops/clk/SM; a hybrid that
// sends part of the taps to L2 as red.global only pays if L2 reds run at a useful rate and do not
// slow the shared atomics down.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_l2red mb_l2red.cu
// Every thread issues `iters` updates at LCG-random addresses:
//   mode 0  ATOMS.ADD (shared, 49152 words)                      -- the spread's resource
//   mode 1  red.global.add.u32 into one shared 64K-word region     (all SMs on the same cells)
//   mode 2  red.global.add.u64 into one shared 64K-word region     (64-bit fixed point, no drains)
//   mode 3  red.global.add.u32 into a per-CTA 64K-word region      (no inter-SM address sharing)
//   mode 4  mixed: per iteration 1 shared atomic + 1 global u32 red (does L2 traffic slow ATOMS?)
//   mode 5  mixed: 3 shared atomics + 1 global u64 red
//   mode 6  red.global.add.v4.f32 (one 16-byte vector red = 4 consecutive cells) into 64K words
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int W = 49152;
constexpr int GW = 65536;

template <int M>
__global__ void __launch_bounds__(1024, 1) k(int iters, int* out, uint32_t* g32, unsigned long long* g64, float* gf) {
  extern __shared__ int sm[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u;
  int chk = 0;
  uint32_t* mine = g32 + (size_t)blockIdx.x * GW;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    const uint32_t r = s >> 8;
    if (M == 0) chk |= atomicAdd(sm + r % W, 1);
    if (M == 1) atomicAdd(g32 + (r & (GW - 1)), 1u);
    if (M == 2) atomicAdd(g64 + (r & (GW / 2 - 1)), 1ull);
    if (M == 3) atomicAdd(mine + (r & (GW - 1)), 1u);
    if (M == 4) {
      chk |= atomicAdd(sm + r % W, 1);
      atomicAdd(g32 + ((r * 7u) & (GW - 1)), 1u);
    }
    if (M == 5) {
      chk |= atomicAdd(sm + r % W, 1);
      chk |= atomicAdd(sm + (r * 3u + 1u) % W, 1);
      chk |= atomicAdd(sm + (r * 5u + 2u) % W, 1);
      atomicAdd(g64 + ((r * 7u) & (GW / 2 - 1)), 1ull);
    }
    if (M == 6) {
      float* p = gf + ((r & (GW / 4 - 1)) * 4);
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(1.f), "f"(0.5f), "f"(0.25f), "f"(0.125f) : "memory");
    }
  }
  __syncthreads();
  if (chk == 0x7fffffff) out[0] = chk;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = sm[5];
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* out; CK(cudaMalloc(&out, 4096 * 4));
  uint32_t* g32; CK(cudaMalloc(&g32, (size_t)sms * GW * 4)); CK(cudaMemset(g32, 0, (size_t)sms * GW * 4));
  unsigned long long* g64; CK(cudaMalloc(&g64, GW * 4)); CK(cudaMemset(g64, 0, GW * 4));
  float* gf; CK(cudaMalloc(&gf, GW * 4)); CK(cudaMemset(gf, 0, GW * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"smem_atoms", "l2_red_u32_shared", "l2_red_u64_shared", "l2_red_u32_perCTA", "mix_1atoms_1red32", "mix_3atoms_1red64", "l2_red_v4f32"};
  const double per_it[] = {1, 1, 1, 1, 2, 4, 4};  // cell updates per iteration
  void (*ks[])(int, int*, uint32_t*, unsigned long long*, float*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>};
  const int iters = 4096;
  for (int rep = 0; rep < 2; ++rep)
    for (int p = 0; p < 7; ++p) {
      CK(cudaFuncSetAttribute(ks[p], cudaFuncAttributeMaxDynamicSharedMemorySize, W * 4));
      cudaEventRecord(e0);
      ks[p]<<<sms, 1024, W * 4>>>(iters, out, g32, g64, gf);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)sms * 1024 * iters;
      printf("%-20s %.3f ms  %.3e instr-lanes/s  %.3e cell-updates/s  %.2f updates/clk/SM @1.965GHz\n", names[p], ms, ops / (ms * 1e-3),
             ops * per_it[p] / (ms * 1e-3), ops * per_it[p] / (ms * 1e-3) / sms / 1.965e9);
    }
  CK(cudaGetLastError());
  return 0;
}
