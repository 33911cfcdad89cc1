// Conflict model of int32 shared-memory ATOMS.ADD on sm_100a: which lane-address patterns cost
// how many cycles (verdict r01 #2 study; decides whether structured spreading layouts pay).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_atoms_pattern mb_atoms_pattern.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
constexpr int W = 49152;  // words of shared memory used (192 KB)

template <int P>
__global__ void __launch_bounds__(1024, 1) k(int iters, int* out) {
  extern __shared__ int sm[];
  for (int i = threadIdx.x; i < W; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t s = threadIdx.x * 2654435761u + blockIdx.x * 97u + 12345u;
  int chk = 0;
  for (int it = 0; it < iters; ++it) {
    s = s * 1664525u + 1013904223u;
    uint32_t r = s >> 8;
    // partner's random number (same for a group of lanes) via shuffle of the group leader's value
    int a;
    if (P == 0) a = r % W;                                                 // 32 random words
    else if (P == 1) a = (__shfl_sync(~0u, r, lane & ~1) % (W / 2)) * 2 + (lane & 1);   // 16 random aligned pairs
    else if (P == 2) a = (__shfl_sync(~0u, r, lane & ~3) % (W / 4)) * 4 + (lane & 3);   // 8 random aligned quads
    else if (P == 3) a = (r % (W / 2)) * 2 + (lane & 1);                      // even lanes even words, odd lanes odd words
    else if (P == 4) a = ((it * 37 + (threadIdx.x >> 5) * 101) & 1023) * 32 + lane;  // consecutive (conflict-free)
    else if (P == 5) a = (__shfl_sync(~0u, r, lane & ~1) % (W - 1)) + (lane & 1);   // 16 random unaligned adjacent pairs
    else if (P == 6) a = (__shfl_sync(~0u, r, lane & ~1) % (W / 64)) * 64 + (lane & 1) * 32 + (r & 31) ;  // pairs 32 words apart (same bank)
    else if (P == 7) a = ((r % (W / 32)) * 32) + lane;                        // lane-ℓ-in-bank-ℓ, random rows
    else if (P == 8) a = (__shfl_sync(~0u, r, lane & ~15) % (W / 16)) * 16 + (lane & 15);  // 2 random 16-word runs
    else if (P == 9) a = (__shfl_sync(~0u, r, lane & ~7) % (W / 8)) * 8 + (lane & 7);      // 4 random 8-word runs
    else if (P == 10) a = (__shfl_sync(~0u, r, lane & ~7) % (W - 8)) + (lane & 7);         // 4 random unaligned 8-word runs
    else a = (__shfl_sync(~0u, r, lane & ~1) % (W / 2)) * 2 + (lane & 1) + 0 * P;          // (unused)
    chk |= atomicAdd(sm + a, 1);
  }
  __syncthreads();
  if (chk == 0x7fffffff) out[0] = chk;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = sm[5];
}

int main() {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int* out; CK(cudaMalloc(&out, 4096 * 4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[] = {"rand32", "pairs_aligned", "quads_aligned", "parity_split", "consecutive", "pairs_unaligned", "pairs_same_bank",
                         "lane_bank_rows", "runs16_x2", "runs8_x4", "runs8_x4_unal"};
  void (*ks[])(int, int*) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>, k<10>};
  const int iters = 8192;
  for (int rep = 0; rep < 2; ++rep)
    for (int p = 0; p < 11; ++p) {
      CK(cudaFuncSetAttribute(ks[p], cudaFuncAttributeMaxDynamicSharedMemorySize, W * 4));
      cudaEventRecord(e0);
      ks[p]<<<sms, 1024, W * 4>>>(iters, out);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double lanes = (double)sms * 1024 * iters;
      printf("%-16s %.3f ms  %.2f lane-atomics/clk/SM @1.965GHz  (%.2f wavefronts per instruction if 1 wf/clk)\n", names[p], ms,
             lanes / (ms * 1e-3) / sms / 1.965e9, 32.0 / (lanes / (ms * 1e-3) / sms / 1.965e9));
    }
  CK(cudaGetLastError());
  return 0;
}
