// Micro-benchmark: cost of bitonic network stages inside one 1024-thread CTA (developer tool).
#include <cstdio>
#include "../../paper_2602_13692_b200/csrc/common.cuh"

// V2: one element per thread, P <= 1024
__device__ __forceinline__ void net1(u64& k, u32& p, int P, u64* sk, u32* sp) {
  const int t = threadIdx.x;
  const bool act = t < P;
  int buf = 0;
  for (int kk = 2; kk <= P; kk <<= 1) {
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const bool take_min = ((t & j) == 0) == ((t & kk) == 0);
      if (j >= 32) {
        if (act) { sk[buf * 1024 + t] = k; sp[buf * 1024 + t] = p; }
        __syncthreads();
        if (act) bitonic_pick(k, p, sk[buf * 1024 + (t ^ j)], sp[buf * 1024 + (t ^ j)], take_min);
        buf ^= 1;
      } else if (act) {
        const u64 ok = __shfl_xor_sync(FULL_MASK, k, j);
        const u32 op = __shfl_xor_sync(FULL_MASK, p, j);
        bitonic_pick(k, p, ok, op, take_min);
      }
    }
  }
}

__global__ void __launch_bounds__(CTA, 1) k_net(int P, int variant, ull* cyc, u64* out) {
  extern __shared__ __align__(16) char dsm[];
  u64* sk = reinterpret_cast<u64*>(dsm);
  u32* sp = reinterpret_cast<u32*>(dsm + 2 * 1024 * 8);
  const int t = threadIdx.x;
  u64 k = (u64)((t * 7919u) % 1031u) << 20;
  u32 p = t;
  __syncthreads();
  ull t0 = clock64();
  if (variant == 0) {
    net1(k, p, P, sk, sp);
  } else if (variant == 1) {                 // shuffle stages only (no smem stages)
    for (int kk = 2; kk <= 32; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        const bool take_min = ((t & j) == 0) == ((t & kk) == 0);
        const u64 ok = __shfl_xor_sync(FULL_MASK, k, j);
        const u32 op = __shfl_xor_sync(FULL_MASK, p, j);
        bitonic_pick(k, p, ok, op, take_min);
      }
  } else {                                   // one barrier, repeated 55 times
    for (int i = 0; i < 55; ++i) __syncthreads();
  }
  __syncthreads();
  ull t1 = clock64();
  if (t == 0) *cyc = t1 - t0;
  out[t] = k ^ p;
}

int main() {
  ull* cyc; u64* out;
  cudaMalloc(&cyc, 8); cudaMalloc(&out, 8 * 1024);
  cudaFuncSetAttribute(k_net, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 1024 * 12);
  const char* names[] = {"net1 (shfl + smem)", "15 shuffle stages only", "55 x __syncthreads"};
  for (int v = 0; v < 3; ++v)
    for (int P : {32, 64, 256, 1024}) {
      ull best = ~0ull;
      for (int r = 0; r < 5; ++r) {
        k_net<<<1, CTA, 2 * 1024 * 12>>>(P, v, cyc, out);
        ull c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        best = c < best ? c : best;
      }
      printf("%-24s P=%5d cycles=%7llu\n", names[v], P, best);
      if (v) break;
    }
  return 0;
}
