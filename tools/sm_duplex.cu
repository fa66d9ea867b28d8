// SM-originated host-link copies, one direction and both at once (developer tool, GPU box).
// Even CTAs copy HBM -> pinned host (mapped), odd CTAs pinned host -> HBM, 128-bit
// loads/stores, grid-stride; compared with the DMA engines (cudaMemcpyAsync) alone and in
// both directions on two streams.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/sm_duplex tools/sm_duplex.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void kcopy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n16,
                      const uint4* __restrict__ c, uint4* __restrict__ dd, size_t m16, int mode) {
  // mode 0: a->b only; 1: c->dd only; 2: even CTAs a->b, odd CTAs c->dd
  int role = mode == 2 ? (blockIdx.x & 1) : mode;
  size_t g = mode == 2 ? gridDim.x / 2 : gridDim.x;
  size_t me = mode == 2 ? blockIdx.x / 2 : blockIdx.x;
  const uint4* src = role == 0 ? a : c;
  uint4* dst = role == 0 ? b : dd;
  size_t n = role == 0 ? n16 : m16;
  for (size_t i = me * blockDim.x + threadIdx.x; i < n; i += g * blockDim.x * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { size_t j = i + k * g * blockDim.x; if (j < n) v[k] = src[j]; }
#pragma unroll
    for (int k = 0; k < 4; ++k) { size_t j = i + k * g * blockDim.x; if (j < n) dst[j] = v[k]; }
  }
}

int main() {
  const size_t bytes = 4ull << 30;
  void *hA, *hB, *dA, *dB;
  cudaHostAlloc(&hA, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&hB, bytes, cudaHostAllocMapped);
  cudaMalloc(&dA, bytes); cudaMalloc(&dB, bytes);
  cudaMemset(dA, 1, bytes); memset(hB, 2, bytes);
  void *hAd, *hBd;
  cudaHostGetDevicePointer(&hAd, hA, 0); cudaHostGetDevicePointer(&hBd, hB, 0);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const size_t n16 = bytes / 16;
  for (int ctas_per_sm : {2, 4}) {
    int grid = sms * ctas_per_sm;
    for (int mode = 0; mode < 3; ++mode) {
      float best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        kcopy<<<mode == 2 ? 2 * grid : grid, 256>>>((const uint4*)dA, (uint4*)hAd, n16, (const uint4*)hBd, (uint4*)dB, n16, mode);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double gb = (mode == 2 ? 2.0 : 1.0) * bytes / 1e9;
      printf("{\"path\": \"sm\", \"ctas_per_sm_per_direction\": %d, \"mode\": \"%s\", \"gbs\": %.1f}\n", ctas_per_sm,
             mode == 0 ? "d2h" : mode == 1 ? "h2d" : "duplex_total", gb / (best * 1e-3));
    }
  }
  cudaStream_t s1, s2; cudaStreamCreate(&s1); cudaStreamCreate(&s2);
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      cudaDeviceSynchronize();
      cudaEventRecord(e0, 0);
      if (mode != 1) cudaMemcpyAsync(hA, dA, bytes, cudaMemcpyDeviceToHost, s1);
      if (mode != 0) cudaMemcpyAsync(dB, hB, bytes, cudaMemcpyHostToDevice, s2);
      cudaDeviceSynchronize();
      cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double gb = (mode == 2 ? 2.0 : 1.0) * bytes / 1e9;
    printf("{\"path\": \"dma\", \"mode\": \"%s\", \"gbs\": %.1f}\n", mode == 0 ? "d2h" : mode == 1 ? "h2d" : "duplex_total", gb / (best * 1e-3));
  }
  printf("done: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
