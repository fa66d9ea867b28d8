// Micro-benchmark of the planner's CTA sorts (developer tool, GPU box):
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I include \
//        -o /tmp/bench_sort tools/micro/bench_sort.cu && /tmp/bench_sort
// Prints SM cycles per cta_sort call for several n and checks the result is the
// stable order.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "../../paper_2602_13692_b200/csrc/common.cuh"

__global__ void __launch_bounds__(CTA, 1) k_bench(u64* ka, u32* va, u64* kb, u32* vb, int n, ull* cyc, int* which, int radix) {
  __shared__ u32 s_big[8192 + 1];
  __shared__ u32 s_tmp[NWARP + 1];
  extern __shared__ __align__(16) char dsm[];
  SortSmem* sm = reinterpret_cast<SortSmem*>(dsm);
  __syncthreads();
  ull t0 = clock64();
  int r = radix ? cta_radix_sort(ka, va, kb, vb, n, s_big, s_tmp) : cta_sort(ka, va, kb, vb, n, s_big, s_tmp, sm);
  ull t1 = clock64();
  if (threadIdx.x == 0) { *cyc = t1 - t0; *which = r; }
}

int main() {
  int ns[] = {16, 32, 64, 128, 256, 384, 512, 513, 1024, 2048, 4096, 5000};
  u64 *ka, *kb; u32 *va, *vb; ull* cyc; int* wh;
  cudaMalloc(&ka, 8 * 8192); cudaMalloc(&kb, 8 * 8192); cudaMalloc(&va, 4 * 8192); cudaMalloc(&vb, 4 * 8192);
  cudaMalloc(&cyc, 8); cudaMalloc(&wh, 4);
  cudaFuncSetAttribute(k_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DSMEM);
  srand(1);
  for (int radix = 0; radix < 2; ++radix)
  for (int n : ns) {
    std::vector<u64> k(n); std::vector<u32> v(n);
    for (int i = 0; i < n; ++i) { k[i] = ((u64)(rand() % 2) << 63) | ((u64)(rand() % 400) << 32) | (rand() % 50); v[i] = i; }
    ull best = ~0ull; int which = 0;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemcpy(ka, k.data(), 8 * n, cudaMemcpyHostToDevice);
      cudaMemcpy(va, v.data(), 4 * n, cudaMemcpyHostToDevice);
      k_bench<<<1, CTA, PLAN_DSMEM>>>(ka, va, kb, vb, n, cyc, wh, radix);
      ull c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&which, wh, 4, cudaMemcpyDeviceToHost);
      best = std::min(best, c);
    }
    std::vector<u64> ko(n); std::vector<u32> vo(n);
    cudaMemcpy(ko.data(), which ? kb : ka, 8 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(vo.data(), which ? vb : va, 4 * n, cudaMemcpyDeviceToHost);
    std::vector<int> idx(n); for (int i = 0; i < n; ++i) idx[i] = i;
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return k[a] < k[b]; });
    bool ok = true;
    for (int i = 0; i < n; ++i) ok &= ko[i] == k[idx[i]] && vo[i] == v[idx[i]];
    printf("%s n=%5d cycles=%8llu (%.2f us at 1965 MHz) %s %s\n", radix ? "radix  " : "cta_sort", n, best, best / 1965.0, ok ? "OK" : "WRONG",
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
