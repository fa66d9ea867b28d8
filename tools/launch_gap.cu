// Launch-gap microbenchmark (developer tool, GPU box): a CUDA graph of dependent kernels
// A -> B -> A -> B ..., each stamping %globaltimer at its first and last instruction
// (thread 0 of CTA 0 and the last CTA to exit), and the gap between one kernel's last
// exit and the next one's first start, for several launch shapes of B.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/launch_gap tools/launch_gap.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

typedef unsigned long long ull;
__device__ __forceinline__ ull gt() { ull t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }

__global__ void kstamp(ull* st, int i, int work_ns, int pdl, int has_smem) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ char sm[];
  if (threadIdx.x == 0) atomicMin(&st[2 * i], gt());
  ull t0 = gt();
  while (gt() - t0 < (ull)work_ns) {}
  if (has_smem) sm[threadIdx.x] = 1;
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&st[2 * i + 1], gt());
}
__global__ void __cluster_dims__(8, 1, 1) kstamp_cl(ull* st, int i, int work_ns, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(&st[2 * i], gt());
  ull t0 = gt();
  while (gt() - t0 < (ull)work_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&st[2 * i + 1], gt());
}
// n_red same-address fire-and-forget atomics at the end (the CTA's stamp precedes them)
__global__ void kred(ull* st, int i, int work_ns, int pdl, int n_red, unsigned* ctr) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicMin(&st[2 * i], gt());
  ull t0 = gt();
  while (gt() - t0 < (ull)work_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&st[2 * i + 1], gt());
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_red; k += gridDim.x * blockDim.x) atomicAdd(ctr + (k & 7), 1u);
}
// a kernel with a local-memory (stack) array, dynamically indexed
__global__ void __launch_bounds__(1024, 1) kloc(ull* st, int i, int work_ns, int idx) {
  if (threadIdx.x == 0) atomicMin(&st[2 * i], gt());
  volatile unsigned loc[64];
  for (int k = 0; k < 64; ++k) loc[k] = k * threadIdx.x;
  ull t0 = gt();
  while (gt() - t0 < (ull)work_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&st[2 * i + 1], gt() + loc[idx & 63]);
}
struct Big { ull* st; unsigned* ctr; ull pad[250]; };
__global__ void kbig(const __grid_constant__ Big b, int i, int work_ns) {
  if (threadIdx.x == 0) atomicMin(&b.st[2 * i], gt());
  ull t0 = gt();
  while (gt() - t0 < (ull)work_ns) {}
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&b.st[2 * i + 1], gt() + b.pad[i]);
}
__global__ void kreset(ull* st, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) st[i] = (i & 1) ? 0ull : ~0ull;
}

struct Shape { const char* name; int grid, block; size_t smem; bool coop, cluster; };

static void launch(const Shape& sh, cudaStream_t s, ull* st, int i, int work, bool pdl) {
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(sh.grid); lc.blockDim = dim3(sh.block); lc.dynamicSmemBytes = sh.smem; lc.stream = s;
  cudaLaunchAttribute at[2]; int n = 0;
  if (sh.coop) { at[n].id = cudaLaunchAttributeCooperative; at[n++].val.cooperative = 1; }
  if (pdl) { at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[n++].val.programmaticStreamSerializationAllowed = 1; }
  lc.attrs = at; lc.numAttrs = n;
  cudaError_t e = sh.cluster ? cudaLaunchKernelEx(&lc, kstamp_cl, st, i, work, (int)pdl)
                             : cudaLaunchKernelEx(&lc, kstamp, st, i, work, (int)pdl, (int)(sh.smem > 0));
  if (e != cudaSuccess) { printf("launch %s: %s\n", sh.name, cudaGetErrorString(e)); exit(1); }
}

int main() {
  cudaFuncSetAttribute(kstamp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(kstamp_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  std::vector<Shape> shapes = {
    {"1x32", 1, 32, 0, false, false},
    {"1x1024", 1, 1024, 0, false, false},
    {"1x1024 smem150K", 1, 1024, 150 * 1024, false, false},
    {"313x256 smem53K", 313, 256, 53 * 1024, false, false},
    {"592x256 coop", 592, 256, 32 * 1024, true, false},
    {"10x1024 coop", 10, 1024, 0, true, false},
    {"8x1024 cluster8 smem150K", 8, 1024, 150 * 1024, false, true},
  };
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const int K = 8;                       // kernels per graph
  ull* st; cudaMalloc(&st, sizeof(ull) * 2 * K);
  for (int pdl = 0; pdl < 2; ++pdl)
  for (const Shape& sh : shapes) {
    for (int work : {2000}) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      kreset<<<1, 64, 0, s>>>(st, 2 * K);
      for (int i = 0; i < K; ++i) launch(sh, s, st, i, work, pdl && i > 0);
      if (cudaStreamEndCapture(s, &g) != cudaSuccess) { printf("capture failed\n"); return 1; }
      if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed %s\n", sh.name); return 1; }
      std::vector<double> gaps, durs;
      for (int rep = 0; rep < 50; ++rep) {
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        ull h[2 * K];
        cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
        if (rep < 5) continue;
        for (int i = 1; i < K; ++i) gaps.push_back(((long long)h[2 * i] - (long long)h[2 * i - 1]) / 1e3);
        for (int i = 0; i < K; ++i) durs.push_back((h[2 * i + 1] - h[2 * i]) / 1e3);
      }
      std::sort(gaps.begin(), gaps.end()); std::sort(durs.begin(), durs.end());
      printf("{\"shape\": \"%s\", \"pdl\": %d, \"work_us\": %.1f, \"gap_us_median\": %.2f, \"gap_us_p90\": %.2f, \"dur_us_median\": %.2f}\n",
             sh.name, pdl, work / 1e3, gaps[gaps.size() / 2], gaps[gaps.size() * 9 / 10], durs[durs.size() / 2]);
      cudaGraphExecDestroy(ge); cudaGraphDestroy(g);
    }
  }
  unsigned* ctr; cudaMalloc(&ctr, 64); cudaMemset(ctr, 0, 64);
  for (int n_red : {0, 1000, 5000, 20000}) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    kreset<<<1, 64, 0, s>>>(st, 2 * K);
    for (int i = 0; i < K; ++i) kred<<<313, 256, 0, s>>>(st, i, 2000, 0, n_red, ctr);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<double> gaps;
    for (int rep = 0; rep < 30; ++rep) {
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      ull h[2 * K]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep < 5) continue;
      for (int i = 1; i < K; ++i) gaps.push_back(((long long)h[2 * i] - (long long)h[2 * i - 1]) / 1e3);
    }
    std::sort(gaps.begin(), gaps.end());
    printf("{\"shape\": \"313x256 + %d same-address REDs (8 addresses) after the end stamp\", \"gap_us_median\": %.2f}\n", n_red, gaps[gaps.size() / 2]);
  }
  {
    Big b = {}; b.st = st; b.ctr = ctr;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    kreset<<<1, 64, 0, s>>>(st, 2 * K);
    for (int i = 0; i < K; ++i) kbig<<<313, 256, 0, s>>>(b, i, 2000);
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<double> gaps;
    for (int rep = 0; rep < 30; ++rep) {
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      ull h[2 * K]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep < 5) continue;
      for (int i = 1; i < K; ++i) gaps.push_back(((long long)h[2 * i] - (long long)h[2 * i - 1]) / 1e3);
    }
    std::sort(gaps.begin(), gaps.end());
    printf("{\"shape\": \"313x256, 2 KB parameter struct\", \"gap_us_median\": %.2f}\n", gaps[gaps.size() / 2]);
  }
  {   // alternating shapes: the front-like grid, then a 1-CTA 1024-thread kernel with 150 KB
    Shape A = {"313x256 smem53K", 313, 256, 53 * 1024, false, false};
    Shape B = {"1x1024 smem150K", 1, 1024, 150 * 1024, false, false};
    Shape Cc = {"8x1024 cluster8 smem150K", 8, 1024, 150 * 1024, false, true};
    Shape D = {"592x256 coop smem32K", 592, 256, 32 * 1024, true, false};
    for (int variant = 0; variant < 2; ++variant) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      kreset<<<1, 64, 0, s>>>(st, 2 * K);
      const Shape* seq[8] = {&A, &B, &Cc, &D, &A, &B, &Cc, &D};
      for (int i = 0; i < K; ++i) launch(*seq[i], s, st, i, 2000, false);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      std::vector<double> gp[8];
      void* fl = nullptr; cudaMalloc(&fl, 256 << 20);
      for (int rep = 0; rep < 30; ++rep) {
        if (variant) cudaMemsetAsync(fl, rep, 256 << 20, s);
        cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
        ull h[2 * K]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
        if (rep < 5) continue;
        for (int i = 1; i < K; ++i) gp[i].push_back(((long long)h[2 * i] - (long long)h[2 * i - 1]) / 1e3);
      }
      cudaFree(fl);
      printf("{\"alternating\": \"front-like -> 1x1024 150K -> cluster8 150K -> coop592 32K\", \"l2_flushed\": %d, \"gaps_us\": [", variant);
      for (int i = 1; i < K; ++i) { std::sort(gp[i].begin(), gp[i].end()); printf("%s%.2f", i > 1 ? ", " : "", gp[i][gp[i].size() / 2]); }
      printf("]}\n");
    }
  }
  {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    kreset<<<1, 64, 0, s>>>(st, 2 * K);
    for (int i = 0; i < K; ++i) {
      if (i & 1) kloc<<<1, 1024, 0, s>>>(st, i, 2000, i);
      else kstamp<<<313, 256, 0, s>>>(st, i, 2000, 0, 0);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    std::vector<double> gaps;
    for (int rep = 0; rep < 30; ++rep) {
      cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
      ull h[2 * K]; cudaMemcpy(h, st, sizeof(h), cudaMemcpyDeviceToHost);
      if (rep < 5) continue;
      for (int i = 1; i < K; ++i) gaps.push_back(((long long)h[2 * i] - (long long)h[2 * i - 1]) / 1e3);
    }
    std::sort(gaps.begin(), gaps.end());
    printf("{\"shape\": \"313x256 <-> 1x1024 with a local-memory array\", \"gap_us_median\": %.2f, \"gap_us_max\": %.2f}\n", gaps[gaps.size() / 2], gaps.back());
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("done: %s\n", cudaGetErrorString(e));
  return 0;
}
