#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_set(cudaGraphConditionalHandle h, int v) { if (threadIdx.x == 0 && h) cudaGraphSetConditional(h, v); }
__global__ void k_body(int* x) { atomicAdd(x, 1); }
__global__ void k_pre(int* x) { atomicAdd(x + 1, 1); }
int main() {
  cudaStream_t s, side; cudaStreamCreate(&s); cudaStreamCreate(&side);
  int* x; cudaMalloc(&x, 8); cudaMemset(x, 0, 8);
  cudaGraph_t g; cudaGraphExec_t ge;
  for (int v = 0; v < 2; ++v) {
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaStreamCaptureStatus st; cudaGraph_t cg; const cudaGraphNode_t* deps; size_t nd;
    cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
    cudaGraphConditionalHandle h;
    printf("create %s\n", cudaGetErrorString(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault)));
    k_pre<<<1, 32, 0, s>>>(x);
    k_set<<<1, 32, 0, s>>>(h, v);
    cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
    cudaGraphNode_t node;
    printf("addnode %s\n", cudaGetErrorString(cudaGraphAddNode(&node, cg, deps, nd, &cp)));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    printf("bcap %s\n", cudaGetErrorString(cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)));
    k_body<<<4, 32, 0, side>>>(x);
    printf("ecap %s\n", cudaGetErrorString(cudaStreamEndCapture(side, &body)));
    printf("upd %s\n", cudaGetErrorString(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies)));
    k_pre<<<1, 32, 0, s>>>(x);
    printf("end %s\n", cudaGetErrorString(cudaStreamEndCapture(s, &g)));
    printf("inst %s\n", cudaGetErrorString(cudaGraphInstantiate(&ge, g, 0)));
    for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    int hx[2]; cudaMemcpy(hx, x, 8, cudaMemcpyDeviceToHost);
    printf("v=%d body_count=%d pre_count=%d err=%s\n", v, hx[0], hx[1], cudaGetErrorString(cudaGetLastError()));
  }
}
