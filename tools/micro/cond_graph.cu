#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_cond(cudaGraphConditionalHandle h, int* cnt, int lim) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < lim ? 1u : 0u);
}
__global__ void k_body(int* x) { atomicAdd(x, 1); }
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add %d\n", (int)e);
  int* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t body = p.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  k_body<<<1,1,0,s>>>(d);
  k_cond<<<1,1,0,s>>>(h, d + 1, 5);
  e = cudaStreamEndCapture(s, &body);
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0);
  printf("inst %d\n", (int)e);
  cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int hv[2]; cudaMemcpy(hv, d, 8, cudaMemcpyDeviceToHost);
  printf("%d %d\n", hv[0], hv[1]);
}
