#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* cnt, cudaGraphConditionalHandle h) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < 10 ? 1u : 0u);
}
int main() {
  int* d; cudaMalloc(&d, 4); cudaMemset(d, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {cudaGraphNodeTypeConditional};
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node; cudaGraphAddNode(&node, g, nullptr, 0, &p);
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  body<<<1,1,0,s>>>(d, h);
  cudaStreamEndCapture(s, &bodyg);
  cudaGraphExec_t ge; cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
  int hcnt; cudaMemcpy(&hcnt, d, 4, cudaMemcpyDeviceToHost);
  printf("count=%d err=%s\n", hcnt, cudaGetErrorString(cudaGetLastError()));
}
