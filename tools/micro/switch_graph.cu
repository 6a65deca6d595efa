// Does a SWITCH conditional node inside a WHILE body (added during stream
// capture) instantiate and run? Minimal repro of the loop graph shape; the
// switch handle is created on the body graph (variant 0) or the top graph (1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 switch_graph.cu -o switch_graph
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { std::printf("  %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
__global__ void setk(cudaGraphConditionalHandle w, cudaGraphConditionalHandle s, int* it) {
  int i = ++*it;
  cudaGraphSetConditional(s, unsigned(i % 3));
  cudaGraphSetConditional(w, i < 6 ? 1u : 0u);
}
__global__ void body_k(int tag, int* it, int* log) { log[*it] = tag; }
int run(int variant, int with_pre) {
  int *it, *log;
  cudaMalloc(&it, 4); cudaMalloc(&log, 64); cudaMemset(it, 0, 4); cudaMemset(log, 0xff, 64);
  cudaStream_t st, st2; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
  cudaGraph_t graph; CK(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle hw; CK(cudaGraphConditionalHandleCreate(&hw, graph, 1u, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp{}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hw;
  cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t wn; CK(cudaGraphAddNode(&wn, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphConditionalHandle hs;
  CK(cudaGraphConditionalHandleCreate(&hs, variant == 0 ? body : graph, 0u, cudaGraphCondAssignDefault));
  CK(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  if (with_pre) setk<<<1, 1, 0, st>>>(hw, hs, it);
  cudaStreamCaptureStatus cs; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  std::printf("  capture graph == body: %d, deps %zu\n", int(g == body), nd);
  cudaGraphNodeParams sp{}; sp.type = cudaGraphNodeTypeConditional; sp.conditional.handle = hs;
  sp.conditional.type = cudaGraphCondTypeSwitch; sp.conditional.size = 3;
  cudaGraphNode_t sn; CK(cudaGraphAddNode(&sn, g, deps, nd, &sp));
  for (int i = 0; i < 3; ++i) {
    cudaGraph_t bg = sp.conditional.phGraph_out[i];
    CK(cudaStreamBeginCaptureToGraph(st2, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body_k<<<1, 1, 0, st2>>>(10 + i, it, log);
    CK(cudaStreamEndCapture(st2, &bg));
  }
  CK(cudaStreamUpdateCaptureDependencies(st, &sn, 1, cudaStreamSetCaptureDependencies));
  if (!with_pre) setk<<<1, 1, 0, st>>>(hw, hs, it);
  CK(cudaStreamEndCapture(st, &body));
  cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, graph, 0));
  CK(cudaGraphLaunch(ex, st)); CK(cudaStreamSynchronize(st));
  int h[16]; cudaMemcpy(h, log, 64, cudaMemcpyDeviceToHost);
  std::printf("  log:"); for (int i = 0; i < 8; ++i) std::printf(" %d", h[i]); std::printf("\n");
  return 0;
}
int main() {
  for (int v = 0; v < 2; ++v) for (int p = 0; p < 2; ++p) { std::printf("variant %d pre %d\n", v, p); run(v, p); }
  return 0;
}
