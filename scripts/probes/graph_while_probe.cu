#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_body(int* cnt, cudaGraphConditionalHandle h, int limit) {
  int v = ++cnt[0];
  cudaGraphSetConditional(h, v < limit ? 1 : 0);
}
int main() {
  int* cnt; cudaMalloc(&cnt, 4); cudaMemset(cnt, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t node;
  cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  printf("add node %s\n", cudaGetErrorString(e));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("begin %s\n", cudaGetErrorString(e));
  k_body<<<1,1,0,s>>>(cnt, h, 7);
  e = cudaStreamEndCapture(s, &body);
  printf("end %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  int c; cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost); printf("launch %s count %d\n", cudaGetErrorString(e), c);
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
  cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost); printf("relaunch count %d\n", c);
}
