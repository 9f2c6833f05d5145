// Per-iteration cost of a CUDA-graph conditional WHILE loop on this GPU (design input for the
// device-resident Nelder-Mead, kde_nm_dev.cu): body = k tiny kernels (1 thread or a full wave),
// the last one counts down and clears the condition.  nvcc -arch=sm_100a tools/graph_loop.cu -o /tmp/gl
#include <cstdio>
#include <cuda_runtime.h>
__global__ void tick(int* c) {}
__global__ void wave(float* x) { x[blockIdx.x * blockDim.x + threadIdx.x] += 1.f; }
__global__ void last(int* cnt, cudaGraphConditionalHandle h) {
  if (--(*cnt) <= 0) cudaGraphSetConditional(h, 0);
}
int main() {
  int* cnt; float* x;
  cudaMalloc(&cnt, 4); cudaMalloc(&x, 148 * 4 * 256 * 4);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int body = 1; body <= 3; ++body) for (int big = 0; big < 2; ++big) {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t node; cudaGraphAddNode(&node, g, nullptr, 0, &cp);
    cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    for (int k = 0; k < body - 1; ++k) { if (big) wave<<<148 * 4, 256, 0, s>>>(x); else tick<<<1, 1, 0, s>>>(cnt); }
    last<<<1, 1, 0, s>>>(cnt, h);
    cudaGraph_t cap; cudaStreamEndCapture(s, &cap);
    cudaGraphExec_t ex; cudaGraphInstantiate(&ex, g, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 3; ++rep) {
      int it = 1000; cudaMemcpy(cnt, &it, 4, cudaMemcpyHostToDevice);
      cudaEventRecord(e0, s); cudaGraphLaunch(ex, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      if (rep == 2) printf("body %d kernels (%s): %.2f us per iteration\n", body, big ? "592-CTA waves + 1-thread" : "1-thread", ms * 1000 / 1000);
    }
  }
  // reference: the same kernels launched from the host with a sync every iteration
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 1000; ++i) { wave<<<148 * 4, 256, 0, s>>>(x); cudaStreamSynchronize(s); }
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("host loop, 1 wave kernel + sync: %.2f us per iteration\n", ms);
  return 0;
}
