// Probe: a conditional IF node inserted into an ongoing stream capture, its body
// captured on a side stream, the condition set from a kernel of the same graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -o cond_graph cond_graph.cu
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_set(cudaGraphConditionalHandle h, const int* flag) {
  if (threadIdx.x == 0) cudaGraphSetConditional(h, *flag ? 1u : 0u);
}
__global__ void k_add(int* x, int v) {
  if (threadIdx.x == 0) *x += v;
}
__global__ void k_big(int* x) {  // a big grid, to time a skipped body
  if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(x, 1000);
}

#define CK(c)                                                                       \
  do {                                                                              \
    cudaError_t e = (c);                                                            \
    if (e != cudaSuccess) {                                                         \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #c, cudaGetErrorString(e));      \
      return 1;                                                                     \
    }                                                                               \
  } while (0)

int main() {
  cudaStream_t s, side;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  int *x, *flag;
  CK(cudaMalloc(&x, 4));
  CK(cudaMalloc(&flag, 4));
  const int STEPS = 50;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int st = 0; st < STEPS; ++st) {
    cudaStreamCaptureStatus cs;
    cudaGraph_t g;
    const cudaGraphNode_t* deps;
    size_t nd;
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    k_add<<<1, 32, 0, s>>>(x, 1);
    k_set<<<1, 32, 0, s>>>(h, flag);
    CK(cudaStreamGetCaptureInfo(s, &cs, nullptr, &g, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, deps, nd, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
    CK(cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    for (int j = 0; j < 6; ++j) k_big<<<4000, 256, 0, side>>>(x);
    CK(cudaStreamEndCapture(side, &body));
    k_add<<<1, 32, 0, s>>>(x, 10);
  }
  cudaGraph_t graph;
  CK(cudaStreamEndCapture(s, &graph));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, graph, 0));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int f = 0; f < 2; ++f) {
    CK(cudaMemset(x, 0, 4));
    CK(cudaMemcpy(flag, &f, 4, cudaMemcpyHostToDevice));
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaMemset(x, 0, 4));
      cudaEventRecord(a, s);
      CK(cudaGraphLaunch(ex, s));
      cudaEventRecord(b, s);
      CK(cudaStreamSynchronize(s));
    }
    int h = 0;
    CK(cudaMemcpy(&h, x, 4, cudaMemcpyDeviceToHost));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("flag=%d x=%d (expect %d) graph %.1f us = %.2f us/step\n", f, h, STEPS * (11 + (f ? 6000 : 0)), ms * 1e3,
           ms * 1e3 / STEPS);
  }
  return 0;
}
