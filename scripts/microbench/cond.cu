#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dec(cudaGraphConditionalHandle h, int* cnt, int lim) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < lim ? 1 : 0);
}
__global__ void k_work(int* x) { atomicAdd(x, 1); }
int main() {
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  printf("add cond: %s\n", cudaGetErrorString(cudaGraphAddNode(&wn, g, nullptr, 0, &cp)));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  int *cnt, *x; cudaMallocManaged(&cnt, 4); cudaMallocManaged(&x, 4); *cnt = 0; *x = 0;
  // body: child graph (work) -> decide
  cudaGraph_t child; cudaGraphCreate(&child, 0);
  cudaKernelNodeParams kp = {}; void* a1[] = {&x}; kp.func = (void*)k_work; kp.gridDim = 1; kp.blockDim = 32; kp.kernelParams = a1;
  cudaGraphNode_t wk; cudaGraphAddKernelNode(&wk, child, nullptr, 0, &kp);
  cudaGraphNode_t cn; printf("child: %s\n", cudaGetErrorString(cudaGraphAddChildGraphNode(&cn, body, nullptr, 0, child)));
  int lim = 5; void* a2[] = {&h, &cnt, &lim};
  cudaKernelNodeParams dp = {}; dp.func = (void*)k_dec; dp.gridDim = 1; dp.blockDim = 1; dp.kernelParams = a2;
  cudaGraphNode_t dn; printf("dec: %s\n", cudaGetErrorString(cudaGraphAddKernelNode(&dn, body, &cn, 1, &dp)));
  cudaGraphExec_t ex; printf("inst: %s\n", cudaGetErrorString(cudaGraphInstantiate(&ex, g, 0)));
  printf("launch: %s\n", cudaGetErrorString(cudaGraphLaunch(ex, 0)));
  cudaDeviceSynchronize();
  printf("cnt=%d x=%d (%s)\n", *cnt, *x, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
