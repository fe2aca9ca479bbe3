// which node kinds instantiate inside a conditional WHILE body (child graph captured from a stream)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dec(cudaGraphConditionalHandle h, int* cnt, int lim) { int c = ++(*cnt); cudaGraphSetConditional(h, c < lim ? 1 : 0); }
__global__ void k_work(int* x) { atomicAdd(x, 1); }
static int try_body(const char* name, int kind) {
  cudaStream_t s; cudaStreamCreate(&s);
  int *cnt, *x, *y; cudaMalloc(&cnt, 4); cudaMalloc(&x, 64); cudaMalloc(&y, 64);
  cudaMemset(cnt, 0, 4); cudaMemset(x, 0, 64);
  cudaGraph_t child;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (kind == 0) k_work<<<1, 32, 0, s>>>(x);
  if (kind == 1) cudaMemsetAsync(x, 0, 64, s);
  if (kind == 2) cudaMemcpyAsync(y, x, 64, cudaMemcpyDeviceToDevice, s);
  if (kind == 3) { void* a[] = {&x}; cudaLaunchCooperativeKernel((void*)k_work, 2, 32, a, 0, s); }
  if (kind == 4) { cudaStream_t s2; cudaStreamCreate(&s2); cudaEvent_t e1, e2; cudaEventCreateWithFlags(&e1, cudaEventDisableTiming); cudaEventCreateWithFlags(&e2, cudaEventDisableTiming);
                   cudaEventRecord(e1, s); cudaStreamWaitEvent(s2, e1); k_work<<<1, 32, 0, s2>>>(x); cudaEventRecord(e2, s2); cudaStreamWaitEvent(s, e2); k_work<<<1,32,0,s>>>(x); }
  cudaStreamEndCapture(s, &child);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t wn; cudaGraphAddNode(&wn, g, nullptr, 0, &cp);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphNode_t cn; cudaError_t e1 = cudaGraphAddChildGraphNode(&cn, body, nullptr, 0, child);
  int lim = 3; void* a2[] = {&h, &cnt, &lim};
  cudaKernelNodeParams dp = {}; dp.func = (void*)k_dec; dp.gridDim = 1; dp.blockDim = 1; dp.kernelParams = a2;
  cudaGraphNode_t dn; cudaGraphAddKernelNode(&dn, body, &cn, 1, &dp);
  cudaGraphExec_t ex; cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
  printf("%-28s addchild=%s instantiate=%s\n", name, cudaGetErrorString(e1), cudaGetErrorString(e2));
  (void)cudaGetLastError();
  return 0;
}
int main() {
  try_body("kernel", 0); try_body("memset", 1); try_body("memcpy d2d", 2); try_body("cooperative kernel", 3);
  try_body("fork/join (events)", 4);
  return 0;
}
