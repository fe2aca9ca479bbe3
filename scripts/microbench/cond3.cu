// device-loop graph shapes: unused handle, nested IF in WHILE setting the outer handle
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_set(cudaGraphConditionalHandle h, int v) { cudaGraphSetConditional(h, v); }
__global__ void k_dec(cudaGraphConditionalHandle hl, cudaGraphConditionalHandle hr, int* cnt, int lim) {
  int c = ++(*cnt); cudaGraphSetConditional(hr, 1); cudaGraphSetConditional(hl, c < lim ? 1 : 0); }
__global__ void k_conf(cudaGraphConditionalHandle hl, int* cnt, int* rep) { ++(*rep); if (*cnt >= 2) cudaGraphSetConditional(hl, 0); }
static void test(int unused_handle, int nested) {
  int *cnt, *rep; cudaMallocManaged(&cnt, 4); cudaMallocManaged(&rep, 4); *cnt = 0; *rep = 0;
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle hl, hu, hr; cudaGraphConditionalHandleCreate(&hl, g, 0, cudaGraphCondAssignDefault);
  cudaGraphNode_t n0; cudaKernelNodeParams kp = {}; int one = 1;
  if (unused_handle) cudaGraphConditionalHandleCreate(&hu, g, 0, cudaGraphCondAssignDefault);
  void* a0[] = {&hl, &one}; kp.func = (void*)k_set; kp.gridDim = 1; kp.blockDim = 1; kp.kernelParams = a0;
  cudaGraphAddKernelNode(&n0, g, nullptr, 0, &kp);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hl;
  cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t wn; cudaGraphAddNode(&wn, g, &n0, 1, &cp);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphConditionalHandleCreate(&hr, body, 0, cudaGraphCondAssignDefault);
  int lim = 4; void* a1[] = {&hl, &hr, &cnt, &lim};
  cudaGraphNode_t dn; kp.func = (void*)k_dec; kp.kernelParams = a1; cudaGraphAddKernelNode(&dn, body, nullptr, 0, &kp);
  if (nested) {
    cudaGraphNodeParams ip = {}; ip.type = cudaGraphNodeTypeConditional; ip.conditional.handle = hr;
    ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
    cudaGraphNode_t in; cudaError_t e = cudaGraphAddNode(&in, body, &dn, 1, &ip);
    cudaGraph_t rb = ip.conditional.phGraph_out[0];
    void* a2[] = {&hl, &cnt, &rep}; cudaGraphNode_t cn; kp.func = (void*)k_conf; kp.kernelParams = a2;
    cudaGraphAddKernelNode(&cn, rb, nullptr, 0, &kp);
    if (e) printf("add if: %s\n", cudaGetErrorString(e));
  }
  cudaGraphExec_t ex; cudaError_t e2 = cudaGraphInstantiate(&ex, g, 0);
  if (!e2) { cudaGraphLaunch(ex, 0); cudaDeviceSynchronize(); }
  printf("unused_handle=%d nested=%d: instantiate=%s cnt=%d rep=%d\n", unused_handle, nested, cudaGetErrorString(e2), *cnt, *rep);
  (void)cudaGetLastError();
}
int main() { test(0, 0); test(1, 0); test(0, 1); test(1, 1); return 0; }
