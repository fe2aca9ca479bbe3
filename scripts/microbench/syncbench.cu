// Latency probes for single-CTA sequential kernels (K5 design): barrier, fp64 divide,
// shared-memory update + barrier.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_sync(int n, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}
__global__ void k_div(int n, long long* out, double* sink) {
  __shared__ double s[1024];
  s[threadIdx.x] = 1.0 + threadIdx.x;
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const double d = s[i & 511];
    const double inv = 1.0 / d;
    acc += inv;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink[0] = acc; }
}
__global__ void k_upd(int n, int k, long long* out, double* sink) {
  extern __shared__ double S[];
  const int ld = k | 1;
  for (int e = threadIdx.x; e < k * ld; e += blockDim.x) S[e] = 1.0 + (e % 7);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
    const int j = it % (k - 1);
    const double inv = 1.0 / S[j * ld + j];
    for (int c = j + 1 + warp; c < k; c += nw) {
      const double lc = S[j * ld + c] * inv;
      for (int i = c + lane; i < k; i += 32) S[c * ld + i] -= S[j * ld + i] * lc * 1e-9;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = t1 - t0; sink[0] = S[5]; }
}
int main() {
  long long* o; double* sk;
  cudaMalloc(&o, 64); cudaMalloc(&sk, 64);
  long long h;
  for (int t : {128, 512, 1024}) {
    k_sync<<<1, t>>>(1000, o); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d: __syncthreads %.1f cycles\n", t, h / 1000.0);
    k_div<<<1, t>>>(1000, o, sk); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("threads %4d: fp64 div + sync %.1f cycles\n", t, h / 1000.0);
    for (int k : {32, 64, 128}) {
      size_t shm = (size_t)k * (k | 1) * 8;
      cudaFuncSetAttribute(k_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      k_upd<<<1, t, shm>>>(1000, k, o, sk); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
      printf("threads %4d k %3d: chol-like step %.1f cycles\n", t, k, h / 1000.0);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
