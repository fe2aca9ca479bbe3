// Latency probes (single warp): dependent DFMA chain, dependent LDS.64 chain, fp64 sqrt and
// division, warp shuffle of a double.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int n, long long* out, double* sink) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 1.0 + 1e-9 * i;
  __syncthreads();
  double a = 1.0 + threadIdx.x * 1e-12, b = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
  long long t1 = clock64();
  int idx = threadIdx.x;
  double acc = 0;
  for (int i = 0; i < n; ++i) { double v = s[idx & 1023]; idx = (int)v + (i & 7); acc += v; }
  long long t2 = clock64();
  double c = 2.0 + threadIdx.x;
  for (int i = 0; i < n; ++i) c = sqrt(c) + 1.0;
  long long t3 = clock64();
  double d = 3.0 + threadIdx.x;
  for (int i = 0; i < n; ++i) d = 7.0 / d + 1.0;
  long long t4 = clock64();
  double e = 1.0 + threadIdx.x;
  for (int i = 0; i < n; ++i) e = __shfl_xor_sync(0xffffffffu, e, 1) + 1.0;
  long long t5 = clock64();
  if (threadIdx.x == 0) {
    out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4;
    sink[0] = a + acc + c + d + e;
  }
}
int main() {
  long long* o; double* sk; cudaMalloc(&o, 64); cudaMalloc(&sk, 64);
  long long h[5];
  const int n = 1000;
  k<<<1, 32>>>(n, o, sk); k<<<1, 32>>>(n, o, sk);
  cudaMemcpy(h, o, 40, cudaMemcpyDeviceToHost);
  const char* nm[5] = {"DFMA dependent", "LDS.64 dependent (+F2I +IADD)", "sqrt(fp64)+1", "7/x+1 (fp64 div)", "shfl double +1"};
  for (int i = 0; i < 5; ++i) printf("%-32s %.1f cycles / iteration\n", nm[i], h[i] / (double)n);
  return 0;
}
