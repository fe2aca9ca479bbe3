// throughput microbenchmarks: independent DFMA / FFMA per warp, LDS.64, with 1 and 16 warps
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_thr(double* out, long long* cyc, int n, double a, double b) {
  __shared__ double sh[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sh[i] = i * 1e-3;
  __syncthreads();
  double x[8];
  float y[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) { x[u] = threadIdx.x * 1e-3 + u; y[u] = (float)x[u]; }
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, b);
  }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) y[u] = fmaf(y[u], (float)a, (float)b);
  }
  long long t2 = clock64();
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) s += sh[(threadIdx.x + 32 * u + i) & 2047];
  }
  long long t3 = clock64();
  double z[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) z[u] = x[u];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) z[u] = z[u] * a;
  }
  long long t4 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  double r = s;
#pragma unroll
  for (int u = 0; u < 8; ++u) r += x[u] + y[u] + z[u];
  out[threadIdx.x] = r;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  const char* nm[] = {"8 indep DFMA", "8 indep FFMA", "8 LDS.64 (+DADD)", "8 indep DMUL"};
  for (int threads : {32, 128, 512}) {
    for (int rep = 0; rep < 2; ++rep) { k_thr<<<1, threads>>>(out, cyc, 1000, 0.999, 1e-3); cudaDeviceSynchronize(); }
    printf("threads=%d (cycles per iteration of 8 ops, thread 0)\n", threads);
    for (int i = 0; i < 4; ++i) printf("  %-22s %.1f\n", nm[i], cyc[i] / 1000.0);
  }
  return 0;
}
