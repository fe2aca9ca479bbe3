// latency microbenchmarks: dependent DFMA / FFMA chains, double shuffles, __syncthreads
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, int n, double a, double b) {
  double x = threadIdx.x * 1e-3;
  float xf = (float)x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, (float)a, (float)b);
  long long t2 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y += __shfl_xor_sync(0xffffffffu, y, 1);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t4 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = sqrt(z + 1.0);
  long long t5 = clock64();
  double w = x + 1.0;
  for (int i = 0; i < n; ++i) w = 1.0 / (w + 1.0);
  long long t6 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  out[threadIdx.x] = x + xf + y + z + w;
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMallocManaged(&cyc, 64);
  const char* nm[] = {"dfma chain", "ffma chain", "shfl.f64+add chain", "__syncthreads", "sqrt(f64) chain", "1/x f64 chain"};
  for (int threads : {32, 512}) {
    for (int rep = 0; rep < 2; ++rep) { k_lat<<<1, threads>>>(out, cyc, 1000, 0.999, 1e-3); cudaDeviceSynchronize(); }
    printf("threads=%d\n", threads);
    for (int i = 0; i < 6; ++i) printf("  %-22s %.1f cycles\n", nm[i], cyc[i] / 1000.0);
  }
  return 0;
}
