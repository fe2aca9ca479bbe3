// latency of the K5 inner recurrences: pc_fast_div chain, twisted D+ step, Sturm step
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double pc_fast_div(double a, double b) {
  const double ab = fabs(b);
  if (ab > 1e-300 && ab < 1e300) {
    double r = (double)__frcp_rn((float)b);
    r = r * fma(-b, r, 2.0);
    r = r * fma(-b, r, 2.0);
    return a * r;
  }
  return a / b;
}
__global__ void k_lat(const double* d, const double* e2, double* out, long long* cyc, int n) {
  __shared__ double sd[256], se[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { sd[i] = d[i]; se[i] = e2[i]; }
  __syncthreads();
  double q = 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) q = 1.0 + pc_fast_div(0.25, q);
  long long t1 = clock64();
  double q2 = 1.5;
  for (int i = 1; i < 256; ++i) {
    q2 = (sd[i] - 0.3) - pc_fast_div(se[i - 1], q2);
    if (fabs(q2) < 1e-300) q2 = -1e-300;
    out[1024 + i] = q2;
  }
  long long t2 = clock64();
  double p0 = 1.0, p1 = sd[0] - 0.3; int cnt = 0;
  for (int i = 1; i < 256; ++i) {
    const double p2 = fma(sd[i] - 0.3, p1, -se[i - 1] * p0);
    cnt += (int)((unsigned)(__double2hiint(p2) ^ __double2hiint(p1)) >> 31);
    p0 = p1; p1 = p2;
    if ((i & 7) == 0) { const int ex = ilogb(p1); if (ex > 256 || ex < -256) { p0 = ldexp(p0, -ex); p1 = ldexp(p1, -ex); } }
  }
  long long t3 = clock64();
  double x = 1.0;
  for (int i = 0; i < n; ++i) x = (double)(float)x + 1e-3;
  long long t4 = clock64();
  float y = 1.0f;
  for (int i = 0; i < n; ++i) y = __frcp_rn(y) + 1.0f;
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
  out[threadIdx.x] = q + q2 + p1 + cnt + x + y;
}
int main() {
  double *d, *e, *out; long long* cyc;
  cudaMalloc(&d, 2048); cudaMalloc(&e, 2048); cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0 + 0.01 * i;
  cudaMemcpy(d, h, 2048, cudaMemcpyHostToDevice); cudaMemcpy(e, h, 2048, cudaMemcpyHostToDevice);
  for (int threads : {32, 256}) {
    for (int r = 0; r < 2; ++r) { k_lat<<<1, threads>>>(d, e, out, cyc, 1000); cudaDeviceSynchronize(); }
    printf("threads=%d: fast_div chain %.1f, twisted D+ step %.1f, sturm step %.1f, f64->f32->f64 %.1f, frcp.f32 chain %.1f cycles\n",
           threads, cyc[0] / 1000.0, cyc[1] / 255.0, cyc[2] / 255.0, cyc[3] / 1000.0, cyc[4] / 1000.0);
  }
  return 0;
}
