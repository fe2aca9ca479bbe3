// variants of the K5 recurrences (latency per step, one thread's clock)
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_approx(double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  return r;
}
__device__ __forceinline__ double div_nr(double a, double b) {   // MUFU.RCP64H + 2 Newton
  double r = rcp_approx(b);
  r = fma(r, fma(-b, r, 1.0), r);
  r = fma(r, fma(-b, r, 1.0), r);
  return a * r;
}
__global__ void k_lat(const double* d, const double* e2, double* out, long long* cyc, int n) {
  __shared__ double sd[256], se[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) { sd[i] = d[i]; se[i] = e2[i]; }
  __syncthreads();
  long long t[8];
  double q = 1.5;
  t[0] = clock64();
  for (int i = 0; i < n; ++i) q = 1.0 + 0.25 / q;                       // IEEE div
  t[1] = clock64();
  double q1 = 1.5;
  for (int i = 0; i < n; ++i) q1 = 1.0 + div_nr(0.25, q1);              // rcp.approx.f64 + NR
  t[2] = clock64();
  // sturm, no rescale
  double p0 = 1.0, p1 = sd[0] - 0.3; int cnt = 0;
#pragma unroll 8
  for (int i = 1; i < 256; ++i) {
    const double p2 = fma(sd[i] - 0.3, p1, -se[i - 1] * p0);
    cnt += (int)((unsigned)(__double2hiint(p2) ^ __double2hiint(p1)) >> 31);
    p0 = p1; p1 = p2;
  }
  t[3] = clock64();
  // sturm with integer exponent check every 8
  double r0 = 1.0, r1 = sd[0] - 0.3; int cnt2 = 0;
  for (int i = 1; i + 8 <= 256; i += 8) {
    double dx[8], ee[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { dx[u] = sd[i + u] - 0.3; ee[u] = se[i + u - 1]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double r2 = fma(dx[u], r1, -ee[u] * r0);
      cnt2 += (int)((unsigned)(__double2hiint(r2) ^ __double2hiint(r1)) >> 31);
      r0 = r1; r1 = r2;
    }
    const int ex = ((__double2hiint(r1) >> 20) & 0x7ff) - 1023;
    if (ex > 256 || ex < -256) {
      const double sc = __hiloint2double((1023 - ex) << 20, 0);
      r0 *= sc; r1 *= sc;
    }
  }
  t[4] = clock64();
  // LDS-dependent loop (no unroll): load + add chain
  double s = 0.0;
  for (int i = 0; i < 255; ++i) s = s * 0.5 + sd[i];
  t[5] = clock64();
  if (threadIdx.x == 0) for (int j = 0; j < 5; ++j) cyc[j] = t[j + 1] - t[j];
  out[threadIdx.x] = q + q1 + p1 + cnt + r1 + cnt2 + s;
}
int main() {
  double *d, *e, *out; long long* cyc;
  cudaMalloc(&d, 2048); cudaMalloc(&e, 2048); cudaMalloc(&out, 4096 * 8); cudaMallocManaged(&cyc, 64);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = 1.0 + 0.01 * i;
  cudaMemcpy(d, h, 2048, cudaMemcpyHostToDevice); cudaMemcpy(e, h, 2048, cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) { k_lat<<<1, 32>>>(d, e, out, cyc, 1000); cudaDeviceSynchronize(); }
  printf("IEEE f64 div chain %.1f | rcp.approx.f64+2NR chain %.1f | sturm (no rescale, unroll 8) %.1f | sturm (int exp check) %.1f | lds+dfma chain %.1f cycles/step\n",
         cyc[0] / 1000.0, cyc[1] / 1000.0, cyc[2] / 255.0, cyc[3] / 255.0, cyc[4] / 255.0);
  return 0;
}
