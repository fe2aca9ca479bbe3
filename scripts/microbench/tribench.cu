// Phase timing of one Householder tridiagonalisation step loop (the k_pc_tri phase 1 code,
// PT threads, k x (k|1) fp64 matrix in shared memory), thread 0's clock at 8 points.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#ifndef PT
#define PT 512
#endif
static constexpr int PNW = PT / 32;
static constexpr int PK_MAX = 160;
__global__ void __launch_bounds__(PT, 1) k_tri(const double* Tg, int k, long long* prof, double* out) {
  extern __shared__ double sm[];
  __shared__ double red[PNW];
  __shared__ double pv[PK_MAX];
  __shared__ double s_norm2;
  const int ld = k | 1;
  double* S = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int quad = threadIdx.x >> 2, ql = threadIdx.x & 3;
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) S[j * ld + i] = 0.5 * (Tg[(size_t)j * k + i] + Tg[(size_t)i * k + j]);
  __syncthreads();
  if (warp == 0) {
    double s2 = 0.0;
    for (int i = 1 + lane; i < k; i += 32) s2 = fma(S[i], S[i], s2);
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) s_norm2 = s2;
  }
  __syncthreads();
  long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int j = 0; j + 2 < k; ++j) {
    long long t0 = clock64();
    const double norm2 = s_norm2;
    const double x0 = S[j * ld + j + 1];
    const double alpha = -copysign(sqrt(norm2), x0);
    const double unorm2 = 2.0 * (norm2 - x0 * alpha);
    const bool skip = !(unorm2 > 0.0) || norm2 == 0.0;
    const double tj = skip ? 0.0 : 2.0 / unorm2;
    const double u0 = x0 - alpha;
    const int j1 = j + 1;
    long long t1 = clock64();
    long long t2 = t1;
    if (!skip) {
      for (int r0 = 0; r0 < k - j1; r0 += PT / 4) {
        const int i = j1 + r0 + quad;
        double sum = 0.0;
        if (i < k) {
          // symmetric: row i of the trailing block = column i, contiguous over l
          const double* ci = S + i * ld;
          const double* uj = S + j * ld;
          double a0 = ql == 0 ? ci[j1] * u0 : 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int l = j1 + 1 + 4 * ql;
          // quad lanes take 4 consecutive l each (16 per quad row), contiguous reads
          for (; l + 3 < k; l += 16) {
            a0 = fma(ci[l], uj[l], a0);
            a1 = fma(ci[l + 1], uj[l + 1], a1);
            a2 = fma(ci[l + 2], uj[l + 2], a2);
            a3 = fma(ci[l + 3], uj[l + 3], a3);
          }
          for (int ll = l; ll < k && ll < l + 4; ++ll) a0 = fma(ci[ll], uj[ll], a0);
          sum = (a0 + a1) + (a2 + a3);
        }
        t2 = clock64();
        sum += __shfl_xor_sync(0xffffffffu, sum, 1);
        sum += __shfl_xor_sync(0xffffffffu, sum, 2);
        double kp = 0.0;
        if (i < k) {
          const double pi = tj * sum;
          if (ql == 0) pv[i] = pi;
          kp = ql == 0 ? (i == j1 ? u0 : S[j * ld + i]) * pi : 0.0;
        }
        kp += __shfl_xor_sync(0xffffffffu, kp, 4);
        kp += __shfl_xor_sync(0xffffffffu, kp, 8);
        kp += __shfl_xor_sync(0xffffffffu, kp, 16);
        if (lane == 0) red[warp] = (r0 == 0 ? 0.0 : red[warp]) + kp;
      }
    }
    long long t3 = clock64();
    __syncthreads();
    long long t4 = clock64();
    if (threadIdx.x == 0 && !skip) S[j * ld + j1] = u0;
    long long t5 = t4, t6 = t4;
    if (!skip) {
      double ksum = 0.0;
      for (int w = 0; w < PNW; ++w) ksum += red[w];
      const double K = 0.5 * tj * ksum;
      constexpr int RT = (PK_MAX + 31) / 32;
      double ur[RT], qr[RT];
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = j1 + lane + 32 * t;
        ur[t] = i < k ? (i == j1 ? u0 : S[j * ld + i]) : 0.0;
        qr[t] = i < k ? pv[i] - K * ur[t] : 0.0;
      }
      t5 = clock64();
      for (int l = j1 + warp; l < k; l += PNW) {
        const double ul = l == j1 ? u0 : S[j * ld + l];
        const double qlv = pv[l] - K * ul;
        double* col = S + l * ld;
        double v[RT];
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j1 + lane + 32 * t;
          v[t] = i < k ? col[i] : 0.0;
        }
        double s2 = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j1 + lane + 32 * t;
          if (i < k) {
            const double nv = v[t] - (ur[t] * qlv + qr[t] * ul);
            col[i] = nv;
            if (i > l) s2 = fma(nv, nv, s2);
          }
        }
        if (l == j1) {
          for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          if (lane == 0) s_norm2 = s2;
        }
      }
      t6 = clock64();
    }
    __syncthreads();
    long long t7 = clock64();
    acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2; acc[3] += t4 - t3; acc[4] += t5 - t4;
    acc[5] += t6 - t5; acc[6] += t7 - t6; acc[7] += t7 - t0;
  }
  if (threadIdx.x == 0) for (int i = 0; i < 8; ++i) prof[i] = acc[i];
  for (int i = threadIdx.x; i < k * ld; i += PT) out[i] = S[i];
}
int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 64;
  double* h = (double*)malloc(sizeof(double) * k * k);
  srand(1);
  for (int i = 0; i < k * k; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  double *d, *o; long long* p;
  cudaMalloc(&d, sizeof(double) * k * k); cudaMalloc(&o, sizeof(double) * k * (k | 1)); cudaMalloc(&p, 64);
  cudaMemcpy(d, h, sizeof(double) * k * k, cudaMemcpyHostToDevice);
  size_t shm = sizeof(double) * k * (k | 1);
  cudaFuncSetAttribute(k_tri, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int r = 0; r < 3; ++r) k_tri<<<1, PT, shm>>>(d, k, p, o);
  long long hp[8];
  cudaMemcpy(hp, p, 64, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"tau", "matvec loop", "shuffles+K partial", "sync A", "ksum+preload", "update cols", "sync B", "total"};
  printf("k=%d PT=%d (cycles per step, thread 0)\n", k, PT);
  for (int i = 0; i < 8; ++i) printf("  %-20s %8.0f\n", nm[i], hp[i] / (double)(k - 2));
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
