// Single-warp Householder tridiagonalisation (k <= 64 rows per lane pair): no block barriers.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
template <int RT>
__global__ void k_tri1(const double* Tg, int k, long long* prof, double* out) {
  extern __shared__ double sm[];
  const int ld = k | 1;
  double* S = sm;
  const int lane = threadIdx.x;
  for (int j = 0; j < k; ++j)
    for (int i = lane; i < k; i += 32) S[j * ld + i] = 0.5 * (Tg[(size_t)j * k + i] + Tg[(size_t)i * k + j]);
  __syncwarp();
  long long t0 = clock64();
  double dsum = 0.0;
  for (int j = 0; j + 2 < k; ++j) {
    const int j1 = j + 1;
    // norm of column j below j+1
    double s2 = 0.0;
#pragma unroll
    for (int t = 0; t < RT; ++t) { const int i = lane + 32 * t; if (i > j1 && i < k) s2 = fma(S[j * ld + i], S[j * ld + i], s2); }
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const double x0 = S[j * ld + j1];
    const double norm2 = s2 + x0 * x0;
    const double alpha = -copysign(sqrt(norm2), x0);
    const double unorm2 = 2.0 * (norm2 - x0 * alpha);
    if (!(unorm2 > 0.0)) continue;
    const double tj = 2.0 / unorm2, u0 = x0 - alpha;
    double u[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) { const int i = lane + 32 * t; u[t] = (i == j1) ? u0 : (i > j1 && i < k ? S[j * ld + i] : 0.0); }
    __syncwarp();
    if (lane == 0) S[j * ld + j1] = u0;
    // matvec p_i = tau sum_l S[l][i] u_l : lane owns rows i = lane + 32 t
    double p[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) p[t] = 0.0;
    for (int l = j1; l < k; ++l) {
      const double ul = __shfl_sync(0xffffffffu, u[(l >> 5)], l & 31);
      const double* col = S + l * ld;
#pragma unroll
      for (int t = 0; t < RT; ++t) { const int i = lane + 32 * t; if (i >= j1 && i < k) p[t] = fma(col[i], ul, p[t]); }
    }
    double kp = 0.0;
#pragma unroll
    for (int t = 0; t < RT; ++t) { p[t] *= tj; kp = fma(u[t], p[t], kp); }
    for (int o = 16; o > 0; o >>= 1) kp += __shfl_xor_sync(0xffffffffu, kp, o);
    const double K = 0.5 * tj * kp;
    double q[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) q[t] = p[t] - K * u[t];
    // update S[l][i] -= u_i q_l + q_i u_l  (i, l >= j1)
    for (int l = j1; l < k; ++l) {
      const double ul = __shfl_sync(0xffffffffu, u[(l >> 5)], l & 31);
      const double ql = __shfl_sync(0xffffffffu, q[(l >> 5)], l & 31);
      double* col = S + l * ld;
#pragma unroll
      for (int t = 0; t < RT; ++t) { const int i = lane + 32 * t; if (i >= j1 && i < k) col[i] -= u[t] * ql + q[t] * ul; }
    }
    __syncwarp();
    dsum += alpha;
  }
  long long t1 = clock64();
  if (lane == 0) { prof[0] = t1 - t0; out[0] = dsum; }
}
int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 64;
  double* h = (double*)malloc(sizeof(double) * k * k);
  srand(1);
  for (int i = 0; i < k * k; ++i) h[i] = rand() / (double)RAND_MAX - 0.5;
  double *d, *o; long long* p;
  cudaMalloc(&d, sizeof(double) * k * k); cudaMalloc(&o, 64); cudaMalloc(&p, 64);
  cudaMemcpy(d, h, sizeof(double) * k * k, cudaMemcpyHostToDevice);
  size_t shm = sizeof(double) * k * (k | 1);
  long long hp;
  if (k <= 64) {
    cudaFuncSetAttribute(k_tri1<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int r = 0; r < 3; ++r) k_tri1<2><<<1, 32, shm>>>(d, k, p, o);
  } else {
    cudaFuncSetAttribute(k_tri1<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    for (int r = 0; r < 3; ++r) k_tri1<4><<<1, 32, shm>>>(d, k, p, o);
  }
  cudaMemcpy(&hp, p, 8, cudaMemcpyDeviceToHost);
  printf("k=%d single warp: %.0f cycles total, %.0f per step, %.1f us at 1.965 GHz  (%s)\n", k, (double)hp,
         hp / (double)(k - 2), hp / 1965.0, cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
