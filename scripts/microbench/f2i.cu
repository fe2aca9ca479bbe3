// throughput of the K7z digit conversion: F2I.S64 (float -> s64) vs bf16 bit manipulation
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k_f2i(const uint32_t* in, unsigned long long* out, long long* cyc, int n, float sc) {
  uint32_t w[8];
  for (int u = 0; u < 8; ++u) w[u] = in[(threadIdx.x + u) & 255];
  unsigned long long acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float x = __uint_as_float((w[u] & 0xffff0000u) ^ (uint32_t)(i << 16));
      acc += (unsigned long long)__float2ll_rz(x * sc) + 0x808080808080ull;
    }
  }
  long long t1 = clock64();
  unsigned long long acc2 = 0;
  const int T = 3;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t b = ((w[u] >> 16) ^ (uint32_t)i) & 0xffffu;          // bf16 bits
      const uint32_t e = (b >> 7) & 0xffu, m = b & 0x7fu;
      const uint32_t mant = e ? (m | 0x80u) : m;
      const int sh = (int)(e ? e : 1u) - 88 - T;
      unsigned long long t = sh >= 0 ? ((unsigned long long)mant << sh) : (unsigned long long)(mant >> min(-sh, 31));
      if (b & 0x8000u) t = 0ull - t;
      acc2 += t + 0x808080808080ull;
    }
  }
  long long t2 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
  out[threadIdx.x] = acc + acc2;
}
int main() {
  uint32_t* in; unsigned long long* out; long long* cyc;
  cudaMalloc(&in, 1024); cudaMalloc(&out, 8 * 1024); cudaMallocManaged(&cyc, 16);
  cudaMemset(in, 0x3f, 1024);
  for (int threads : {128, 512}) {
    for (int r = 0; r < 2; ++r) { k_f2i<<<1, threads>>>(in, out, cyc, 1000, 1024.0f); cudaDeviceSynchronize(); }
    const double per = 8.0 * threads * 1000;
    printf("threads=%d: F2I.S64 path %.3f cycles/elem/SM, integer path %.3f cycles/elem/SM\n", threads,
           cyc[0] / per, cyc[1] / per);
  }
  return 0;
}
