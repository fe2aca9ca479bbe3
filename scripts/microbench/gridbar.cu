// Grid-wide per-step exchange patterns of the Hessenberg kernel (148 co-resident CTAs):
//  A: atomicMax key + red.release counter, poll, read key, read winner row (current K3)
//  B: per-CTA tagged slots (plain stores + st.release), warp polls all slots, read row
//  C: like B without the row read (poll + fold only)
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ void st_rel(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__global__ void k_A(unsigned* cnt, unsigned long long* key, double* rows, int k, int steps, long long* out) {
  const int G = gridDim.x, c = blockIdx.x;
  __shared__ double prow[256];
  __shared__ unsigned long long skey;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) rows[((size_t)(s & 1) * G + c) * k + i] = s + c + i;
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicMax(&key[s], (unsigned long long)((c * 7919u) % 1000u) << 32 | c);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned g;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(cnt) : "memory"); } while (g < (unsigned)(s + 1) * G);
    }
    __syncthreads();
    if (threadIdx.x == 0) skey = __ldcg(&key[s]);
    __syncthreads();
    const int owner = (int)(skey & 0xffffffffu);
    for (int i = threadIdx.x; i < k; i += blockDim.x) prow[i] = __ldcg(&rows[((size_t)(s & 1) * G + owner) * k + i]);
    __syncthreads();
  }
  if (c == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  if (prow[0] < -1) out[1] = 1;
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v;
}
// barrier only: red.release + poll (mode 0), + atomicMax/key read (mode 1)
__global__ void k_bar(unsigned* cnt, unsigned long long* key, int steps, int mode, long long* out) {
  const int G = gridDim.x, c = blockIdx.x;
  __shared__ unsigned long long skey;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (mode == 1) atomicMax(&key[s], (unsigned long long)c);
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
      unsigned g;
      do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(cnt) : "memory"); } while (g < (unsigned)(s + 1) * G);
      if (mode == 1) skey = __ldcg(&key[s]);
    }
    __syncthreads();
  }
  if (c == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  if (skey == 12345) out[1] = 1;
}
__global__ void k_C(unsigned long long* slot, double* rows, int k, int steps, int readrow, long long* out) {
  const int G = gridDim.x, c = blockIdx.x;
  __shared__ double prow[256];
  __shared__ int sown;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int b = s & 1;
    for (int i = threadIdx.x; i < k; i += blockDim.x) rows[((size_t)b * G + c) * k + i] = s + c + i;
    __syncthreads();
    const unsigned long long tag = (unsigned long long)(s + 1) << 48;
    if (threadIdx.x == 0) st_rel(&slot[b * G + c], tag | ((unsigned long long)((c * 7919u + s) % 1000u) << 16) | c);
    if (threadIdx.x < 32) {
      unsigned long long v[5];
      bool done;
      do {
        done = true;
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const int q = threadIdx.x + 32 * u;
          v[u] = q < G ? ld_rlx(&slot[b * G + q]) : tag;
          if ((v[u] >> 48) != (unsigned long long)(s + 1)) done = false;
        }
        done = __all_sync(0xffffffffu, done);
      } while (!done);
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      unsigned long long best = 0;
#pragma unroll
      for (int u = 0; u < 5; ++u) { const unsigned long long kk = (threadIdx.x + 32 * u < G) ? (v[u] & 0xffffffffffffull) : 0; best = kk > best ? kk : best; }
      for (int o = 16; o > 0; o >>= 1) { const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o); best = x > best ? x : best; }
      if (threadIdx.x == 0) sown = (int)(best & 0xffff);
    }
    __syncthreads();
    if (readrow) {
      const int owner = sown;
      for (int i = threadIdx.x; i < k; i += blockDim.x) prow[i] = __ldcg(&rows[((size_t)b * G + owner) * k + i]);
      __syncthreads();
    }
  }
  if (c == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  if (prow[0] < -1) out[1] = 1;
}
__global__ void k_cg(int steps, long long* out) {
  cooperative_groups::grid_group g = cooperative_groups::this_grid();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) g.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}
__global__ void k_B(unsigned long long* slot, double* rows, int k, int steps, int readrow, long long* out) {
  const int G = gridDim.x, c = blockIdx.x;
  __shared__ double prow[256];
  __shared__ int sown;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int b = s & 1;
    for (int i = threadIdx.x; i < k; i += blockDim.x) rows[((size_t)b * G + c) * k + i] = s + c + i;
    __syncthreads();
    const unsigned long long tag = (unsigned long long)(s + 1) << 48;
    if (threadIdx.x == 0) st_rel(&slot[b * G + c], tag | ((unsigned long long)((c * 7919u + s) % 1000u) << 16) | c);
    if (threadIdx.x < 32) {
      unsigned long long best = 0;
      bool done;
      do {
        done = true;
        best = 0;
        for (int q = threadIdx.x; q < G; q += 32) {
          const unsigned long long v = ld_acq(&slot[b * G + q]);
          if ((v >> 48) != (unsigned long long)(s + 1)) done = false;
          const unsigned long long kk = v & 0xffffffffffffull;
          best = kk > best ? kk : best;
        }
        done = __all_sync(0xffffffffu, done);
      } while (!done);
      for (int o = 16; o > 0; o >>= 1) { const unsigned long long x = __shfl_xor_sync(0xffffffffu, best, o); best = x > best ? x : best; }
      if (threadIdx.x == 0) sown = (int)(best & 0xffff);
    }
    __syncthreads();
    if (readrow) {
      const int owner = sown;
      for (int i = threadIdx.x; i < k; i += blockDim.x) prow[i] = __ldcg(&rows[((size_t)b * G + owner) * k + i]);
      __syncthreads();
    }
  }
  if (c == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
  if (prow[0] < -1) out[1] = 1;
}
int main() {
  int k = 64, steps = 200;
  unsigned* cnt; unsigned long long *key; long long* out;
  cudaMalloc(&cnt, 4); cudaMalloc(&key, 8 * steps); cudaMallocManaged(&out, 16);
  for (int G : {8, 16, 32, 64, 96, 128, 148}) {
    for (int mode = 0; mode < 2; ++mode) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(cnt, 0, 4); cudaMemset(key, 0, 8 * steps);
        int threads = 256;
        void* a[] = {&cnt, &key, &steps, &mode, &out};
        cudaLaunchCooperativeKernel((void*)k_bar, G, threads, a, 0, 0); cudaDeviceSynchronize();
      }
      printf("G=%3d barrier%s: %.0f cycles/step\n", G, mode ? " + atomicMax + key read" : "", out[0] / (double)steps);
    }
  }
  (void)k;
  return 0;
}
