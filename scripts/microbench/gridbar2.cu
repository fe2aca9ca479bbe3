// grid barrier variants, 148 co-resident CTAs (cycles per barrier, CTA 0's clock)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_bar(unsigned* cnt, int steps, int mode, long long* out) {
  const unsigned G = gridDim.x;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)(s + 1) * G;
      if (mode == 0) {            // red.release + ld.acquire poll (current K3)
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned g;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(cnt) : "memory"); } while (g < target);
      } else if (mode == 1) {     // fence + relaxed red; relaxed poll + fence
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned g;
        do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(cnt) : "memory"); } while (g < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else if (mode == 2) {     // as 0 with nanosleep backoff in the poll
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(cnt) : "memory");
        unsigned g;
        while (true) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(cnt) : "memory");
          if (g >= target) break;
          __nanosleep(32);
        }
      } else {                     // atom.add returning (arrival order); last arriver flips a flag
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
        volatile unsigned* flag = cnt + 32;
        if (old == target - 1) {
          asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(cnt + 32), "r"((unsigned)(s + 1)) : "memory");
        } else {
          unsigned f;
          do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(cnt + 32) : "memory"); } while (f < (unsigned)(s + 1));
        }
        (void)flag;
      }
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = clock64() - t0;
}
int main() {
  unsigned* cnt; long long* out;
  cudaMalloc(&cnt, 256); cudaMallocManaged(&out, 16);
  const char* nm[] = {"red.release + ld.acquire poll", "fence + relaxed red/poll + fence", "acquire poll + nanosleep(32)",
                      "atom.acq_rel + last-arriver flag"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaMemset(cnt, 0, 256);
      int steps = 200, G = 148, threads = 256;
      void* a[] = {&cnt, &steps, &mode, &out};
      cudaLaunchCooperativeKernel((void*)k_bar, G, threads, a, 0, 0);
      cudaDeviceSynchronize();
    }
    printf("%-36s %.0f cycles/barrier\n", nm[mode], out[0] / 200.0);
  }
  return 0;
}
