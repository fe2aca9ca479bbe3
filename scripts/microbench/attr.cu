#include <cstdio>
#include <cuda_runtime.h>
#include <dlfcn.h>
int main(int argc, char** argv) {
  void* h = dlopen(argv[1], RTLD_NOW);
  if (!h) { printf("dlopen failed %s\n", dlerror()); return 1; }
  for (int i = 2; i < argc; ++i) {
    void* f = dlsym(h, argv[i]);
    if (!f) { printf("no symbol %s\n", argv[i]); continue; }
    cudaFuncAttributes a;
    cudaError_t e = cudaFuncGetAttributes(&a, f);
    printf("%s: %s regs %d maxThreads %d shared %zu local %zu\n", argv[i], cudaGetErrorString(e), a.numRegs,
           a.maxThreadsPerBlock, a.sharedSizeBytes, a.localSizeBytes);
  }
  return 0;
}
