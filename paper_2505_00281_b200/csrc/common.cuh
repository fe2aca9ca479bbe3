// common.cuh -- format codes, exact-rounding helpers and sm_100a PTX wrappers
// (mbarrier, TMA, tcgen05) shared by the OFRR B200 kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_fp8.h>
#include <stdint.h>
#include <atomic>
#include "../../include/ofrr_b200.h"

namespace ofrr {

// Format codes: ofrr/precision.py:20-25 (F16=0, F32=1, F64=2) + BF16=3, FP8_E4M3=4.
enum Fmt : int { F16 = OFRR_F16, F32 = OFRR_F32, F64 = OFRR_F64, BF16 = OFRR_BF16, FP8 = OFRR_FP8E4M3 };

__host__ __device__ inline int fmt_bytes(int f) {
  return f == F64 ? 8 : f == F32 ? 4 : f == FP8 ? 1 : 2;
}

// ---------------------------------------------------------------------------------
// Exact rounding into a format, mirroring ofrr/halfround.h (RNE, overflow -> inf,
// subnormals kept).  A double is rounded to binary16/bfloat16 via binary32, which is
// exact by the 2p+2 bound (ofrr/halfround.h:4-9).  FP8 e4m3 has no inf; values that
// round beyond 448 are reported as +-inf so the overflow diagnostic fires.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ float rnd_f16f(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ float rnd_bf16f(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
__device__ __forceinline__ float rnd_fp8f(float x) {
  if (x != x) return x;
  if (fabsf(x) > 464.0f) return copysignf(INFINITY, x);  // > 464 rounds past 448 (464 ties to 448)
  __nv_fp8_e4m3 v(x);  // RNE, satfinite
  return float(v);
}
__device__ __forceinline__ double rnd(double x, int f) {
  switch (f) {
    case F64: return x;
    case F32: return (double)__double2float_rn(x);
    case F16: return (double)rnd_f16f(__double2float_rn(x));
    case BF16: return (double)rnd_bf16f(__double2float_rn(x));
    default: return (double)rnd_fp8f(__double2float_rn(x));
  }
}
// float-input variant (x already representable in f32)
__device__ __forceinline__ float rndf(float x, int f) {
  switch (f) {
    case F16: return rnd_f16f(x);
    case BF16: return rnd_bf16f(x);
    case FP8: return rnd_fp8f(x);
    default: return x;
  }
}

// Typed load / store of one element of format f (as double).
__device__ __forceinline__ double ld_fmt(const void* p, long i, int f) {
  switch (f) {
    case F64: return ((const double*)p)[i];
    case F32: return (double)((const float*)p)[i];
    case F16: return (double)__half2float(((const __half*)p)[i]);
    case BF16: return (double)__bfloat162float(((const __nv_bfloat16*)p)[i]);
    default: { __nv_fp8_e4m3 v; v.__x = ((const __nv_fp8_storage_t*)p)[i]; return (double)float(v); }
  }
}
// Stores a value that is already representable in f (exact conversion).
__device__ __forceinline__ void st_fmt(void* p, long i, int f, double v) {
  switch (f) {
    case F64: ((double*)p)[i] = v; break;
    case F32: ((float*)p)[i] = (float)v; break;
    case F16: ((__half*)p)[i] = __float2half_rn((float)v); break;
    case BF16: ((__nv_bfloat16*)p)[i] = __float2bfloat16_rn((float)v); break;
    default: {
      float fv = (float)v;
      __nv_fp8_e4m3 q(fv);
      if (isinf(fv)) q.__x = fv > 0 ? 0x7e : 0xfe;  // saturate storage; flag carries the overflow
      ((__nv_fp8_storage_t*)p)[i] = q.__x;
    }
  }
}

// element <-> double for the storage types (exact for representable values)
__device__ __forceinline__ double to_d(double x) { return x; }
__device__ __forceinline__ double to_d(float x) { return (double)x; }
__device__ __forceinline__ double to_d(__half x) { return (double)__half2float(x); }
__device__ __forceinline__ double to_d(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
__device__ __forceinline__ double to_d(__nv_fp8_e4m3 x) { return (double)float(x); }
template <typename T> __device__ __forceinline__ T from_d(double v);
template <> __device__ __forceinline__ double from_d<double>(double v) { return v; }
template <> __device__ __forceinline__ float from_d<float>(double v) { return (float)v; }
template <> __device__ __forceinline__ __half from_d<__half>(double v) { return __float2half_rn((float)v); }
template <> __device__ __forceinline__ __nv_bfloat16 from_d<__nv_bfloat16>(double v) { return __float2bfloat16_rn((float)v); }

// Compute-format arithmetic (exactly one rounding per op into format c), used by the
// elementwise steps that the reference rounds explicitly: ofrr/precision.py:159-180.
__device__ __forceinline__ double c_div(double a, double b, int c) {
  if (c == F64) return __ddiv_rn(a, b);
  return rnd((double)__fdiv_rn((float)a, (float)b), c);  // f32 division; f16/bf16 via f32 (2p+2)
}
__device__ __forceinline__ double c_mul(double a, double b, int c) {
  if (c == F64) return __dmul_rn(a, b);
  return rnd((double)__fmul_rn((float)a, (float)b), c);
}
__device__ __forceinline__ double c_sub(double a, double b, int c) {
  if (c == F64) return __dsub_rn(a, b);
  return rnd((double)__fsub_rn((float)a, (float)b), c);
}

// ---------------------------------------------------------------------------------
// PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1,
                                            uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// multicast to the CTAs of ctaMask in the cluster: same smem offset and mbarrier offset in
// each destination CTA
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar,
                                               uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5, %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "h"(mask), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tm)) : "memory");
}

// tcgen05 -------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
// commit arriving on the mbarrier at this offset in every CTA of ctaMask
__device__ __forceinline__ void tc_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16/fp16 inputs, fp32 accumulate)
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// kind::f8f6f4 (e4m3 inputs, fp32 accumulate)
__device__ __forceinline__ void mma_f8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 ld_shared_v2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
// Warp-wide issue: the whole warp runs the issue loop and one elected lane issues.  With the
// warp index made visibly warp-uniform (warp_index() below) ptxas keeps the descriptors in
// uniform registers and emits back-to-back UTC*MMA; issuing from `if (lane == 0)` instead wraps
// every MMA in a per-lane waterfall (ELECT + five R2UR + branch) -- the issuing thread, not the
// tensor pipe, then paces a kernel whose MMAs are short.
__device__ __forceinline__ int warp_index() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }
#define OFRR_MMA_WS(NAME, KIND)                                                                  \
  __device__ __forceinline__ void NAME(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, \
                                       uint32_t accumulate) {                                       \
    asm volatile(                                                                                   \
        "{\n\t.reg .pred p, e;\n\t"                                                               \
        "elect.sync _|e, 0xffffffff;\n\t"                                                          \
        "setp.ne.b32 p, %4, 0;\n\t"                                                                \
        "@e tcgen05.mma.cta_group::1.kind::" KIND " [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),      \
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));                                        \
  }
OFRR_MMA_WS(mma_f16_ws, "f16")
OFRR_MMA_WS(mma_f8_ws, "f8f6f4")
OFRR_MMA_WS(mma_i8_ws, "i8")
#undef OFRR_MMA_WS
__device__ __forceinline__ void tc_commit_ws(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc_ws(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B apart
// (SBO), version 1 (Blackwell), base offset 0 (stage buffers are 1024 B aligned).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// order-preserving max of non-negative floats via their bit patterns
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
}
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace ofrr

// error plumbing shared by all translation units
void ofrr_set_error(const char* fmt, ...);
#define OFRR_CUDA_TRY(expr)                                                              \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      ofrr_set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
      return OFRR_ERR_CUDA;                                                              \
    }                                                                                    \
  } while (0)
#define OFRR_CHECK_LAUNCH()                                                                   \
  do {                                                                                        \
    cudaError_t _e = cudaGetLastError();                                                      \
    if (_e != cudaSuccess) {                                                                  \
      ofrr_set_error("%s:%d kernel launch: %s", __FILE__, __LINE__, cudaGetErrorString(_e)); \
      return OFRR_ERR_CUDA;                                                                   \
    }                                                                                         \
  } while (0)
