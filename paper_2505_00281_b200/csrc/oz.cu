// oz.cu -- K7z: FP64-accurate A * V for a 16/8-bit operator on the int8 tensor cores
// (Ozaki scheme: error-free integer slices, exact int32 accumulation).
//
// Replaces the FP64 product inside the reference's residual report
// (ofrr/projection.py:136-147: A @ v in numpy float64 on to_dense_f64(A)).
//
// Representation.  Every row i of A gets a power-of-two scale 2^T_i > max_l |a_il|, every
// column j of V a scale 2^F_j > max_l |v_lj|.  An entry becomes the fixed-point integer
// t = trunc(a 2^(46 - T_i)), |t| < 2^46, written in balanced base 256: six signed bytes,
// most significant first,
//     a_il = 2^(T_i - 46) * sum_P d^(P)_il 256^(5 - P),   d in [-128, 127]
// (byte P of t + 0x808080808080, minus 128: slicing is an add and byte extraction).  A
// bf16/fp16/e4m3 entry is exact unless it is 2^-23 below its row maximum.  Digit products
// are exact in int8 x int8 -> int32 (tcgen05.mma kind::i8), and a level sum
//     D_L = sum_{P + Q = L} sum_l a^(P)_il v^(Q)_lj,   L = 0..5 (21 products)
// cannot overflow while a chunk of K covers at most 16384 terms (6 * 128^2 * 16384 < 2^31).
// Then  (A V)_ij = 2^(T_i + F_j) * sum_L D_L 2^(-8 L - 12)  up to the dropped levels L > 5
// and the truncated tails, both of random sign: ~2^-46 relative to |A| |V| per term (an
// FP64 GEMM: ~2^-53); the level sums are combined in fp64.
//
// Kernels: k_oz_slices_a (row scales + the six byte planes of A; HBM-bound),
// k_oz_slices_v (column scales + bytes of V), k_oz_gemm (tcgen05 int8, TMA, TMEM int32
// accumulators for the six levels, stream-K over (row tile, K chunk) with fp64 partials),
// k_oz_resid (deterministic partial sums -> (A v_j - lambda_j y_j) column sums of squares).
#include "common.cuh"
#include <vector>
#include <mutex>
#include <algorithm>
#include <climits>
#include <cstdlib>

namespace ofrr {

// in-kernel timing of k_ozk_gemm for the bench roofline (the K1 scheme, gemm_tc.cu): every CTA
// stamps its entry (min) and exit (max) in globaltimer ns; the k_oz_resid launch that follows
// adds the interval to a running sum and re-arms the stamps
// min start, max end, then (sum, count) per tier: [2..3] every product, [4..5] FP64-accurate
// (6 levels), [6..7] lite (4 levels), [8..9] 5 levels -- the k_oz_resid launch passes the tier
__device__ unsigned long long g_oz_stamp[10] = {~0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
static bool g_oz_stamp_on = false;
__device__ __forceinline__ unsigned long long oz_gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
int oz_stamp_enable(int on) {
  g_oz_stamp_on = on != 0;
  if (on) {
    const unsigned long long z[10] = {~0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
    if (cudaMemcpyToSymbol(g_oz_stamp, z, sizeof(z)) != cudaSuccess) return OFRR_ERR_CUDA;
  }
  return OFRR_OK;
}
int oz_stamp_read(double* sum_ms, long long* count, int tier) {   // tier 0 all, 1 FP64-accurate, 2 lite, 3 5-level
  unsigned long long v[10];
  if (tier < 0 || tier > 3) return OFRR_ERR_INVALID;
  if (cudaMemcpyFromSymbol(v, g_oz_stamp, sizeof(v)) != cudaSuccess) return OFRR_ERR_CUDA;
  *sum_ms = (double)v[2 + 2 * tier] * 1e-6;
  *count = (long long)v[3 + 2 * tier];
  return OFRR_OK;
}

static constexpr int OZ_D = 6;            // digits per operand
static constexpr int OZ_TM = 128;         // rows per tile (UMMA M = 128)
static constexpr int OZ_KB = 128;         // K per k-block (int8: one 128B swizzle row)
static constexpr int OZ_THREADS = 192;    // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
static constexpr int OZ_MAXCHUNK = 128;   // k-blocks per accumulation chunk (16384 terms)
static constexpr int OZ_BAD = INT_MIN;    // scale marker: the row / column has inf or NaN
static constexpr int OZR_CG = 8;          // k_oz_resid: columns per CTA (8: ~60 registers, 2x the resident warps of 16)

template <int BN>
struct OzCfg {
  static constexpr int A_BYTES = OZ_TM * OZ_KB;            // one digit plane tile of A, 16 KB
  static constexpr int V_BYTES = OZ_D * BN * OZ_KB;        // the six digit tiles of V for a k-block
  static constexpr int A_STAGES_RAW = (200 * 1024 - 2 * V_BYTES) / A_BYTES;
  static constexpr int A_STAGES = A_STAGES_RAW > 8 ? 8 : A_STAGES_RAW;
  static constexpr int TMEM_COLS = OZ_D * BN <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = 1024 + 2 * V_BYTES + A_STAGES * A_BYTES + 256;
};

// idesc for kind::i8: D = S32 (bits 4-5 = 2), A / B signed (1) or unsigned (0) 8-bit
// (bits 7-9 / 10-12), K-major, N >> 3 at bit 17, M >> 4 at bit 24.
__host__ __device__ inline uint32_t oz_idesc(int n, bool a_signed, bool b_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_ld16i(uint32_t taddr, int* v) {
  float f[16];
  tmem_ld16(taddr, f);
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __float_as_int(f[i]);
}

// scale exponent E with |x| < 2^E for m = max |x| (0 for m == 0, OZ_BAD for inf/NaN)
__device__ __forceinline__ int oz_scale(double m) {
  if (!(m <= 1.7976931348623157e308)) return OZ_BAD;
  if (m == 0.0) return 0;
  return ilogb(m) + 1;
}
// 4 x 4 byte transpose: in[e] holds bytes (b0, b1, b2, b3) of entry e; out[b] holds byte b
// of entries 0..3 (entry e in byte e)
__device__ __forceinline__ void oz_t4(const uint32_t (&in)[4], uint32_t (&out)[4]) {
  const uint32_t a01 = __byte_perm(in[0], in[1], 0x5140), b01 = __byte_perm(in[0], in[1], 0x7362);
  const uint32_t a23 = __byte_perm(in[2], in[3], 0x5140), b23 = __byte_perm(in[2], in[3], 0x7362);
  out[0] = __byte_perm(a01, a23, 0x5410);
  out[1] = __byte_perm(a01, a23, 0x7632);
  out[2] = __byte_perm(b01, b23, 0x5410);
  out[3] = __byte_perm(b01, b23, 0x7632);
}
// balanced base-256 digit planes (most significant first) of four fixed-point words given
// as biased (lo, hi) = t + 0x808080808080: digit = byte - 128 = byte ^ 0x80
__device__ __forceinline__ void oz_planes4(const uint32_t (&lo)[4], const uint32_t (&hi)[4], uint32_t (&w)[OZ_D]) {
  uint32_t tl[4], th[4];
  oz_t4(lo, tl);
  oz_t4(hi, th);
  w[0] = th[1] ^ 0x80808080u;   // byte 5
  w[1] = th[0] ^ 0x80808080u;   // byte 4
  w[2] = tl[3] ^ 0x80808080u;
  w[3] = tl[2] ^ 0x80808080u;
  w[4] = tl[1] ^ 0x80808080u;
  w[5] = tl[0] ^ 0x80808080u;
}
// plain two's-complement bytes of four fixed-point words (lo, hi) = t: byte 5 (signed: the
// sign lives there since |t| < 2^46) first, bytes 4..0 unsigned -- the A digits of the
// in-kernel product (no bias add, no byte flip; the MMA takes plane 0 as s8, 1..5 as u8)
__device__ __forceinline__ void oz_planes4u(const uint32_t (&lo)[4], const uint32_t (&hi)[4], uint32_t (&w)[OZ_D]) {
  uint32_t tl[4], th[4];
  oz_t4(lo, tl);
  oz_t4(hi, th);
  w[0] = th[1];
  w[1] = th[0];
  w[2] = tl[3];
  w[3] = tl[2];
  w[4] = tl[1];
  w[5] = tl[0];
}
__device__ __forceinline__ void oz_bias(uint32_t& lo, uint32_t& hi) {
  const uint32_t l = lo + 0x80808080u;
  hi = hi + 0x8080u + (l < lo ? 1u : 0u);
  lo = l;
}
// fp64 x on the 46-bit window below 2^E -> biased two's-complement (lo, hi)
__device__ __forceinline__ void oz_fixed64(double x, int E, uint32_t& lo, uint32_t& hi) {
  long long t = 0;
  if (E != OZ_BAD && x != 0.0) {
    t = (long long)ldexp(fabs(x), 46 - E);   // < 2^46, truncated toward zero
    if (x < 0.0) t = -t;
  }
  lo = (uint32_t)(unsigned long long)t;
  hi = (uint32_t)((unsigned long long)t >> 32);
  oz_bias(lo, hi);
}

// ---------------------------------------------------------------------------------
// A (rows x cols, row-major, 16/8-bit) -> T[rows_pad], planes[6][rows_pad][cols_pad] int8.
// One CTA per row.  Entries go through their f32 bit pattern (exact for bf16 / f16 /
// e4m3): value = M 2^(e - 150) with the 24-bit significand M, so the fixed-point word is
// t = M << (e - 108 - T) (or >> when negative) -- integer ops only.  The row maximum is
// an integer max over |bits| (positive float patterns order like their values; NaN
// patterns sort above inf).  Padding rows get zero digits.
// ---------------------------------------------------------------------------------
template <int FMT>
__device__ __forceinline__ float oz_ld_f(const void* A, int64_t i) {
  if constexpr (FMT == BF16) return __bfloat162float(((const __nv_bfloat16*)A)[i]);
  else if constexpr (FMT == F16) return __half2float(((const __half*)A)[i]);
  else { __nv_fp8_e4m3 v; v.__x = ((const __nv_fp8_storage_t*)A)[i]; return float(v); }
}
// f32 bit pattern b (exact value of a bf16 / f16 / e4m3 entry) on the 46-bit window
// below 2^T -> biased two's-complement (lo, hi): value = M 2^(e - 150), t = M << (e - 104 - T)
__device__ __forceinline__ void oz_fixed32(uint32_t b, int T, uint32_t& lo, uint32_t& hi) {
  const uint32_t ab = b & 0x7fffffffu;
  const int e = (int)(ab >> 23);
  const uint32_t M = (ab & 0x7fffffu) | (e ? 0x800000u : 0u);
  const int sh = (e ? e : 1) - 104 - T;                 // <= 22
  const uint32_t s = (uint32_t)max(sh, 0), r = (uint32_t)min(max(-sh, 0), 31);
  uint32_t l = (M << s) >> r;
  uint32_t h = s ? (M >> (32u - s)) : 0u;
  if (b >> 31) {                                         // two's-complement negate (lo, hi)
    h = ~h + (l == 0u ? 1u : 0u);
    l = 0u - l;
  }
  lo = l;
  hi = h;
  oz_bias(lo, hi);
}

template <int FMT>
__device__ __forceinline__ void oz_ld8(const void* A, int64_t base, int64_t l0, int64_t cols, bool vec, float (&x)[8]) {
  if (vec && l0 + 8 <= cols) {
    if constexpr (FMT == FP8) {
      const uint2 v = *reinterpret_cast<const uint2*>((const uint8_t*)A + base + l0);
      const uint32_t w[2] = {v.x, v.y};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        __nv_fp8_e4m3 q;
        q.__x = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
        x[e] = float(q);
      }
    } else {
      const uint4 v = *reinterpret_cast<const uint4*>((const uint16_t*)A + base + l0);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint16_t h = (uint16_t)(w[e >> 1] >> (16 * (e & 1)));
        if constexpr (FMT == BF16) x[e] = __uint_as_float((uint32_t)h << 16);
        else x[e] = __half2float(__ushort_as_half(h));
      }
    }
  } else {
#pragma unroll
    for (int e = 0; e < 8; ++e) x[e] = l0 + e < cols ? oz_ld_f<FMT>(A, base + l0 + e) : 0.0f;
  }
}

template <int FMT>
__global__ void __launch_bounds__(256)
    k_oz_slices_a(const void* __restrict__ A, int64_t rows, int64_t cols, int64_t lda, int* __restrict__ T,
                  int8_t* __restrict__ planes, int64_t rows_pad, int64_t cols_pad) {
  const int64_t i = blockIdx.x;
  __shared__ uint32_t red[8];
  const size_t plane = (size_t)rows_pad * cols_pad;
  int8_t* row0 = planes + (size_t)i * cols_pad;
  if (i >= rows) {
    for (int64_t l = 4 * (int64_t)threadIdx.x; l < cols_pad; l += 4 * (int64_t)blockDim.x)
      for (int p = 0; p < OZ_D; ++p) *reinterpret_cast<uint32_t*>(row0 + p * plane + l) = 0u;
    if (threadIdx.x == 0) T[i] = 0;
    return;
  }
  const int64_t base = i * lda;
  const int eb = FMT == FP8 ? 1 : 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(A) + (uintptr_t)(base * eb)) & 15) == 0;
  uint32_t m = 0;
  for (int64_t l0 = 8 * (int64_t)threadIdx.x; l0 < cols; l0 += 8 * (int64_t)blockDim.x) {
    float x[8];
    oz_ld8<FMT>(A, base, l0, cols, vec, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t b = __float_as_uint(x[e]) & 0x7fffffffu;
      m = b > m ? b : m;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t om = __shfl_xor_sync(0xffffffffu, m, o);
    m = om > m ? om : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < 8; ++w) m = red[w] > m ? red[w] : m;
  const int E = oz_scale((double)__uint_as_float(m));
  if (threadIdx.x == 0) T[i] = E;
  // the scale 2^(46 - E) as an f32 (normal range) -> conversion path; else the bit path
  const bool fast = E != OZ_BAD && 46 - E <= 127 && 46 - E >= -126;
  const float sc = fast ? __int_as_float((46 - E + 127) << 23) : 0.0f;
  // 8 consecutive entries per thread step -> one 64-bit word per plane (cols_pad % 16 == 0)
  for (int64_t l0 = 8 * (int64_t)threadIdx.x; l0 < cols_pad; l0 += 8 * (int64_t)blockDim.x) {
    uint32_t w0[OZ_D] = {0, 0, 0, 0, 0, 0}, w1[OZ_D] = {0, 0, 0, 0, 0, 0};
    if (E != OZ_BAD) {
      float x[8];
      oz_ld8<FMT>(A, base, l0, cols, vec, x);
      uint32_t lo[4], hi[4];
      if (fast) {
        // t = trunc(x 2^(46 - E)): exact scaling in f32, one f32 -> s64 conversion
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const long long t = __float2ll_rz(x[4 * h + e] * sc);
            lo[e] = (uint32_t)(unsigned long long)t;
            hi[e] = (uint32_t)((unsigned long long)t >> 32);
            oz_bias(lo[e], hi[e]);
          }
          oz_planes4(lo, hi, h ? w1 : w0);
        }
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) oz_fixed32(__float_as_uint(x[e]), E, lo[e], hi[e]);
        oz_planes4(lo, hi, w0);
#pragma unroll
        for (int e = 0; e < 4; ++e) oz_fixed32(__float_as_uint(x[4 + e]), E, lo[e], hi[e]);
        oz_planes4(lo, hi, w1);
      }
    }
#pragma unroll
    for (int p = 0; p < OZ_D; ++p) *reinterpret_cast<uint2*>(row0 + p * plane + l0) = make_uint2(w0[p], w1[p]);
  }
}

// V (cols x n fp64, column j contiguous, ld ldv) -> F[npad], digits[6][npad][cols_pad]
__global__ void __launch_bounds__(256)
    k_oz_slices_v(const double* __restrict__ V, int64_t ldv, int64_t cols, int n, int* __restrict__ F,
                  int8_t* __restrict__ dig, int npad, int64_t cols_pad) {
  const int j = blockIdx.x;
  __shared__ double red[8];
  __shared__ int sE;
  const size_t plane = (size_t)npad * cols_pad;
  int8_t* row0 = dig + (size_t)j * cols_pad;
  if (j >= n) {
    for (int64_t l = threadIdx.x; l < cols_pad; l += blockDim.x)
      for (int p = 0; p < OZ_D; ++p) row0[p * plane + l] = 0;
    if (threadIdx.x == 0) F[j] = 0;
    return;
  }
  const double* v = V + (size_t)j * ldv;
  double m = 0.0;
  for (int64_t l = threadIdx.x; l < cols; l += blockDim.x) {
    const double a = fabs(v[l]);
    m = (a != a || a > m) ? a : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double om = __shfl_xor_sync(0xffffffffu, m, o);
    m = (om != om || om > m) ? om : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mm = (red[w] != red[w] || red[w] > mm) ? red[w] : mm;
    sE = oz_scale(mm);
    F[j] = sE;
  }
  __syncthreads();
  const int E = sE;
  for (int64_t l0 = 4 * (int64_t)threadIdx.x; l0 < cols_pad; l0 += 4 * (int64_t)blockDim.x) {
    uint32_t w[OZ_D], lo[4], hi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) oz_fixed64(l0 + e < cols ? v[l0 + e] : 0.0, E, lo[e], hi[e]);
    oz_planes4(lo, hi, w);
#pragma unroll
    for (int p = 0; p < OZ_D; ++p) *reinterpret_cast<uint32_t*>(row0 + p * plane + l0) = w[p];
  }
}

// The same split over (column, segment) CTAs: the column maxima first (bit patterns of
// non-negative doubles order like the values, NaN above inf -> OZ_BAD as above), then the
// digits of each segment -- one CTA per column left most SMs idle on this streaming pass.
__global__ void __launch_bounds__(256)
    k_oz_vmax(const double* __restrict__ V, int64_t ldv, int64_t cols, int n, unsigned long long* __restrict__ vmax,
              int64_t seg) {
  const int j = blockIdx.x;
  if (j >= n) return;
  const double* v = V + (size_t)j * ldv;
  const int64_t l1 = std::min<int64_t>(cols, ((int64_t)blockIdx.y + 1) * seg);
  unsigned long long m = 0ull;
  for (int64_t l = (int64_t)blockIdx.y * seg + threadIdx.x; l < l1; l += blockDim.x) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(v[l]));
    m = b > m ? b : m;
  }
  const unsigned hi = (unsigned)(m >> 32), lo = (unsigned)m;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  if ((threadIdx.x & 31) == 0) atomicMax(&vmax[j], ((unsigned long long)mhi << 32) | mlo);
}

__global__ void __launch_bounds__(256)
    k_oz_slices_vs(const double* __restrict__ V, int64_t ldv, int64_t cols, int n,
                   const unsigned long long* __restrict__ vmax, int* __restrict__ F, int8_t* __restrict__ dig, int npad,
                   int64_t cols_pad, int64_t seg) {
  const int j = blockIdx.x;
  const size_t plane = (size_t)npad * cols_pad;
  int8_t* row0 = dig + (size_t)j * cols_pad;
  const int64_t s0 = (int64_t)blockIdx.y * seg, s1 = std::min<int64_t>(cols_pad, s0 + seg);
  if (j >= n) {
    for (int64_t l = s0 + threadIdx.x; l < s1; l += blockDim.x)
      for (int p = 0; p < OZ_D; ++p) row0[p * plane + l] = 0;
    if (blockIdx.y == 0 && threadIdx.x == 0) F[j] = 0;
    return;
  }
  const double* v = V + (size_t)j * ldv;
  const int E = oz_scale(__longlong_as_double((long long)vmax[j]));
  if (blockIdx.y == 0 && threadIdx.x == 0) F[j] = E;
  for (int64_t l0 = s0 + 4 * (int64_t)threadIdx.x; l0 < s1; l0 += 4 * (int64_t)blockDim.x) {
    uint32_t w[OZ_D], lo[4], hi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) oz_fixed64(l0 + e < cols ? v[l0 + e] : 0.0, E, lo[e], hi[e]);
    oz_planes4(lo, hi, w);
#pragma unroll
    for (int p = 0; p < OZ_D; ++p) *reinterpret_cast<uint32_t*>(row0 + p * plane + l0) = w[p];
  }
}

// ---------------------------------------------------------------------------------
// The int8 tensor-core product.  Work unit = one k-block of a virtual tile vt = (row tile,
// K chunk); stream-K splits the units evenly over the grid.  Per unit the V digit tiles
// (6 x BN x 128 B) are staged once (double-buffered) and the six A digit-plane tiles
// stream through a ring; digit p of A meets digits q = 1..7-p of V in one or two MMAs that
// write the contiguous TMEM levels p+q (level L at column (L - 2) BN, int32).
// ---------------------------------------------------------------------------------
template <int BN>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmV,
              double* __restrict__ ws, int kbc, int nchunks, long long total_units, int max_slots,
              int rows_pad, int npad, int col0) {
  using C = OzCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* vbuf = smem;                               // [2][V_BYTES]
  uint8_t* abuf = smem + 2 * C::V_BYTES;              // [A_STAGES][A_BYTES]
  uint64_t* afull = reinterpret_cast<uint64_t*>(abuf + C::A_STAGES * C::A_BYTES);
  uint64_t* aempty = afull + C::A_STAGES;
  uint64_t* vfull = aempty + C::A_STAGES;
  uint64_t* vempty = vfull + 2;
  uint64_t* tfull = vempty + 2;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = warp_index(), lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  const long long u0 = (long long)blockIdx.x * total_units / G;
  const long long u1 = ((long long)blockIdx.x + 1) * total_units / G;
  const int vt_first = (int)(u0 / kbc);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::A_STAGES; ++s) { mbar_init(&afull[s], 1); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_barrier_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmV);
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_a = policy_evict_first(), pol_v = policy_evict_last();
      int as = 0, vs = 0;
      uint32_t aph = 0, vph = 0;
      for (long long u = u0; u < u1; ++u) {
        const int vt = (int)(u / kbc);
        const int kb = (vt % nchunks) * kbc + (int)(u % kbc);
        const int mt = vt / nchunks;
        mbar_wait(&vempty[vs], vph ^ 1);
        mbar_expect_tx(&vfull[vs], C::V_BYTES);
        for (int q = 0; q < OZ_D; ++q)
          tma_load_2d(vbuf + vs * C::V_BYTES + q * BN * OZ_KB, &tmV, kb * OZ_KB, q * npad + col0, &vfull[vs], pol_v);
        if (++vs == 2) { vs = 0; vph ^= 1; }
        for (int p = 0; p < OZ_D; ++p) {
          mbar_wait(&aempty[as], aph ^ 1);
          mbar_expect_tx(&afull[as], C::A_BYTES);
          tma_load_2d(abuf + as * C::A_BYTES, &tmA, kb * OZ_KB, p * rows_pad + mt * OZ_TM, &afull[as], pol_a);
          if (++as == C::A_STAGES) { as = 0; aph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ===== MMA issuer (warp-wide loop, elected lane issues) =====
      int as = 0, vs = 0;
      uint32_t aph = 0, vph = 0, acc_phase = 0;
      long long u = u0;
      while (u < u1) {
        const int vt = (int)(u / kbc);
        const long long seg_end = std::min<long long>(u1, (long long)(vt + 1) * kbc);
        const long long seg_start = u;
        mbar_wait(tempty, acc_phase ^ 1);
        tc_fence_after();
        for (; u < seg_end; ++u) {
          mbar_wait(&vfull[vs], vph);
          tc_fence_after();
          const uint64_t dv = umma_desc_sw128(smem_u32(vbuf + vs * C::V_BYTES));
          for (int p = 0; p < OZ_D; ++p) {
            mbar_wait(&afull[as], aph);
            tc_fence_after();
            const uint64_t da = umma_desc_sw128(smem_u32(abuf + as * C::A_BYTES));
            const int nq = OZ_D - p;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              // the segment's first unit, plane 0, k 0 initialises every level
              const uint32_t acc = (u > seg_start || p > 0 || k > 0) ? 1u : 0u;
              for (int q0 = 0; q0 < nq; q0 += 256 / BN) {
                const int ng = std::min(256 / BN, nq - q0);
                mma_i8_ws(tmem + (uint32_t)((p + q0) * BN), da + (uint64_t)(k * 2),
                       dv + (uint64_t)((q0 * BN * OZ_KB) >> 4) + (uint64_t)(k * 2), oz_idesc(ng * BN, true, true),
                       acc);
              }
            }
            tc_commit_ws(&aempty[as]);
            if (++as == C::A_STAGES) { as = 0; aph ^= 1; }
          }
          tc_commit_ws(&vempty[vs]);
          if (++vs == 2) { vs = 0; vph ^= 1; }
        }
        tc_commit_ws(tfull);
        acc_phase ^= 1;
      }
    }
  } else {
    // ===== epilogue warps 2..5: TMEM int32 levels -> fp64 partial tile (column-major) =====
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t acc_phase = 0;
    long long u = u0;
    while (u < u1) {
      const int vt = (int)(u / kbc);
      u = std::min<long long>(u1, (long long)(vt + 1) * kbc);
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      double* dst = ws + ((size_t)blockIdx.x * max_slots + (vt - vt_first)) * (size_t)(OZ_TM * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        double s[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) s[i] = 0.0;
#pragma unroll 1
        for (int lv = OZ_D - 1; lv >= 0; --lv) {     // lowest weight first
          int d[16];
          tmem_ld16i(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(lv * BN + c0), d);
          const double w = ldexp(1.0, -8 * lv - 12);
#pragma unroll
          for (int i = 0; i < 16; ++i) s[i] = fma((double)d[i], w, s[i]);   // exact product
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[(size_t)(c0 + i) * OZ_TM + row] = s[i];
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------------
// Row scales of A and the sparse tails of its 3-digit heads (the in-kernel slicing path
// below converts A on the fly).
//
// Head / tail split: with |a| < 2^T (T = row scale), the in-kernel product multiplies the
// 24-bit head h = trunc(a 2^(22 - T)) (three int8 digits: byte 2 signed, bytes 1, 0
// unsigned -- the top three of the six 46-bit digits, same weights) and the tail
// a - h 2^(T - 22) (the bits of a below 2^(T - 22): |tail| < 2^(T - 22), same sign, at most
// 8 significant bits, exact in f32) is applied exactly in fp64 from a per-row list.  For
// 16/8-bit entries the tail is non-zero only for entries ~2^-15 below their row maximum (a
// handful per row), so 15 digit products (p <= 2, p + q <= 5) replace 21 with no loss.
// A row whose tails overflow OZ_TAIL_CAP, or whose scale leaves the f32 range of the
// conversion, sets the operator's `full` flag: every product with it then uses all six
// digits (the previous scheme).  Tails are listed in ascending column order (ordered
// block compaction): deterministic sums.
// ---------------------------------------------------------------------------------
static constexpr int OZ_TAIL_CAP = 32;      // tail entries kept per row

struct OzOpLayout {
  int64_t rows_pad;
  size_t off_T, off_full, off_cnt, off_col, off_val, bytes;
};
static OzOpLayout oz_op_layout(int64_t rows) {
  OzOpLayout L;
  L.rows_pad = (rows + OZ_TM - 1) / OZ_TM * OZ_TM;
  size_t b = 0;
  auto take = [&](size_t n) { size_t o = b; b += (n + 255) & ~size_t(255); return o; };
  L.off_T = take((size_t)L.rows_pad * 4);
  L.off_full = take(16);
  L.off_cnt = take((size_t)L.rows_pad * 4);
  L.off_col = take((size_t)L.rows_pad * OZ_TAIL_CAP * 4);
  L.off_val = take((size_t)L.rows_pad * OZ_TAIL_CAP * 4);
  L.bytes = b;
  return L;
}

static constexpr int OZ_RS_THREADS = 128;    // k_oz_rowscale: one CTA per row, one 32-entry group per thread step

// mantissa bits of the 16/8-bit formats: an entry with exponent e has no bit below 2^(e - MB)
template <int FMT> __device__ __forceinline__ constexpr int oz_mant_bits() { return FMT == BF16 ? 7 : FMT == F16 ? 10 : 3; }
// unbiased exponent of a non-negative 16-bit pattern (bf16 / f16); subnormals count as the
// lowest normal exponent minus one (conservative for the candidate test)
template <int FMT> __device__ __forceinline__ int oz_exp16(uint32_t p) {
  if constexpr (FMT == BF16) return (int)(p >> 7) - 127;
  else return (int)(p >> 10) - 15;
}
template <int FMT> __device__ __forceinline__ float oz_val16(uint32_t p) {
  if constexpr (FMT == BF16) return __uint_as_float(p << 16);
  else return __half2float(__ushort_as_half((unsigned short)p));
}

// Row scale T (|a| < 2^T), and the row's tails (see above).  Pass 1 reads the row once
// (32 entries per thread step, four 16-byte loads in flight): the row maximum and, per
// 32-entry group, the smallest non-zero magnitude -- as packed 16-bit SIMD max / min on the
// bit patterns for bf16 / f16 (positive float patterns order like their values).  Pass 2
// (warp 0 only) revisits just the groups whose smallest entry can hold bits below
// 2^(T - 22): their indices are compacted in order from shared memory, then one lane per
// candidate group re-reads its 32 entries and the tails are written in ascending column
// order (warp scan of the per-group counts).
template <int FMT>
__global__ void __launch_bounds__(OZ_RS_THREADS)
    k_oz_rowscale(const void* __restrict__ A, int64_t rows, int64_t cols, int64_t lda, int* __restrict__ T,
                  int* __restrict__ full, int* __restrict__ tcnt, int* __restrict__ tcol, float* __restrict__ tval) {
  constexpr int NW = OZ_RS_THREADS / 32;
  constexpr bool P16 = FMT != FP8;
  extern __shared__ int gsh[];               // per 32-entry group: smallest exponent (then: candidate list)
  const int64_t i = blockIdx.x;
  __shared__ uint32_t red[NW];
  if (i >= rows) {
    if (threadIdx.x == 0) {
      T[i] = 0;
      if (tcnt) tcnt[i] = 0;
    }
    return;
  }
  const int64_t base = i * lda;
  const int eb = FMT == FP8 ? 1 : 2;
  const bool vec = ((reinterpret_cast<uintptr_t>(A) + (uintptr_t)(base * eb)) & 15) == 0;
  const int64_t step = 32 * (int64_t)OZ_RS_THREADS;
  const int64_t ngroups = (cols + 31) / 32;
  uint32_t m = 0;                            // max |a| as f32 bits
  for (int64_t c0 = 0; c0 < cols; c0 += step) {
    const int64_t l0 = c0 + 32 * (int64_t)threadIdx.x;
    if (l0 >= cols) continue;
    int emin = 127;
    if (P16 && vec && l0 + 32 <= cols) {
      const uint4* src = reinterpret_cast<const uint4*>((const uint16_t*)A + base + l0);
      uint4 w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = __ldcs(src + u);
      uint32_t vmax = 0u, vmin = 0xffffffffu;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t ww[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t av = ww[q] & 0x7fff7fffu;
          vmax = __vmaxu2(vmax, av);
          vmin = __vminu2(vmin, av | __vcmpeq2(av, 0u));
        }
      }
      const uint32_t pmax = max(vmax & 0xffffu, vmax >> 16);
      const uint32_t pmin = min(vmin & 0xffffu, vmin >> 16);
      const uint32_t fb = __float_as_uint(oz_val16<FMT>(pmax));
      m = fb > m ? fb : m;
      if (pmin != 0xffffu) emin = oz_exp16<FMT>(pmin);
    } else {
      for (int e = 0; e < 32 && l0 + e < cols; ++e) {
        const uint32_t bb = __float_as_uint(oz_ld_f<FMT>(A, base + l0 + e)) & 0x7fffffffu;
        m = bb > m ? bb : m;
        if (bb) emin = min(emin, bb >= 0x00800000u ? (int)(bb >> 23) - 127 : -127);
      }
    }
    if (tcnt) gsh[l0 >> 5] = emin;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint32_t om = __shfl_xor_sync(0xffffffffu, m, o);
    m = om > m ? om : m;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x >= 32) return;             // pass 2 is warp 0's
  m = red[0];
  for (int w = 1; w < NW; ++w) m = red[w] > m ? red[w] : m;
  const int E = oz_scale((double)__uint_as_float(m));
  const int lane = threadIdx.x;
  if (lane == 0) T[i] = E;
  if (!tcnt) return;
  if (E == OZ_BAD) {                         // non-finite row: its products are NaN anyway
    if (lane == 0) tcnt[i] = 0;
    return;
  }
  if (22 - E > 127 || 22 - E < -126 || E - 22 < -126) {   // scale outside the f32 conversion range
    if (lane == 0) { tcnt[i] = 0; atomicOr(full, 1); }
    return;
  }
  const float sc = __int_as_float((22 - E + 127) << 23);      // 2^(22 - E)
  const float isc = __int_as_float((E - 22 + 127) << 23);     // 2^(E - 22)
  const int ecut = E - 22 + oz_mant_bits<FMT>();              // a group can hold a tail iff its min exponent < ecut
  // ordered list of candidate groups, compacted in place (slot ncand <= g: no overlap)
  int ncand = 0;
  for (int64_t g0 = 0; g0 < ngroups; g0 += 32) {
    const int64_t g = g0 + lane;
    const bool c = g < ngroups && gsh[g] < ecut;
    const uint32_t bal = __ballot_sync(0xffffffffu, c);
    __syncwarp();
    if (c) gsh[ncand + __popc(bal & ((1u << lane) - 1u))] = (int)g;
    ncand += __popc(bal);
    __syncwarp();
  }
  int total = 0;
  for (int c0 = 0; c0 < ncand; c0 += 32) {
    uint32_t mask = 0;
    int64_t l0 = 0;
    float tl[32];
    if (c0 + lane < ncand) {
      l0 = (int64_t)gsh[c0 + lane] * 32;
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float x = l0 + e < cols ? oz_ld_f<FMT>(A, base + l0 + e) : 0.0f;
        const int h = __float2int_rz(x * sc);
        tl[e] = x - __int2float_rn(h) * isc;           // the tail (exact, see above)
        mask |= (tl[e] != 0.0f ? 1u : 0u) << e;
      }
    }
    const int nt = __popc(mask);
    int inc = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    int pos = total + inc - nt;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      if ((mask >> e) & 1u) {
        if (pos < OZ_TAIL_CAP) {
          tcol[i * OZ_TAIL_CAP + pos] = (int)(l0 + e);
          tval[i * OZ_TAIL_CAP + pos] = tl[e];
        }
        ++pos;
      }
    }
    total += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    tcnt[i] = total < OZ_TAIL_CAP ? total : OZ_TAIL_CAP;
    if (total > OZ_TAIL_CAP) atomicOr(full, 1);
  }
}

// The tails times one column pass of V: Wt[row * BN + j] = sum_e tail_e V[col_e, j0 + j]
// (fp64, list order).  A warp per row, lanes over the pass's columns: each tail entry reads
// one contiguous row of Vt.
__global__ void __launch_bounds__(256)
    k_oz_tailmul(int64_t rows, const int* __restrict__ full, const int* __restrict__ tcnt,
                 const int* __restrict__ tcol, const float* __restrict__ tval, const double* __restrict__ Vt,
                 int ldvt, int j0, int ncols, int BN, double* __restrict__ Wt) {
  if (*full) return;
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int cnt = tcnt[row];
  const int mc = lane < cnt ? tcol[row * OZ_TAIL_CAP + lane] : 0;
  const double mv = lane < cnt ? (double)tval[row * OZ_TAIL_CAP + lane] : 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};                // columns lane + 32 t, BN <= 128
  for (int e = 0; e < cnt; ++e) {
    const int c = __shfl_sync(0xffffffffu, mc, e);
    const double v = __shfl_sync(0xffffffffu, mv, e);
    const double* vr = Vt + (int64_t)c * ldvt + j0;
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (lane + 32 * t < ncols) acc[t] = fma(v, vr[lane + 32 * t], acc[t]);
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if (lane + 32 * t < BN) Wt[row * BN + lane + 32 * t] = acc[t];
}

// V (fp64, column j contiguous with ld ldv, n rows x r columns) -> Vt row-major (row l holds
// V[l, 0..r), leading dimension ldt): the tails read one contiguous row of V per entry
__global__ void __launch_bounds__(256)
    k_oz_vt(const double* __restrict__ V, int64_t ldv, int64_t n, int r, double* __restrict__ Vt, int ldt) {
  __shared__ double tile[32][33];
  const int64_t l0 = (int64_t)blockIdx.x * 32;
  const int j0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;      // 32 x 8
  for (int jj = ty; jj < 32; jj += 8) {
    const int j = j0 + jj;
    const int64_t l = l0 + tx;
    tile[jj][tx] = (j < r && l < n) ? V[(int64_t)j * ldv + l] : 0.0;
  }
  __syncthreads();
  for (int ll = ty; ll < 32; ll += 8) {
    const int64_t l = l0 + ll;
    const int j = j0 + tx;
    if (l < n && j < r) Vt[l * ldt + j] = tile[tx][ll];
  }
}

// ---------------------------------------------------------------------------------
// The int8 tensor-core product with the A digits made on the fly (no digit planes in HBM):
// A is read once in its own format.  64-byte k-blocks (SWIZZLE_64B tiles: a full digit set
// of one k-block is 6 x 8 KB), 8 converter warps turn the bf16/f16/e4m3 tile into the six
// balanced base-256 digit tiles in shared memory (triple-buffered) while warp 1 issues the
// tcgen05 int8 MMAs of the previous k-block and warp 0 streams the V digit tiles by TMA.
// Same digits and exact integer level sums as k_oz_gemm: identical results.
// ---------------------------------------------------------------------------------
static constexpr int OZK_KB = 64;          // K elements (= int8 bytes) per k-block
static constexpr int OZK_CONV_WARPS = 16;
static constexpr int OZK_THREADS = 192 + 32 * OZK_CONV_WARPS;
// k-blocks per chunk (8192 terms): with u8 A digits (<= 255) x s8 V digits a level sums up
// to 6 products of |d| <= 255 * 128 per term -- 6 * 32640 * 8192 < 2^31
static constexpr int OZK_MAXCHUNK = 128;
// the 3-plane (heads) variants sum at most 3 digit products per level: 3 * 128^2 * 32768 < 2^31,
// so their chunks are twice as long (half the fp64 partial tiles for k_oz_resid)
static constexpr int OZK_MAXCHUNK_H = 256;

// NL = accumulation levels kept (digit products with p + q < NL): 6 -> ~2^-46 of |A||x| per
// term (FP64-accurate); 4 -> ~2^-30 (the "lite" products of the full-f64-lite rung), which
// frees TMEM for BN = 128 columns per launch (4 levels x 128 = 512 TMEM columns).
template <int BN, int NP = OZ_D, int NL = OZ_D>
struct OzkCfg {
  static constexpr int A_TILE = OZ_TM * OZK_KB;         // 8 KB per digit plane
  static constexpr int A_SET = NP * A_TILE;             // NP digit planes per k-block (48 / 24 KB)
  static constexpr int V_SET = NL * BN * OZK_KB;        // the NL V digit tiles a product needs
  // the 3-digit heads free half of each A stage: deeper rings on both operands
  static constexpr int A_STAGES = NP == OZ_D ? 3 : (BN == 128 ? 4 : 5);
  static constexpr int V_STAGES = NP == OZ_D ? 2 : (BN == 128 ? 2 : (BN == 64 ? 3 : 4));
  static constexpr int TMEM_COLS = NL * BN <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = 1024 + A_STAGES * A_SET + V_STAGES * V_SET + 256;
  static_assert(SMEM_BYTES <= 227 * 1024, "ozk shared memory");
  static_assert(NL * BN <= 512, "ozk TMEM");
};

// UMMA shared-memory descriptor: K-major, 64B swizzle, 8-row groups 512 B apart
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int FMT>
__device__ __forceinline__ void ozk_load32(const void* A, int64_t off, bool ok_vec, int64_t l0, int64_t cols,
                                           bool row_ok, uint4 (&raw)[4]) {
  // 32 consecutive entries (64 B for 16-bit, 32 B for e4m3) of one row, zero outside
  constexpr int EB = FMT == FP8 ? 1 : 2;
  constexpr int NV = 32 * EB / 16;
#pragma unroll
  for (int v = 0; v < 4; ++v) raw[v] = make_uint4(0, 0, 0, 0);
  if (!row_ok) return;
  if (ok_vec && l0 + 32 <= cols) {
    const uint4* src = reinterpret_cast<const uint4*>((const uint8_t*)A + (off + l0) * EB);
#pragma unroll
    for (int v = 0; v < NV; ++v) raw[v] = __ldcs(src + v);
  } else {
    uint8_t* dst = reinterpret_cast<uint8_t*>(raw);
    for (int e = 0; e < 32; ++e) {
      if (l0 + e < cols) {
        if (EB == 2) {
          const uint16_t h = ((const uint16_t*)A)[off + l0 + e];
          dst[2 * e] = (uint8_t)h;
          dst[2 * e + 1] = (uint8_t)(h >> 8);
        } else {
          dst[e] = ((const uint8_t*)A)[off + l0 + e];
        }
      }
    }
  }
}
template <int FMT>
__device__ __forceinline__ float ozk_elem(const uint4 (&raw)[2], int e) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(raw);
  if constexpr (FMT == BF16) {
    return __uint_as_float(((w[e >> 1] >> (16 * (e & 1))) & 0xffffu) << 16);
  } else if constexpr (FMT == F16) {
    return __half2float(__ushort_as_half((uint16_t)(w[e >> 1] >> (16 * (e & 1)))));
  } else {
    __nv_fp8_e4m3 q;
    q.__x = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
    return float(q);
  }
}

// NP = digit planes of A: 3 (the 24-bit heads; tails applied by k_oz_resid) or 6 (all of A).
// Both variants are launched back to back; the one that does not match the operator's
// `full` flag (set by its prepare pass) exits at once -- the choice stays on the device
// (CUDA graphs) and the MMA issue loop stays fully unrolled.
template <int FMT, int BN, int NP, int NL>
__global__ void __launch_bounds__(OZK_THREADS, 1)
    k_ozk_gemm(const void* __restrict__ A, int64_t rows, int64_t cols, int64_t lda, const int* __restrict__ Tg,
               const __grid_constant__ CUtensorMap tmV, double* __restrict__ ws, int kbc, int nchunks,
               long long total_units, int max_slots, int npad, int col0, int stamp,
               const int* __restrict__ full_flag) {
  using C = OzkCfg<BN, NP, NL>;
  constexpr bool full = NP == OZ_D;
  if (full_flag != nullptr && ((*full_flag != 0) != full)) return;
  if (stamp && threadIdx.x == 0) atomicMin(&g_oz_stamp[0], oz_gtimer_ns());
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* abuf = smem;                                  // [A_STAGES][6][128 x 64 B]
  uint8_t* vbuf = smem + C::A_STAGES * C::A_SET;         // [V_STAGES][6][BN x 64 B]
  uint64_t* afull = reinterpret_cast<uint64_t*>(vbuf + C::V_STAGES * C::V_SET);
  uint64_t* aempty = afull + C::A_STAGES;
  uint64_t* vfull = aempty + C::A_STAGES;
  uint64_t* vempty = vfull + C::V_STAGES;
  uint64_t* tfull = vempty + C::V_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = warp_index(), lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  const long long u0 = (long long)blockIdx.x * total_units / G;
  const long long u1 = ((long long)blockIdx.x + 1) * total_units / G;
  const int vt_first = (int)(u0 / kbc);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::A_STAGES; ++s) { mbar_init(&afull[s], OZK_CONV_WARPS); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < C::V_STAGES; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_barrier_init();
    prefetch_tmap(&tmV);
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: V digit tiles =====
      const uint64_t pol_v = policy_evict_last();
      int vs = 0;
      uint32_t vph = 0;
      int vt = (int)(u0 / kbc), rem = (int)(u0 % kbc);     // (tile, k-block) of u, no divisions per step
      for (long long u = u0; u < u1; ++u) {
        const int kb = (vt % nchunks) * kbc + rem;
        if (++rem == kbc) { rem = 0; ++vt; }
        mbar_wait(&vempty[vs], vph ^ 1);
        mbar_expect_tx(&vfull[vs], C::V_SET);
        for (int q = 0; q < NL; ++q)
          tma_load_2d(vbuf + vs * C::V_SET + q * BN * OZK_KB, &tmV, kb * OZK_KB, q * npad + col0, &vfull[vs], pol_v);
        if (++vs == C::V_STAGES) { vs = 0; vph ^= 1; }
      }
    }
  } else if (warp == 1) {
    {
      // ===== MMA issuer (warp-wide loop, elected lane issues) =====
      int as = 0, vs = 0;
      uint32_t aph = 0, vph = 0, acc_phase = 0;
      long long u = u0;
      while (u < u1) {
        const int vt = (int)(u / kbc);
        const long long seg_end = std::min<long long>(u1, (long long)(vt + 1) * kbc);
        const long long seg_start = u;
        mbar_wait(tempty, acc_phase ^ 1);
        tc_fence_after();
        for (; u < seg_end; ++u) {
          mbar_wait(&vfull[vs], vph);
          mbar_wait(&afull[as], aph);
          tc_fence_after();
          const uint32_t sa = smem_u32(abuf + as * C::A_SET);
          const uint64_t dv = umma_desc_sw64(smem_u32(vbuf + vs * C::V_SET));
#pragma unroll
          for (int p = 0; p < (NP < NL ? NP : NL); ++p) {
            const uint64_t da = umma_desc_sw64(sa + p * C::A_TILE);
            const int nq = NL - p;
            // both K halves of a k-block back to back on the same accumulator columns
            for (int q0 = 0; q0 < nq; q0 += 256 / BN) {
              const int ng = std::min(256 / BN, nq - q0);
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const uint32_t acc = (u > seg_start || p > 0 || k > 0) ? 1u : 0u;
                mma_i8_ws(tmem + (uint32_t)((p + q0) * BN), da + (uint64_t)(k * 2),
                       dv + (uint64_t)((q0 * BN * OZK_KB) >> 4) + (uint64_t)(k * 2), oz_idesc(ng * BN, p == 0, true),
                       acc);
              }
            }
          }
          tc_commit_ws(&aempty[as]);
          tc_commit_ws(&vempty[vs]);
          if (++as == C::A_STAGES) { as = 0; aph ^= 1; }
          if (++vs == C::V_STAGES) { vs = 0; vph ^= 1; }
        }
        tc_commit_ws(tfull);
        acc_phase ^= 1;
      }
    }
  } else if (warp < 6) {
    // ===== epilogue warps 2..5: TMEM int32 levels -> fp64 partial tile (column-major) =====
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t acc_phase = 0;
    long long u = u0;
    while (u < u1) {
      const int vt = (int)(u / kbc);
      u = std::min<long long>(u1, (long long)(vt + 1) * kbc);
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      double* dst = ws + ((size_t)blockIdx.x * max_slots + (vt - vt_first)) * (size_t)(OZ_TM * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        double s[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) s[i] = 0.0;
#pragma unroll 1
        for (int lv = NL - 1; lv >= 0; --lv) {
          int d[16];
          tmem_ld16i(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(lv * BN + c0), d);
          const double w = ldexp(1.0, -8 * lv - 12);
#pragma unroll
          for (int i = 0; i < 16; ++i) s[i] = fma((double)d[i], w, s[i]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[(size_t)(c0 + i) * OZ_TM + row] = s[i];
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  } else {
    // ===== converter warps: A tile (128 rows x 64 entries) -> six digit tiles ===========
    // thread -> (row, 16-entry quarter of the k-block): one 16-byte chunk per digit plane
    const int ct = threadIdx.x - 192;        // 0..511
    const int r = ct >> 2, qt = ct & 3;
    constexpr int EB = FMT == FP8 ? 1 : 2;
    int as = 0;
    uint32_t aph = 0;
    int cur_vt = -1;
    int E = 0;
    float sc = 0.0f;
    bool fast = false, row_ok = false;
    // (tile, k-block) of the next fetch, advanced without 64-bit divisions (they were a
    // fifth of the converters' instructions)
    int fvt = (int)(u0 / kbc), frem = (int)(u0 % kbc);
    // the fetch position's row, chunk start and row base address, refreshed only when the
    // virtual tile changes (no divisions per k-block)
    int fch = fvt % nchunks;
    int64_t fgrow = (int64_t)(fvt / nchunks) * OZ_TM + r;
    const uint8_t* frow = (const uint8_t*)A + (fgrow * lda + qt * 16) * EB;
    auto fetch = [&](long long /*u*/, uint4 (&raw)[2]) {
      const int kb = fch * kbc + frem;
      const int64_t grow = fgrow;
      const uint8_t* src = frow + (int64_t)kb * OZK_KB * EB;
      if (++frem == kbc) {
        frem = 0;
        ++fvt;
        if (++fch == nchunks) { fch = 0; fgrow += OZ_TM; frow += (int64_t)OZ_TM * lda * EB; }
      }
      raw[0] = raw[1] = make_uint4(0, 0, 0, 0);
      if (grow >= rows) return;
      const int64_t l0 = (int64_t)kb * OZK_KB + qt * 16;
      if (l0 + 16 <= cols && ((reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        raw[0] = __ldcs(reinterpret_cast<const uint4*>(src));
        if (EB == 2) raw[1] = __ldcs(reinterpret_cast<const uint4*>(src) + 1);
      } else {
        uint8_t* dst = reinterpret_cast<uint8_t*>(raw);
        for (int e = 0; e < 16; ++e)
          if (l0 + e < cols)
            for (int bb = 0; bb < EB; ++bb) dst[EB * e + bb] = src[EB * e + bb];
      }
    };
    int lvt = (int)(u0 / kbc), lrem = (int)(u0 % kbc);
    const uint32_t abase = smem_u32(abuf);
    // one k-block: convert `raw`, refill it with the entries two k-blocks ahead (`refill`),
    // then wait for the stage and store the digit planes
    auto step = [&](uint4 (&raw)[2], bool refill) {
      const int vt = lvt;
      if (++lrem == kbc) { lrem = 0; ++lvt; }
      if (vt != cur_vt) {
        cur_vt = vt;
        const int64_t grow = (int64_t)(vt / nchunks) * OZ_TM + r;
        row_ok = grow < rows;
        E = row_ok ? Tg[grow] : 0;
        fast = row_ok && E != OZ_BAD && 46 - E <= 127 && 46 - E >= -126;
        sc = fast ? __int_as_float((46 - E + 127) << 23) : 0.0f;
        if constexpr (!full) {                // heads: h = trunc(a 2^(22 - E)) (prepare checked the range)
          fast = row_ok && E != OZ_BAD;
          sc = fast ? __int_as_float((22 - E + 127) << 23) : 0.0f;
        }
      }
      uint32_t w[OZ_D][4];
      if constexpr (!full) {
        // 24-bit heads: byte 2 (signed) and bytes 1, 0 of the int32 h are the three digits
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t hw[4], tw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) hw[e] = (uint32_t)__float2int_rz(ozk_elem<FMT>(raw, 4 * g + e) * sc);
          oz_t4(hw, tw);
          w[0][g] = tw[2];
          w[1][g] = tw[1];
          w[2][g] = tw[0];
        }
      } else if (fast) {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const unsigned long long t = (unsigned long long)__float2ll_rz(ozk_elem<FMT>(raw, 4 * g + e) * sc);
            lo[e] = (uint32_t)t;
            hi[e] = (uint32_t)(t >> 32);
          }
          uint32_t pw[OZ_D];
          oz_planes4u(lo, hi, pw);
#pragma unroll
          for (int p = 0; p < OZ_D; ++p) w[p][g] = pw[p];
        }
      } else {
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint32_t lo[4], hi[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (row_ok && E != OZ_BAD) {
              oz_fixed32(__float_as_uint(ozk_elem<FMT>(raw, 4 * g + e)), E, lo[e], hi[e]);
              // back to the plain two's-complement word (oz_fixed32 returns it biased)
              const unsigned long long t = (((unsigned long long)hi[e] << 32) | lo[e]) - 0x808080808080ull;
              lo[e] = (uint32_t)t;
              hi[e] = (uint32_t)(t >> 32);
            } else {
              lo[e] = 0u;
              hi[e] = 0u;
            }
          }
          uint32_t pw[OZ_D];
          oz_planes4u(lo, hi, pw);
#pragma unroll
          for (int p = 0; p < OZ_D; ++p) w[p][g] = pw[p];
        }
      }
      // the global loads two k-blocks ahead go out now: a one-deep prefetch left the
      // converters waiting on HBM latency every k-block
      if (refill) fetch(0, raw);
      mbar_wait(&aempty[as], aph ^ 1);
      const uint32_t slot = abase + as * C::A_SET;
      const int pos = (r >> 3) * 512 + (r & 7) * 64 + ((qt ^ ((r >> 1) & 3)) << 4);
#pragma unroll
      for (int p = 0; p < OZ_D; ++p)
        if (p < NP) st_shared_v4(slot + p * C::A_TILE + pos, w[p][0], w[p][1], w[p][2], w[p][3]);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[as]);
      if (++as == C::A_STAGES) { as = 0; aph ^= 1; }
    };
    uint4 pa[2], pb[2];
    if (u0 < u1) fetch(u0, pa);
    if (u0 + 1 < u1) fetch(u0 + 1, pb);
    for (long long u = u0; u < u1; u += 2) {
      step(pa, u + 2 < u1);
      if (u + 1 < u1) step(pb, u + 3 < u1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (stamp && threadIdx.x == 0) atomicMax(&g_oz_stamp[1], oz_gtimer_ns());
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---- K7z heads with the digit planes of A in tensor memory ------------------------------
// The shared-memory kernel above moves ~148 KB through shared memory per k-block (A digit
// planes written by the converters and read once per MMA group, V digit tiles written by TMA
// and read by every group): at ~75% of the SM's shared-memory bandwidth that, not the tensor
// pipe, set its pace.  Here the converters store the three head planes straight into TMEM
// (tcgen05.st) and the MMAs take A from there (tcgen05.mma ... [a-tmem]), so shared memory only
// carries the V tiles: 84 KB per k-block, below the MMA floor.  Stages are half k-blocks (the
// 32 entries of one MMA: 8 TMEM columns per plane) in the columns the level accumulators leave
// free.  Heads only (NP = 3); the six-plane variant stays on the shared-memory kernel.
template <int BN, int NL, int EB>
struct OzkTsCfg {
  static constexpr int HALF_COLS = 3 * 8;                  // 3 planes x 32 int8 entries per row
  static constexpr int ACC_COLS = NL * BN;
  static constexpr int A_TSTAGES = (512 - ACC_COLS) / HALF_COLS < 8 ? (512 - ACC_COLS) / HALF_COLS : 8;
  static constexpr int R_SET = OZ_TM * OZK_KB * EB;        // one raw A tile (TMA, 128 / 64 B swizzle)
  static constexpr int R_STAGES = 6;
  static constexpr int V_SET = NL * BN * OZK_KB;
  static constexpr int V_STAGES = (216 * 1024 - R_STAGES * R_SET) / V_SET < 8 ? (216 * 1024 - R_STAGES * R_SET) / V_SET : 8;
  static constexpr int SMEM_BYTES = 1024 + R_STAGES * R_SET + V_STAGES * V_SET + 512;
  static_assert(A_TSTAGES >= 3, "ozk-ts: TMEM stages");
  static_assert(SMEM_BYTES <= 227 * 1024, "ozk-ts shared memory");
};

__device__ __forceinline__ void mma_i8_ts_ws(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
// 16 lanes x 256 bits: thread t -> lanes t/4 (v[0], v[1]) and t/4 + 8 (v[2], v[3]), columns
// 2 (t % 4) and 2 (t % 4) + 1
__device__ __forceinline__ void tmem_st_16x256(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.16x256b.x1.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

static constexpr int OZK_TS_THREADS = OZK_THREADS + 32;   // + warp 22: the raw A producer

template <int FMT, int BN, int NL>
__global__ void __launch_bounds__(OZK_TS_THREADS, 1)
    k_ozk_ts(const __grid_constant__ CUtensorMap tmA, int64_t rows, const int* __restrict__ Tg,
             const __grid_constant__ CUtensorMap tmV, double* __restrict__ ws, int kbc, int nchunks,
             long long total_units, int max_slots, int npad, int col0, int stamp, const int* __restrict__ full_flag) {
  constexpr int EB = FMT == FP8 ? 1 : 2;
  using C = OzkTsCfg<BN, NL, EB>;
  if (full_flag != nullptr && *full_flag != 0) return;     // the operator needs all six planes
  if (stamp && threadIdx.x == 0) atomicMin(&g_oz_stamp[0], oz_gtimer_ns());
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* rbuf = smem;                                  // [R_STAGES][128 rows x 64 entries] raw A
  uint8_t* vbuf = smem + C::R_STAGES * C::R_SET;         // [V_STAGES][NL][BN x 64 B]
  uint64_t* afull = reinterpret_cast<uint64_t*>(vbuf + C::V_STAGES * C::V_SET);
  uint64_t* aempty = afull + C::A_TSTAGES;
  uint64_t* vfull = aempty + C::A_TSTAGES;
  uint64_t* vempty = vfull + C::V_STAGES;
  uint64_t* rfull = vempty + C::V_STAGES;
  uint64_t* rempty = rfull + C::R_STAGES;
  uint64_t* tfull = rempty + C::R_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = warp_index(), lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  const long long u0 = (long long)blockIdx.x * total_units / G;
  const long long u1 = ((long long)blockIdx.x + 1) * total_units / G;
  const int vt_first = (int)(u0 / kbc);

  if (threadIdx.x == 0) {
    // a half-stage is written by the 8 converter warps holding its two 16-entry quarters
    for (int s = 0; s < C::A_TSTAGES; ++s) { mbar_init(&afull[s], OZK_CONV_WARPS / 2); mbar_init(&aempty[s], 1); }
    for (int s = 0; s < C::V_STAGES; ++s) { mbar_init(&vfull[s], 1); mbar_init(&vempty[s], 1); }
    for (int s = 0; s < C::R_STAGES; ++s) { mbar_init(&rfull[s], 1); mbar_init(&rempty[s], OZK_CONV_WARPS); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_barrier_init();
    prefetch_tmap(&tmV);
    prefetch_tmap(&tmA);
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: V digit tiles (the raw A tiles have their own warp: one thread
      // serving both rings held the raw tiles back behind a full V ring) =====
      const uint64_t pol_v = policy_evict_last();
      int vs = 0;
      uint32_t vph = 0;
      int vt = (int)(u0 / kbc), rem = (int)(u0 % kbc);
      for (long long u = u0; u < u1; ++u) {
        const int kb = (vt % nchunks) * kbc + rem;
        if (++rem == kbc) { rem = 0; ++vt; }
        mbar_wait(&vempty[vs], vph ^ 1);
        mbar_expect_tx(&vfull[vs], C::V_SET);
        for (int q = 0; q < NL; ++q)
          tma_load_2d(vbuf + vs * C::V_SET + q * BN * OZK_KB, &tmV, kb * OZK_KB, q * npad + col0, &vfull[vs], pol_v);
        if (++vs == C::V_STAGES) { vs = 0; vph ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ===== MMA issuer (warp-wide loop, elected lane issues) =====
    int hs = 0, vs = 0;
    uint32_t hph = 0, vph = 0, acc_phase = 0;
    long long u = u0;
    while (u < u1) {
      const int vt = (int)(u / kbc);
      const long long seg_end = std::min<long long>(u1, (long long)(vt + 1) * kbc);
      const long long seg_start = u;
      mbar_wait(tempty, acc_phase ^ 1);
      tc_fence_after();
      for (; u < seg_end; ++u) {
        mbar_wait(&vfull[vs], vph);
        const uint64_t dv = umma_desc_sw64(smem_u32(vbuf + vs * C::V_SET));
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&afull[hs], hph);
          tc_fence_after();
          const uint32_t ta = tmem + (uint32_t)(C::ACC_COLS + hs * C::HALF_COLS);
#pragma unroll
          for (int p = 0; p < (NL < 3 ? NL : 3); ++p) {
            const int nq = NL - p;
#pragma unroll
            for (int q0 = 0; q0 < nq; q0 += 256 / BN) {
              const int ng = (256 / BN < nq - q0) ? 256 / BN : nq - q0;
              const uint32_t acc = (u > seg_start || p > 0 || h > 0) ? 1u : 0u;
              mma_i8_ts_ws(tmem + (uint32_t)((p + q0) * BN), ta + (uint32_t)(p * 8),
                           dv + (uint64_t)((q0 * BN * OZK_KB) >> 4) + (uint64_t)(h * 2), oz_idesc(ng * BN, p == 0, true),
                           acc);
            }
          }
          tc_commit_ws(&aempty[hs]);
          if (++hs == C::A_TSTAGES) { hs = 0; hph ^= 1; }
        }
        tc_commit_ws(&vempty[vs]);
        if (++vs == C::V_STAGES) { vs = 0; vph ^= 1; }
      }
      tc_commit_ws(tfull);
      acc_phase ^= 1;
    }
  } else if (warp == 22) {
    if (lane == 0) {
      // ===== TMA producer: raw A tiles =====
      const uint64_t pol_a = policy_evict_first();
      int rs = 0;
      uint32_t rph = 0;
      int vt = (int)(u0 / kbc), rem = (int)(u0 % kbc);
      for (long long u = u0; u < u1; ++u) {
        const int kb = (vt % nchunks) * kbc + rem;
        const int mt = vt / nchunks;
        if (++rem == kbc) { rem = 0; ++vt; }
        mbar_wait(&rempty[rs], rph ^ 1);
        mbar_expect_tx(&rfull[rs], C::R_SET);
        tma_load_2d(rbuf + rs * C::R_SET, &tmA, kb * OZK_KB, mt * OZ_TM, &rfull[rs], pol_a);
        if (++rs == C::R_STAGES) { rs = 0; rph ^= 1; }
      }
    }
  } else if (warp < 6) {
    // ===== epilogue warps 2..5: TMEM int32 levels -> fp64 partial tile (column-major) =====
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    uint32_t acc_phase = 0;
    long long u = u0;
    while (u < u1) {
      const int vt = (int)(u / kbc);
      u = std::min<long long>(u1, (long long)(vt + 1) * kbc);
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      double* dst = ws + ((size_t)blockIdx.x * max_slots + (vt - vt_first)) * (size_t)(OZ_TM * BN);
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 16) {
        double s[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) s[i] = 0.0;
#pragma unroll 1
        for (int lv = NL - 1; lv >= 0; --lv) {
          int d[16];
          tmem_ld16i(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(lv * BN + c0), d);
          const double w = ldexp(1.0, -8 * lv - 12);
#pragma unroll
          for (int i = 0; i < 16; ++i) s[i] = fma((double)d[i], w, s[i]);
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) dst[(size_t)(c0 + i) * OZ_TM + row] = s[i];
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  } else {
    // ===== converter warps: raw A tile (smem) -> three head digit planes in TMEM ==========
    // warp -> TMEM lane quarter Q = warp % 4, half k-block h and 16-lane half of the quarter;
    // one tcgen05.st 16x256b per plane covers its 16 rows x 8 columns (32 entries): thread t
    // holds rows t/4 and t/4 + 8 of them, entries 8(t%4) .. +8 (two TMEM columns).  The raw
    // tile arrives by TMA (a four-deep ring: register prefetch left HBM latency exposed).
    const int cw = warp - 6;                   // 0..15
    const int quarter = warp & 3;
    const int sub = (cw >> 2) & 1;             // 16-lane half of the quarter
    const int h = cw >> 3;                     // half k-block = TMEM stage parity
    const int t0 = lane & 3, t1 = lane >> 2;
    const int r = quarter * 32 + sub * 16 + t1;           // first row; the second is r + 8
    const uint32_t tbase = tmem + ((uint32_t)(quarter * 32 + sub * 16) << 16) + (uint32_t)C::ACC_COLS;
    // byte offsets of this thread's 8 entries in the two rows of a swizzled raw tile
    constexpr int P = OZK_KB * EB;             // row pitch: 128 B (bf16/f16, 128B swizzle), 64 B (fp8)
    auto roff = [&](int row) {
      const int b = (h * 32 + t0 * 8) * EB;
      return row * P + ((((b >> 4) ^ ((row * P >> 7) & (P / 16 - 1)))) << 4) + (b & 15);
    };
    const uint32_t offa = (uint32_t)roff(r), offb = (uint32_t)roff(r + 8);
    const uint32_t rbase = smem_u32(rbuf);
    int hs = h, hph = 0;                       // this warp's half-stage: global half index 2j + h
    int rs = 0;
    uint32_t rph = 0;
    int cur_vt = -1;
    float sca = 0.0f, scb = 0.0f;
    auto elem = [&](const uint4& v, int e) -> float {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
      if constexpr (FMT == BF16) {
        return __uint_as_float(((w[e >> 1] >> (16 * (e & 1))) & 0xffffu) << 16);
      } else if constexpr (FMT == F16) {
        return __half2float(__ushort_as_half((uint16_t)(w[e >> 1] >> (16 * (e & 1)))));
      } else {
        __nv_fp8_e4m3 q;
        q.__x = (uint8_t)(w[e >> 2] >> (8 * (e & 3)));
        return float(q);
      }
    };
    int lvt = (int)(u0 / kbc), lrem = (int)(u0 % kbc);
    for (long long u = u0; u < u1; ++u) {
      const int vt = lvt;
      if (++lrem == kbc) { lrem = 0; ++lvt; }
      if (vt != cur_vt) {
        cur_vt = vt;
        // heads: h = trunc(a 2^(22 - E)) (the prepare pass checked the range)
        const int64_t ga = (int64_t)(vt / nchunks) * OZ_TM + r;
        const int Ea = ga < rows ? Tg[ga] : OZ_BAD;
        const int Eb = ga + 8 < rows ? Tg[ga + 8] : OZ_BAD;
        sca = Ea != OZ_BAD ? __int_as_float((22 - Ea + 127) << 23) : 0.0f;
        scb = Eb != OZ_BAD ? __int_as_float((22 - Eb + 127) << 23) : 0.0f;
      }
      uint4 raw[2];
      mbar_wait(&rfull[rs], rph);
      const uint32_t rb = rbase + rs * C::R_SET;
      if constexpr (EB == 2) {
        raw[0] = ld_shared_v4(rb + offa);
        raw[1] = ld_shared_v4(rb + offb);
      } else {
        const uint2 qa = ld_shared_v2(rb + offa), qb = ld_shared_v2(rb + offb);
        raw[0] = make_uint4(qa.x, qa.y, 0, 0);
        raw[1] = make_uint4(qb.x, qb.y, 0, 0);
      }
      // w[p] = {row a: columns 2 t0, 2 t0 + 1; row b: the same columns}
      uint32_t w[3][4];
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const float sc = rr == 0 ? sca : scb;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          uint32_t hw[4], tw[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) hw[e] = (uint32_t)__float2int_rz(elem(raw[rr], 4 * g + e) * sc);
          oz_t4(hw, tw);
          w[0][2 * rr + g] = tw[2];
          w[1][2 * rr + g] = tw[1];
          w[2][2 * rr + g] = tw[0];
        }
      }
      mbar_wait(&aempty[hs], hph ^ 1);
      tc_fence_after();
      const uint32_t ta = tbase + (uint32_t)(hs * C::HALF_COLS);
      tmem_st_16x256(ta, w[0]);
      tmem_st_16x256(ta + 8, w[1]);
      tmem_st_16x256(ta + 16, w[2]);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      // both stages are released only after the TMEM stores completed: their source registers
      // (hence the shared loads of the raw stage) are then consumed for certain
      if (lane == 0) {
        mbar_arrive(&afull[hs]);
        mbar_arrive(&rempty[rs]);
      }
      if (++rs == C::R_STAGES) { rs = 0; rph ^= 1; }
      hs += 2;
      if (hs >= C::A_TSTAGES) { hs -= C::A_TSTAGES; hph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (stamp && threadIdx.x == 0) atomicMax(&g_oz_stamp[1], oz_gtimer_ns());
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

__device__ __forceinline__ long long oz_seg_begin(long long c, long long T, long long G) { return c * T / G; }

// Sum the partials of row tile t over its K chunks and stream-K segments (fixed order),
// scale to (A V)_ij and form the residual column sums of squares of this tile:
//   part[t * ldp + j0 + j] = sum_i ((A V)_ij - lambda_j Y_ij)^2
// (with W: write W = A V (fp64) instead).  One thread per row, 16 columns at a time.
__global__ void __launch_bounds__(OZ_TM)
    k_oz_resid(const double* __restrict__ ws, int BN, int kbc, int nchunks, long long total_units, int G,
               int max_slots, int64_t rows, int ncols, int j0, const int* __restrict__ T, const int* __restrict__ F,
               const double* __restrict__ vals, const int* __restrict__ r_dev, const double* __restrict__ Y,
               int64_t ldy, double* __restrict__ part, int ldp, void* __restrict__ W, int64_t ldw, int out_fmt,
               double* __restrict__ colmax, int* __restrict__ flags, void* __restrict__ W2, int64_t ldw2,
               int out_fmt2, int stamp, const int* __restrict__ full, const double* __restrict__ Wt,
               int kbc_h, int nchunks_h, long long total_h, int slots_h) {
  __shared__ double red[4][OZR_CG];
  // the heads variant ran (full == 0): its own, longer chunks
  if (full && !*full) {
    kbc = kbc_h;
    nchunks = nchunks_h;
    total_units = total_h;
    max_slots = slots_h;
  }
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {   // the product kernel is done
    const unsigned long long t0 = g_oz_stamp[0], t1 = g_oz_stamp[1];
    if (t1 > t0) {
      g_oz_stamp[2] += t1 - t0;
      g_oz_stamp[3] += 1;
      g_oz_stamp[2 + 2 * stamp] += t1 - t0;
      g_oz_stamp[3 + 2 * stamp] += 1;
    }
    g_oz_stamp[0] = ~0ull;
    g_oz_stamp[1] = 0ull;
  }
  const int t = blockIdx.x;
  const int row = threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t grow = (int64_t)t * OZ_TM + row;
  const bool valid = grow < rows;
  const int Ti = valid ? T[grow] : 0;
  const int nvalid = r_dev ? min(j0 + ncols, *r_dev) : j0 + ncols;
  // the partial tiles of this row tile (per chunk, the CTA segments covering it, in
  // ascending order): thread 0 resolves them once per block (64-bit divisions), every thread
  // reads the table -- the summation order is unchanged
  constexpr int MAXE = 512;
  __shared__ long long s_base[MAXE];
  __shared__ int s_ne;
  if (threadIdx.x == 0) {
    int ne = 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      const long long vt = (long long)t * nchunks + ch;
      const long long x0 = vt * kbc, x1 = x0 + kbc - 1;
      long long lo = x0 * G / total_units, hi = x1 * G / total_units;
      while (lo + 1 < G && oz_seg_begin(lo + 1, total_units, G) <= x0) ++lo;
      while (lo > 0 && oz_seg_begin(lo, total_units, G) > x0) --lo;
      while (hi + 1 < G && oz_seg_begin(hi + 1, total_units, G) <= x1) ++hi;
      while (hi > 0 && oz_seg_begin(hi, total_units, G) > x1) --hi;
      for (long long c = lo; c <= hi; ++c) {
        const int slot = (int)(vt - oz_seg_begin(c, total_units, G) / kbc);
        if (ne < MAXE) s_base[ne] = ((long long)c * max_slots + slot) * (long long)(OZ_TM * BN);
        ++ne;
      }
    }
    s_ne = ne;
  }
  __syncthreads();
  const int ne = s_ne;
  // the exact fp64 tail products of this row (3-digit heads in the product kernel)
  const double* wt = (Wt && valid && !*full) ? Wt + grow * BN : nullptr;
  for (int jb = OZR_CG * blockIdx.y; jb < ncols; jb += OZR_CG * gridDim.y) {   // OZR_CG columns per y-block
    double s[OZR_CG], tl[OZR_CG];
#pragma unroll
    for (int q = 0; q < OZR_CG; ++q) {
      s[q] = 0.0;
      tl[q] = (wt && jb + q < ncols) ? wt[jb + q] : 0.0;
    }
    if (ne <= MAXE) {
      for (int e = 0; e < ne; ++e) {
        const double* src = ws + s_base[e] + row;
#pragma unroll
        for (int q = 0; q < OZR_CG; ++q)
          if (jb + q < ncols) s[q] += src[(size_t)(jb + q) * OZ_TM];
      }
    } else {                                  // more segments than the table: resolve per thread
      for (int ch = 0; ch < nchunks; ++ch) {
        const long long vt = (long long)t * nchunks + ch;
        const long long x0 = vt * kbc, x1 = x0 + kbc - 1;
        long long lo = x0 * G / total_units, hi = x1 * G / total_units;
        while (lo + 1 < G && oz_seg_begin(lo + 1, total_units, G) <= x0) ++lo;
        while (lo > 0 && oz_seg_begin(lo, total_units, G) > x0) --lo;
        while (hi + 1 < G && oz_seg_begin(hi + 1, total_units, G) <= x1) ++hi;
        while (hi > 0 && oz_seg_begin(hi, total_units, G) > x1) --hi;
        for (long long c = lo; c <= hi; ++c) {
          const int slot = (int)(vt - oz_seg_begin(c, total_units, G) / kbc);
          const double* src = ws + ((size_t)c * max_slots + slot) * (size_t)(OZ_TM * BN) + row;
#pragma unroll
          for (int q = 0; q < OZR_CG; ++q)
            if (jb + q < ncols) s[q] += src[(size_t)(jb + q) * OZ_TM];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < OZR_CG; ++q) {
      const int j = jb + q, gj = j0 + j;
      double r2 = 0.0;
      if (valid && j < ncols && gj < nvalid) {
        const int Fj = F[j];
        const double av = (Ti == OZ_BAD || Fj == OZ_BAD) ? __longlong_as_double(0x7ff8000000000000ll)
                                                          : ldexp(s[q], Ti + Fj) + tl[q];
        if (W) {
          // the product rounded to the output format; r2 carries |w| for the column max
          const double w = rnd(av, out_fmt);
          st_fmt(W, (long)((int64_t)gj * ldw + grow), out_fmt, w);
          if (W2) st_fmt(W2, (long)((int64_t)gj * ldw2 + grow), out_fmt2, rnd(av, out_fmt2));
          if (!isfinite(w) && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
          r2 = (w != w) ? INFINITY : fabs(w);
        } else {
          const double d = av - vals[gj] * Y[(int64_t)gj * ldy + grow];
          r2 = d * d;
        }
      }
      if (W) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2 = fmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      }
      if (lane == 0) red[warp][q] = r2;
    }
    __syncthreads();
    if (threadIdx.x < OZR_CG && jb + threadIdx.x < ncols) {
      const double* rr = &red[0][0];
      if (W) {
        const double m = fmax(fmax(rr[threadIdx.x], rr[OZR_CG + threadIdx.x]),
                              fmax(rr[2 * OZR_CG + threadIdx.x], rr[3 * OZR_CG + threadIdx.x]));
        if (colmax) atomic_max_nonneg(&colmax[j0 + jb + threadIdx.x], m);
      } else {
        part[(int64_t)t * ldp + j0 + jb + threadIdx.x] =
            ((red[0][threadIdx.x] + red[1][threadIdx.x]) + red[2][threadIdx.x]) + red[3][threadIdx.x];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_oz)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int oz_make_tmap_u8(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                    uint32_t box_inner, uint32_t box_outer);   // gemm_tc.cu

struct OzPlan {
  int bn, npass, m_tiles, kblocks, nchunks, kbc, grid, max_slots;
  int64_t rows_pad, cols_pad;
  int npad;
  long long total;
  // operator workspace (per A): row scales + digit planes
  size_t op_T, op_planes, op_bytes;
  // product workspace (per call): column scales, digits of V, partials, residual partials
  size_t off_F, off_dig, off_ws, off_part, bytes;
};

static OzPlan oz_plan(int64_t rows, int64_t cols, int r) {
  OzPlan p;
  r = std::max(r, 1);
  p.bn = r <= 32 ? 32 : 64;
  p.npass = (r + p.bn - 1) / p.bn;
  p.npad = p.npass * p.bn;
  p.rows_pad = (rows + OZ_TM - 1) / OZ_TM * OZ_TM;
  p.cols_pad = (cols + 15) / 16 * 16;
  p.m_tiles = (int)(p.rows_pad / OZ_TM);
  p.kblocks = (int)((cols + OZ_KB - 1) / OZ_KB);
  p.nchunks = (p.kblocks + OZ_MAXCHUNK - 1) / OZ_MAXCHUNK;
  p.kbc = (p.kblocks + p.nchunks - 1) / p.nchunks;
  p.total = (long long)p.m_tiles * p.nchunks * p.kbc;   // work units (k-blocks)
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  p.grid = (int)std::max<long long>(1, std::min<long long>(sms, p.total));
  const long long per = (p.total + p.grid - 1) / p.grid;
  p.max_slots = (int)((per + p.kbc - 1) / p.kbc) + 1;
  size_t b = 0;
  auto take = [&](size_t n) { size_t o = b; b += (n + 1023) & ~size_t(1023); return o; };
  p.op_T = take((size_t)p.rows_pad * 4);
  p.op_planes = take((size_t)OZ_D * p.rows_pad * p.cols_pad);
  p.op_bytes = b;
  b = 0;
  p.off_F = take((size_t)p.npad * 4);
  p.off_dig = take((size_t)OZ_D * p.npad * p.cols_pad);
  p.off_ws = take((size_t)p.grid * p.max_slots * OZ_TM * p.bn * sizeof(double));
  p.off_part = take((size_t)p.m_tiles * r * sizeof(double));
  p.bytes = b;
  return p;
}

size_t oz_op_ws(int64_t rows, int64_t cols) { return oz_plan(rows, cols, 1).op_bytes; }
size_t oz_prod_ws(int64_t rows, int64_t cols, int r) { return oz_plan(rows, cols, r).bytes; }
// one-shot workspace (operator + product) of the residual entry points
size_t ozx_op_ws(int64_t rows, int64_t cols);
size_t ozx_prod_ws(int64_t rows, int64_t cols, int r);
size_t oz_ws(int64_t rows, int64_t cols, int r) {
  return ((ozx_op_ws(rows, cols) + 1023) & ~size_t(1023)) + ozx_prod_ws(rows, cols, r);
}
int oz_nblocks(int64_t rows) { return (int)((rows + OZ_TM - 1) / OZ_TM); }

template <int BN>
static int oz_launch(const CUtensorMap& tA, const CUtensorMap& tV, const OzPlan& p, double* ws, int col0,
                     cudaStream_t st) {
  using C = OzCfg<BN>;
  static std::atomic<bool> attr{false};   // set once; concurrent callers may both set it (idempotent)
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_oz_gemm<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr = true;
  }
  k_oz_gemm<BN><<<p.grid, OZ_THREADS, C::SMEM_BYTES, st>>>(tA, tV, ws, p.kbc, p.nchunks, p.total, p.max_slots,
                                                           (int)p.rows_pad, p.npad, col0);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// K7z stage 1: the row scales and digit planes of A (rows x cols row-major, F16 / BF16 /
// FP8) into the operator workspace; reusable for any number of products with this A.
int oz_prepare(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, void* op_ws, size_t op_bytes,
               cudaStream_t st) {
  if (a_fmt != BF16 && a_fmt != F16 && a_fmt != FP8) {
    ofrr_set_error("ozaki: A format %d not supported (16/8-bit operators)", a_fmt);
    return OFRR_ERR_UNSUPPORTED;
  }
  const OzPlan p = oz_plan(rows, cols, 1);
  if (!op_ws || op_bytes < p.op_bytes) { ofrr_set_error("ozaki: operator workspace too small (%zu < %zu)", op_bytes, p.op_bytes); return OFRR_ERR_INVALID; }
  uint8_t* base = (uint8_t*)op_ws;
  int* T = (int*)(base + p.op_T);
  int8_t* planes = (int8_t*)(base + p.op_planes);
  if (a_fmt == BF16)
    k_oz_slices_a<BF16><<<(unsigned)p.rows_pad, 256, 0, st>>>(A, rows, cols, lda, T, planes, p.rows_pad, p.cols_pad);
  else if (a_fmt == F16)
    k_oz_slices_a<F16><<<(unsigned)p.rows_pad, 256, 0, st>>>(A, rows, cols, lda, T, planes, p.rows_pad, p.cols_pad);
  else
    k_oz_slices_a<FP8><<<(unsigned)p.rows_pad, 256, 0, st>>>(A, rows, cols, lda, T, planes, p.rows_pad, p.cols_pad);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// K7z stage 2: (A V) with a prepared operator.  Residual mode (W == nullptr):
// part[m_tile * r + j] = sum over the tile's rows of ((A V)_ij - vals_j Y_ij)^2.  Product
// mode: W = A V rounded to out_fmt (+ W2 in out_fmt2, colmax |= max |W|, flags on non-finite).
int oz_apply(const void* op_ws, int64_t rows, int64_t cols, const double* V, int64_t ldv, int r,
             const double* vals, const int* r_dev, const double* Y, int64_t ldy, void* W, int64_t ldw, int out_fmt,
             double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2, double** part_out, void* ws,
             size_t ws_bytes, cudaStream_t st) {
  const OzPlan p = oz_plan(rows, cols, r);
  if (!ws || ws_bytes < p.bytes) { ofrr_set_error("ozaki: workspace too small (%zu < %zu)", ws_bytes, p.bytes); return OFRR_ERR_INVALID; }
  const uint8_t* obase = (const uint8_t*)op_ws;
  const int* T = (const int*)(obase + p.op_T);
  const int8_t* planes = (const int8_t*)(obase + p.op_planes);
  uint8_t* base = (uint8_t*)ws;
  int* F = (int*)(base + p.off_F);
  int8_t* dig = (int8_t*)(base + p.off_dig);
  double* pws = (double*)(base + p.off_ws);
  double* part = (double*)(base + p.off_part);
  k_oz_slices_v<<<(unsigned)p.npad, 256, 0, st>>>(V, ldv, cols, r, F, dig, p.npad, p.cols_pad);
  OFRR_CHECK_LAUNCH();
  CUtensorMap tA, tV;
  int rc = oz_make_tmap_u8(&tA, planes, (uint64_t)cols, (uint64_t)OZ_D * p.rows_pad, (uint64_t)p.cols_pad, OZ_KB, OZ_TM);
  if (rc) return rc;
  rc = oz_make_tmap_u8(&tV, dig, (uint64_t)cols, (uint64_t)OZ_D * p.npad, (uint64_t)p.cols_pad, OZ_KB, (uint32_t)p.bn);
  if (rc) return rc;
  for (int ps = 0; ps < p.npass; ++ps) {
    const int j0 = ps * p.bn;
    rc = p.bn == 32 ? oz_launch<32>(tA, tV, p, pws, j0, st) : oz_launch<64>(tA, tV, p, pws, j0, st);
    if (rc) return rc;
    k_oz_resid<<<dim3(p.m_tiles, (unsigned)((std::min(p.bn, r - j0) + OZR_CG - 1) / OZR_CG)), OZ_TM, 0, st>>>(pws, p.bn, p.kbc, p.nchunks, p.total, p.grid, p.max_slots, rows,
                                           std::min(p.bn, r - j0), j0, T, F + j0, vals, r_dev, Y, ldy, part, r, W,
                                           ldw, out_fmt, colmax, flags, W2, ldw2, out_fmt2, g_oz_stamp_on ? 1 : 0, nullptr, nullptr,
                                           p.kbc, p.nchunks, p.total, p.max_slots);
    OFRR_CHECK_LAUNCH();
  }
  if (part_out) *part_out = part;
  return OFRR_OK;
}

// ---- in-kernel slicing path (default): operator workspace = row scales only ----------
int oz_make_tmap_a(CUtensorMap* tm, const void* base, int a_fmt, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                   uint32_t box_inner, uint32_t box_outer);
int oz_make_tmap_u8_sw64(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                         uint32_t box_inner, uint32_t box_outer);   // gemm_tc.cu

static bool oz_use_planes() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("OFRR_OZ_PLANES"); v = (e && atoi(e) == 1) ? 1 : 0; }
  return v == 1;
}

struct OzkPlan {
  int bn, npass, npad, m_tiles, kblocks, nchunks, kbc, grid, max_slots, ldvt;
  int nchunks_h, kbc_h, slots_h;      // the heads variants' chunking (OZK_MAXCHUNK_H)
  int64_t rows_pad, cols_pad;
  long long total, total_h;
  size_t off_F, off_dig, off_ws, off_part, off_vt, off_wt, off_vmax, bytes;
};

// OFRR_OZK_TMEM_A=0: the heads on the shared-memory kernel (comparison runs)
static bool ozk_use_tmem_a() {       // read per launch: the tests compare both kernels in one process
  const char* e = getenv("OFRR_OZK_TMEM_A");
  return !(e && e[0] == '0');
}

static OzkPlan ozk_plan(int64_t rows, int64_t cols, int r, int levels = OZ_D) {
  OzkPlan p;
  r = std::max(r, 1);
  // lite tier: 128-column passes on the shared-memory kernel (64-column passes with the digit
  // planes in TMEM read A twice: 5.2 vs 4.4 ms per A pass at C3)
  static int lite_bn = -1;                 // OFRR_OZK_LITE_BN=64: lite passes of 64 columns (comparison runs)
  if (lite_bn < 0) { const char* e = getenv("OFRR_OZK_LITE_BN"); lite_bn = e ? atoi(e) : 128; }
  p.bn = levels >= 5 ? (r <= 32 ? 32 : 64) : (r <= 64 || lite_bn == 64 ? 64 : 128);
  p.npass = (r + p.bn - 1) / p.bn;
  p.npad = p.npass * p.bn;
  p.rows_pad = (rows + OZ_TM - 1) / OZ_TM * OZ_TM;
  p.cols_pad = (cols + 15) / 16 * 16;
  p.m_tiles = (int)(p.rows_pad / OZ_TM);
  p.kblocks = (int)((cols + OZK_KB - 1) / OZK_KB);
  p.nchunks = (p.kblocks + OZK_MAXCHUNK - 1) / OZK_MAXCHUNK;
  p.kbc = (p.kblocks + p.nchunks - 1) / p.nchunks;
  p.total = (long long)p.m_tiles * p.nchunks * p.kbc;
  p.nchunks_h = (p.kblocks + OZK_MAXCHUNK_H - 1) / OZK_MAXCHUNK_H;
  p.kbc_h = (p.kblocks + p.nchunks_h - 1) / p.nchunks_h;
  p.total_h = (long long)p.m_tiles * p.nchunks_h * p.kbc_h;
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  p.grid = (int)std::max<long long>(1, std::min<long long>(sms, std::min(p.total, p.total_h)));
  const long long per = (p.total + p.grid - 1) / p.grid;
  p.max_slots = (int)((per + p.kbc - 1) / p.kbc) + 1;
  const long long per_h = (p.total_h + p.grid - 1) / p.grid;
  p.slots_h = (int)((per_h + p.kbc_h - 1) / p.kbc_h) + 1;
  size_t b = 0;
  auto take = [&](size_t n) { size_t o = b; b += (n + 1023) & ~size_t(1023); return o; };
  p.off_F = take((size_t)p.npad * 4);
  p.off_dig = take((size_t)OZ_D * p.npad * p.cols_pad);
  p.off_ws = take((size_t)p.grid * std::max(p.max_slots, p.slots_h) * OZ_TM * p.bn * sizeof(double));
  p.off_part = take((size_t)p.m_tiles * r * sizeof(double));
  p.ldvt = p.npad;
  p.off_vt = take((size_t)cols * p.ldvt * sizeof(double));     // V row-major for the tails
  p.off_wt = take((size_t)p.rows_pad * p.bn * sizeof(double));  // tails x V of one column pass
  p.off_vmax = take((size_t)p.npad * sizeof(unsigned long long));   // column maxima of |V| (bits)
  p.bytes = b;
  return p;
}

template <int FMT, int BN, int NL>
static int ozk_launch(const void* A, int64_t rows, int64_t cols, int64_t lda, const int* T, const CUtensorMap& tV,
                      const OzkPlan& p, double* ws, int col0, const int* full, cudaStream_t st) {
  using C3 = OzkCfg<BN, 3, NL>;
  using C = OzkCfg<BN, OZ_D, NL>;
  static std::once_flag attr;
  cudaError_t ae = cudaSuccess;
  std::call_once(attr, [&] {
    ae = cudaFuncSetAttribute(k_ozk_gemm<FMT, BN, 3, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, C3::SMEM_BYTES);
    if (ae == cudaSuccess)
      ae = cudaFuncSetAttribute(k_ozk_gemm<FMT, BN, OZ_D, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::SMEM_BYTES);
  });
  OFRR_CUDA_TRY(ae);
  const int stamp = g_oz_stamp_on ? 1 : 0;
  if (full) {
    bool ts = false;
    if constexpr (NL * BN <= 384) {
      CUtensorMap tA;
      // TMA needs a 16-byte aligned base and row pitch; otherwise the shared-memory kernel
      const int eb = FMT == FP8 ? 1 : 2;
      if (ozk_use_tmem_a() && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && ((uint64_t)lda * eb) % 16 == 0 &&
          oz_make_tmap_a(&tA, A, FMT, (uint64_t)cols, (uint64_t)rows, (uint64_t)lda, OZK_KB, OZ_TM) == OFRR_OK) {
        using CT = OzkTsCfg<BN, NL, FMT == FP8 ? 1 : 2>;
        static std::once_flag attr_ts;
        std::call_once(attr_ts, [&] {
          ae = cudaFuncSetAttribute(k_ozk_ts<FMT, BN, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, CT::SMEM_BYTES);
        });
        OFRR_CUDA_TRY(ae);
        k_ozk_ts<FMT, BN, NL><<<p.grid, OZK_TS_THREADS, CT::SMEM_BYTES, st>>>(tA, rows, T, tV, ws, p.kbc_h,
                                                                         p.nchunks_h, p.total_h, p.slots_h, p.npad,
                                                                         col0, stamp,
                                                                         full);
        OFRR_CHECK_LAUNCH();
        ts = true;
      }
    }
    if (!ts) {
      k_ozk_gemm<FMT, BN, 3, NL><<<p.grid, OZK_THREADS, C3::SMEM_BYTES, st>>>(A, rows, cols, lda, T, tV, ws, p.kbc_h,
                                                                             p.nchunks_h, p.total_h, p.slots_h, p.npad,
                                                                             col0, stamp, full);
      OFRR_CHECK_LAUNCH();
    }
  }
  k_ozk_gemm<FMT, BN, OZ_D, NL><<<p.grid, OZK_THREADS, C::SMEM_BYTES, st>>>(A, rows, cols, lda, T, tV, ws, p.kbc,
                                                                           p.nchunks, p.total, p.max_slots, p.npad,
                                                                           col0, stamp, full);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

size_t ozx_op_ws(int64_t rows, int64_t cols) {
  return oz_use_planes() ? oz_plan(rows, cols, 1).op_bytes : oz_op_layout(rows).bytes + 1024;
}
static bool oz_no_tails() {     // OFRR_OZ_FULL=1: all six digits of A in every product (diagnostics)
  static int v = -1;
  if (v < 0) { const char* e = getenv("OFRR_OZ_FULL"); v = (e && atoi(e) == 1) ? 1 : 0; }
  return v == 1;
}
size_t ozx_prod_ws(int64_t rows, int64_t cols, int r) {
  // sized for either product accuracy (6 levels, 64-column passes; 4 levels, 128-column passes)
  return oz_use_planes() ? oz_plan(rows, cols, r).bytes
                         : std::max(ozk_plan(rows, cols, r).bytes, ozk_plan(rows, cols, r, 4).bytes);
}

int ozx_info(const void* op_ws, int64_t rows, int* full, long long* tails) {
  if (oz_use_planes()) { *full = 1; *tails = 0; return OFRR_OK; }
  const OzOpLayout L = oz_op_layout(rows);
  const uint8_t* b = (const uint8_t*)op_ws;
  OFRR_CUDA_TRY(cudaDeviceSynchronize());
  OFRR_CUDA_TRY(cudaMemcpy(full, b + L.off_full, sizeof(int), cudaMemcpyDeviceToHost));
  std::vector<int> c((size_t)rows);
  OFRR_CUDA_TRY(cudaMemcpy(c.data(), b + L.off_cnt, (size_t)rows * sizeof(int), cudaMemcpyDeviceToHost));
  long long t = 0;
  for (int v : c) t += v;
  *tails = t;
  return OFRR_OK;
}

int ozx_prepare(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, void* op_ws, size_t op_bytes,
                cudaStream_t st) {
  if (oz_use_planes()) return oz_prepare(A, rows, cols, lda, a_fmt, op_ws, op_bytes, st);
  if (a_fmt != BF16 && a_fmt != F16 && a_fmt != FP8) {
    ofrr_set_error("ozaki: A format %d not supported (16/8-bit operators)", a_fmt);
    return OFRR_ERR_UNSUPPORTED;
  }
  if (!op_ws || op_bytes < ozx_op_ws(rows, cols)) { ofrr_set_error("ozaki: operator workspace too small"); return OFRR_ERR_INVALID; }
  const OzOpLayout L = oz_op_layout(rows);
  const unsigned g = (unsigned)L.rows_pad;
  uint8_t* b = (uint8_t*)op_ws;
  int* T = (int*)(b + L.off_T);
  int* full = (int*)(b + L.off_full);
  int* tcnt = (int*)(b + L.off_cnt);
  int* tcol = (int*)(b + L.off_col);
  float* tval = (float*)(b + L.off_val);
  const int one = oz_no_tails() ? 1 : 0;
  const size_t gbytes = (size_t)((cols + 31) / 32) * sizeof(int);   // per-group minimum exponents (pass 1 -> pass 2)
  if (gbytes > 48 * 1024) {
    static std::once_flag big;
    cudaError_t e = cudaSuccess;
    std::call_once(big, [&] {
      e = cudaFuncSetAttribute(k_oz_rowscale<BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k_oz_rowscale<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e == cudaSuccess) e = cudaFuncSetAttribute(k_oz_rowscale<FP8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    OFRR_CUDA_TRY(e);
    if (gbytes > 200 * 1024) { ofrr_set_error("ozaki: %lld columns exceed the row-scale pass", (long long)cols); return OFRR_ERR_UNSUPPORTED; }
  }
  OFRR_CUDA_TRY(cudaMemsetAsync(full, 0, sizeof(int), st));
  if (one) OFRR_CUDA_TRY(cudaMemsetAsync(full, 0x01, 1, st));
  if (a_fmt == BF16) k_oz_rowscale<BF16><<<g, OZ_RS_THREADS, gbytes, st>>>(A, rows, cols, lda, T, full, tcnt, tcol, tval);
  else if (a_fmt == F16) k_oz_rowscale<F16><<<g, OZ_RS_THREADS, gbytes, st>>>(A, rows, cols, lda, T, full, tcnt, tcol, tval);
  else k_oz_rowscale<FP8><<<g, OZ_RS_THREADS, gbytes, st>>>(A, rows, cols, lda, T, full, tcnt, tcol, tval);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

int ozx_apply(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* op_ws, const double* V,
              int64_t ldv, int r, const double* vals, const int* r_dev, const double* Y, int64_t ldy, void* W,
              int64_t ldw, int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
              double** part_out, void* ws, size_t ws_bytes, cudaStream_t st, int levels) {
  if (levels < 3 || levels > OZ_D) {
    ofrr_set_error("ozaki: levels must be 3..6 (got %d)", levels);
    return OFRR_ERR_INVALID;
  }
  if (oz_use_planes())
    return oz_apply(op_ws, rows, cols, V, ldv, r, vals, r_dev, Y, ldy, W, ldw, out_fmt, colmax, flags, W2, ldw2,
                    out_fmt2, part_out, ws, ws_bytes, st);
  const OzkPlan p = ozk_plan(rows, cols, r, levels);
  if (!ws || ws_bytes < p.bytes) { ofrr_set_error("ozaki: workspace too small (%zu < %zu)", ws_bytes, p.bytes); return OFRR_ERR_INVALID; }
  const OzOpLayout OL = oz_op_layout(rows);
  const uint8_t* ob = (const uint8_t*)op_ws;
  const int* T = (const int*)(ob + OL.off_T);
  const int* full = (const int*)(ob + OL.off_full);
  const int* tcnt = (const int*)(ob + OL.off_cnt);
  const int* tcol = (const int*)(ob + OL.off_col);
  const float* tval = (const float*)(ob + OL.off_val);
  uint8_t* base = (uint8_t*)ws;
  int* F = (int*)(base + p.off_F);
  int8_t* dig = (int8_t*)(base + p.off_dig);
  double* pws = (double*)(base + p.off_ws);
  double* part = (double*)(base + p.off_part);
  double* Vt = (double*)(base + p.off_vt);
  double* Wt = (double*)(base + p.off_wt);
  {
    unsigned long long* vmax = (unsigned long long*)(base + p.off_vmax);
    const int64_t seg = 4096;                                   // multiple of 4 (digit groups)
    const unsigned nseg = (unsigned)((p.cols_pad + seg - 1) / seg);
    OFRR_CUDA_TRY(cudaMemsetAsync(vmax, 0, (size_t)p.npad * sizeof(unsigned long long), st));
    k_oz_vmax<<<dim3((unsigned)p.npad, nseg), 256, 0, st>>>(V, ldv, cols, r, vmax, seg);
    OFRR_CHECK_LAUNCH();
    k_oz_slices_vs<<<dim3((unsigned)p.npad, nseg), 256, 0, st>>>(V, ldv, cols, r, vmax, F, dig, p.npad, p.cols_pad,
                                                                 seg);
    OFRR_CHECK_LAUNCH();
  }
  k_oz_vt<<<dim3((unsigned)((cols + 31) / 32), (unsigned)((r + 31) / 32)), 256, 0, st>>>(V, ldv, cols, r, Vt, p.ldvt);
  OFRR_CHECK_LAUNCH();
  CUtensorMap tV;
  int rc = oz_make_tmap_u8_sw64(&tV, dig, (uint64_t)cols, (uint64_t)OZ_D * p.npad, (uint64_t)p.cols_pad, OZK_KB,
                                (uint32_t)p.bn);
  if (rc) return rc;
  for (int ps = 0; ps < p.npass; ++ps) {
    const int j0 = ps * p.bn;
#define OZK_CASE(F)                                                                              \
    if (levels == OZ_D)                                                                          \
      rc = p.bn == 32 ? ozk_launch<F, 32, OZ_D>(A, rows, cols, lda, T, tV, p, pws, j0, full, st)  \
                      : ozk_launch<F, 64, OZ_D>(A, rows, cols, lda, T, tV, p, pws, j0, full, st); \
    else if (levels == 5)                                                                        \
      rc = p.bn == 32 ? ozk_launch<F, 32, 5>(A, rows, cols, lda, T, tV, p, pws, j0, full, st)     \
                      : ozk_launch<F, 64, 5>(A, rows, cols, lda, T, tV, p, pws, j0, full, st);    \
    else if (levels == 3)                                                                        \
      rc = p.bn == 64 ? ozk_launch<F, 64, 3>(A, rows, cols, lda, T, tV, p, pws, j0, full, st)     \
                      : ozk_launch<F, 128, 3>(A, rows, cols, lda, T, tV, p, pws, j0, full, st);   \
    else                                                                                         \
      rc = p.bn == 64 ? ozk_launch<F, 64, 4>(A, rows, cols, lda, T, tV, p, pws, j0, full, st)     \
                      : ozk_launch<F, 128, 4>(A, rows, cols, lda, T, tV, p, pws, j0, full, st);
    if (a_fmt == BF16) { OZK_CASE(BF16) } else if (a_fmt == F16) { OZK_CASE(F16) } else { OZK_CASE(FP8) }
#undef OZK_CASE
    if (rc) return rc;
    k_oz_tailmul<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, full, tcnt, tcol, tval, Vt, p.ldvt, j0,
                                                             std::min(p.bn, r - j0), p.bn, Wt);
    OFRR_CHECK_LAUNCH();
    k_oz_resid<<<dim3(p.m_tiles, (unsigned)((std::min(p.bn, r - j0) + OZR_CG - 1) / OZR_CG)), OZ_TM, 0, st>>>(pws, p.bn, p.kbc, p.nchunks, p.total, p.grid, p.max_slots, rows,
                                           std::min(p.bn, r - j0), j0, T, F + j0, vals, r_dev, Y, ldy, part, r, W,
                                           ldw, out_fmt, colmax, flags, W2, ldw2, out_fmt2,
                                           g_oz_stamp_on ? (levels == OZ_D ? 1 : levels == 5 ? 3 : 2) : 0, full, Wt,
                                           p.kbc_h, p.nchunks_h, p.total_h, p.slots_h);
    OFRR_CHECK_LAUNCH();
  }
  if (part_out) *part_out = part;
  return OFRR_OK;
}

// one-shot residual product (prepare + apply in one workspace)
int oz_product(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const double* V, int64_t ldv,
               int r, const double* vals, const int* r_dev, const double* Y, int64_t ldy, double* W, int64_t ldw,
               double** part_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  const size_t opb = (ozx_op_ws(rows, cols) + 1023) & ~size_t(1023);
  const size_t pb = ozx_prod_ws(rows, cols, r);
  if (!ws || ws_bytes < opb + pb) { ofrr_set_error("ozaki product: workspace too small (%zu < %zu)", ws_bytes, opb + pb); return OFRR_ERR_INVALID; }
  int rc = ozx_prepare(A, rows, cols, lda, a_fmt, ws, opb, st);
  if (rc) return rc;
  return ozx_apply(A, rows, cols, lda, a_fmt, ws, V, ldv, r, vals, r_dev, Y, ldy, W, ldw, F64, nullptr, nullptr,
                   nullptr, 0, F64, part_out, (uint8_t*)ws + opb, ws_bytes - opb, st, OZ_D);
}

}  // namespace ofrr
