// gemm_tc.cu -- K1: W = A * X on the 5th-generation tensor cores (tcgen05 + TMA + TMEM).
//
// Replaces the reference's A.V pass: ofrr/matrix.py:242-254 (apply_dense) ->
// ofrr/precision.py:122-135 (mixed_gemm) -> ofrr/_kernels.pyx:60-84 (gemm_mixed).
//
// Shape: A is rows x cols row-major (K-major for the MMA), X is cols x k column-major
// (K-major B operand), k <= 256.  A is streamed exactly once from HBM; the X panel
// (n x k, a few MB) is re-read from L2 by every CTA.
//
// Design (one CTA per SM, persistent, stream-K):
//   * tile = 256 rows x BN (BN = k rounded up to 32/64/128/256), two M=128 UMMAs
//     per K-step share the B (X) tile, halving L2 traffic for X.
//   * BLOCK_K = 128 bytes (64 bf16/f16, 128 e4m3) so every smem row is one
//     128B-swizzle atom; 4 UMMAs (32 bytes of K each) per stage.
//   * the flattened (tile, k-block) iteration space is split evenly over the grid
//     (stream-K), so all 148 SMs stream A for the whole kernel; each (tile, CTA)
//     segment is written as an fp32 partial, and k_finalize sums the partials of a
//     tile in ascending CTA order (deterministic), rounds to the storage format,
//     and produces the per-column inf-norms for the column scaling (K2).
//   * warp roles: warp 0 = TMA producer, warp 1 = MMA issuer (+ TMEM owner),
//     warps 2..5 = epilogue (TMEM -> registers -> fp32 partials, coalesced).
#include "common.cuh"
#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <vector>
#include <utility>

namespace ofrr {

static constexpr int TILE_M = 256;          // rows per tile (2 x UMMA_M=128)
static constexpr int KBYTES = 128;          // bytes of K per stage (one SW128 atom row)
static constexpr int A_STAGE = TILE_M * KBYTES;  // 32 KB
static constexpr int SMEM_BUDGET = 200 * 1024;
static constexpr int THREADS = 192;

// MH = M halves per tile: 2 (256 rows, the two M=128 UMMAs share each B tile, BN <= 256),
// or 1 ("wide": 128 rows, BN up to 512 fp32 TMEM columns as two N chunks of <= 256 that share
// each A tile -- one pass over A for N = 3k up to 510, e.g. the fp32 split at k = 128)
template <int BN, int MH = 2>
struct TcCfg {
  static constexpr int TM = 128 * MH;               // rows per tile
  static constexpr int A_ST = TM * KBYTES;
  static constexpr int B_STAGE = BN * KBYTES;
  static constexpr int STAGE = A_ST + B_STAGE;
  static constexpr int STAGES_RAW = SMEM_BUDGET / STAGE;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  // MH accumulators of BN fp32 columns; allocation is a power of two >= 32
  static constexpr int TMEM_COLS = (MH * BN) <= 32 ? 32 : (MH * BN) <= 64 ? 64 : (MH * BN) <= 128 ? 128
                                   : (MH * BN) <= 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE + 256;
  static constexpr int XBOX = BN <= 256 ? BN : 128;    // rows per TMA box of the B operand
};

// Instruction descriptor (kind::f16 / kind::f8f6f4): c_format=F32 (bits 4-5), a/b formats
// (bits 7-9 / 10-12), K-major A and B, N>>3 (bits 17-22), M>>4 (bits 24-28).
static inline uint32_t make_idesc(int a_fmt, int n) {
  uint32_t ab = (a_fmt == BF16) ? 1u : 0u;  // F16 = 0, BF16 = 1; E4M3 = 0 for f8f6f4
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

struct Segments {
  long long it0, it1;
  int kblocks;
};

// ---- in-kernel timing of k_gemm_av_tc for the bench roofline (works inside CUDA graphs
// with device-side loops, where event nodes are not allowed): every CTA stamps its entry
// (min) and exit (max) in globaltimer ns; the launch's k_finalize (stream-ordered after it)
// adds the interval to a running sum and re-arms the stamps. ----
__device__ unsigned long long g_k1_stamp[4] = {~0ull, 0ull, 0ull, 0ull};   // min start, max end, sum, count
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// CL = 2 (wide tile only): a cluster of two CTAs works on a pair of 128-row tiles with the
// same k-block sequence; each loads its own A tile and half of the B tile, multicast into
// both CTAs' shared memory (X is read from L2 once per 256 rows, as in the MH = 2 tile),
// and each MMA commit releases the stage in both CTAs.
template <int BN, bool FP8K, int MH = 2, int CL = 1>
__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_av_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmX,
                 float* __restrict__ ws, int kblocks, long long total_iters, int max_slots,
                 uint32_t idesc, int stamp, uint32_t idesc2, int m_tiles) {
  using C = TcCfg<BN, MH>;
  constexpr int TMR = C::TM;
  static_assert(CL == 1 || MH == 1, "cluster pairs use the wide tile");
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  if (stamp && threadIdx.x == 0) atomicMin(&g_k1_stamp[0], gtimer_ns());
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = warp_index(), lane = threadIdx.x & 31;
  const long long G = gridDim.x / CL;                          // work units are split per cluster
  const long long cidx = blockIdx.x / CL;
  const long long it0 = cidx * total_iters / G;
  const long long it1 = (cidx + 1) * total_iters / G;
  const int t_first = (int)(it0 / kblocks);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], CL); }
    mbar_init(tfull, 1);
    mbar_init(tempty, 128);
    fence_barrier_init();
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmX);
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();                   // peers' barriers initialised
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_a = policy_evict_first(), pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (long long it = it0; it < it1; ++it) {
        const int t = (int)(it / kblocks), kb = (int)(it % kblocks);
        mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* sa = smem + stage * C::STAGE;
        mbar_expect_tx(&full[stage], C::STAGE);
        const int kcoord = FP8K ? kb * 128 : kb * 64;
        tma_load_2d(sa, &tmA, kcoord, (t * CL + crank) * TMR, &full[stage], pol_a);
        if constexpr (CL == 1) {
#pragma unroll
          for (int xb = 0; xb < BN; xb += C::XBOX)
            tma_load_2d(sa + C::A_ST + xb * KBYTES, &tmX, kcoord, xb, &full[stage], pol_x);
        } else {
#pragma unroll
          for (int xb = 0; xb < BN; xb += C::XBOX)
            if ((xb / C::XBOX) % CL == crank)
              tma_load_2d_mc(sa + C::A_ST + xb * KBYTES, &tmX, kcoord, xb, &full[stage], (uint16_t)((1u << CL) - 1u),
                             pol_x);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
      if constexpr (CL > 1) {
        // drain: every stage's last release (this CTA's and the peer's commits) has landed
        // before the cluster may exit
        for (int i = 0; i < C::STAGES; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ===== MMA issuer (warp-wide, elected lane issues) =====
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      long long it = it0;
      while (it < it1) {
        const int kb0 = (int)(it % kblocks);
        const int kb1 = (int)std::min<long long>(kblocks, kb0 + (it1 - it));
        mbar_wait(tempty, acc_phase ^ 1);
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + C::A_ST);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t acc = (kb > kb0 || k > 0) ? 1u : 0u;
            if constexpr (MH == 2) {
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                // +32 B of K per step (>>4 = 2); second M half starts 128 rows (16 KB) later
                const uint64_t a = da + (uint64_t)(k * 2 + h * (16384 >> 4));
                const uint64_t b = db + (uint64_t)(k * 2);
                if (FP8K) mma_f8_ws(tmem + h * BN, a, b, idesc, acc);
                else mma_f16_ws(tmem + h * BN, a, b, idesc, acc);
              }
            } else {
              // one M=128 half, N in chunks of 256 columns sharing the A tile; the second
              // chunk's B rows start 256 rows (32 KB) into the B stage
              const uint64_t a = da + (uint64_t)(k * 2);
              if (FP8K) mma_f8_ws(tmem, a, db + (uint64_t)(k * 2), idesc, acc);
              else mma_f16_ws(tmem, a, db + (uint64_t)(k * 2), idesc, acc);
              if constexpr (BN > 256) {
                const uint64_t b2 = db + (uint64_t)(k * 2 + ((256 * KBYTES) >> 4));
                if (FP8K) mma_f8_ws(tmem + 256, a, b2, idesc2, acc);
                else mma_f16_ws(tmem + 256, a, b2, idesc2, acc);
              }
            }
          }
          if constexpr (CL > 1) tc_commit_mc_ws(&empty[stage], (uint16_t)((1u << CL) - 1u));
          else tc_commit_ws(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        tc_commit_ws(tfull);
        acc_phase ^= 1;
      }
    }
  } else {
    // ===== epilogue warps 2..5: TMEM -> fp32 partial tiles (column-major 256 x BN) =====
    const int q = warp & 3;                // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;         // row within the 128-row accumulator
    uint32_t acc_phase = 0;
    long long it = it0;
    while (it < it1) {
      const int t = (int)(it / kblocks);
      const int kb0 = (int)(it % kblocks);
      const int kb1 = (int)std::min<long long>(kblocks, kb0 + (it1 - it));
      it += kb1 - kb0;
      mbar_wait(tfull, acc_phase);
      tc_fence_after();
      float* dst = ws + ((size_t)blockIdx.x * max_slots + (t - t_first)) * (size_t)(TMR * BN);
      const bool live = (long long)t * CL + crank < m_tiles;       // odd tile count: the pair's 2nd may not exist
#pragma unroll
      for (int h = 0; h < MH; ++h) {
        if (!live) break;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float v[16];
          tmem_ld16(tmem + ((uint32_t)(q * 32) << 16) + h * BN + c0, v);
#pragma unroll
          for (int i = 0; i < 16; ++i) dst[(size_t)(c0 + i) * TMR + h * 128 + row] = v[i];
        }
      }
      tc_fence_before();
      mbar_arrive(tempty);
      acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();
  if (stamp && threadIdx.x == 0) atomicMax(&g_k1_stamp[1], gtimer_ns());
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Sum the stream-K partials of one 256-row tile in ascending CTA order, round to the
// output format, write W (column-major) and the per-column inf-norm.
__device__ __forceinline__ long long seg_begin(long long c, long long T, long long G) { return c * T / G; }

static constexpr int FIN_COLS = 16;   // columns per finalize block

__global__ void __launch_bounds__(256)
    k_finalize(const float* __restrict__ ws, int BN, int kblocks, long long total_iters, int G,
               int max_slots, int64_t rows, int k, void* __restrict__ W, int64_t ldw, int out_fmt,
               double* __restrict__ colmax, int* __restrict__ flags, void* __restrict__ W2, int64_t ldw2,
               int out_fmt2, int nsplit, int stamp, int TMR, int CLN) {
  if (stamp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {   // the product kernel is done
    const unsigned long long t0 = g_k1_stamp[0], t1 = g_k1_stamp[1];
    if (t1 > t0) { g_k1_stamp[2] += t1 - t0; g_k1_stamp[3] += 1; }
    g_k1_stamp[0] = ~0ull;
    g_k1_stamp[1] = 0ull;
  }
  // nsplit > 1: the product was taken against [X_hi | X_mid | X_lo] (bf16 slices of an fp32
  // block, see k_split_bf16); output column j sums tile columns j + s*k, lowest slice first
  __shared__ float smax[8][FIN_COLS];
  const int t = blockIdx.x;
  const int j0 = blockIdx.y * FIN_COLS;
  const int row = threadIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // cluster pairs (CLN = 2): tile t is rank t % 2 of pair t / 2, work split per cluster
  const int tu = t / CLN, trank = t % CLN;
  G /= CLN;
  const long long x0 = (long long)tu * kblocks, x1 = x0 + kblocks - 1;
  // the CTAs owning the tile's iterations and their partial slots: thread 0 resolves them
  // once per block (64-bit divisions), every thread reads the table
  constexpr int MAXC = 160;
  __shared__ long long s_base[MAXC];
  __shared__ int s_nc;
  if (threadIdx.x == 0) {
    // CTA owning iteration x: largest c with seg_begin(c) <= x
    long long c_lo = x0 * G / total_iters, c_hi = x1 * G / total_iters;
    while (c_lo + 1 < G && seg_begin(c_lo + 1, total_iters, G) <= x0) ++c_lo;
    while (c_lo > 0 && seg_begin(c_lo, total_iters, G) > x0) --c_lo;
    while (c_hi + 1 < G && seg_begin(c_hi + 1, total_iters, G) <= x1) ++c_hi;
    while (c_hi > 0 && seg_begin(c_hi, total_iters, G) > x1) --c_hi;
    int nc = 0;
    for (long long c = c_lo; c <= c_hi && nc < MAXC; ++c, ++nc) {
      const int slot = tu - (int)(seg_begin(c, total_iters, G) / kblocks);
      s_base[nc] = ((long long)(c * CLN + trank) * max_slots + slot) * (long long)(TMR * BN);
    }
    s_nc = nc;
  }
  __syncthreads();
  const int nc = s_nc;
  const int64_t grow = (int64_t)t * TMR + row;
  const bool valid = grow < rows;
  float s[FIN_COLS];
#pragma unroll
  for (int i = 0; i < FIN_COLS; ++i) s[i] = 0.f;
  for (int sl = nsplit - 1; sl >= 0; --sl) {
    for (int q = 0; q < nc; ++q) {
      const float* src = ws + s_base[q] + row + (size_t)sl * k * TMR;
#pragma unroll
      for (int i = 0; i < FIN_COLS; ++i)
        if (j0 + i < k) s[i] += src[(size_t)(j0 + i) * TMR];
    }
  }
  int bad = 0;
#pragma unroll
  for (int i = 0; i < FIN_COLS; ++i) {
    const int j = j0 + i;
    float a = 0.f;
    if (valid && j < k) {
      const float w = rndf(s[i], out_fmt);
      st_fmt(W, (int64_t)j * ldw + grow, out_fmt, (double)w);
      if (W2) st_fmt(W2, (int64_t)j * ldw2 + grow, out_fmt2, (double)rndf(s[i], out_fmt2));
      if (!isfinite(w)) bad = 1;
      a = (w != w) ? INFINITY : fabsf(w);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (lane == 0) smax[warp][i] = a;
  }
  __syncthreads();
  if (colmax && threadIdx.x < FIN_COLS && j0 + threadIdx.x < k) {
    float a = smax[0][threadIdx.x];
    for (int w8 = 1; w8 < (int)(blockDim.x >> 5); ++w8) a = fmaxf(a, smax[w8][threadIdx.x]);
    atomic_max_nonneg(&colmax[j0 + threadIdx.x], (double)a);
  }
  if (bad && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
}

// ---------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

static int make_tmap_2d(CUtensorMap* tm, const void* base, int a_fmt, uint64_t inner, uint64_t outer,
                        uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer,
                        CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled enc = get_encode();
  if (!enc) { ofrr_set_error("cuTensorMapEncodeTiled unavailable"); return OFRR_ERR_CUDA; }
  CUtensorMapDataType dt = a_fmt == BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                         : a_fmt == F16  ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                         : CU_TENSOR_MAP_DATA_TYPE_UINT8;
  const int eb = fmt_bytes(a_fmt);
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * (uint64_t)eb};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    ofrr_set_error("cuTensorMapEncodeTiled failed (%d): dims %llu x %llu ld %llu box %u x %u", (int)r,
                   (unsigned long long)inner, (unsigned long long)outer, (unsigned long long)ld_elems,
                   box_inner, box_outer);
    return OFRR_ERR_INVALID;
  }
  return OFRR_OK;
}

// 2-D uint8 map with 128B swizzle (the int8 digit planes of oz.cu)
int oz_make_tmap_u8(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                    uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(tm, base, FP8, inner, outer, ld_bytes, box_inner, box_outer);
}

// raw operator rows for the K7z converters: 64 entries x 128 rows, 128B swizzle (64B for fp8)
int oz_make_tmap_a(CUtensorMap* tm, const void* base, int a_fmt, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                   uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(tm, base, a_fmt, inner, outer, ld_elems, box_inner, box_outer,
                      a_fmt == FP8 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B);
}

int oz_make_tmap_u8_sw64(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t ld_bytes,
                         uint32_t box_inner, uint32_t box_outer) {
  return make_tmap_2d(tm, base, FP8, inner, outer, ld_bytes, box_inner, box_outer, CU_TENSOR_MAP_SWIZZLE_64B);
}

// N of the UMMA = k rounded up to a multiple of 32 (M=128 needs N % 16 == 0, N <= 256)
// ---- kernel-only timing of k_gemm_av_tc (bench.py roofline): a pair of CUDA events
// recorded on the launching stream immediately around each launch.  Eager launches take a
// pair from a free pool and queue it as pending; launches captured into a CUDA graph
// (pairs still pending when the caller claims them) become a group owned by the graph,
// re-recorded by every replay and harvested after it.  Durations accumulate in launch
// order and are read back after the timed region. ----
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_prof_ev;
static std::vector<int> g_prof_free, g_prof_pending;
static std::vector<std::vector<int>> g_prof_groups;
static std::vector<float> g_prof_acc;

static cudaEvent_t* prof_slot() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return nullptr;
  int idx;
  if (!g_prof_free.empty()) {
    idx = g_prof_free.back();
    g_prof_free.pop_back();
  } else {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return nullptr;
    g_prof_ev.push_back({a, b});
    idx = (int)g_prof_ev.size() - 1;
  }
  g_prof_pending.push_back(idx);
  return &g_prof_ev[idx].first;
}

static int prof_harvest(const std::vector<int>& idx) {
  for (int i : idx) {
    float t = 0.f;
    if (cudaEventSynchronize(g_prof_ev[i].second) != cudaSuccess ||
        cudaEventElapsedTime(&t, g_prof_ev[i].first, g_prof_ev[i].second) != cudaSuccess) {
      (void)cudaGetLastError();   // timing is best effort: never poison later launch checks
      return -1;
    }
    g_prof_acc.push_back(t);
  }
  return 0;
}

// record a timing event; inside a stream capture as an external event node, so that every
// replay of the graph records it
static void prof_record(cudaEvent_t ev, cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
  else
    cudaEventRecord(ev, st);
}

void prof_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  g_prof_acc.clear();
  for (int i : g_prof_pending) g_prof_free.push_back(i);
  g_prof_pending.clear();
}
int prof_active() { return g_prof_on ? 1 : 0; }

// pending (eager) pairs -> accumulated durations; the pairs return to the pool
int prof_collect() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int rc = prof_harvest(g_prof_pending);
  for (int i : g_prof_pending) g_prof_free.push_back(i);
  g_prof_pending.clear();
  return rc;
}
// the pending pairs were captured into a graph: make them a group, return its id
int prof_claim() {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g_prof_pending.empty()) return -1;
  g_prof_groups.push_back(g_prof_pending);
  g_prof_pending.clear();
  return (int)g_prof_groups.size() - 1;
}
// after a replay of the graph owning group g (and a synchronisation)
int prof_collect_group(int g) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (g < 0 || g >= (int)g_prof_groups.size()) return 0;
  if (!g_prof_on) return 0;
  return prof_harvest(g_prof_groups[g]);
}

static bool g_stamp_on = false;
int stamp_enable(int on) {
  g_stamp_on = on != 0;
  if (on) {
    const unsigned long long z[4] = {~0ull, 0ull, 0ull, 0ull};
    if (cudaMemcpyToSymbol(g_k1_stamp, z, sizeof(z)) != cudaSuccess) return OFRR_ERR_CUDA;
  }
  return OFRR_OK;
}
int stamp_read(double* sum_ms, long long* count) {
  unsigned long long v[4];
  if (cudaMemcpyFromSymbol(v, g_k1_stamp, sizeof(v)) != cudaSuccess) return OFRR_ERR_CUDA;
  *sum_ms = (double)v[2] * 1e-6;
  *count = (long long)v[3];
  return OFRR_OK;
}

int prof_read(float* ms, int max) {
  if (prof_collect() != 0) return -1;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int n = 0;
  for (size_t i = 0; i < g_prof_acc.size() && n < max; ++i) ms[n++] = g_prof_acc[i];
  return n;
}

static int pick_bn(int k) { return k <= 32 ? 32 : ((k + 31) / 32) * 32; }
static int g_no_cluster = -1;   // OFRR_K1_NO_CLUSTER=1: the wide tile without the cluster pairs

// N > 256 (up to 512): the wide one-M-half tile (TcCfg MH = 1), BN a multiple of 128
static bool wide_n(int k) { return k > 256; }

struct TcPlan {
  int bn, m_tiles, kblocks, grid, max_slots, tm, cl;
  long long total;
  size_t ws_bytes;
};

static TcPlan plan_tc(int64_t rows, int64_t cols, int k, int a_fmt) {
  if (g_no_cluster < 0) { const char* e = getenv("OFRR_K1_NO_CLUSTER"); g_no_cluster = (e && atoi(e) == 1) ? 1 : 0; }
  TcPlan p;
  const bool wide = wide_n(k);
  p.bn = wide ? ((k + 127) / 128) * 128 : pick_bn(k);
  p.tm = wide ? 128 : TILE_M;
  const int kel = (a_fmt == FP8) ? 128 : 64;
  p.m_tiles = (int)((rows + p.tm - 1) / p.tm);
  p.kblocks = (int)((cols + kel - 1) / kel);
  // the wide tile runs as cluster pairs (two 128-row tiles share each B tile by multicast)
  p.cl = (wide && p.m_tiles >= 2 && !g_no_cluster) ? 2 : 1;
  p.total = (long long)((p.m_tiles + p.cl - 1) / p.cl) * p.kblocks;   // work units per cluster
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  const long long nclus = std::min<long long>(sms / p.cl, p.total);
  p.grid = (int)std::max<long long>(1, nclus) * p.cl;
  const long long per = (p.total + p.grid / p.cl - 1) / (p.grid / p.cl);
  p.max_slots = (int)((per + p.kblocks - 1) / p.kblocks) + 1;
  p.ws_bytes = (size_t)p.grid * p.max_slots * p.tm * p.bn * sizeof(float);
  return p;
}

size_t tc_workspace(int64_t rows, int64_t cols, int k, int a_fmt) {
  return plan_tc(rows, cols, k, a_fmt).ws_bytes;
}

template <int BN, bool FP8K, int MH, int CL>
static int launch_tc_bn(const CUtensorMap& tA, const CUtensorMap& tX, const TcPlan& p, float* ws,
                        uint32_t idesc, uint32_t idesc2, cudaStream_t st) {
  using C = TcCfg<BN, MH>;
  auto kern = k_gemm_av_tc<BN, FP8K, MH, CL>;
  static std::atomic<bool> attr_done{false};
  if (!attr_done) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES));
    attr_done = true;
  }
  cudaEvent_t* ev = prof_slot();
  if (ev) prof_record(ev[0], st);
  const int stamp = g_stamp_on ? 1 : 0;
  if constexpr (CL == 1) {
    kern<<<p.grid, THREADS, C::SMEM_BYTES, st>>>(tA, tX, ws, p.kblocks, p.total, p.max_slots, idesc, stamp, idesc2,
                                                 p.m_tiles);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(p.grid);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = C::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    OFRR_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tA, tX, ws, p.kblocks, p.total, p.max_slots, idesc, stamp, idesc2,
                                     p.m_tiles));
  }
  if (ev) prof_record(ev[1], st);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

int tc_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* X,
               int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags,
               void* ws, size_t ws_bytes, cudaStream_t st, void* W2, int64_t ldw2, int out_fmt2, int nsplit) {
  TcPlan p = plan_tc(rows, cols, k, a_fmt);
  if (ws_bytes < p.ws_bytes || ws == nullptr) {
    ofrr_set_error("gemm_av: workspace too small (%zu < %zu)", ws_bytes, p.ws_bytes);
    return OFRR_ERR_INVALID;
  }
  if (k > 512) { ofrr_set_error("gemm_av: k=%d > 512 on the tensor-core path", k); return OFRR_ERR_INVALID; }
  const bool fp8 = a_fmt == FP8;
  const bool wide = wide_n(k);
  const uint32_t kel = fp8 ? 128 : 64;
  CUtensorMap tA, tX;
  int rc = make_tmap_2d(&tA, A, a_fmt, (uint64_t)cols, (uint64_t)rows, (uint64_t)lda, kel, (uint32_t)p.tm);
  if (rc) return rc;
  rc = make_tmap_2d(&tX, X, a_fmt, (uint64_t)cols, (uint64_t)k, (uint64_t)ldx, kel,
                    (uint32_t)(wide ? 128 : p.bn));
  if (rc) return rc;
  const uint32_t idesc = make_idesc(a_fmt, wide ? 256 : p.bn);
  const uint32_t idesc2 = wide ? make_idesc(a_fmt, p.bn - 256) : 0u;
#define TC_CASE(B) case B: rc = fp8 ? launch_tc_bn<B, true, 2, 1>(tA, tX, p, (float*)ws, idesc, idesc2, st) \
                                  : launch_tc_bn<B, false, 2, 1>(tA, tX, p, (float*)ws, idesc, idesc2, st); break;
#define TC_WIDE(B) case B: if (p.cl == 2) { rc = fp8 ? launch_tc_bn<B, true, 1, 2>(tA, tX, p, (float*)ws, idesc, idesc2, st) \
                                               : launch_tc_bn<B, false, 1, 2>(tA, tX, p, (float*)ws, idesc, idesc2, st); } \
                           else { rc = fp8 ? launch_tc_bn<B, true, 1, 1>(tA, tX, p, (float*)ws, idesc, idesc2, st) \
                                           : launch_tc_bn<B, false, 1, 1>(tA, tX, p, (float*)ws, idesc, idesc2, st); } break;
  if (wide) {
    switch (p.bn) {
      TC_WIDE(384)
      default: TC_WIDE(512)
    }
  } else {
    switch (p.bn) {
      TC_CASE(32) TC_CASE(64) TC_CASE(96) TC_CASE(128) TC_CASE(160) TC_CASE(192) TC_CASE(224)
      default: TC_CASE(256)
    }
  }
#undef TC_CASE
#undef TC_WIDE
  if (rc) return rc;
  k_finalize<<<dim3(p.m_tiles, (k / nsplit + FIN_COLS - 1) / FIN_COLS), p.tm, 0, st>>>((const float*)ws, p.bn, p.kblocks, p.total, p.grid, p.max_slots,
                                        rows, k / nsplit, W, ldw, out_fmt, colmax, flags, W2, ldw2, out_fmt2,
                                        nsplit, g_stamp_on ? 1 : 0, p.tm, p.cl);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// ---------------------------------------------------------------------------------
// fp32 blocks on the bf16 tensor cores: X (n x k fp32, column-major) -> [X_hi|X_mid|X_lo]
// (n x 3k bf16): x_hi = bf16(x), x_mid = bf16(x - x_hi), x_lo = bf16(x - x_hi - x_mid).  The
// residues are exact in fp32, so the three slices carry the full 24-bit significand and
// A (bf16) times each slice is an exact-product, fp32-accumulated tensor-core product.
// ---------------------------------------------------------------------------------
// slices = 2 ("lite": x_hi + x_mid, a 16-bit significand, N = 2k) keeps the product at the
// HBM roofline for k <= 125 (N <= 251 flop/B at bf16) where 3 slices are tensor-bound; slices
// = 1 (x_hi only) for a product whose block needs no more (the random start block).
__global__ void k_split_bf16(const float* __restrict__ X, int64_t ldx, int64_t n, int k,
                             __nv_bfloat16* __restrict__ Xs, int64_t lds, int slices) {
  const int j = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float x = X[(int64_t)j * ldx + i];
    const __nv_bfloat16 h = __float2bfloat16_rn(x);
    const float r1 = x - __bfloat162float(h);
    const __nv_bfloat16 m = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(m);
    Xs[(int64_t)j * lds + i] = h;
    if (slices >= 2) Xs[(int64_t)(k + j) * lds + i] = m;
    if (slices == 3) Xs[(int64_t)(2 * k + j) * lds + i] = __float2bfloat16_rn(r2);
  }
}

// columns per pass: 3 * 170 = 510 <= 512 (one pass over A up to k = 170; the wide tile
// for 85 < k, the two-M-half tile up to 85); 2 slices: 2 * 256
static constexpr int SPLIT_KC = 170;
static int split_kc(int slices) { return slices == 1 ? 384 : slices == 2 ? 256 : SPLIT_KC; }

size_t split_workspace(int64_t rows, int64_t cols, int k) {
  size_t best = 0;
  for (int slices = 1; slices <= 3; ++slices) {
    const int kc = std::min(k, split_kc(slices));
    const int64_t lds = (cols + 63) / 64 * 64;
    best = std::max(best, (size_t)slices * kc * lds * 2 + 1024 + tc_workspace(rows, cols, slices * kc, BF16));
  }
  return best;
}

// k <= 170: one pass over A with N = 3k.  k > 170: column chunks of <= 170, one pass each
// (full fp32 semantics at the price of ceil(k / 170) passes).
int tc_gemm_av_split(const void* A, int64_t rows, int64_t cols, int64_t lda, const float* X, int64_t ldx, int k,
                     void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* ws, size_t ws_bytes,
                     cudaStream_t st, void* W2, int64_t ldw2, int out_fmt2, int slices) {
  if (slices < 1 || slices > 3) { ofrr_set_error("gemm_av split: slices must be 1, 2 or 3"); return OFRR_ERR_INVALID; }
  if (ws_bytes < split_workspace(rows, cols, k)) { ofrr_set_error("gemm_av split: workspace too small"); return OFRR_ERR_INVALID; }
  const int64_t lds = (cols + 63) / 64 * 64;
  const int KC = split_kc(slices);
  const int kcmax = std::min(k, KC);
  __nv_bfloat16* Xs = (__nv_bfloat16*)ws;
  uint8_t* rest = (uint8_t*)ws + (((size_t)slices * kcmax * lds * 2 + 1023) & ~size_t(1023));
  const size_t rest_bytes = ws_bytes - (rest - (uint8_t*)ws);
  const int ob = fmt_bytes(out_fmt), ob2 = fmt_bytes(out_fmt2);
  for (int j0 = 0; j0 < k; j0 += KC) {
    const int kc = std::min(KC, k - j0);
    unsigned gx = (unsigned)std::min<int64_t>((cols + 255) / 256, 64);
    k_split_bf16<<<dim3(gx, kc), 256, 0, st>>>(X + (int64_t)j0 * ldx, ldx, cols, kc, Xs, lds, slices);
    OFRR_CHECK_LAUNCH();
    const int rc = tc_gemm_av(A, rows, cols, lda, BF16, Xs, lds, slices * kc, (uint8_t*)W + (size_t)j0 * ldw * ob,
                              ldw, out_fmt, colmax ? colmax + j0 : nullptr, flags, rest, rest_bytes, st,
                              W2 ? (uint8_t*)W2 + (size_t)j0 * ldw2 * ob2 : nullptr, ldw2, out_fmt2, slices);
    if (rc) return rc;
  }
  return OFRR_OK;
}

}  // namespace ofrr
