// gram.cu -- K4: projected matrices G1 = U^T W and G2 = U^T U for the OFRR pencil.
//
// Replaces ofrr/projection.py:56-61 (_project) as called from ofrr_eig (:79-80) and
// ofrr_svd (:109-111).  Tall-skinny reduction over the n rows:
//   stage 1: grid (row chunks x 64x64 output tiles); each CTA stages a 32-row slab of
//            U and [W U] in shared memory as fp64 (register-prefetched one slab ahead) and
//            accumulates with fp64 tensor-core MMA (DMMA m8n8k4; storage values have <= 24
//            significant bits, so every product is exact in fp64; only the sums round);
//   stage 2: fixed-order sum of the chunk partials (deterministic), rounding to the
//            projection output format (ofrr/projection.py:42-53), non-finite check.
#include "common.cuh"
#include <algorithm>
#include <cstdlib>

namespace ofrr {

static constexpr int GT = 64;   // output tile
static constexpr int GR = 32;   // rows per smem slab

// fp64 tensor-core MMA (DMMA), m8n8k4: A row-major 8x4, B col-major 4x8, C 8x8 fp64.
// Fragments (lane = 4 g + t): a = A[g][t], b = B[t][g], c = C[g][2t .. 2t+1].
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

static constexpr int GS = GR + 4;   // smem row stride (doubles): conflict-free fragment reads

template <typename T>
__global__ void __launch_bounds__(256)
    k_gram_partial(const T* __restrict__ U, int64_t ldu, const T* __restrict__ W, int64_t ldw, int64_t n,
                   int k, int kw, int64_t rows_per_chunk, double* __restrict__ part) {
  // output columns: [0, kw) -> U^T W, [kw, kw + k) -> U^T U.  Slabs are staged column-major
  // ([column][row], stride GS) as fp64; each warp owns a 16 x 32 block of the 64 x 64 tile
  // (2 x 4 DMMA tiles) and walks the slab 4 rows per MMA.
  __shared__ double Us[GT][GS];
  __shared__ double Vs[GT][GS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
  const int i0 = blockIdx.y * GT;      // rows of the Gram (columns of U)
  const int j0 = blockIdx.z * GT;      // columns of the Gram ([W U])
  const int ncols = kw + k;
  // U^T U is symmetric: with tile-aligned blocks (kw % GT == 0) the tiles below its diagonal
  // are not computed; k_gram_reduce mirrors them (the pencil symmetrises M anyway)
  if (kw % GT == 0 && j0 >= kw && (j0 - kw) / GT < i0 / GT) return;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_chunk;
  const int64_t re = std::min<int64_t>(n, rb + rows_per_chunk);
  double acc[2][4][2] = {};
  // software pipeline: the next slab's 8 + 8 raw elements per thread are loaded into registers
  // (branch-free, clamped addresses + validity masks, converted only when staged) while the
  // current slab is multiplied out of shared memory -- all 16 loads are in flight at once
  constexpr int PER = GR * GT / 256;
  T pu[PER], pv[PER];
  unsigned okm = 0;
  auto fetch = [&](int64_t l0) {
    okm = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + 256 * q;
      const int c = e / GR, rr = e % GR;   // contiguous along rows (column-major inputs)
      const int64_t l = l0 + rr;
      const bool lin = l < re;
      const bool uok = lin && i0 + c < k;
      const int jc = j0 + c;
      const bool vok = lin && jc < ncols;
      const T* vp = jc < kw ? W + (int64_t)jc * ldw : U + (int64_t)(jc - kw) * ldu;
      pu[q] = U[uok ? (int64_t)(i0 + c) * ldu + l : 0];
      pv[q] = vok ? vp[l] : U[0];
      okm |= (uok ? 1u : 0u) << q | (vok ? 1u : 0u) << (q + 16);
    }
  };
  if (rb < re) fetch(rb);
  for (int64_t l0 = rb; l0 < re; l0 += GR) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int e = tid + 256 * q;
      Us[e / GR][e % GR] = (okm >> q & 1u) ? to_d(pu[q]) : 0.0;
      Vs[e / GR][e % GR] = (okm >> (q + 16) & 1u) ? to_d(pv[q]) : 0.0;
    }
    __syncthreads();
    if (l0 + GR < re) fetch(l0 + GR);
#pragma unroll
    for (int kk = 0; kk < GR; kk += 4) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = Us[wm + 8 * i + g][kk + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Vs[wn + 8 * j + g][kk + t];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  // partial layout: [chunk][ncols][k] column-major per chunk
  double* dst = part + (int64_t)blockIdx.x * ncols * k;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gi = i0 + wm + 8 * i + g, gj = j0 + wn + 8 * j + 2 * t + h;
        if (gi < k && gj < ncols) dst[(int64_t)gj * k + gi] = acc[i][j][h];
      }
}

// 32 output elements x 8 chunk lanes per CTA: each lane sums its chunks c = g, g+8, ... in
// order, then lane 0 adds the 8 lane sums in order -- a fixed summation order (deterministic)
// with 8x the memory-level parallelism of one thread per element
__global__ void __launch_bounds__(256) k_gram_reduce(const double* __restrict__ part, int nchunks, int k, int kw,
                                                     int out_fmt, double* __restrict__ G1, double* __restrict__ G2,
                                                     int* __restrict__ flags) {
  __shared__ double red[8][33];
  const int ncols = kw + k;
  const int64_t total = (int64_t)ncols * k;
  const int lx = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = (int64_t)blockIdx.x * 32 + lx;
  int64_t es = e;                                   // the partials' element (mirrored tiles of U^T U)
  if (e < total && kw % GT == 0) {
    const int gj = (int)(e / k), gi = (int)(e % k);
    if (gj >= kw && (gj - kw) / GT < gi / GT) es = (int64_t)(kw + gi) * k + (gj - kw);
  }
  double s = 0.0;
  if (e < total) {
#pragma unroll 4
    for (int c = g; c < nchunks; c += 8) s += part[(int64_t)c * total + es];
  }
  red[g][lx] = s;
  __syncthreads();
  if (g != 0 || e >= total) return;
  s = red[0][lx];
#pragma unroll
  for (int j = 1; j < 8; ++j) s += red[j][lx];
  s = rnd(s, out_fmt);
  if (!isfinite(s) && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
  const int gj = (int)(e / k), gi = (int)(e % k);
  if (gj < kw) { if (G1) G1[(int64_t)gj * k + gi] = s; }
  else if (G2) G2[(int64_t)(gj - kw) * k + gi] = s;
}

struct GramPlan { int nchunks; int64_t rows_per; };
static GramPlan gram_plan(int64_t n, int k, int kw) {
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  const int kt = (k + GT - 1) / GT;
  // computed tiles: U^T U below its diagonal is mirrored (k_gram_partial) when tile-aligned
  const int tiles = kt * ((kw + k + GT - 1) / GT) - (kw % GT == 0 ? kt * (kt - 1) / 2 : 0);
  // ~4 CTAs per SM (each has one slab of loads in flight; more CTAs hide the latency),
  // at least 4 slabs per chunk (the partials are re-read by the reduce)
  int64_t chunks = std::max<int64_t>(1, (4 * sms + tiles - 1) / tiles);
  if (const char* e = getenv("OFRR_GRAM_CHUNKS")) chunks = atoi(e);   // tuning override
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, n / (4 * GR)));
  int64_t rows_per = (n + chunks - 1) / chunks;
  rows_per = (rows_per + GR - 1) / GR * GR;
  chunks = std::max<int64_t>(1, (n + rows_per - 1) / rows_per);
  return {(int)chunks, rows_per};
}

size_t gram_ws(int64_t n, int k, int kw) {
  GramPlan p = gram_plan(n, k, kw);
  return (size_t)p.nchunks * (size_t)(kw + k) * k * sizeof(double);
}

template <typename T>
static int launch_gram(const void* U, int64_t ldu, const void* W, int64_t ldw, int64_t n, int k, int kw, int out_fmt,
                       double* G1, double* G2, int* flags, double* part, cudaStream_t st) {
  GramPlan p = gram_plan(n, k, kw);
  dim3 grid(p.nchunks, (k + GT - 1) / GT, (kw + k + GT - 1) / GT);
  k_gram_partial<T><<<grid, 256, 0, st>>>((const T*)U, ldu, (const T*)W, ldw, n, k, kw, p.rows_per, part);
  OFRR_CHECK_LAUNCH();
  const int64_t total = (int64_t)(kw + k) * k;
  k_gram_reduce<<<(unsigned)((total + 31) / 32), 256, 0, st>>>(part, p.nchunks, k, kw, out_fmt,
                                                                                      G1, G2, flags);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

int gram(const void* U, int64_t ldu, const void* W, int64_t ldw, int64_t n, int k, int kw, int storage, int out_fmt,
         double* G1, double* G2, int* flags, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!W) kw = 0;
  if (ws_bytes < gram_ws(n, k, kw)) { ofrr_set_error("gram: workspace too small"); return OFRR_ERR_INVALID; }
  double* part = (double*)ws;
  switch (storage) {
    case F64: return launch_gram<double>(U, ldu, W, ldw, n, k, kw, out_fmt, G1, G2, flags, part, st);
    case F32: return launch_gram<float>(U, ldu, W, ldw, n, k, kw, out_fmt, G1, G2, flags, part, st);
    case F16: return launch_gram<__half>(U, ldu, W, ldw, n, k, kw, out_fmt, G1, G2, flags, part, st);
    case BF16: return launch_gram<__nv_bfloat16>(U, ldu, W, ldw, n, k, kw, out_fmt, G1, G2, flags, part, st);
    case FP8: return launch_gram<__nv_fp8_e4m3>(U, ldu, W, ldw, n, k, kw, out_fmt, G1, G2, flags, part, st);
    default: ofrr_set_error("gram: storage format %d unsupported", storage); return OFRR_ERR_UNSUPPORTED;
  }
}

}  // namespace ofrr
