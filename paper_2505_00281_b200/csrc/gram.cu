// gram.cu -- K4: projected matrices G1 = U^T W and G2 = U^T U for the OFRR pencil.
//
// Replaces ofrr/projection.py:56-61 (_project) as called from ofrr_eig (:79-80) and
// ofrr_svd (:109-111).  Tall-skinny reduction over the n rows:
//   stage 1: grid (row chunks x 64x64 output tiles); each CTA stages a 32-row slab of
//            U and [W U] in shared memory as fp64 and accumulates 4x4 outputs per thread
//            with fp64 FMA (storage values have <= 24 significant bits, so every product
//            is exact in fp64; only the sums round);
//   stage 2: fixed-order sum of the chunk partials (deterministic), rounding to the
//            projection output format (ofrr/projection.py:42-53), non-finite check.
#include "common.cuh"
#include <algorithm>

namespace ofrr {

static constexpr int GT = 64;   // output tile
static constexpr int GR = 32;   // rows per smem slab

template <typename T>
__global__ void __launch_bounds__(256)
    k_gram_partial(const T* __restrict__ U, int64_t ldu, const T* __restrict__ W, int64_t ldw, int64_t n,
                   int k, int kw, int64_t rows_per_chunk, double* __restrict__ part) {
  // output columns: [0, kw) -> U^T W, [kw, kw + k) -> U^T U
  __shared__ double Us[GR][GT + 1];
  __shared__ double Vs[GR][GT + 1];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int i0 = blockIdx.y * GT;      // rows of the Gram (columns of U)
  const int j0 = blockIdx.z * GT;      // columns of the Gram ([W U])
  const int ncols = kw + k;
  const int64_t rb = (int64_t)blockIdx.x * rows_per_chunk;
  const int64_t re = std::min<int64_t>(n, rb + rows_per_chunk);
  double acc[4][4] = {};
  for (int64_t l0 = rb; l0 < re; l0 += GR) {
    for (int e = tid; e < GR * GT; e += 256) {
      const int c = e / GR, rr = e % GR;   // contiguous along rows (column-major inputs)
      const int64_t l = l0 + rr;
      double u = 0.0, v = 0.0;
      if (l < re) {
        if (i0 + c < k) u = to_d(U[(int64_t)(i0 + c) * ldu + l]);
        const int jc = j0 + c;
        if (jc < kw) v = to_d(W[(int64_t)jc * ldw + l]);
        else if (jc < ncols) v = to_d(U[(int64_t)(jc - kw) * ldu + l]);
      }
      Us[rr][c] = u;
      Vs[rr][c] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < GR; ++rr) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Us[rr][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Vs[rr][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  // partial layout: [chunk][ncols][k] column-major per chunk
  double* dst = part + (int64_t)blockIdx.x * ncols * k;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = i0 + ty + 16 * i, gj = j0 + tx + 16 * j;
      if (gi < k && gj < ncols) dst[(int64_t)gj * k + gi] = acc[i][j];
    }
}

__global__ void k_gram_reduce(const double* __restrict__ part, int nchunks, int k, int kw, int out_fmt,
                              double* __restrict__ G1, double* __restrict__ G2, int* __restrict__ flags) {
  const int ncols = kw + k;
  const int64_t total = (int64_t)ncols * k;
  int bad = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += part[(int64_t)c * total + e];
    s = rnd(s, out_fmt);
    if (!isfinite(s)) bad = 1;
    const int gj = (int)(e / k), gi = (int)(e % k);
    if (gj < kw) { if (G1) G1[(int64_t)gj * k + gi] = s; }
    else if (G2) G2[(int64_t)(gj - kw) * k + gi] = s;
  }
  if (bad && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
}

struct GramPlan { int nchunks; int64_t rows_per; };
static GramPlan gram_plan(int64_t n, int k, int kw) {
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  const int tiles = ((k + GT - 1) / GT) * ((kw + k + GT - 1) / GT);
  int64_t chunks = std::max<int64_t>(1, (2 * sms + tiles - 1) / tiles);
  chunks = std::min<int64_t>(chunks, (n + GR - 1) / GR);
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
  k_gram_reduce<<<(unsigned)std::min<int64_t>((total + 255) / 256, 1024), 256, 0, st>>>(part, p.nchunks, k, kw, out_fmt,
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
