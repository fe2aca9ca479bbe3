// simt.cu -- CUDA-core kernels of the OFRR hot path:
//   * k_gemm_simt: W = op(A) X for F32 / F64 storage (tensor cores have no exact fp32/fp64
//     path; kind::tf32 is not fp32), and the FP64 residual products (K7);
//   * k_scale_columns (K2), k_convert.
#include "common.cuh"
#include <algorithm>
#include <cstdlib>

namespace ofrr {

template <typename T> struct Ld;
template <> struct Ld<double> { __device__ static double get(const void* p, long i) { return ((const double*)p)[i]; } };
template <> struct Ld<float> { __device__ static double get(const void* p, long i) { return (double)((const float*)p)[i]; } };
template <> struct Ld<__half> { __device__ static double get(const void* p, long i) { return (double)__half2float(((const __half*)p)[i]); } };
template <> struct Ld<__nv_bfloat16> { __device__ static double get(const void* p, long i) { return (double)__bfloat162float(((const __nv_bfloat16*)p)[i]); } };
template <> struct Ld<__nv_fp8_storage_t> {
  __device__ static double get(const void* p, long i) {
    __nv_fp8_e4m3 v; v.__x = ((const __nv_fp8_storage_t*)p)[i]; return (double)float(v);
  }
};

// ---------------------------------------------------------------------------------
// C (m x n) = op(A) (m x K) * B (K x n).  A row-major (rows x cols, lda); op(A) = A or A^T.
// B column-major (ldb).  Tiles 64 x 64 x 16, 256 threads, 4x4 register blocking.
// MODE 0: store C rounded to out_fmt (column-major, ldc) + colmax + non-finite flag.
// MODE 1: residual partials  part[blockIdx.x * n + j] = sum_i (C[i,j] - vals[j] * Y[i,j])^2
// ---------------------------------------------------------------------------------
static constexpr int SBM = 64, SBN = 64, SBK = 16;

template <typename TA, typename TB, typename ACC, int MODE>
__global__ void __launch_bounds__(256)
    k_gemm_simt(const void* __restrict__ A, int64_t lda, int transpose, int64_t m, int64_t K,
                const void* __restrict__ B, int64_t ldb, int n, void* __restrict__ C, int64_t ldc,
                int out_fmt, double* __restrict__ colmax, int* __restrict__ flags,
                const double* __restrict__ Y, int64_t ldy, const double* __restrict__ vals,
                const int* __restrict__ r_dev, double* __restrict__ part, void* __restrict__ C2, int64_t ldc2,
                int out_fmt2) {
  __shared__ ACC As[SBK][SBM + 1];
  __shared__ ACC Bs[SBK][SBN + 1];
  __shared__ double cmax[SBN];
  __shared__ double csum[16][SBN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;  // 16 x 16 threads, each 4 x 4 outputs
  const int64_t m0 = (int64_t)blockIdx.x * SBM;
  const int n0 = blockIdx.y * SBN;
  int nvalid = n;
  if (MODE == 1 && r_dev) nvalid = min(n, *r_dev);
  ACC acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = ACC(0);

  for (int64_t k0 = 0; k0 < K; k0 += SBK) {
    // A tile: 64 rows x 16 k  (1024 elements, 4 per thread)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      int r, kk;
      if (!transpose) { r = idx >> 4; kk = idx & 15; }   // contiguous along k
      else { kk = idx >> 6; r = idx & 63; }               // contiguous along m
      const int64_t gr = m0 + r, gk = k0 + kk;
      ACC v = ACC(0);
      if (gr < m && gk < K)
        v = (ACC)Ld<TA>::get(A, transpose ? gk * lda + gr : gr * lda + gk);
      As[kk][r] = v;
    }
    // B tile: 16 k x 64 cols (column-major: contiguous along k)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      const int c = idx >> 4, kk = idx & 15;
      const int64_t gk = k0 + kk;
      const int gc = n0 + c;
      ACC v = ACC(0);
      if (gk < K && gc < n) v = (ACC)Ld<TB>::get(B, (int64_t)gc * ldb + gk);
      Bs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SBK; ++kk) {
      ACC a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }

  if (MODE == 0) {
    if (tid < SBN) cmax[tid] = 0.0;
    __syncthreads();
    int bad = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = n0 + tx + 16 * j;
      double lm = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t gr = m0 + ty + 16 * i;
        if (gr < m && gc < n) {
          const double w = rnd((double)acc[i][j], out_fmt);
          st_fmt(C, (int64_t)gc * ldc + gr, out_fmt, w);
          if (C2) st_fmt(C2, (int64_t)gc * ldc2 + gr, out_fmt2, rnd((double)acc[i][j], out_fmt2));
          if (!isfinite(w)) { bad = 1; lm = INFINITY; }
          else lm = fmax(lm, fabs(w));
        }
      }
      if (gc < n) atomic_max_nonneg(&cmax[tx + 16 * j], lm);
    }
    __syncthreads();
    if (colmax && tid < SBN && n0 + tid < n) atomic_max_nonneg(&colmax[n0 + tid], cmax[tid]);
    if (bad && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
  } else {
    // residual partial sums of squares, fixed order (rows ty, ty+16, ... then over ty)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gc = n0 + tx + 16 * j;
      double s = 0.0;
      if (gc < nvalid) {
        const double lam = vals[gc];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t gr = m0 + ty + 16 * i;
          if (gr < m) {
            const double r = (double)acc[i][j] - lam * Y[(int64_t)gc * ldy + gr];
            s += r * r;
          }
        }
      }
      csum[ty][tx + 16 * j] = s;
    }
    __syncthreads();
    if (tid < SBN) {
      double s = 0.0;
      for (int y = 0; y < 16; ++y) s += csum[y][tid];
      if (n0 + tid < n) part[(int64_t)blockIdx.x * n + n0 + tid] = s;
    }
  }
}

// ---------------------------------------------------------------------------------
// FP64 residual product (K7), tuned: C = A (rows x K, row-major, any storage format,
// promoted exactly to fp64) * V (K x r, column-major fp64), epilogue
// part[block, j] = sum_rows (C[i,j] - vals[j] * Y[i,j])^2.
// CTA tile 128 x 64, BK = 32, 256 threads, 8 x 4 fp64 accumulators per thread,
// double-buffered shared memory (A staged transposed as fp64 so a warp's A reads are
// broadcasts), 16-byte global loads.  FP64-FMA bound.
// ---------------------------------------------------------------------------------
static constexpr int RBM = 128, RBN = 64, RBK = 32;

// Raw global staging of one k-tile (kept in registers while the previous tile computes):
// A: thread -> (row tid & 127, k half tid >> 7) : 16 consecutive elements of one row
// B: thread -> (col tid >> 2, k quarter tid & 3): 8 consecutive fp64 of one column
template <typename TA>
struct ResidStage {
  uint4 araw[2];   // 16 x 16-bit values (vector path)
  TA a[16];        // scalar path
  double b[8];
  bool vec;
};

template <typename TA>
__device__ __forceinline__ void resid_fetch(const TA* __restrict__ A, int64_t lda, const double* __restrict__ V,
                                            int64_t ldv, int64_t m0, int n0, int64_t k0, int64_t m, int64_t K, int n,
                                            int tid, ResidStage<TA>& st) {
  const int r = tid & 127, kh = (tid >> 7) * 16;
  const int64_t gr = m0 + r;
  st.vec = false;
  if constexpr (sizeof(TA) == 2) {
    if (gr < m && k0 + kh + 16 <= K) {
      const uint4* p = reinterpret_cast<const uint4*>(A + gr * lda + k0 + kh);
      st.araw[0] = __ldg(p);
      st.araw[1] = __ldg(p + 1);
      st.vec = true;
    }
  }
  if (!st.vec) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int64_t gk = k0 + kh + e;
      st.a[e] = (gr < m && gk < K) ? A[gr * lda + gk] : from_d<TA>(0.0);
    }
  }
  const int c = tid >> 2, kq = (tid & 3) * 8;
  const int gc = n0 + c;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int64_t gk = k0 + kq + e;
    st.b[e] = (gc < n && gk < K) ? V[(int64_t)gc * ldv + gk] : 0.0;
  }
}

// converts (exactly) to fp64 only here, after the previous tile's math, so the global
// loads of resid_fetch stay in flight across the compute loop
template <typename TA>
__device__ __forceinline__ void resid_store(double (*As)[RBM + 1], double (*Bs)[RBN + 1], int tid,
                                            const ResidStage<TA>& st) {
  const int r = tid & 127, kh = (tid >> 7) * 16;
  if constexpr (sizeof(TA) == 2) {
    if (st.vec) {
      const uint32_t w[8] = {st.araw[0].x, st.araw[0].y, st.araw[0].z, st.araw[0].w,
                             st.araw[1].x, st.araw[1].y, st.araw[1].z, st.araw[1].w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        TA lo, hi;
        const uint16_t l16 = (uint16_t)(w[e] & 0xffffu), h16 = (uint16_t)(w[e] >> 16);
        memcpy(&lo, &l16, 2);
        memcpy(&hi, &h16, 2);
        As[kh + 2 * e][r] = to_d(lo);        // a warp: 32 consecutive rows
        As[kh + 2 * e + 1][r] = to_d(hi);
      }
    }
  }
  if (!st.vec) {
#pragma unroll
    for (int e = 0; e < 16; ++e) As[kh + e][r] = to_d(st.a[e]);
  }
  const int c = tid >> 2, kq = (tid & 3) * 8;
#pragma unroll
  for (int e = 0; e < 8; ++e) Bs[kq + e][c] = st.b[e];
}

template <typename TA>
__global__ void __launch_bounds__(256, 1)
    k_resid64(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t K, const double* __restrict__ V, int64_t ldv,
              int n, const double* __restrict__ Y, int64_t ldy, const double* __restrict__ vals,
              const int* __restrict__ r_dev, double* __restrict__ part) {
  extern __shared__ double rsm[];
  double (*As)[RBM + 1] = reinterpret_cast<double (*)[RBM + 1]>(rsm);                       // [2][RBK][RBM+1]
  double (*Bs)[RBN + 1] = reinterpret_cast<double (*)[RBN + 1]>(rsm + 2 * RBK * (RBM + 1));  // [2][RBK][RBN+1]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * RBM;
  const int n0 = blockIdx.y * RBN;
  const int nvalid = r_dev ? min(n, *r_dev) : n;
  // thread (ty, tx) owns rows ty + 16 i (i < 8) and columns tx + 16 j (j < 4): smem reads
  // of a warp are broadcasts (A) or 16 consecutive doubles (B) -- bank-conflict free
  double acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int nk = (int)((K + RBK - 1) / RBK);
  ResidStage<TA> st;
  resid_fetch<TA>(A, lda, V, ldv, m0, n0, 0, m, K, n, tid, st);
  resid_store<TA>(As, Bs, tid, st);
  __syncthreads();
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    double (*Ac)[RBM + 1] = As + cur * RBK;
    double (*Bc)[RBN + 1] = Bs + cur * RBK;
    const bool more = t + 1 < nk;
    if (more) resid_fetch<TA>(A, lda, V, ldv, m0, n0, (int64_t)(t + 1) * RBK, m, K, n, tid, st);
#pragma unroll 8
    for (int kk = 0; kk < RBK; ++kk) {
      double a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Ac[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bc[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    if (more) resid_store<TA>(As + (cur ^ 1) * RBK, Bs + (cur ^ 1) * RBK, tid, st);
    __syncthreads();
  }
  // epilogue: per-column sums of squares over this CTA's rows, fixed order
  double* csum = rsm;   // reuse: [16][RBN]
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int gc = n0 + tx + 16 * j;
    double s = 0.0;
    if (gc < nvalid) {
      const double lam = vals[gc];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t gr = m0 + ty + 16 * i;
        if (gr < m) {
          const double d = acc[i][j] - lam * Y[(int64_t)gc * ldy + gr];
          s = fma(d, d, s);
        }
      }
    }
    csum[ty * RBN + tx + 16 * j] = s;
  }
  __syncthreads();
  if (tid < RBN && n0 + tid < n) {
    double s = 0.0;
    for (int y = 0; y < 16; ++y) s += csum[y * RBN + tid];
    part[(int64_t)blockIdx.x * n + n0 + tid] = s;
  }
}

// ---------------------------------------------------------------------------------
// FP64 residual product on the FP64 tensor cores (DMMA, mma.sync m8n8k4 f64):
// CTA tile 128 x 64, 8 warps as 4 (rows) x 2 (cols), warp tile 32 x 32 = 4 x 4 DMMA tiles,
// k-tile 32 staged as As[m][k] / Bs[n][k] (k contiguous, padded to 36: fragment loads
// are bank-conflict free), register-staged prefetch of the next k-tile.
// Fragments (PTX m8n8k4 .f64): a = A[lane/4][lane%4], b = B[lane%4][lane/4],
// c[2] = C[lane/4][2*(lane%4) + {0,1}].
// ---------------------------------------------------------------------------------
static constexpr int DBM = 128, DBN = 64, DBK = 32, DLK = 36;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename TA>
__global__ void __launch_bounds__(256, 1)
    k_resid_dmma(const TA* __restrict__ A, int64_t lda, int64_t m, int64_t K, const double* __restrict__ V,
                 int64_t ldv, int n, const double* __restrict__ Y, int64_t ldy, const double* __restrict__ vals,
                 const int* __restrict__ r_dev, double* __restrict__ part) {
  extern __shared__ double dsh[];
  double* As = dsh;                        // [2][DBM][DLK]
  double* Bs = dsh + 2 * DBM * DLK;        // [2][DBN][DLK]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;   // warp tile origin: rows 32*wm, cols 32*wn
  const int64_t m0 = (int64_t)blockIdx.x * DBM;
  const int n0 = blockIdx.y * DBN;
  const int nvalid = r_dev ? min(n, *r_dev) : n;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // staging: A tile 128 x 32 -> thread (row tid/2, 16 k); V tile 64 cols x 32 k -> thread (col tid/4, 8 k)
  uint4 araw[2];
  double areg[16], breg[8];
  bool avec = false;
  auto fetch = [&](int64_t k0) {
    const int r = tid >> 1, kh = (tid & 1) * 16;
    const int64_t gr = m0 + r;
    avec = false;
    if constexpr (sizeof(TA) == 2) {
      if (gr < m && k0 + kh + 16 <= K) {
        const uint4* pp = reinterpret_cast<const uint4*>(A + gr * lda + k0 + kh);
        araw[0] = __ldg(pp);
        araw[1] = __ldg(pp + 1);
        avec = true;
      }
    }
    if (!avec) {
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t gk = k0 + kh + e;
        areg[e] = (gr < m && gk < K) ? to_d(A[gr * lda + gk]) : 0.0;
      }
    }
    const int c = tid >> 2, kq = (tid & 3) * 8;
    const int gc = n0 + c;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t gk = k0 + kq + e;
      breg[e] = (gc < n && gk < K) ? V[(int64_t)gc * ldv + gk] : 0.0;
    }
  };
  auto store = [&](int buf) {
    const int r = tid >> 1, kh = (tid & 1) * 16;
    double* Ab = As + buf * DBM * DLK + r * DLK + kh;
    if constexpr (sizeof(TA) == 2) {
      if (avec) {
        const uint32_t w[8] = {araw[0].x, araw[0].y, araw[0].z, araw[0].w, araw[1].x, araw[1].y, araw[1].z, araw[1].w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          TA lo, hi;
          const uint16_t l16 = (uint16_t)(w[e] & 0xffffu), h16 = (uint16_t)(w[e] >> 16);
          memcpy(&lo, &l16, 2);
          memcpy(&hi, &h16, 2);
          Ab[2 * e] = to_d(lo);
          Ab[2 * e + 1] = to_d(hi);
        }
      }
    }
    if (!avec) {
#pragma unroll
      for (int e = 0; e < 16; ++e) Ab[e] = areg[e];
    }
    const int c = tid >> 2, kq = (tid & 3) * 8;
    double* Bb = Bs + buf * DBN * DLK + c * DLK + kq;
#pragma unroll
    for (int e = 0; e < 8; ++e) Bb[e] = breg[e];
  };
  const int nk = (int)((K + DBK - 1) / DBK);
  fetch(0);
  store(0);
  __syncthreads();
  const int fr = lane >> 2, fk = lane & 3;
  for (int t = 0; t < nk; ++t) {
    const int cur = t & 1;
    const bool more = t + 1 < nk;
    if (more) fetch((int64_t)(t + 1) * DBK);
    const double* Ab = As + cur * DBM * DLK + (32 * wm + fr) * DLK + fk;
    const double* Bb = Bs + cur * DBN * DLK + (32 * wn + fr) * DLK + fk;
#pragma unroll
    for (int kk = 0; kk < DBK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Ab[i * 8 * DLK + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bb[j * 8 * DLK + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    if (more) store(cur ^ 1);
    __syncthreads();
  }
  // epilogue: C[row][col] = acc[i][j][e] at row 32 wm + 8 i + lane/4, col 32 wn + 8 j + 2 (lane%4) + e
  double* csum = dsh;   // [4 (wm)][DBN] partial column sums (reuse smem after the final barrier)
  for (int e = tid; e < 4 * DBN; e += blockDim.x) csum[e] = 0.0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int lc = 32 * wn + 8 * j + 2 * (lane & 3) + h;
      const int gc = n0 + lc;
      double s = 0.0;
      if (gc < nvalid) {
        const double lam = vals[gc];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t gr = m0 + 32 * wm + 8 * i + (lane >> 2);
          if (gr < m) {
            const double d = acc[i][j][h] - lam * Y[(int64_t)gc * ldy + gr];
            s = fma(d, d, s);
          }
        }
      }
      // reduce over the 8 lanes sharing this column (lane>>2 varies), fixed order
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if ((lane >> 2) == 0) csum[wm * DBN + lc] = s;
    }
  __syncthreads();
  if (tid < DBN && n0 + tid < n) {
    const double s = ((csum[tid] + csum[DBN + tid]) + csum[2 * DBN + tid]) + csum[3 * DBN + tid];
    part[(int64_t)blockIdx.x * n + n0 + tid] = s;
  }
}

template <typename TA>
static int launch_resid_dmma(const void* A, int64_t lda, int64_t m, int64_t K, const double* V, int64_t ldv, int n,
                             const double* Y, int64_t ldy, const double* vals, const int* r_dev, double* part,
                             cudaStream_t st) {
  const size_t shm = (size_t)2 * (DBM + DBN) * DLK * sizeof(double);
  static std::atomic<bool> attr{false};   // set once; concurrent callers may both set it (idempotent)
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_resid_dmma<TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr = true;
  }
  dim3 grid((unsigned)((m + DBM - 1) / DBM), (unsigned)((n + DBN - 1) / DBN));
  k_resid_dmma<TA><<<grid, 256, shm, st>>>((const TA*)A, lda, m, K, V, ldv, n, Y, ldy, vals, r_dev, part);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

template <typename TA>
static int launch_resid64(const void* A, int64_t lda, int64_t m, int64_t K, const double* V, int64_t ldv, int n,
                          const double* Y, int64_t ldy, const double* vals, const int* r_dev, double* part,
                          cudaStream_t st) {
  const size_t shm = (size_t)2 * RBK * ((RBM + 1) + (RBN + 1)) * sizeof(double);
  static std::atomic<bool> attr{false};   // set once; concurrent callers may both set it (idempotent)
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_resid64<TA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm));
    attr = true;
  }
  dim3 grid((unsigned)((m + RBM - 1) / RBM), (unsigned)((n + RBN - 1) / RBN));
  k_resid64<TA><<<grid, 256, shm, st>>>((const TA*)A, lda, m, K, V, ldv, n, Y, ldy, vals, r_dev, part);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// res[j] = sqrt(sum_b part[b, j]) / |vals[j]|  (inf for vals[j] == 0), fixed order.
// one warp per column: lane l sums blocks l, l + 32, ... (ascending), then a fixed
// butterfly -- a fixed summation order (deterministic) with the latency of nblocks / 32 adds
__global__ void k_residual_reduce(const double* __restrict__ part, int nblocks, int n,
                                  const double* __restrict__ vals, const int* __restrict__ r_dev,
                                  double* __restrict__ res, int accumulate_max) {
  const int j = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (j >= n) return;
  // accumulate_max: 0 -> res = ||r|| / |lambda|; 1 -> res = max(res, ||r|| / |lambda|);
  //                 2 -> res = raw sum of squares (row-partitioned runs all-reduce it first)
  const int nvalid = r_dev ? min(n, *r_dev) : n;
  if (j >= nvalid) { if (accumulate_max != 1 && lane == 0) res[j] = 0.0; return; }
  double s = 0.0;
  for (int b = lane; b < nblocks; b += 32) s += part[(int64_t)b * n + j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane != 0) return;
  if (accumulate_max == 2) { res[j] = s; return; }
  const double lam = vals[j];
  const double r = lam == 0.0 ? INFINITY : sqrt(s) / fabs(lam);
  res[j] = accumulate_max ? fmax(res[j], r) : r;
}

template <typename TA, typename TB, typename ACC, int MODE>
static int launch_simt(const void* A, int64_t lda, int transpose, int64_t m, int64_t K, const void* B,
                       int64_t ldb, int n, void* C, int64_t ldc, int out_fmt, double* colmax, int* flags,
                       const double* Y, int64_t ldy, const double* vals, const int* r_dev, double* part,
                       cudaStream_t st, void* C2 = nullptr, int64_t ldc2 = 0, int out_fmt2 = 0) {
  dim3 grid((unsigned)((m + SBM - 1) / SBM), (unsigned)((n + SBN - 1) / SBN));
  k_gemm_simt<TA, TB, ACC, MODE><<<grid, 256, 0, st>>>(A, lda, transpose, m, K, B, ldb, n, C, ldc, out_fmt,
                                                       colmax, flags, Y, ldy, vals, r_dev, part, C2, ldc2, out_fmt2);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

int simt_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose,
                 const void* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax,
                 int* flags, cudaStream_t st, void* W2, int64_t ldw2, int out_fmt2) {
  const int64_t m = transpose ? cols : rows, K = transpose ? rows : cols;
  if (a_fmt == F64)
    return launch_simt<double, double, double, 0>(A, lda, transpose, m, K, X, ldx, k, W, ldw, out_fmt, colmax,
                                                  flags, nullptr, 0, nullptr, nullptr, nullptr, st, W2, ldw2, out_fmt2);
  if (a_fmt == F32)
    return launch_simt<float, float, float, 0>(A, lda, transpose, m, K, X, ldx, k, W, ldw, out_fmt, colmax,
                                               flags, nullptr, 0, nullptr, nullptr, nullptr, st, W2, ldw2, out_fmt2);
  ofrr_set_error("simt_gemm_av: format %d not supported on the CUDA-core path", a_fmt);
  return OFRR_ERR_UNSUPPORTED;
}

int residual_reduce(const double* part, int nblocks, int n, const double* vals, const int* r_dev, double* res,
                    int mode, cudaStream_t st) {
  k_residual_reduce<<<(n + 3) / 4, 128, 0, st>>>(part, nblocks, n, vals, r_dev, res, mode);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

size_t residual_ws(int64_t rows, int r) {
  return (size_t)((rows + SBM - 1) / SBM) * (size_t)r * sizeof(double);
}

size_t oz_ws(int64_t rows, int64_t cols, int r);
int oz_product(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const double* V, int64_t ldv,
               int r, const double* vals, const int* r_dev, const double* Y, int64_t ldy, double* W, int64_t ldw,
               double** part_out, void* ws, size_t ws_bytes, cudaStream_t st);
int oz_nblocks(int64_t rows);

// The FP64-accurate residual product runs on the int8 tensor cores (oz.cu) for 16/8-bit
// operators; OFRR_RESID_DMMA=1 forces the FP64 DMMA kernel (and OFRR_RESID_SIMT=1 the
// CUDA-core one) for comparison.
static bool use_ozaki(int a_fmt, int transpose) {
  static int force = -1;
  if (force < 0) {
    const char* e = getenv("OFRR_RESID_DMMA");
    const char* f = getenv("OFRR_RESID_SIMT");
    force = ((e && atoi(e) == 1) || (f && atoi(f) == 1)) ? 1 : 0;
  }
  return !force && !transpose && (a_fmt == BF16 || a_fmt == F16 || a_fmt == FP8);
}

size_t residual_ws2(int64_t rows, int64_t cols, int r, int a_fmt, int transpose) {
  const int64_t m = transpose ? cols : rows;
  if (use_ozaki(a_fmt, transpose)) return oz_ws(rows, cols, r);
  return residual_ws(m, r);
}

int simt_residual(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose,
                  const double* Xv, int64_t ldx, const double* Yv, int64_t ldy, const double* vals,
                  const int* r_dev, int r_max, double* res, int accumulate_max, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  const int64_t m = transpose ? cols : rows, K = transpose ? rows : cols;
  if (use_ozaki(a_fmt, transpose)) {
    double* part = nullptr;
    const int rc = oz_product(A, rows, cols, lda, a_fmt, Xv, ldx, r_max, vals, r_dev, Yv, ldy, nullptr, 0, &part,
                              ws, ws_bytes, st);
    if (rc) return rc;
    k_residual_reduce<<<(r_max + 3) / 4, 128, 0, st>>>(part, oz_nblocks(m), r_max, vals, r_dev, res,
                                                           accumulate_max);
    OFRR_CHECK_LAUNCH();
    return OFRR_OK;
  }
  const size_t need = residual_ws(m, r_max);
  if (!ws || ws_bytes < need) { ofrr_set_error("residual: workspace too small (%zu < %zu)", ws_bytes, need); return OFRR_ERR_INVALID; }
  double* part = (double*)ws;
  int rc;
  if (!transpose && a_fmt != FP8) {
    static int use_simt = -1;
    if (use_simt < 0) { const char* e = getenv("OFRR_RESID_SIMT"); use_simt = (e && atoi(e) == 1) ? 1 : 0; }
    if (use_simt) {
      switch (a_fmt) {
        case F64: rc = launch_resid64<double>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        case F32: rc = launch_resid64<float>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        case F16: rc = launch_resid64<__half>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        default: rc = launch_resid64<__nv_bfloat16>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
      }
    } else {
      switch (a_fmt) {
        case F64: rc = launch_resid_dmma<double>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        case F32: rc = launch_resid_dmma<float>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        case F16: rc = launch_resid_dmma<__half>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
        default: rc = launch_resid_dmma<__nv_bfloat16>(A, lda, m, K, Xv, ldx, r_max, Yv, ldy, vals, r_dev, part, st); break;
      }
    }
    if (rc) return rc;
    const int nb = (int)((m + RBM - 1) / RBM);
    k_residual_reduce<<<(r_max + 3) / 4, 128, 0, st>>>(part, nb, r_max, vals, r_dev, res, accumulate_max);
    OFRR_CHECK_LAUNCH();
    return OFRR_OK;
  }
  switch (a_fmt) {
    case F64: rc = launch_simt<double, double, double, 1>(A, lda, transpose, m, K, Xv, ldx, r_max, nullptr, 0, 0, nullptr, nullptr, Yv, ldy, vals, r_dev, part, st); break;
    case F32: rc = launch_simt<float, double, double, 1>(A, lda, transpose, m, K, Xv, ldx, r_max, nullptr, 0, 0, nullptr, nullptr, Yv, ldy, vals, r_dev, part, st); break;
    case F16: rc = launch_simt<__half, double, double, 1>(A, lda, transpose, m, K, Xv, ldx, r_max, nullptr, 0, 0, nullptr, nullptr, Yv, ldy, vals, r_dev, part, st); break;
    case BF16: rc = launch_simt<__nv_bfloat16, double, double, 1>(A, lda, transpose, m, K, Xv, ldx, r_max, nullptr, 0, 0, nullptr, nullptr, Yv, ldy, vals, r_dev, part, st); break;
    default: rc = launch_simt<__nv_fp8_storage_t, double, double, 1>(A, lda, transpose, m, K, Xv, ldx, r_max, nullptr, 0, 0, nullptr, nullptr, Yv, ldy, vals, r_dev, part, st); break;
  }
  if (rc) return rc;
  const int nb = (int)((m + SBM - 1) / SBM);
  k_residual_reduce<<<(r_max + 3) / 4, 128, 0, st>>>(part, nb, r_max, vals, r_dev, res, accumulate_max);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// ---------------------------------------------------------------------------------
// K2: X[:,j] <- round_s(round_c(X[:,j] / colmax[j]))   (ofrr/precision.py:159-169)
// ---------------------------------------------------------------------------------
__global__ void k_scale_columns(void* __restrict__ X, int64_t n, int k, int64_t ldx, int storage,
                                int compute, const double* __restrict__ colmax) {
  const int j = blockIdx.y;
  const double m = (double)colmax[j];
  if (m == 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = (int64_t)j * ldx + i;
    const double x = ld_fmt(X, o, storage);
    st_fmt(X, o, storage, rnd(c_div(x, m, compute), storage));
  }
}

// the same for 4-byte / 8-byte storage with four elements in flight per thread (the generic
// kernel above runs one dependent load per iteration and is latency-bound at C3)
template <typename T>
__global__ void __launch_bounds__(256) k_scale_columns4(T* __restrict__ X, int64_t n, int64_t ldx, int storage,
                                                        int compute, const double* __restrict__ colmax) {
  const int j = blockIdx.y;
  const double m = (double)colmax[j];
  if (m == 0.0) return;
  T* col = X + (int64_t)j * ldx;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = i0 + u * stride < n ? (double)col[i0 + u * stride] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (i0 + u * stride < n) col[i0 + u * stride] = (T)rnd(c_div(x[u], m, compute), storage);
  }
}

int scale_columns(void* X, int64_t n, int k, int64_t ldx, int storage, int compute, const double* colmax,
                  cudaStream_t st) {
  if (k <= 0 || n <= 0) return OFRR_OK;
  unsigned gx = (unsigned)std::min<int64_t>((n + 255) / 256, 64);
  if (storage == F32 || storage == F64) {
    const unsigned g4 = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 1023) / 1024, 16));
    if (storage == F32)
      k_scale_columns4<float><<<dim3(g4, k), 256, 0, st>>>((float*)X, n, ldx, storage, compute, colmax);
    else
      k_scale_columns4<double><<<dim3(g4, k), 256, 0, st>>>((double*)X, n, ldx, storage, compute, colmax);
    OFRR_CHECK_LAUNCH();
    return OFRR_OK;
  }
  k_scale_columns<<<dim3(gx, k), 256, 0, st>>>(X, n, k, ldx, storage, compute, colmax);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

__global__ void k_convert(const void* __restrict__ src, int sf, int64_t lds, void* __restrict__ dst, int df,
                          int64_t ldd, int64_t n, int64_t k, int* __restrict__ flags) {
  int bad = 0;
  const int64_t total = n * k;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e - j * n;
    const double x = ld_fmt(src, j * lds + i, sf);
    const double v = rnd(x, df);
    if (!isfinite(v)) bad |= OFRR_FLAG_NONFINITE;
    if (v != x && x == x) bad |= OFRR_FLAG_INEXACT;
    st_fmt(dst, j * ldd + i, df, v);
  }
  if (bad && flags) atomicOr(flags, bad);
}

// dst (row-major rows x cols, ldd) <- round(src (column-major rows x cols, lds)): uploads of
// the reference's F-order float64 operators into the device's row-major storage layout.
__global__ void k_transpose_convert(const void* __restrict__ src, int sf, int64_t lds, void* __restrict__ dst, int df,
                                    int64_t ldd, int64_t rows, int64_t cols, int* __restrict__ flags) {
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, r = r0 + threadIdx.x;
    tile[y][threadIdx.x] = (c < cols && r < rows) ? ld_fmt(src, c * lds + r, sf) : 0.0;
  }
  __syncthreads();
  int bad = 0;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = r0 + y, c = c0 + threadIdx.x;
    if (r < rows && c < cols) {
      const double x = tile[threadIdx.x][y];
      const double v = rnd(x, df);
      if (!isfinite(v)) bad |= OFRR_FLAG_NONFINITE;
      if (v != x && x == x) bad |= OFRR_FLAG_INEXACT;
      st_fmt(dst, r * ldd + c, df, v);
    }
  }
  if (bad && flags) atomicOr(flags, bad);
}

int transpose_convert(const void* src, int sf, int64_t lds, void* dst, int df, int64_t ldd, int64_t rows, int64_t cols,
                      int* flags, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return OFRR_OK;
  for (int64_t rb = 0; rb < rows; rb += 32 * 65535) {
    const int64_t rr = std::min<int64_t>(rows - rb, 32 * 65535);
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rr + 31) / 32));
    k_transpose_convert<<<grid, dim3(32, 8), 0, st>>>((const uint8_t*)src + rb * fmt_bytes(sf), sf, lds,
                                                      (uint8_t*)dst + rb * ldd * fmt_bytes(df), df, ldd, rr, cols,
                                                      flags);
    OFRR_CHECK_LAUNCH();
  }
  return OFRR_OK;
}

int convert(const void* src, int sf, int64_t lds, void* dst, int df, int64_t ldd, int64_t n, int64_t k,
            int* flags, cudaStream_t st) {
  if (n <= 0 || k <= 0) return OFRR_OK;
  const int64_t total = n * k;
  unsigned g = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_convert<<<g, 256, 0, st>>>(src, sf, lds, dst, df, ldd, n, k, flags);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
