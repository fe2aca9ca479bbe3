// ritz.cu -- K6 (Ritz-vector recovery) and K8 (synthetic symmetric generator).
#include "common.cuh"
#include <algorithm>

namespace ofrr {

// ---------------------------------------------------------------------------------
// K6: Ut = scale * U[:, :kp] * Y[:kp, :r]  in fp64, fused with the storage rounding of
// the restart block (and, for A-pass reuse, the column inf-norms of the rounded block).
// Replaces ofrr/projection.py:86 / :129-130 and ofrr/driver.py:109.  On the fp64 tensor
// cores (DMMA m8n8k4): 64 x 64 output tile per CTA, each warp a 16 x 32 block (2 x 4 MMA
// tiles), kp in slabs of 16 staged in shared memory as fp64 (storage values are exact).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void dmma884r(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
template <typename T>
__global__ void __launch_bounds__(256)
    k_ritz_dmma(const T* __restrict__ U, int64_t ldu, int64_t n, int kp, const double* __restrict__ Y, int ldy,
                const int* __restrict__ r_dev, int r_max, double scale, double* __restrict__ Ut64, int64_t ldo64,
                void* __restrict__ Xout, int64_t ldx, int x_fmt, int* __restrict__ flags,
                double* __restrict__ colmax) {
  constexpr int RS = 16 + 4;                 // Us row stride (doubles)
  __shared__ double Us[64][RS];              // [row][l]
  __shared__ double Ys[16][64 + 4];          // [l][col]
  __shared__ double cm[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;
  const int64_t m0 = (int64_t)blockIdx.x * 64;
  const int n0 = blockIdx.y * 64;
  const int r = r_dev ? min(r_max, *r_dev) : r_max;
  double acc[2][4][2] = {};
  for (int l0 = 0; l0 < kp; l0 += 16) {
    for (int e = tid; e < 16 * 64; e += 256) {
      const int rr = e & 63, ll = e >> 6;
      const int64_t gi = m0 + rr;
      Us[rr][ll] = (gi < n && l0 + ll < kp) ? to_d(U[(int64_t)(l0 + ll) * ldu + gi]) : 0.0;
      const int gj = n0 + rr;
      Ys[ll][rr] = (gj < r && l0 + ll < kp) ? Y[(int64_t)gj * ldy + l0 + ll] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) a[i] = Us[wm + 8 * i + g][kk + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ys[kk + t][wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884r(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  if (colmax && tid < 64) cm[tid] = 0.0;
  if (colmax) __syncthreads();
  int bad = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    double cmx[2] = {0.0, 0.0};
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gi = m0 + wm + 8 * i + g;
        const int gj = n0 + wn + 8 * j + 2 * t + h;
        if (gi >= n || gj >= r_max) continue;
        const double v = gj < r ? scale * acc[i][j][h] : 0.0;
        if (Ut64) Ut64[(int64_t)gj * ldo64 + gi] = v;
        if (Xout) {
          const double xv = rnd(v, x_fmt);
          if (!isfinite(xv)) bad = 1;
          st_fmt(Xout, (int64_t)gj * ldx + gi, x_fmt, xv);
          cmx[h] = fmax(cmx[h], fabs(xv));
        }
      }
    if (colmax) {
#pragma unroll
      for (int h = 0; h < 2; ++h) atomic_max_nonneg(&cm[wn + 8 * j + 2 * t + h], cmx[h]);
    }
  }
  if (bad && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
  if (colmax) {
    __syncthreads();
    if (tid < 64 && n0 + tid < r_max) atomic_max_nonneg(&colmax[n0 + tid], cm[tid]);
  }
}

int ritz_recover(const void* U, int64_t ldu, int u_fmt, int64_t n, int kp, const double* Y, int ldy, const int* r_dev,
                 int r_max, double scale, double* Ut64, int64_t ldo64, void* Xout, int64_t ldx, int x_fmt, int* flags,
                 cudaStream_t st, double* colmax) {
  if (n <= 0 || r_max <= 0) return OFRR_OK;
  dim3 grid((unsigned)((n + 63) / 64), (unsigned)((r_max + 63) / 64));
  switch (u_fmt) {
    case F64: k_ritz_dmma<double><<<grid, 256, 0, st>>>((const double*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags, colmax); break;
    case F32: k_ritz_dmma<float><<<grid, 256, 0, st>>>((const float*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags, colmax); break;
    case F16: k_ritz_dmma<__half><<<grid, 256, 0, st>>>((const __half*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags, colmax); break;
    case BF16: k_ritz_dmma<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags, colmax); break;
    case FP8: k_ritz_dmma<__nv_fp8_e4m3><<<grid, 256, 0, st>>>((const __nv_fp8_e4m3*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags, colmax); break;
    default: ofrr_set_error("ritz: basis format %d unsupported", u_fmt); return OFRR_ERR_UNSUPPORTED;
  }
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// ---------------------------------------------------------------------------------
// K7e: residual estimate for the per-iteration convergence test.
//   r_j = || (W - lambda_j U) y_j ||_2      with W = A U kept in the accumulation format
// (fp32 from the tensor cores, fp64 on the fp64 path) -- since A (U y) = (A U) y, this is
// the Ritz residual up to the accumulation error of W, without another pass over A.
// Partial sums of squares per 64-row block -> part[block * r_max + j] (fixed order).
// ---------------------------------------------------------------------------------
// On the fp64 tensor cores (DMMA m8n8k4): 32 rows x 32 Ritz columns per 128-thread CTA,
// each warp a 16 x 16 block of both products (U y and W y, 2 x 2 MMA tiles each), kp in
// slabs of 32 staged in shared memory as fp64 (storage values are exact).  At C2
// (n = 16384, r = 32) that is 512 CTAs, all resident at once; no work past column r.
// The per-column sums of squares reduce over the 8 row lanes of each MMA tile by a fixed
// butterfly, then over the CTA's 4 row groups in fixed order.
constexpr int RE_BM = 32, RE_BN = 32, RE_KC = 32, RE_RS = RE_KC + 4;

template <typename TU, typename TW>
__global__ void __launch_bounds__(128)
    k_resid_est(const TU* __restrict__ U, int64_t ldu, const TW* __restrict__ W, int64_t ldw, int64_t n,
                int kp, const double* __restrict__ Y, int ldy, const int* __restrict__ r_dev,
                int r_max, const double* __restrict__ vals, double* __restrict__ part) {
  __shared__ double Us[RE_BM][RE_RS];        // [row][l]
  __shared__ double Ws[RE_BM][RE_RS];
  __shared__ double Ys[RE_KC][RE_BN + 4];    // [l][col]
  __shared__ double csum[2][RE_BN];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 16;
  const int64_t m0 = (int64_t)blockIdx.x * RE_BM;
  const int n0 = blockIdx.y * RE_BN;
  const int r = r_dev ? min(r_max, *r_dev) : r_max;
  double au[2][2][2] = {}, aw[2][2][2] = {};
  if (n0 < r) {
    for (int l0 = 0; l0 < kp; l0 += RE_KC) {
#pragma unroll
      for (int q = 0; q < RE_KC * RE_BM / 128; ++q) {
        const int e = tid + 128 * q, rr = e & 31, ll = e >> 5;
        const int64_t gi = m0 + rr;
        const bool ok = gi < n && l0 + ll < kp;
        Us[rr][ll] = ok ? to_d(U[(int64_t)(l0 + ll) * ldu + gi]) : 0.0;
        Ws[rr][ll] = ok ? to_d(W[(int64_t)(l0 + ll) * ldw + gi]) : 0.0;
        // Y is k x r column-major (ldy): the fast index runs down a column
        const int gj = n0 + ll;
        Ys[rr][ll] = (gj < r && l0 + rr < kp) ? Y[(int64_t)gj * ldy + l0 + rr] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < RE_KC; kk += 4) {
        double a[2], w[2], b[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) { a[i] = Us[wm + 8 * i + g][kk + t]; w[i] = Ws[wm + 8 * i + g][kk + t]; }
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j] = Ys[kk + t][wn + 8 * j + g];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) { dmma884r(au[i][j], a[i], b[j]); dmma884r(aw[i][j], w[i], b[j]); }
      }
      __syncthreads();
    }
  }
  // thread holds rows wm + 8i + g, columns wn + 8j + 2t + h
#pragma unroll
  for (int j = 0; j < 2; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int gj = n0 + wn + 8 * j + 2 * t + h;
      double s = 0.0;
      if (gj < r) {
        const double lam = vals[gj];
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (m0 + wm + 8 * i + g < n) {
            const double d = aw[i][j][h] - lam * au[i][j][h];
            s += d * d;
          }
      }
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      s += __shfl_xor_sync(0xffffffffu, s, 8);
      s += __shfl_xor_sync(0xffffffffu, s, 16);
      if (g == 0) csum[warp >> 1][wn + 8 * j + 2 * t + h] = s;
    }
  __syncthreads();
  if (tid < RE_BN && n0 + tid < r_max) part[(int64_t)blockIdx.x * r_max + n0 + tid] = csum[0][tid] + csum[1][tid];
}

int residual_reduce(const double* part, int nblocks, int n, const double* vals, const int* r_dev, double* res,
                    int mode, cudaStream_t st);

size_t resid_est_ws(int64_t n, int r) { return (size_t)((n + RE_BM - 1) / RE_BM) * (size_t)r * sizeof(double); }

int resid_est(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n, int kp,
              const double* Y, int ldy, const double* vals, const int* r_dev, int r_max, double* res, int mode,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n <= 0 || r_max <= 0) return OFRR_OK;
  if (ws_bytes < resid_est_ws(n, r_max)) { ofrr_set_error("residual estimate: workspace too small"); return OFRR_ERR_INVALID; }
  const int nb = (int)((n + RE_BM - 1) / RE_BM);
  dim3 grid((unsigned)nb, (unsigned)((r_max + RE_BN - 1) / RE_BN));
  double* part = (double*)ws;
  auto go = [&](auto tu, auto tw) {
    using TU = decltype(tu);
    using TW = decltype(tw);
    k_resid_est<TU, TW><<<grid, 128, 0, st>>>((const TU*)U, ldu, (const TW*)W, ldw, n, kp, Y, ldy, r_dev, r_max,
                                              vals, part);
  };
  auto with_u = [&](auto tw) {
    switch (u_fmt) {
      case F64: go(double(), tw); break;
      case F32: go(float(), tw); break;
      case F16: go(__half(), tw); break;
      case BF16: go(__nv_bfloat16(), tw); break;
      default: go(__nv_fp8_e4m3(), tw); break;
    }
  };
  switch (w_fmt) {
    case F64: with_u(double()); break;
    case F32: with_u(float()); break;
    default: ofrr_set_error("residual estimate: W format %d (want F32 or F64)", w_fmt); return OFRR_ERR_UNSUPPORTED;
  }
  OFRR_CHECK_LAUNCH();
  return residual_reduce((double*)ws, nb, r_max, vals, r_dev, res, mode, st);
}

// ---------------------------------------------------------------------------------
// Start block X0 = numpy default_rng(seed).random((n, k)) rounded to the storage format
// (ofrr/driver.py:97-99), generated on the device bit for bit: numpy's PCG64 is a 128-bit
// LCG (state <- state * M + inc) with the XSL-RR output; random() = (next64 >> 11) * 2^-53,
// drawn in C order (element [i, j] is draw i*k + j).  Each thread jumps its private copy of
// the LCG to its first draw (O(log) square-and-multiply, pcg_advance_lcg_128) and walks a
// contiguous run of draws.
// ---------------------------------------------------------------------------------
typedef unsigned __int128 u128;

__device__ __forceinline__ u128 lcg_advance(u128 state, u128 delta, u128 mult, u128 plus) {
  u128 acc_mult = 1, acc_plus = 0;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= mult;
      acc_plus = acc_plus * mult + plus;
    }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__global__ void k_pcg64_block(unsigned long long s_hi, unsigned long long s_lo, unsigned long long i_hi,
                              unsigned long long i_lo, int64_t n, int k, void* __restrict__ X, int64_t ldx, int fmt,
                              int per_thread) {
  const u128 M = ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
  const u128 inc = ((u128)i_hi << 64) | (u128)i_lo;
  const int64_t total = n * (int64_t)k;
  const int64_t d0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * per_thread;
  if (d0 >= total) return;
  u128 s = lcg_advance(((u128)s_hi << 64) | (u128)s_lo, (u128)d0, M, inc);
  const int64_t d1 = d0 + per_thread < total ? d0 + per_thread : total;
  for (int64_t d = d0; d < d1; ++d) {
    s = s * M + inc;
    const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
    const unsigned rot = (unsigned)(s >> 122);
    const unsigned long long x = hi ^ lo;
    const unsigned long long out = (x >> rot) | (x << ((64u - rot) & 63u));
    const double v = (double)(out >> 11) * (1.0 / 9007199254740992.0);
    const int64_t i = d / k, j = d - i * k;
    st_fmt(X, (int64_t)j * ldx + i, fmt, rnd(v, fmt));
  }
}

int start_block_pcg64(unsigned long long s_hi, unsigned long long s_lo, unsigned long long i_hi,
                      unsigned long long i_lo, int64_t n, int k, void* X, int64_t ldx, int fmt, cudaStream_t st) {
  const int64_t total = n * (int64_t)k;
  if (total <= 0) return OFRR_OK;
  const int per = 64;
  const int64_t threads = (total + per - 1) / per;
  k_pcg64_block<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(s_hi, s_lo, i_hi, i_lo, n, k, X, ldx, fmt, per);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

// ---------------------------------------------------------------------------------
// K8: A[i, j] = base(i, j) + sum_s (Wf[i,s] Mf[j,s] + Mf[i,s] Wf[j,s]), FP64 in a fixed
// order (no FMA contraction), rounded once to a_fmt.  base = s_i s_j c[i ^ j] (Walsh-
// Hadamard diagonalised) or diag(c).  Rows [row0, row0 + rows) written row-major.
// ---------------------------------------------------------------------------------
__global__ void k_generate_sym(int64_t n, int64_t row0, int64_t rows, int hadamard, const double* __restrict__ c,
                               const double* __restrict__ sgn, const double* __restrict__ Wf,
                               const double* __restrict__ Mf, int r, void* __restrict__ A, int64_t lda, int a_fmt) {
  const int64_t i = row0 + blockIdx.y;
  if (blockIdx.y >= rows) return;
  extern __shared__ double wi[];   // [2 r]: Wf[i, :], Mf[i, :]
  for (int s = threadIdx.x; s < r; s += blockDim.x) { wi[s] = Wf[(int64_t)s * n + i]; wi[r + s] = Mf[(int64_t)s * n + i]; }
  __syncthreads();
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double acc;
    if (hadamard) acc = __dmul_rn(__dmul_rn(sgn[i], sgn[j]), c[i ^ j]);
    else acc = (i == j) ? c[i] : 0.0;
    for (int s = 0; s < r; ++s) {
      acc = __dadd_rn(acc, __dmul_rn(wi[s], Mf[(int64_t)s * n + j]));
      acc = __dadd_rn(acc, __dmul_rn(wi[r + s], Wf[(int64_t)s * n + j]));
    }
    st_fmt(A, (int64_t)blockIdx.y * lda + j, a_fmt, rnd(acc, a_fmt));
  }
}

int generate_sym(int64_t n, int64_t row0, int64_t rows, int hadamard, const double* c, const double* s,
                 const double* Wf, const double* Mf, int r, void* A, int64_t lda, int a_fmt, cudaStream_t st) {
  if (rows <= 0) return OFRR_OK;
  for (int64_t done = 0; done < rows; done += 65535) {
    const int64_t chunk = std::min<int64_t>(65535, rows - done);
    const int64_t bytes_off = done * lda * fmt_bytes(a_fmt);
    dim3 grid((unsigned)std::min<int64_t>((n + 255) / 256, 8), (unsigned)chunk);
    k_generate_sym<<<grid, 256, 2 * r * sizeof(double), st>>>(n, row0 + done, chunk, hadamard, c, s, Wf, Mf, r,
                                                             (uint8_t*)A + bytes_off, lda, a_fmt);
    OFRR_CHECK_LAUNCH();
  }
  return OFRR_OK;
}

}  // namespace ofrr
