// ritz.cu -- K6 (Ritz-vector recovery) and K8 (synthetic symmetric generator).
#include "common.cuh"
#include <algorithm>

namespace ofrr {

// ---------------------------------------------------------------------------------
// K6: Ut = scale * U[:, :kp] * Y[:kp, :r]  in fp64, fused with the storage rounding of
// the restart block.  Replaces ofrr/projection.py:86 / :129-130 and ofrr/driver.py:109.
// Block = 64 rows x 64 columns, 256 threads (4 x 4 outputs each), kp in slabs of 16.
// ---------------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
    k_ritz(const T* __restrict__ U, int64_t ldu, int64_t n, int kp, const double* __restrict__ Y, int ldy,
           const int* __restrict__ r_dev, int r_max, double scale, double* __restrict__ Ut64, int64_t ldo64,
           void* __restrict__ Xout, int64_t ldx, int x_fmt, int* __restrict__ flags) {
  __shared__ double Us[16][65];
  __shared__ double Ys[16][65];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = (int64_t)blockIdx.x * 64;
  const int n0 = blockIdx.y * 64;
  const int r = r_dev ? min(r_max, *r_dev) : r_max;
  double acc[4][4] = {};
  for (int l0 = 0; l0 < kp; l0 += 16) {
    for (int e = tid; e < 16 * 64; e += 256) {
      const int rr = e & 63, ll = e >> 6;
      const int64_t gi = m0 + rr;
      Us[ll][rr] = (gi < n && l0 + ll < kp) ? to_d(U[(int64_t)(l0 + ll) * ldu + gi]) : 0.0;
      const int cc = e & 63;
      const int gj = n0 + cc;
      Ys[ll][cc] = (gj < r && l0 + ll < kp) ? Y[(int64_t)gj * ldy + l0 + ll] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ll = 0; ll < 16; ++ll) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = Us[ll][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Ys[ll][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  int bad = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gi = m0 + ty + 16 * i;
      const int gj = n0 + tx + 16 * j;
      if (gi >= n || gj >= r_max) continue;
      const double v = gj < r ? scale * acc[i][j] : 0.0;
      if (Ut64) Ut64[(int64_t)gj * ldo64 + gi] = v;
      if (Xout) {
        const double xv = rnd(v, x_fmt);
        if (!isfinite(xv)) bad = 1;
        st_fmt(Xout, (int64_t)gj * ldx + gi, x_fmt, xv);
      }
    }
  if (bad && flags) atomicOr(flags, OFRR_FLAG_NONFINITE);
}

int ritz_recover(const void* U, int64_t ldu, int u_fmt, int64_t n, int kp, const double* Y, int ldy, const int* r_dev,
                 int r_max, double scale, double* Ut64, int64_t ldo64, void* Xout, int64_t ldx, int x_fmt, int* flags,
                 cudaStream_t st) {
  if (n <= 0 || r_max <= 0) return OFRR_OK;
  dim3 grid((unsigned)((n + 63) / 64), (unsigned)((r_max + 63) / 64));
  switch (u_fmt) {
    case F64: k_ritz<double><<<grid, 256, 0, st>>>((const double*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags); break;
    case F32: k_ritz<float><<<grid, 256, 0, st>>>((const float*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags); break;
    case F16: k_ritz<__half><<<grid, 256, 0, st>>>((const __half*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags); break;
    case BF16: k_ritz<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)U, ldu, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags); break;
    default: ofrr_set_error("ritz: basis format %d unsupported", u_fmt); return OFRR_ERR_UNSUPPORTED;
  }
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
