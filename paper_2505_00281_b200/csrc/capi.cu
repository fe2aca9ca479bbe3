// capi.cu -- the extern "C" boundary of libofrr_b200.so (see include/ofrr_b200.h).
#include "common.cuh"
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>

namespace ofrr {
// implemented in the kernel translation units
size_t tc_workspace(int64_t rows, int64_t cols, int k, int a_fmt);
int tc_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* X, int64_t ldx, int k,
               void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* ws, size_t ws_bytes, cudaStream_t st,
               void* W2, int64_t ldw2, int out_fmt2, int nsplit);
size_t split_workspace(int64_t rows, int64_t cols, int k);
int tc_gemm_av_split(const void* A, int64_t rows, int64_t cols, int64_t lda, const float* X, int64_t ldx, int k,
                     void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* ws, size_t ws_bytes,
                     cudaStream_t st, void* W2, int64_t ldw2, int out_fmt2, int slices);
int simt_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose, const void* X,
                 int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, cudaStream_t st,
                 void* W2, int64_t ldw2, int out_fmt2);
size_t resid_est_ws(int64_t n, int r);
int resid_est(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n, int kp,
              const double* Y, int ldy, const double* vals, const int* r_dev, int r_max, double* res, int mode,
              void* ws, size_t ws_bytes, cudaStream_t st);
size_t residual_ws(int64_t rows, int r);
size_t residual_ws2(int64_t rows, int64_t cols, int r, int a_fmt, int transpose);
size_t ozx_op_ws(int64_t rows, int64_t cols);
size_t ozx_prod_ws(int64_t rows, int64_t cols, int r);
int ozx_info(const void* op_ws, int64_t rows, int* full, long long* tails);
int gaussian_kernel(const double* px, int64_t n, const double* py, int64_t m, double f, double l, double s,
                    void* out, int64_t ld, int fmt, cudaStream_t st);
size_t gram_schmidt_ws(int64_t n, int k);
int gram_schmidt(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, int accumulate,
                 double drop_tol, int method, int reorth, void* Q, int64_t ldq, int* kept, int* n_kept, void* ws,
                 size_t ws_bytes, cudaStream_t st);
int ozx_prepare(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, void* op_ws, size_t op_bytes,
                cudaStream_t st);
int ozx_apply(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* op_ws, const double* V,
              int64_t ldv, int r, const double* vals, const int* r_dev, const double* Y, int64_t ldy, void* W,
              int64_t ldw, int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
              double** part_out, void* ws, size_t ws_bytes, cudaStream_t st, int levels);
int oz_nblocks(int64_t rows);
int residual_reduce(const double* part, int nblocks, int n, const double* vals, const int* r_dev, double* res,
                    int mode, cudaStream_t st);
int simt_residual(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose, const double* Xv,
                  int64_t ldx, const double* Yv, int64_t ldy, const double* vals, const int* r_dev, int r_max,
                  double* res, int accumulate_max, void* ws, size_t ws_bytes, cudaStream_t st);
int scale_columns(void* X, int64_t n, int k, int64_t ldx, int storage, int compute, const double* colmax, cudaStream_t st);
int convert(const void* src, int sf, int64_t lds, void* dst, int df, int64_t ldd, int64_t n, int64_t k, int* flags,
            cudaStream_t st);
size_t restart_ws(int64_t n, int t);
int restart(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n, int kp,
            const double* Y, int ldy, const int* r_dev, int r_max, void* Xu, int64_t ldxu, int xu_fmt, int* flags_u,
            double* U64, int64_t ld64, void* Xw, int64_t ldxw, int xw_fmt, int* flags_w, double* colmax,
            const double* vals, int t, double* res, int mode, void* ws, size_t ws_bytes, cudaStream_t st);
int upload_sym(const void* host, int64_t ld_host, void* A, int64_t lda, int64_t n, int fmt, int uplo,
               int64_t block_rows, long long* bytes, cudaStream_t st);
int transpose_convert(const void* src, int sf, int64_t lds, void* dst, int df, int64_t ldd, int64_t rows, int64_t cols,
                      int* flags, cudaStream_t st);
size_t hessenberg_ws(int64_t n, int k, int storage);
int hessenberg(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, double tol, void* Q,
               int64_t ldq, int64_t* pivots, int* kept, int* n_kept, void* ws, size_t ws_bytes, cudaStream_t st);
size_t gram_ws(int64_t n, int k, int kw);
int gram(const void* U, int64_t ldu, const void* W, int64_t ldw, int64_t n, int k, int kw, int storage, int out_fmt,
         double* G1, double* G2, int* flags, void* ws, size_t ws_bytes, cudaStream_t st);
size_t small_eig_ws(int k);
int small_eig(int mode, const double* A, const double* M, int k, double raw_tol, int raw_sweeps, double* values,
              double* vectors, int* n_out, int* status, double* off_out, int* sweeps_out, void* ws, size_t ws_bytes,
              cudaStream_t st);
int ritz_recover(const void* U, int64_t ldu, int u_fmt, int64_t n, int kp, const double* Y, int ldy, const int* r_dev,
                 int r_max, double scale, double* Ut64, int64_t ldo64, void* Xout, int64_t ldx, int x_fmt, int* flags,
                 cudaStream_t st, double* colmax = nullptr);
int generate_sym(int64_t n, int64_t row0, int64_t rows, int hadamard, const double* c, const double* s,
                 const double* Wf, const double* Mf, int r, void* A, int64_t lda, int a_fmt, cudaStream_t st);
int start_block_pcg64(unsigned long long s_hi, unsigned long long s_lo, unsigned long long i_hi,
                      unsigned long long i_lo, int64_t n, int k, void* X, int64_t ldx, int fmt, cudaStream_t st);
}  // namespace ofrr

using namespace ofrr;

static thread_local char g_err[1024] = {0};

void ofrr_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }
static inline bool valid_fmt(int f) { return f >= 0 && f <= 4; }
static inline bool tc_fmt(int f) { return f == BF16 || f == F16 || f == FP8; }

extern "C" {

int ofrr_abi_version(void) { return 1; }
const char* ofrr_last_error(void) { return g_err; }

int ofrr_device_sm_count(int device) {
  static int cached[16] = {0};
  int dev = device;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < 16 && cached[dev] > 0) return cached[dev];
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  if (dev >= 0 && dev < 16) cached[dev] = sms;
  return sms;
}

size_t ofrr_gemm_av_workspace(int64_t rows, int64_t cols, int k, int a_fmt, int transpose) {
  if (tc_fmt(a_fmt) && !transpose && k <= 256) return tc_workspace(rows, cols, k, a_fmt);
  return 256;
}

int ofrr_gemm_av2(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose, const void* X,
                  int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* W2,
                  int64_t ldw2, int out_fmt2, void* workspace, size_t workspace_bytes, void* stream) {
  if (!valid_fmt(a_fmt) || !valid_fmt(out_fmt) || !valid_fmt(out_fmt2) || k < 0 || rows < 0 || cols < 0) {
    ofrr_set_error("gemm_av: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  if (rows == 0 || cols == 0 || k == 0) {
    // empty inner dimension -> zeros (ofrr/_kernels.pyx:70-74)
    const int64_t m = transpose ? cols : rows;
    if (m > 0 && k > 0 && cols * rows == 0) {
      OFRR_CUDA_TRY(cudaMemset2DAsync(W, ldw * fmt_bytes(out_fmt), 0, m * fmt_bytes(out_fmt), k, S(stream)));
      if (W2) OFRR_CUDA_TRY(cudaMemset2DAsync(W2, ldw2 * fmt_bytes(out_fmt2), 0, m * fmt_bytes(out_fmt2), k, S(stream)));
    }
    return OFRR_OK;
  }
  if (tc_fmt(a_fmt) && !transpose) {
    if (k > 256) { ofrr_set_error("gemm_av: k=%d > 256 on the tensor-core path", k); return OFRR_ERR_UNSUPPORTED; }
    if ((lda * fmt_bytes(a_fmt)) % 16 || (ldx * fmt_bytes(a_fmt)) % 16) {
      ofrr_set_error("gemm_av: leading dimensions must be multiples of 16 bytes for TMA");
      return OFRR_ERR_INVALID;
    }
    return tc_gemm_av(A, rows, cols, lda, a_fmt, X, ldx, k, W, ldw, out_fmt, colmax, flags, workspace,
                      workspace_bytes, S(stream), W2, ldw2, out_fmt2, 1);
  }
  return simt_gemm_av(A, rows, cols, lda, a_fmt, transpose, X, ldx, k, W, ldw, out_fmt, colmax, flags, S(stream),
                      W2, ldw2, out_fmt2);
}

size_t ofrr_gemm_av_split_workspace(int64_t rows, int64_t cols, int k) { return split_workspace(rows, cols, k); }

static int gemm_av_split_impl(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const float* X, int64_t ldx,
                       int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2,
                       int out_fmt2, void* workspace, size_t workspace_bytes, void* stream, int slices) {
  if (a_fmt != BF16) { ofrr_set_error("gemm_av_split: A must be bf16"); return OFRR_ERR_UNSUPPORTED; }
  if (rows <= 0 || cols <= 0 || k <= 0) return OFRR_OK;
  if ((lda * 2) % 16) { ofrr_set_error("gemm_av_split: lda must be a multiple of 8"); return OFRR_ERR_INVALID; }
  return tc_gemm_av_split(A, rows, cols, lda, X, ldx, k, W, ldw, out_fmt, colmax, flags, workspace, workspace_bytes,
                          S(stream), W2, ldw2, out_fmt2, slices);
}

int ofrr_gemm_av_split(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const float* X, int64_t ldx,
                       int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2,
                       int out_fmt2, void* workspace, size_t workspace_bytes, void* stream) {
  return gemm_av_split_impl(A, rows, cols, lda, a_fmt, X, ldx, k, W, ldw, out_fmt, colmax, flags, W2, ldw2, out_fmt2,
                            workspace, workspace_bytes, stream, 3);
}
int ofrr_gemm_av_split_slices(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const float* X,
                              int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags,
                              void* W2, int64_t ldw2, int out_fmt2, int slices, void* workspace,
                              size_t workspace_bytes, void* stream) {
  return gemm_av_split_impl(A, rows, cols, lda, a_fmt, X, ldx, k, W, ldw, out_fmt, colmax, flags, W2, ldw2, out_fmt2,
                            workspace, workspace_bytes, stream, slices);
}

int ofrr_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose, const void* X,
                 int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax, int* flags, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return ofrr_gemm_av2(A, rows, cols, lda, a_fmt, transpose, X, ldx, k, W, ldw, out_fmt, colmax, flags, nullptr, 0,
                       out_fmt, workspace, workspace_bytes, stream);
}

int ofrr_scale_columns(void* X, int64_t n, int k, int64_t ldx, int storage, int compute, const double* colmax,
                       void* stream) {
  return scale_columns(X, n, k, ldx, storage, compute, colmax, S(stream));
}

size_t ofrr_hessenberg_workspace(int64_t n, int k, int storage) { return hessenberg_ws(n, k, storage); }

int ofrr_hessenberg(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, double tol, void* Q,
                    int64_t ldq, int64_t* pivots, int* kept, int* n_kept, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (k <= 0 || n <= 0) { ofrr_set_error("hessenberg: no input columns"); return OFRR_ERR_EMPTY_BASIS; }
  return hessenberg(X, n, k, ldx, storage, compute, tol, Q, ldq, pivots, kept, n_kept, workspace, workspace_bytes,
                    S(stream));
}

size_t ofrr_gram_workspace(int64_t n, int k, int kw) { return gram_ws(n, k, kw); }

int ofrr_gram(const void* U, int64_t ldu, const void* W, int64_t ldw, int64_t n, int k, int kw, int storage,
              int out_fmt, double* G1, double* G2, int* flags, void* workspace, size_t workspace_bytes, void* stream) {
  return gram(U, ldu, W, ldw, n, k, kw, storage, out_fmt, G1, G2, flags, workspace, workspace_bytes, S(stream));
}

size_t ofrr_small_eig_workspace(int k) { return small_eig_ws(k); }

int ofrr_sym_def_gen_eig(const double* B, const double* M, int k, double* values, double* vectors, int* n_out,
                         int* status, void* workspace, size_t workspace_bytes, void* stream) {
  return small_eig(2, B, M, k, 0.0, 0, values, vectors, n_out, status, nullptr, nullptr, workspace, workspace_bytes,
                   S(stream));
}

int ofrr_sym_eig(const double* Sm, int k, double* values, double* vectors, int* status, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return small_eig(0, Sm, nullptr, k, 0.0, 0, values, vectors, nullptr, status, nullptr, nullptr, workspace,
                   workspace_bytes, S(stream));
}

int ofrr_ritz_recover(const void* U, int64_t ldu, int u_fmt, int64_t n, int kp, const double* Y, int ldy,
                      const int* r_dev, int r_max, double scale, double* Ut64, int64_t ldo64, void* Xout, int64_t ldx,
                      int x_fmt, int* flags, void* stream) {
  return ritz_recover(U, ldu, u_fmt, n, kp, Y, ldy, r_dev, r_max, scale, Ut64, ldo64, Xout, ldx, x_fmt, flags,
                      S(stream));
}

int ofrr_reuse_power(const void* W, int64_t ldw, int w_fmt, int64_t n, int kp, const double* Y, int ldy,
                     const int* r_dev, int r_max, void* Xout, int64_t ldx, int x_fmt, double* colmax, int* flags,
                     void* stream) {
  if (!Xout || !colmax || !valid_fmt(x_fmt)) { ofrr_set_error("reuse_power: invalid arguments"); return OFRR_ERR_INVALID; }
  return ritz_recover(W, ldw, w_fmt, n, kp, Y, ldy, r_dev, r_max, 1.0, nullptr, 0, Xout, ldx, x_fmt, flags, S(stream),
                      colmax);
}

size_t ofrr_restart_workspace(int64_t n, int t) { return restart_ws(n, t); }
int ofrr_restart(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n, int kp,
                 const double* Y, int ldy, const int* r_dev, int r_max, void* Xu, int64_t ldxu, int xu_fmt,
                 int* flags_u, double* U64, int64_t ld64, void* Xw, int64_t ldxw, int xw_fmt, int* flags_w,
                 double* colmax, const double* vals, int t, double* res, int mode, void* workspace,
                 size_t workspace_bytes, void* stream) {
  if (!valid_fmt(u_fmt) || (W && !valid_fmt(w_fmt)) || (Xu && !valid_fmt(xu_fmt)) || (Xw && !valid_fmt(xw_fmt)) ||
      n < 0 || kp < 0 || r_max < 0 || t < 0) {
    ofrr_set_error("restart: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  return restart(U, ldu, u_fmt, W, ldw, w_fmt, n, kp, Y, ldy, r_dev, r_max, Xu, ldxu, xu_fmt, flags_u, U64, ld64, Xw,
                 ldxw, xw_fmt, flags_w, colmax, vals, t, res, mode, workspace, workspace_bytes, S(stream));
}

size_t ofrr_residual_workspace(int64_t rows, int r) { return residual_ws(rows, r); }
size_t ofrr_residual_workspace2(int64_t rows, int64_t cols, int r, int a_fmt, int transpose) {
  return residual_ws2(rows, cols, r, a_fmt, transpose);
}

size_t ofrr_ozaki_operator_workspace(int64_t rows, int64_t cols) { return ozx_op_ws(rows, cols); }
size_t ofrr_ozaki_workspace(int64_t rows, int64_t cols, int r) { return ozx_prod_ws(rows, cols, r); }
size_t ofrr_orthonormalize_workspace(int64_t n, int k) { return gram_schmidt_ws(n, k); }
int ofrr_orthonormalize(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, int accumulate,
                        double drop_tol, int method, int reorth, void* Q, int64_t ldq, int* kept, int* n_kept,
                        void* workspace, size_t workspace_bytes, void* stream) {
  if (!valid_fmt(storage) || !valid_fmt(compute) || !valid_fmt(accumulate)) {
    ofrr_set_error("orthonormalize: invalid format");
    return OFRR_ERR_INVALID;
  }
  return gram_schmidt(X, n, k, ldx, storage, compute, accumulate, drop_tol, method, reorth, Q, ldq, kept, n_kept,
                      workspace, workspace_bytes, S(stream));
}
int ofrr_gaussian_kernel(const double* px, int64_t n, const double* py, int64_t m, double f, double l, double s,
                         void* out, int64_t ld, int out_fmt, void* stream) {
  if (!valid_fmt(out_fmt)) { ofrr_set_error("gaussian_kernel: invalid format"); return OFRR_ERR_INVALID; }
  return gaussian_kernel(px, n, py, m, f, l, s, out, ld, out_fmt, S(stream));
}
int ofrr_ozaki_operator_info(const void* op_ws, int64_t rows, int* full, long long* tails) {
  return ozx_info(op_ws, rows, full, tails);
}

int ofrr_ozaki_prepare(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, void* op_ws,
                       size_t op_bytes, void* stream) {
  if (rows <= 0 || cols <= 0) { ofrr_set_error("ozaki_prepare: empty operator"); return OFRR_ERR_INVALID; }
  return ozx_prepare(A, rows, cols, lda, a_fmt, op_ws, op_bytes, S(stream));
}

int ofrr_ozaki_gemm(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* op_ws,
                    const double* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax,
                    int* flags, void* W2, int64_t ldw2, int out_fmt2, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (!valid_fmt(out_fmt) || !valid_fmt(out_fmt2) || k <= 0 || !W) { ofrr_set_error("ozaki_gemm: invalid arguments"); return OFRR_ERR_INVALID; }
  return ozx_apply(A, rows, cols, lda, a_fmt, op_ws, X, ldx, k, nullptr, nullptr, nullptr, 0, W, ldw, out_fmt, colmax,
                   flags, W2, ldw2, out_fmt2, nullptr, workspace, workspace_bytes, S(stream), 6);
}

int ofrr_ozaki_gemm_levels(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* op_ws,
                           const double* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt, double* colmax,
                           int* flags, void* W2, int64_t ldw2, int out_fmt2, int levels, void* workspace,
                           size_t workspace_bytes, void* stream) {
  if (!valid_fmt(out_fmt) || !valid_fmt(out_fmt2) || k <= 0 || !W) { ofrr_set_error("ozaki_gemm: invalid arguments"); return OFRR_ERR_INVALID; }
  return ozx_apply(A, rows, cols, lda, a_fmt, op_ws, X, ldx, k, nullptr, nullptr, nullptr, 0, W, ldw, out_fmt, colmax,
                   flags, W2, ldw2, out_fmt2, nullptr, workspace, workspace_bytes, S(stream), levels);
}

int ofrr_ozaki_residual(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, const void* op_ws,
                        const double* Xv, int64_t ldx, const double* Yv, int64_t ldy, const double* vals,
                        const int* r_dev, int r_max, double* res, int accumulate_max, void* workspace,
                        size_t workspace_bytes, void* stream) {
  double* part = nullptr;
  int rc = ozx_apply(A, rows, cols, lda, a_fmt, op_ws, Xv, ldx, r_max, vals, r_dev, Yv, ldy, nullptr, 0, F64, nullptr,
                     nullptr, nullptr, 0, F64, &part, workspace, workspace_bytes, S(stream), 6);
  if (rc) return rc;
  return residual_reduce(part, oz_nblocks(rows), r_max, vals, r_dev, res, accumulate_max, S(stream));
}

size_t ofrr_residual_estimate_workspace(int64_t n, int r) { return resid_est_ws(n, r); }

int ofrr_residual_estimate(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n,
                           int kp, const double* Y, int ldy, const double* vals, const int* r_dev, int r_max,
                           double* res, int mode, void* workspace, size_t workspace_bytes, void* stream) {
  return resid_est(U, ldu, u_fmt, W, ldw, w_fmt, n, kp, Y, ldy, vals, r_dev, r_max, res, mode, workspace,
                   workspace_bytes, S(stream));
}

int ofrr_residual_eig(const void* A, int64_t n, int64_t lda, int a_fmt, const double* V, int64_t ldv,
                      const double* vals, const int* r_dev, int r_max, double* res, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return simt_residual(A, n, n, lda, a_fmt, 0, V, ldv, V, ldv, vals, r_dev, r_max, res, 0, workspace,
                       workspace_bytes, S(stream));
}

int ofrr_residual_pair(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose,
                       const double* Xv, int64_t ldx, const double* Yv, int64_t ldy, const double* vals,
                       const int* r_dev, int r_max, double* res, int accumulate_max, void* workspace,
                       size_t workspace_bytes, void* stream) {
  return simt_residual(A, rows, cols, lda, a_fmt, transpose, Xv, ldx, Yv, ldy, vals, r_dev, r_max, res,
                       accumulate_max, workspace, workspace_bytes, S(stream));
}

int ofrr_generate_sym(int64_t n, int64_t row0, int64_t rows, int hadamard, const double* c, const double* s,
                      const double* Wf, const double* Mf, int r, void* A, int64_t lda, int a_fmt, void* stream) {
  return generate_sym(n, row0, rows, hadamard, c, s, Wf, Mf, r, A, lda, a_fmt, S(stream));
}

int ofrr_start_block_pcg64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t n, int k,
                           void* X, int64_t ldx, int fmt, void* stream) {
  if (!valid_fmt(fmt) || n < 0 || k < 0) { ofrr_set_error("start_block: invalid arguments"); return OFRR_ERR_INVALID; }
  return start_block_pcg64(state_hi, state_lo, inc_hi, inc_lo, n, k, X, ldx, fmt, S(stream));
}

int ofrr_convert(const void* src, int src_fmt, int64_t ld_src, void* dst, int dst_fmt, int64_t ld_dst, int64_t n,
                 int64_t k, int* flags, void* stream) {
  return convert(src, src_fmt, ld_src, dst, dst_fmt, ld_dst, n, k, flags, S(stream));
}

int ofrr_transpose_convert(const void* src, int src_fmt, int64_t ld_src, void* dst, int dst_fmt, int64_t ld_dst,
                           int64_t rows, int64_t cols, int* flags, void* stream) {
  return transpose_convert(src, src_fmt, ld_src, dst, dst_fmt, ld_dst, rows, cols, flags, S(stream));
}

int ofrr_upload_sym(const void* host, int64_t ld_host, void* A, int64_t lda, int64_t n, int fmt, int uplo,
                    int64_t block_rows, long long* bytes, void* stream) {
  return upload_sym(host, ld_host, A, lda, n, fmt, uplo, block_rows, bytes, S(stream));
}

// ---------------------------------------------------------------------------------
// host-buffer plugin entry points (ofrr/_kernels.pyx signatures)
// ---------------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
  cudaError_t alloc(size_t b) { return cudaMalloc(&p, b ? b : 16); }
};

int ofrr_host_gemm_mixed(const double* a, int64_t ars, int64_t acs, const double* b, int64_t brs, int64_t bcs,
                         int64_t m, int64_t k, int64_t n, int compute, int accumulate, int out_fmt, double* c) {
  if (m < 0 || k < 0 || n < 0 || !valid_fmt(compute) || !valid_fmt(accumulate) || !valid_fmt(out_fmt)) {
    ofrr_set_error("gemm_mixed: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  if (m == 0 || n == 0) return OFRR_OK;
  if (k == 0) { memset(c, 0, sizeof(double) * m * n); return OFRR_OK; }
  // device format of the operands: 16-bit/8-bit compute -> tensor cores, else fp32/fp64 FMA
  const int dfmt = (compute == F64 || accumulate == F64) ? F64 : compute == F32 ? F32 : compute;
  const int64_t lda = (k + 63) / 64 * 64, ldx = lda;
  std::vector<double> ha((size_t)m * lda, 0.0), hb((size_t)n * ldx, 0.0);
  for (int64_t i = 0; i < m; ++i)
    for (int64_t l = 0; l < k; ++l) ha[(size_t)i * lda + l] = a[i * ars + l * acs];
  for (int64_t j = 0; j < n; ++j)
    for (int64_t l = 0; l < k; ++l) hb[(size_t)j * ldx + l] = b[l * brs + j * bcs];
  DevBuf d64a, d64b, da, db, dw, d64w, dws;
  const int eb = fmt_bytes(dfmt);
  OFRR_CUDA_TRY(d64a.alloc(ha.size() * 8));
  OFRR_CUDA_TRY(d64b.alloc(hb.size() * 8));
  OFRR_CUDA_TRY(da.alloc(ha.size() * eb));
  OFRR_CUDA_TRY(db.alloc(hb.size() * eb));
  OFRR_CUDA_TRY(dw.alloc((size_t)m * n * 8));
  OFRR_CUDA_TRY(d64w.alloc((size_t)m * n * 8));
  cudaStream_t st = 0;
  OFRR_CUDA_TRY(cudaMemcpyAsync(d64a.p, ha.data(), ha.size() * 8, cudaMemcpyHostToDevice, st));
  OFRR_CUDA_TRY(cudaMemcpyAsync(d64b.p, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, st));
  int rc = convert(d64a.p, F64, lda, da.p, dfmt, lda, lda, m, nullptr, st);
  if (!rc) rc = convert(d64b.p, F64, ldx, db.p, dfmt, ldx, ldx, n, nullptr, st);
  if (rc) return rc;
  const size_t wsb = ofrr_gemm_av_workspace(m, k, (int)n, dfmt, 0);
  OFRR_CUDA_TRY(dws.alloc(wsb));
  if (tc_fmt(dfmt) && n > 256) {
    // wide right-hand sides: column panels of 256
    for (int64_t j0 = 0; j0 < n; j0 += 256) {
      const int nj = (int)std::min<int64_t>(256, n - j0);
      rc = ofrr_gemm_av(da.p, m, k, lda, dfmt, 0, (uint8_t*)db.p + (size_t)j0 * ldx * eb, ldx, nj,
                        (uint8_t*)dw.p + (size_t)j0 * m * 8, m, F64, nullptr, nullptr, dws.p, wsb, st);
      if (rc) return rc;
    }
  } else {
    rc = ofrr_gemm_av(da.p, m, k, lda, dfmt, 0, db.p, ldx, (int)n, dw.p, m, F64, nullptr, nullptr, dws.p, wsb, st);
    if (rc) return rc;
  }
  rc = convert(dw.p, F64, m, d64w.p, out_fmt, m, m, n, nullptr, st);
  if (rc) return rc;
  // round to out_fmt then widen back to fp64 for the host (F-order m x n)
  rc = convert(d64w.p, out_fmt, m, dw.p, F64, m, m, n, nullptr, st);
  if (rc) return rc;
  OFRR_CUDA_TRY(cudaMemcpyAsync(c, dw.p, (size_t)m * n * 8, cudaMemcpyDeviceToHost, st));
  OFRR_CUDA_TRY(cudaStreamSynchronize(st));
  return OFRR_OK;
}

int ofrr_host_jacobi_eig(const double* a, int64_t n, int max_sweeps, double tol, double* vals, double* vecs,
                         int* sweeps, double* off) {
  if (n < 0 || n > 512) { ofrr_set_error("jacobi_eig: n=%lld outside [0, 512]", (long long)n); return OFRR_ERR_INVALID; }
  if (n == 0) { if (sweeps) *sweeps = 0; if (off) *off = 0.0; return OFRR_OK; }
  std::vector<double> cm((size_t)n * n);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) cm[(size_t)j * n + i] = a[i * n + j];
  DevBuf dA, dvals, dvecs, dint, doff, dws;
  const size_t wsb = small_eig_ws((int)n);
  OFRR_CUDA_TRY(dA.alloc(cm.size() * 8));
  OFRR_CUDA_TRY(dvals.alloc(n * 8));
  OFRR_CUDA_TRY(dvecs.alloc(cm.size() * 8));
  OFRR_CUDA_TRY(dint.alloc(16));
  OFRR_CUDA_TRY(doff.alloc(8));
  OFRR_CUDA_TRY(dws.alloc(wsb));
  cudaStream_t st = 0;
  OFRR_CUDA_TRY(cudaMemcpyAsync(dA.p, cm.data(), cm.size() * 8, cudaMemcpyHostToDevice, st));
  int rc = small_eig(1, (double*)dA.p, nullptr, (int)n, tol, max_sweeps, (double*)dvals.p, (double*)dvecs.p, nullptr,
                     (int*)dint.p, (double*)doff.p, (int*)dint.p + 1, dws.p, wsb, st);
  if (rc) return rc;
  std::vector<double> hv((size_t)n * n);
  int hi[2];
  OFRR_CUDA_TRY(cudaMemcpyAsync(vals, dvals.p, n * 8, cudaMemcpyDeviceToHost, st));
  OFRR_CUDA_TRY(cudaMemcpyAsync(hv.data(), dvecs.p, hv.size() * 8, cudaMemcpyDeviceToHost, st));
  OFRR_CUDA_TRY(cudaMemcpyAsync(hi, dint.p, 8, cudaMemcpyDeviceToHost, st));
  double ho = 0.0;
  OFRR_CUDA_TRY(cudaMemcpyAsync(&ho, doff.p, 8, cudaMemcpyDeviceToHost, st));
  OFRR_CUDA_TRY(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = 0; p < n; ++p) vecs[i * n + p] = hv[(size_t)p * n + i];
  if (sweeps) *sweeps = hi[1];
  if (off) *off = ho;
  return OFRR_OK;
}

}  // extern "C"

namespace ofrr { int k5_profile(long long* out); }
extern "C" int ofrr_debug_k5_profile(long long* out8) { return ofrr::k5_profile(out8); }
namespace ofrr { int hess_profile(unsigned long long* out); int pc_profile(unsigned long long* out); }
extern "C" int ofrr_debug_pencil_profile(unsigned long long* out16) { return ofrr::pc_profile(out16); }
extern "C" int ofrr_debug_hess_profile(unsigned long long* out8) { return ofrr::hess_profile(out8); }
namespace ofrr { int hess_mode(int force_global, int pb); }
extern "C" int ofrr_debug_hess_mode(int force_global, int pb) { return ofrr::hess_mode(force_global, pb); }

namespace ofrr {
void prof_enable(int on); int prof_read(float* ms, int max); int prof_active(); int prof_collect();
int prof_claim(); int prof_collect_group(int g);
}
extern "C" void ofrr_prof_gemm_enable(int on) { ofrr::prof_enable(on); }
extern "C" int ofrr_prof_gemm_read(float* ms, int max) { return ofrr::prof_read(ms, max); }
extern "C" int ofrr_prof_gemm_active(void) { return ofrr::prof_active(); }
extern "C" int ofrr_prof_gemm_collect(void) { return ofrr::prof_collect(); }
extern "C" int ofrr_prof_gemm_claim(void) { return ofrr::prof_claim(); }
extern "C" int ofrr_prof_gemm_collect_group(int group) { return ofrr::prof_collect_group(group); }
namespace ofrr { int stamp_enable(int on); int stamp_read(double* sum_ms, long long* count); }
extern "C" int ofrr_prof_k1_stamp(int on) { return ofrr::stamp_enable(on); }
extern "C" int ofrr_prof_k1_read(double* sum_ms, long long* count) { return ofrr::stamp_read(sum_ms, count); }
namespace ofrr { int oz_stamp_enable(int on); int oz_stamp_read(double* sum_ms, long long* count, int tier); }
extern "C" int ofrr_prof_oz_stamp(int on) { return ofrr::oz_stamp_enable(on); }
extern "C" int ofrr_prof_oz_read(double* sum_ms, long long* count) { return ofrr::oz_stamp_read(sum_ms, count, 0); }
extern "C" int ofrr_prof_oz_read_tier(int tier, double* sum_ms, long long* count) {
  return ofrr::oz_stamp_read(sum_ms, count, tier);
}
