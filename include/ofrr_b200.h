/*
 * ofrr_b200.h -- C ABI of libofrr_b200.so, the B200 (sm_100a) OFRR hot path.
 *
 * Drop-in boundary for the reference's kernel plugin slot (`ofrr.backend.kernels`,
 * /root/reference/pkg/src/ofrr/backend.py:14-22) and for the device-resident driver
 * steps of ofrr/driver.py:84-173.  Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *  - Format codes follow ofrr/precision.py:20-25 (F16=0, F32=1, F64=2) and extend them
 *    with BF16=3, FP8_E4M3=4.
 *  - "Device" entry points take device pointers and an explicit cudaStream_t (passed as
 *    void*; NULL = legacy default stream).  They enqueue work and return immediately.
 *  - Matrices: A is row-major (rows x cols, leading dimension lda in elements); blocks
 *    X/W/U/Q are column-major (n x k, leading dimension ld >= n), i.e. the reference's
 *    Fortran order (ofrr/matrix.py:25-31).
 *  - Every call returns an ofrr status (0 = OK).  Errors map 1:1 onto the reference's
 *    exceptions (see OFRR_ERR_*); ofrr_last_error() gives the message.
 *  - The library never frees caller memory.  Workspaces are caller-owned; the
 *    *_workspace() queries give their sizes in bytes.
 *  - Thread safety: entry points are re-entrant; concurrent calls must use distinct
 *    workspaces (the reference's CLI calls drivers from a thread pool,
 *    ofrr/cli.py:399-401).
 */
#ifndef OFRR_B200_H
#define OFRR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* formats: ofrr/precision.py:20-25 (+ extensions) */
#define OFRR_F16 0
#define OFRR_F32 1
#define OFRR_F64 2
#define OFRR_BF16 3
#define OFRR_FP8E4M3 4

/* status codes */
#define OFRR_OK 0
#define OFRR_ERR_INVALID 1      /* ValueError (argument validation) */
#define OFRR_ERR_CUDA 2         /* CUDA runtime failure */
#define OFRR_ERR_OVERFLOW 3     /* OverflowDiagnostic: ofrr/projection.py:24-25, driver.py:73-75 */
#define OFRR_ERR_EMPTY_BASIS 4  /* EmptyBasisError: ofrr/basis.py:41-42 */
#define OFRR_ERR_EMPTY_PENCIL 5 /* EmptyPencilError: ofrr/projection.py:28-29 */
#define OFRR_ERR_CONVERGENCE 6  /* ConvergenceError: ofrr/smallsolve.py:20-25 */
#define OFRR_ERR_UNSUPPORTED 7  /* format / shape combination this build does not run */

/* device-side flag bits written by kernels (int32, OR-ed) */
#define OFRR_FLAG_NONFINITE 1
#define OFRR_FLAG_NOCONV 2
#define OFRR_FLAG_INEXACT 4 /* ofrr_transpose_convert: some value was not representable */

int ofrr_abi_version(void);
const char* ofrr_last_error(void);
int ofrr_device_sm_count(int device);

/* ---------------------------------------------------------------------------------
 * K1: block product W = A * X  (or A^T * X when transpose != 0)
 * Replaces ofrr/matrix.py:242-254 apply_dense -> ofrr/precision.py:122-135 mixed_gemm
 *          -> ofrr/_kernels.pyx:60-84 gemm_mixed.
 * A: rows x cols row-major, format a_fmt (BF16/F16: tcgen05 tensor cores, fp32 TMEM
 *    accumulation; FP8E4M3: tcgen05 kind::f8f6f4; F32/F64: CUDA-core FMA).
 * X: (transpose ? rows : cols) x k column-major, same format as A.
 * W: (transpose ? cols : rows) x k column-major, rounded to out_fmt.
 * colmax (device double[k], may be NULL): max |W[:,j]| after rounding (for the inf-norm
 *    column scaling, ofrr/precision.py:159-169).  flags (device int, may be NULL):
 *    OR-ed with OFRR_FLAG_NONFINITE when W has non-finite entries
 *    (ofrr/driver.py:73-75).  Deterministic: fixed-order split-K reduction.
 * ------------------------------------------------------------------------------- */
size_t ofrr_gemm_av_workspace(int64_t rows, int64_t cols, int k, int a_fmt, int transpose);
int ofrr_gemm_av(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose,
                 const void* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt,
                 double* colmax, int* flags, void* workspace, size_t workspace_bytes,
                 void* stream);

/* K1 with a second output: W2 = the same product rounded to out_fmt2 (e.g. the fp32
 * accumulator itself, kept for the residual estimate of ofrr_residual_estimate). */
int ofrr_gemm_av2(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, int transpose,
                  const void* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt,
                  double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
                  void* workspace, size_t workspace_bytes, void* stream);

/* K1, fp32 block on the bf16 tensor cores: W = A X with A bf16 and X fp32.  X is split into
 * three bf16 slices [X_hi | X_mid | X_lo] (exact: 3 x 8 bits = the fp32 significand), the
 * n x 3k product runs in ONE pass over A (3k <= 256), and the slices are summed in fp32 in
 * the finalize.  This is the device form of the reference's full-f32 policy
 * (ofrr/precision.py:79) for an operator stored in bf16 -- fp32-accurate products at
 * bf16 HBM traffic. */
size_t ofrr_gemm_av_split_workspace(int64_t rows, int64_t cols, int k);
int ofrr_gemm_av_split(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                       const float* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt,
                       double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
                       void* workspace, size_t workspace_bytes, void* stream);
/* The same with 2 or 3 bf16 slices of the fp32 block: slices = 2 keeps a 16-bit significand
 * (x_hi + x_mid; N = 2k, HBM-bound for k <= 125) -- the products of the full-f32-lite ladder
 * rung; slices = 3 is ofrr_gemm_av_split. */
int ofrr_gemm_av_split_slices(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                              const float* X, int64_t ldx, int k, void* W, int64_t ldw, int out_fmt,
                              double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2, int slices,
                              void* workspace, size_t workspace_bytes, void* stream);

/* Kernel-only timing of the K1 tensor-core kernel (measurement support): while enabled,
 * every k_gemm_av_tc launch is bracketed by CUDA events on its stream; read returns the
 * durations (ms) of the launches since enable.  Launches captured into a CUDA graph:
 * claim (right after the capture) turns the captured event pairs into a group whose
 * durations collect_group appends after each replay; collect harvests eager launches. */
void ofrr_prof_gemm_enable(int on);
int ofrr_prof_gemm_read(float* ms, int max);
int ofrr_prof_gemm_active(void);
int ofrr_prof_gemm_collect(void);
int ofrr_prof_gemm_claim(void);
int ofrr_prof_gemm_collect_group(int group);
/* The same measurement from inside the kernels (usable inside CUDA graphs with device-side
 * loops, which cannot hold event nodes): while enabled (at launch/capture time), each
 * k_gemm_av_tc launch stamps its first CTA entry and last CTA exit (globaltimer) and its
 * k_finalize accumulates the interval; read returns the summed ms and the launch count. */
int ofrr_prof_k1_stamp(int on);
int ofrr_prof_k1_read(double* sum_ms, long long* count);
/* The same in-kernel stamps for k_ozk_gemm (K7z, the FP64-accurate int8 Ozaki product),
 * closed by the k_oz_resid launch that follows each product. */
int ofrr_prof_oz_stamp(int on);
int ofrr_prof_oz_read(double* sum_ms, long long* count);
/* the same split by product tier: 1 = FP64-accurate (6 levels), 2 = lite (4 levels), 3 = 5 levels, 0 = all */
int ofrr_prof_oz_read_tier(int tier, double* sum_ms, long long* count);

/* ---------------------------------------------------------------------------------
 * Device-side outer loop (ofrr/driver.py:101-111 with the tol extension) as one CUDA graph:
 *   init -> first(iteration graph, e.g. with the start block's MatVec) -> decide
 *        -> [copy first_out -> steady_in] -> WHILE(continue) { steady iteration -> decide
 *        -> IF(report) { FP64 report graph -> confirm } }
 * decide reads the iteration's status word (int32[8], driver layout) and the leading
 * `top` residual estimates: non-finite / empty / narrowed basis or a pencil error stop the
 * loop with a state for the host; otherwise it requests the FP64 report when the estimate
 * passes tol, stalls (> 0.5x the previous, < 16 tol) or the iteration is the m-th; confirm
 * stops the loop when the FP64 residuals pass.  ctl (device, ofrr_loop_ctl_bytes) holds the
 * state, iteration count and per-iteration estimate / FP64 histories.  The graphs are
 * cudaGraph_t handles (e.g. torch.cuda.CUDAGraph(keep_graph=True).raw_cuda_graph()); the
 * result is an instantiated cudaGraphExec_t (launch / destroy below).
 * ------------------------------------------------------------------------------- */
#define OFRR_LOOP_RUNNING 0
#define OFRR_LOOP_CONVERGED 1       /* FP64 residuals of the leading `top` pairs < tol */
#define OFRR_LOOP_EXHAUSTED 2       /* m iterations, report made, not converged */
#define OFRR_LOOP_HOST 3            /* a case the host loop handles (status error, narrowed
                                       basis, report requested after the first iteration) */
size_t ofrr_loop_ctl_bytes(void);
int ofrr_loop_build(void* first_graph, void* steady_graph, void* report_graph, const int* st_first,
                    const double* est_first, const int* st_steady, const double* est_steady,
                    const double* res_report, const void* copy_src, void* copy_dst, size_t copy_bytes,
                    void* ctl, int m, int top, int k, double tol, void** exec_out);
/* A precision-ladder rung's loop (driver.py EigEngine.run with stop_estimate): the first and
 * steady iteration graphs, no report; the rung stops when its worst leading estimate falls
 * below `sw` or stops halving -> state OFRR_LOOP_RUNG_DONE, the restart block and the next
 * iterate are the last iteration's outputs. */
#define OFRR_LOOP_RUNG_DONE 4
int ofrr_loop_build_rung(void* first_graph, void* steady_graph, const int* st_first,
                         const double* est_first, const int* st_steady, const double* est_steady,
                         const void* copy_src, void* copy_dst, size_t copy_bytes, void* ctl, int m,
                         int top, int k, double sw, void** exec_out);
int ofrr_loop_launch(void* exec, void* stream);
int ofrr_loop_destroy(void* exec);

/* K2: X[:,j] <- round_s(round_c(X[:,j] / colmax[j])) for colmax[j] != 0, in place.
 * Replaces ofrr/precision.py:159-169 scale_columns_inf. */
int ofrr_scale_columns(void* X, int64_t n, int k, int64_t ldx, int storage, int compute,
                       const double* colmax, void* stream);

/* ---------------------------------------------------------------------------------
 * K3: Hessenberg (LU with partial pivoting) basis of X (n x k, format `storage`).
 * Replaces ofrr/basis.py:151-204 hessenberg_basis (layouts "left"/"right" give the
 * identical update sequence, tests/test_basis.py:92-98).  Arithmetic follows the
 * reference exactly: axpy in the compute format rounded to storage
 * (ofrr/precision.py:172-180), pivot = largest |v| over non-pivot rows, lowest index
 * on ties (ofrr/basis.py:199-204), columns with |pivot| < tol are skipped.
 * Outputs (device): Q (n x k, kept columns compacted to the front, ldq),
 * pivots (int64[k], first n_kept valid), kept (int32[k] 0/1), n_kept (int32 scalar).
 * ------------------------------------------------------------------------------- */
size_t ofrr_hessenberg_workspace(int64_t n, int k, int storage);
int ofrr_hessenberg(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute,
                    double tol, void* Q, int64_t ldq, int64_t* pivots, int* kept, int* n_kept,
                    void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * K4: Grams G1 = U^T W and G2 = U^T U (k x k each, column-major fp64 outputs, values
 * rounded to out_fmt: F32 for F16 storage, F64 otherwise -- ofrr/projection.py:42-53).
 * Replaces ofrr/projection.py:56-61 _project (x2 in ofrr_eig, :79-80).  W may be NULL
 * (only G2 is formed) and G2 may be NULL.  Products are exact (storage formats of
 * <= 24 significant bits multiply exactly in fp64), sums in fp64 with a
 * fixed-order two-stage reduction.  `k` columns of U, `kw` columns of W.
 * ------------------------------------------------------------------------------- */
size_t ofrr_gram_workspace(int64_t n, int k, int kw);
int ofrr_gram(const void* U, int64_t ldu, const void* W, int64_t ldw, int64_t n, int k, int kw,
              int storage, int out_fmt, double* G1, double* G2, int* flags, void* workspace,
              size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * K5: symmetric-definite pencil B y = lambda M y in fp64 (k x k, column-major).
 * Replaces ofrr/smallsolve.py:64-88 sym_def_gen_eig (with sym_eig :34-49 and the
 * Jacobi kernel ofrr/_kernels.pyx:105-150): symmetrize, eig(M), keep
 * mu > k*eps*mu_max, T = D^-1/2 P^T B P D^-1/2, eig(T), y = P D^-1/2 Z, sort
 * descending (stable) with the largest-|entry|-positive sign rule.
 * Outputs: values (fp64[k], first *n_out valid), vectors (k x k col-major, first
 * *n_out columns valid), n_out (device int32), status (device int32:
 * 0 ok, OFRR_ERR_CONVERGENCE, OFRR_ERR_EMPTY_PENCIL when nothing is retained).
 * sym_eig alone: ofrr_sym_eig (same sort/sign rules).
 * ------------------------------------------------------------------------------- */
size_t ofrr_small_eig_workspace(int k);
int ofrr_sym_def_gen_eig(const double* B, const double* M, int k, double* values,
                         double* vectors, int* n_out, int* status, void* workspace,
                         size_t workspace_bytes, void* stream);
int ofrr_sym_eig(const double* S, int k, double* values, double* vectors, int* status,
                 void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * K6: Ritz recovery  Ut = scale * U * Y[:, :r]  (n x k' times k' x r, fp64 math).
 * Replaces ofrr/projection.py:86 (u.data @ eig.vectors) and :129-130 (sqrt(2)*U*Y),
 * fused with ofrr/driver.py:109 round_to(..., mv.storage).
 * r_dev (device int32, may be NULL -> r_max) gives the number of valid columns.
 * Outputs (either may be NULL): Ut64 (n x r_max fp64, ldo64), Xout (n x r_max in
 * x_fmt, ldx; columns >= r are zero-filled), flags |= NONFINITE on Xout.
 * ------------------------------------------------------------------------------- */
int ofrr_ritz_recover(const void* U, int64_t ldu, int u_fmt, int64_t n, int kp, const double* Y,
                      int ldy, const int* r_dev, int r_max, double scale, double* Ut64,
                      int64_t ldo64, void* Xout, int64_t ldx, int x_fmt, int* flags,
                      void* stream);

/* ---------------------------------------------------------------------------------
 * A-pass reuse (IterConfig.reuse_av, an extension): the next power step A X with
 * X = U Y taken from the projection's block product, A X = (A U) Y = W Y.  Replaces the
 * MatVec of ofrr/driver.py:102-104 that follows the restart of :109.
 * Xout = round(W Y[:, :r], x_fmt) (columns >= r zero-filled), colmax[j] = max |Xout[:, j]|
 * (atomic max: zero it first; the input of ofrr_scale_columns), flags |= NONFINITE.
 * ------------------------------------------------------------------------------- */
int ofrr_reuse_power(const void* W, int64_t ldw, int w_fmt, int64_t n, int kp, const double* Y,
                     int ldy, const int* r_dev, int r_max, void* Xout, int64_t ldx, int x_fmt,
                     double* colmax, int* flags, void* stream);

/* ---------------------------------------------------------------------------------
 * K6f: the restart step of one outer iteration in one pass over (U, W) -- ofrr_ritz_recover
 * (Xu = round(U Y), U64 = U Y), ofrr_reuse_power (Xw = round(W Y), colmax) and
 * ofrr_residual_estimate (columns < t, mode as there) fused: both products of a row tile
 * on the fp64 tensor cores from one Y slab.  Every output is optional (NULL); Xu / U64 / Xw
 * are bitwise those of the separate entries.  Replaces ofrr/projection.py:86 and
 * ofrr/driver.py:102-109 of the next iteration (A-pass reuse) plus the convergence estimate.
 * W (w_fmt F32 or F64) may be NULL when only Xu / U64 are asked for.  The workspace
 * (ofrr_restart_workspace(n, t) bytes) holds the per-row-block residual sums.
 * ------------------------------------------------------------------------------- */
size_t ofrr_restart_workspace(int64_t n, int t);
int ofrr_restart(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n,
                 int kp, const double* Y, int ldy, const int* r_dev, int r_max, void* Xu, int64_t ldxu,
                 int xu_fmt, int* flags_u, double* U64, int64_t ld64, void* Xw, int64_t ldxw, int xw_fmt,
                 int* flags_w, double* colmax, const double* vals, int t, double* res, int mode,
                 void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * K7: FP64 residuals  res[j] = || A v_j - lambda_j v_j ||_2 / |lambda_j|  (inf when
 * lambda_j == 0).  Replaces ofrr/projection.py:136-147 residual_report (eig branch).
 * A (rows x cols row-major, a_fmt) is promoted to fp64 exactly.  For the SVD branch
 * (:148-157) call twice: ofrr_residual_pair with (A, V, U) and (A^T, U, V).
 * ofrr_residual_pair: res[j] = max(res[j], ||op(A) x_j - s_j y_j|| / s_j).
 * ------------------------------------------------------------------------------- */
size_t ofrr_residual_workspace(int64_t rows, int r);
/* Workspace of ofrr_residual_eig / ofrr_residual_pair for a rows x cols operator in a_fmt.
 * For a 16/8-bit operator (not transposed) the FP64-accurate product runs on the int8
 * tensor cores (Ozaki scheme: six 7-bit digit planes of A and of the vectors, exact int32
 * level sums); the workspace then holds the digit planes (~6 bytes per entry of A). */
size_t ofrr_residual_workspace2(int64_t rows, int64_t cols, int r, int a_fmt, int transpose);

/* FP64-accurate products with a 16/8-bit operator on the int8 tensor cores (Ozaki scheme,
 * see ofrr_residual_workspace2), split into a per-operator stage and per-product calls:
 *   prepare   the row scales of A into op_ws (ofrr_ozaki_operator_workspace bytes); the
 *             digits of A are made on the fly inside the product kernel (A is read once
 *             in its own format); OFRR_OZ_PLANES=1 selects the variant that stores six
 *             balanced base-256 digit planes of A (~6 bytes per entry) instead;
 *   gemm      W = A X for an fp64 block X (cols x k, ldx), W rounded to out_fmt (ldw),
 *             optional W2 in out_fmt2, colmax[j] = max(colmax[j], max_i |W_ij|), flags |=
 *             NONFINITE -- the F64-policy block product of ofrr/_kernels.pyx:60-84 without an
 *             fp64 copy of A;
 *   residual  res[j] as ofrr_residual_pair (A not transposed) with the prepared operator.
 * Products agree with an FP64 GEMM to ~2^-46 relative to |A| |X| per term (random-sign
 * truncation), not bitwise. */
/* Diagnostics of a prepared operator (synchronous): *full = 1 when its products use all six
 * digit planes of A (some row's tails overflowed the per-row list or its scale left the f32
 * range), 0 when they use the 3-digit heads plus the exact fp64 tails; *tails = number of
 * tail entries listed over all rows. */
int ofrr_ozaki_operator_info(const void* op_ws, int64_t rows, int* full, long long* tails);
size_t ofrr_ozaki_operator_workspace(int64_t rows, int64_t cols);
size_t ofrr_ozaki_workspace(int64_t rows, int64_t cols, int r);
int ofrr_ozaki_prepare(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt, void* op_ws,
                       size_t op_bytes, void* stream);
int ofrr_ozaki_gemm(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                    const void* op_ws, const double* X, int64_t ldx, int k, void* W, int64_t ldw,
                    int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
                    void* workspace, size_t workspace_bytes, void* stream);
/* The same product with a chosen accuracy: levels = 6 is ofrr_ozaki_gemm (digit products
 * with p + q < 6, ~2^-46 of |A||x| per term); levels = 4 keeps p + q < 4 (~2^-30 per term,
 * ~40% of the int8 work, 128 columns per pass) -- the products of the full-f64-lite ladder
 * rung, which hands over to full FP64 before the residuals need more. */
int ofrr_ozaki_gemm_levels(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                           const void* op_ws, const double* X, int64_t ldx, int k, void* W, int64_t ldw,
                           int out_fmt, double* colmax, int* flags, void* W2, int64_t ldw2, int out_fmt2,
                           int levels, void* workspace, size_t workspace_bytes, void* stream);
int ofrr_ozaki_residual(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                        const void* op_ws, const double* Xv, int64_t ldx, const double* Yv,
                        int64_t ldy, const double* vals, const int* r_dev, int r_max, double* res,
                        int accumulate_max, void* workspace, size_t workspace_bytes, void* stream);
int ofrr_residual_eig(const void* A, int64_t n, int64_t lda, int a_fmt, const double* V,
                      int64_t ldv, const double* vals, const int* r_dev, int r_max, double* res,
                      void* workspace, size_t workspace_bytes, void* stream);
int ofrr_residual_pair(const void* A, int64_t rows, int64_t cols, int64_t lda, int a_fmt,
                       int transpose, const double* Xv, int64_t ldx, const double* Yv,
                       int64_t ldy, const double* vals, const int* r_dev, int r_max,
                       double* res, int accumulate_max, void* workspace,
                       size_t workspace_bytes, void* stream);

/* K7e: per-iteration residual estimate without another pass over A:
 *   res[j] = || (W - lambda_j U) y_j ||_2 / |lambda_j|,  W = A U in its accumulation format
 * (mode 0; mode 2 returns raw sums of squares for a cross-rank all-reduce).  Used only to
 * decide when to stop; the reported residuals are always the FP64 ones of K7. */
size_t ofrr_residual_estimate_workspace(int64_t n, int r);
int ofrr_residual_estimate(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt,
                           int64_t n, int kp, const double* Y, int ldy, const double* vals,
                           const int* r_dev, int r_max, double* res, int mode, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * K8: synthetic symmetric matrix A = S C S + Wf Mf^T + Mf Wf^T (FP64, rounded once to
 * a_fmt, row-major), where C[i,j] = c[i xor j] (n a power of two; Walsh-Hadamard
 * diagonalisation) or C = diag(c) otherwise.  Row block [row0, row0+rows).
 * The host computes c, s, Wf, Mf (ofrr_b200/matrix.py); the device evaluates the
 * elementwise formula in a fixed order, so the oracle reproduces it bit for bit.
 * ------------------------------------------------------------------------------- */
int ofrr_generate_sym(int64_t n, int64_t row0, int64_t rows, int hadamard, const double* c,
                      const double* s, const double* Wf, const double* Mf, int r, void* A,
                      int64_t lda, int a_fmt, void* stream);

/* Start block X0 = numpy.random.default_rng(seed).random((n, k)) rounded to fmt
 * (ofrr/driver.py:97-99, ofrr/driver.py:150-152), generated on the device bit for bit from
 * the PCG64 state (state, inc) that numpy's SeedSequence derives from the seed. */
int ofrr_start_block_pcg64(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           int64_t n, int k, void* X, int64_t ldx, int fmt, void* stream);

/* utility: round/convert a column-major block between formats (ofrr/precision.py:90-104) */
int ofrr_convert(const void* src, int src_fmt, int64_t ld_src, void* dst, int dst_fmt,
                 int64_t ld_dst, int64_t n, int64_t k, int* flags, void* stream);

/* utility: dst (row-major rows x cols) <- round(src (column-major rows x cols)); uploads the
 * reference's F-order operators (ofrr/matrix.py:25-31) into the row-major device layout */
int ofrr_transpose_convert(const void* src, int src_fmt, int64_t ld_src, void* dst, int dst_fmt,
                           int64_t ld_dst, int64_t rows, int64_t cols, int* flags, void* stream);

/* utility: symmetric operator upload from a HOST row-major n x n array already in the
 * storage format `fmt`.  Only one triangle is read (uplo 0: entries (i, j >= i); uplo 1:
 * (i, j <= i) -- the dsyev(uplo) convention; the eigen path ofrr/driver.py:84-111 is defined
 * for symmetric A): it crosses PCIe as 2-D copies of `block_rows`-row blocks (0: 2048) on
 * `stream`, and a side stream mirrors each block into the other triangle as it lands.
 * *bytes = host bytes copied.  `host` should be pinned for the copies to be asynchronous. */
int ofrr_upload_sym(const void* host, int64_t ld_host, void* A, int64_t lda, int64_t n, int fmt, int uplo,
                    int64_t block_rows, long long* bytes, void* stream);

/* ---------------------------------------------------------------------------------
 * Host-buffer plugin entry points: the exact signatures of the reference's kernel
 * module (ofrr/_kernels.pyx) so `ofrr.backend.kernels` can bind them.
 * Host float64 in, host float64 out; copies run inside the call.
 * ------------------------------------------------------------------------------- */
/* ofrr/_kernels.pyx:60-84 gemm_mixed(a, b, compute, accumulate, out_fmt): a is m x k
 * with element strides (ars, acs), b is k x n with (brs, bcs), c is m x n F-order.
 * The device computes with exact products (tensor cores for 16-bit values) and fp32
 * (F16/BF16/F32 accumulate) or fp64 accumulation. */
int ofrr_host_gemm_mixed(const double* a, int64_t ars, int64_t acs, const double* b,
                         int64_t brs, int64_t bcs, int64_t m, int64_t k, int64_t n, int compute,
                         int accumulate, int out_fmt, double* c);
/* ofrr/_kernels.pyx:105-150 jacobi_eig(a, max_sweeps, tol) -> (vals, vecs, sweeps, off)
 * a: n x n row-major; vals[n]; vecs n x n row-major (vecs[i*n+p] = V[i,p]). */
int ofrr_host_jacobi_eig(const double* a, int64_t n, int max_sweeps, double tol, double* vals,
                         double* vecs, int* sweeps, double* off);

/* K8b: the reference's Gaussian-kernel test matrix (ofrr/matrix.py:97-113) evaluated on the
 * device, FP64 in the reference's operation order, rounded once to out_fmt and written
 * row-major (leading dimension ld >= m).  px: n x 2 points (row-major, device); py: m x 2
 * column points (cross kernel, no diagonal term) or NULL (square kernel: py = px, + s on the
 * diagonal).  Replaces the host generation in ofrr/cli.py:163-189 for the harness. */
int ofrr_gaussian_kernel(const double* px, int64_t n, const double* py, int64_t m, double f, double l, double s,
                         void* out, int64_t ld, int out_fmt, void* stream);

/* Gram-Schmidt basis builders, the classical comparators that OFRR + Hessenberg replaces
 * (SURVEY.md 8(f) rank 4).  Replaces ofrr/basis.py:65-148 (orthonormalize with
 * method = 0 mgs-l, 1 mgs-r, 2 cgs, 3 cgs2; reorth as the reference's keyword).  Q receives
 * the kept columns first (n_kept of them, zeros after), kept[k] marks the input columns
 * kept.  Element arithmetic per the policy (storage / compute / accumulate), sums in
 * parallel order: agrees with the reference to the accumulate format's rounding.
 * k <= 512.  Returns OFRR_OK (an empty basis is *n_kept == 0; the caller raises). */
size_t ofrr_orthonormalize_workspace(int64_t n, int k);
int ofrr_orthonormalize(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, int accumulate,
                        double drop_tol, int method, int reorth, void* Q, int64_t ldq, int* kept, int* n_kept,
                        void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OFRR_B200_H */
