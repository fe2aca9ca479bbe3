// small_eig.cu -- K5: fp64 solve of the projected OFRR pencil  B y = lambda M y.
//
// Replaces ofrr/smallsolve.py:34-88 (sym_eig, _sorted_desc, sym_def_gen_eig) and the
// cyclic Jacobi of ofrr/_kernels.pyx:105-161.  One CTA of 1024 threads, everything in
// shared memory when it fits:
//
//  * Jacobi, round-robin (tournament) parallel ordering: each round rotates k/2 disjoint
//    (p,q) pairs.  One warp owns a pair: it forms (c, s) from a_pp, a_qq, a_pq with the
//    reference's formula (_kernels.pyx:124-130), applies the row rotation to rows p,q,
//    [barrier], then the column rotation to columns p,q and to V, and zeroes a_pq / a_qp
//    exactly (:141-142) [barrier].  Two barriers per round, no integer division, pair
//    tables precomputed.  Same skip threshold off/k^2, stopping rule
//    off <= 1e-14 ||S||_F and 30-sweep cap as the reference (smallsolve.py:17,45-48).
//  * sym_def_gen_eig (smallsolve.py:64-88): the reference whitens M through eig(M) and
//    drops the directions with mu <= k eps mu_max.  When M is certifiably above that
//    cutoff -- Cholesky M = R^T R succeeds and 1/||R^-1||_F^2 > 4 k eps ||M||_F, which
//    bounds mu_min from below and mu_max from above -- nothing is dropped, and whitening
//    with R gives the same pencil eigenpairs (eigenvalues identical, M-orthonormal
//    eigenvectors identical up to sign, fixed by the sign rule).  Otherwise the
//    reference's eig(M) path runs.  Then eig(T), back-transform, stable descending sort
//    and the largest-|entry|-positive sign rule (smallsolve.py:52-61).
#include "common.cuh"
#include <algorithm>

namespace ofrr {

static constexpr int ET = 1024;
static constexpr int NW = ET / 32;
static constexpr int MAXK = 512;
static constexpr int JACOBI_MAX_SWEEPS = 30;   // ofrr/smallsolve.py:17

struct EigScratch {
  double c[MAXK / 2], s[MAXK / 2];
  int p[MAXK / 2], q[MAXK / 2], act[MAXK / 2];
  double red[NW];
  double vals[MAXK];
  double dis[MAXK];
  int order[MAXK];
  int flag;
};

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    double t = threadIdx.x < NW ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// S is column-major with leading dimension ld (element (i,j) at S[j*ld + i]).
__device__ double off_norm(const double* S, int k, int ld, double* red) {
  double v = 0.0;
  for (int j = threadIdx.x >> 5; j < k; j += NW)
    for (int i = threadIdx.x & 31; i < k; i += 32)
      if (i != j) v += S[j * ld + i] * S[j * ld + i];
  return sqrt(block_sum(v, red));
}

__device__ double fro_norm(const double* S, int k, int ld, double* red) {
  double v = 0.0;
  for (int j = threadIdx.x >> 5; j < k; j += NW)
    for (int i = threadIdx.x & 31; i < k; i += 32) v += S[j * ld + i] * S[j * ld + i];
  return sqrt(block_sum(v, red));
}

// Parallel-order cyclic Jacobi on S (k x k, ld); V (k x k, ldv) <- accumulated rotations.
// Returns the final off-diagonal norm; *sweeps_out (thread 0) receives the sweep count.
__device__ double jacobi_parallel(double* S, int ld, double* V, int ldv, int k, double tol, int max_sweeps,
                                  EigScratch& sc, int* sweeps_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < k; j += NW)
    for (int i = lane; i < k; i += 32) V[j * ldv + i] = (i == j) ? 1.0 : 0.0;
  double off = off_norm(S, k, ld, sc.red);
  const int kk = k + (k & 1), np = kk / 2, m = kk - 1;
  int sweeps = 0;
  while (off > tol && sweeps < max_sweeps) {
    const double skip = off / ((double)k * (double)k);
    for (int r = 0; r < m; ++r) {
      // ---- phase A: every warp forms the rotations of its pairs, rotates their rows ----
      // (a warp handles pairs w, w + NW, ...; k <= 2*NW*...: loop)
      int my_act = 0;
      for (int t = warp; t < np; t += NW) {
        if (lane != 0) continue;
        int a, b;
        if (t == 0) { a = m; b = r; }
        else {
          a = r + t; if (a >= m) a -= m;
          b = r - t; if (b < 0) b += m;
        }
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        int ac = 0;
        if (q < k) {
          const double apq = S[q * ld + p];
          if (fabs(apq) > skip) {
            const double app = S[p * ld + p], aqq = S[q * ld + q];
            const double theta = (aqq - app) / (2.0 * apq);
            const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(tt * tt + 1.0);
            s = tt * c;
            ac = 1;
          }
        }
        sc.c[t] = c; sc.s[t] = s; sc.p[t] = p; sc.q[t] = q; sc.act[t] = ac;
        my_act |= ac;
      }
      // barrier: every warp has read its a_pp, a_qq, a_pq before any row changes; a round
      // in which every pair is below the skip threshold does nothing (uniform branch)
      if (!__syncthreads_or(my_act)) continue;
      for (int t = warp; t < np; t += NW) {
        if (!sc.act[t]) continue;
        const int p = sc.p[t], q = sc.q[t];
        const double c = sc.c[t], s = sc.s[t];
        for (int j = lane; j < k; j += 32) {       // rows p, q  (_kernels.pyx:131-135)
          const double tp = S[j * ld + p], tq = S[j * ld + q];
          S[j * ld + p] = c * tp - s * tq;
          S[j * ld + q] = s * tp + c * tq;
        }
      }
      __syncthreads();
      // ---- phase B: columns p, q (:136-140), zero a_pq (:141-142), V (:143-147) -------
      for (int t = warp; t < np; t += NW) {
        if (!sc.act[t]) continue;
        const int p = sc.p[t], q = sc.q[t];
        const double c = sc.c[t], s = sc.s[t];
        for (int i = lane; i < k; i += 32) {
          const double tp = S[p * ld + i], tq = S[q * ld + i];
          S[p * ld + i] = c * tp - s * tq;
          S[q * ld + i] = s * tp + c * tq;
          const double vp = V[p * ldv + i], vq = V[q * ldv + i];
          V[p * ldv + i] = c * vp - s * vq;
          V[q * ldv + i] = s * vp + c * vq;
        }
        __syncwarp();
        if (lane == 0) { S[q * ld + p] = 0.0; S[p * ld + q] = 0.0; }
      }
      __syncthreads();
    }
    off = off_norm(S, k, ld, sc.red);
    ++sweeps;
  }
  if (sweeps_out && threadIdx.x == 0) *sweeps_out = sweeps;
  return off;
}

// ofrr/smallsolve.py:52-61: stable descending sort of vals (length nv) with the columns of
// Vin (rows x nv, ld ldi) -> Vout (ld ldo); then the largest-|entry|-positive sign rule.
__device__ void sorted_desc(const double* vals_in, const double* Vin, int ldi, int rows, int nv, double* vals_out,
                            double* Vout, int ldo, EigScratch& sc) {
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    const double vi = vals_in[i];
    int rank = 0;
    for (int j = 0; j < nv; ++j) {
      const double vj = vals_in[j];
      if (vj > vi || (vj == vi && j < i)) ++rank;
    }
    sc.order[rank] = i;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) sc.vals[i] = vals_in[sc.order[i]];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < nv; j += NW)
    for (int r = lane; r < rows; r += 32) Vout[j * ldo + r] = Vin[sc.order[j] * ldi + r];
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) vals_out[i] = sc.vals[i];
  for (int j = warp; j < nv; j += NW) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = lane; r < rows; r += 32) {
      const double a = fabs(Vout[j * ldo + r]);
      if (a > best) { best = a; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const bool neg = Vout[j * ldo + bi] < 0.0;
    __syncwarp();
    if (neg)
      for (int r = lane; r < rows; r += 32) Vout[j * ldo + r] = -Vout[j * ldo + r];
  }
  __syncthreads();
}

// C (m x n, ldc) = op(A) * op(B) with column-major operands; block-wide, fp64.
__device__ void mm(const double* A, int lda, bool ta, const double* B, int ldb, bool tb, double* C, int ldc, int m,
                   int n, int kd, double alpha = 1.0) {
  for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
    const int i = e % m, j = e / m;
    double s = 0.0;
    for (int l = 0; l < kd; ++l) {
      const double a = ta ? A[i * lda + l] : A[l * lda + i];
      const double b = tb ? B[l * ldb + j] : B[j * ldb + l];
      s = fma(a, b, s);
    }
    C[j * ldc + i] = alpha * s;
  }
  __syncthreads();
}

// In-place Cholesky (lower) of the k x k SPD matrix L (ld); returns false if a pivot <= 0.
__device__ bool cholesky(double* L, int ld, int k, EigScratch& sc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) sc.flag = 1;
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const double d = L[j * ld + j];
    if (!(d > 0.0)) {
      if (threadIdx.x == 0) sc.flag = 0;
      __syncthreads();
      return false;
    }
    const double r = sqrt(d);
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) L[j * ld + i] /= r;
    if (threadIdx.x == 0) L[j * ld + j] = r;
    __syncthreads();
    // trailing update (lower triangle): L[i, c] -= L[i, j] L[c, j], c in (j, k), i >= c
    for (int c = j + 1 + warp; c < k; c += NW) {
      const double lc = L[j * ld + c];
      for (int i = c + lane; i < k; i += 32) L[c * ld + i] -= L[j * ld + i] * lc;
    }
    __syncthreads();
  }
  return sc.flag != 0;
}

// Rinv (lower-triangular inverse of L, ld) written into X (ld), X zero above the diagonal.
__device__ void tri_inverse_lower(const double* L, int ld, double* X, int ldx, int k) {
  // column j of L^-1: forward substitution L x = e_j (independent per column)
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    for (int i = 0; i < j; ++i) X[j * ldx + i] = 0.0;
    X[j * ldx + j] = 1.0 / L[j * ld + j];
    for (int i = j + 1; i < k; ++i) {
      double s = 0.0;
      for (int l = j; l < i; ++l) s = fma(L[l * ld + i], X[j * ldx + l], s);
      X[j * ldx + i] = -s / L[i * ld + i];
    }
  }
  __syncthreads();
}

struct EigBufs { double *S, *V, *P, *T; };

__device__ long long g_k5prof[8];   // phase timestamps of the last pencil solve (debug)
int k5_profile(long long* out) { return cudaMemcpyFromSymbol(out, g_k5prof, sizeof(g_k5prof)) == cudaSuccess ? 0 : 2; }

// Every k x k work buffer uses the padded leading dimension L = k | 1 (odd): row walks of a
// column-major fp64 matrix then hit distinct shared-memory banks.
__host__ __device__ inline int pad_k(int k) { return (k % 2 == 0) ? k + 1 : k; }

// mode 0: sym_eig(A)      -> values[k], vectors (k x k)            (smallsolve.py:34-49)
// mode 1: raw jacobi_eig  -> values = diag (unsorted), vectors = V  (_kernels.pyx:105-150)
// mode 2: sym_def_gen_eig(B=A, M=Mm)                                 (smallsolve.py:64-88)
// Inputs/outputs are column-major with leading dimension k.
__global__ void __launch_bounds__(ET, 1)
    k_small_eig(int mode, const double* __restrict__ A, const double* __restrict__ Mm, int k, double raw_tol,
                int raw_sweeps, double* __restrict__ values, double* __restrict__ vectors, int* __restrict__ n_out,
                int* __restrict__ status, double* __restrict__ off_out, int* __restrict__ sweeps_out, EigBufs gb,
                int nsm) {
  extern __shared__ double dsm[];
  __shared__ EigScratch sc;
  __shared__ double tau[MAXK];
  __shared__ int kp_s;
  const int L = pad_k(k);
  const size_t kL = (size_t)k * L;
  // buffers: the first `nsm` of {S, V, P, T} live in shared memory
  double* S = nsm >= 1 ? dsm : gb.S;
  double* V = nsm >= 2 ? dsm + kL : gb.V;
  double* P = nsm >= 3 ? dsm + 2 * kL : gb.P;
  double* T = nsm >= 4 ? dsm + 3 * kL : gb.T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (k == 0) {
    if (threadIdx.x == 0) { if (n_out) *n_out = 0; if (status) *status = mode == 2 ? OFRR_ERR_EMPTY_PENCIL : 0; }
    return;
  }
  // S <- input (mode 1) or its symmetric part (modes 0 / 2: M for the pencil)
  const double* src = mode == 2 ? Mm : A;
  for (int j = warp; j < k; j += NW)
    for (int i = lane; i < k; i += 32)
      S[j * L + i] = mode == 1 ? src[(size_t)j * k + i] : (src[(size_t)j * k + i] + src[(size_t)i * k + j]) / 2.0;
  __syncthreads();
  if (mode == 1) {
    double off = jacobi_parallel(S, L, V, L, k, raw_tol, raw_sweeps, sc, sweeps_out);
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) values[i] = S[i * L + i];
    for (int j = warp; j < k; j += NW)
      for (int i = lane; i < k; i += 32) vectors[(size_t)j * k + i] = V[j * L + i];
    if (threadIdx.x == 0) { if (off_out) *off_out = off; if (status) *status = 0; }
    return;
  }
  if (mode == 0) {
    const double nrm = fro_norm(S, k, L, sc.red), tol = 1e-14 * nrm;
    const double off = jacobi_parallel(S, L, V, L, k, tol, JACOBI_MAX_SWEEPS, sc, nullptr);
    if (off > tol && nrm > 0.0) {
      if (threadIdx.x == 0) { *status = OFRR_ERR_CONVERGENCE; if (off_out) *off_out = off; }
      return;
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) tau[i] = S[i * L + i];
    __syncthreads();
    sorted_desc(tau, V, L, k, k, values, vectors, k, sc);
    if (threadIdx.x == 0) { *status = 0; if (n_out) *n_out = k; }
    return;
  }

  // ======================= mode 2: the pencil ===========================================
  if (threadIdx.x == 0) g_k5prof[0] = clock64();
  // ---- fast whitening: Cholesky, certified above the safeguard cutoff ----
  const double mnorm = fro_norm(S, k, L, sc.red);   // ||M||_F >= mu_max
  for (int j = warp; j < k; j += NW)
    for (int i = lane; i < k; i += 32) P[j * L + i] = S[j * L + i];
  __syncthreads();
  bool chol = mnorm > 0.0 && cholesky(P, L, k, sc);
  if (threadIdx.x == 0) g_k5prof[1] = clock64();
  int kp = k;
  if (chol) {
    tri_inverse_lower(P, L, T, L, k);                // T = L^-1 (= R^-T)
    if (threadIdx.x == 0) g_k5prof[2] = clock64();
    const double inv2 = fro_norm(T, k, L, sc.red);   // ||R^-1||_F ; mu_min >= 1/||R^-1||_F^2
    chol = (1.0 / (inv2 * inv2)) > 4.0 * (double)k * 2.220446049250313e-16 * mnorm;
  }
  if (chol) {
    for (int j = warp; j < k; j += NW)                // V <- Bs = (B + B^T)/2
      for (int i = lane; i < k; i += 32) V[j * L + i] = (A[(size_t)j * k + i] + A[(size_t)i * k + j]) / 2.0;
    __syncthreads();
    mm(T, L, false, V, L, false, P, L, k, k, k);     // P <- L^-1 Bs
    mm(P, L, false, T, L, true, V, L, k, k, k);      // V <- (L^-1 Bs) L^-T
    if (threadIdx.x == 0) g_k5prof[3] = clock64();
  } else {
    // ---- the reference's eigen-whitening (smallsolve.py:75-88) ----
    const double tol = 1e-14 * mnorm;
    const double off = jacobi_parallel(S, L, V, L, k, tol, JACOBI_MAX_SWEEPS, sc, nullptr);
    if (off > tol && mnorm > 0.0) {
      if (threadIdx.x == 0) { *status = OFRR_ERR_CONVERGENCE; *n_out = 0; if (off_out) *off_out = off; }
      return;
    }
    for (int i = threadIdx.x; i < k; i += blockDim.x) tau[i] = S[i * L + i];
    __syncthreads();
    sorted_desc(tau, V, L, k, k, sc.dis, P, L, sc);   // mu (desc) in sc.dis, P = eigvecs of M
    const double mu_max = sc.dis[0];
    if (threadIdx.x == 0) {
      int c = 0;
      const double thr = (double)k * 2.220446049250313e-16 * mu_max;
      if (mu_max > 0.0) while (c < k && sc.dis[c] > thr) ++c;
      kp_s = c;
    }
    __syncthreads();
    kp = kp_s;
    if (kp == 0) {
      if (threadIdx.x == 0) { *status = OFRR_ERR_EMPTY_PENCIL; *n_out = 0; }
      return;
    }
    for (int i = threadIdx.x; i < kp; i += blockDim.x) sc.dis[i] = 1.0 / sqrt(sc.dis[i]);
    for (int j = warp; j < k; j += NW)                // S <- Bs
      for (int i = lane; i < k; i += 32) S[j * L + i] = (A[(size_t)j * k + i] + A[(size_t)i * k + j]) / 2.0;
    __syncthreads();
    mm(S, L, false, P, L, false, T, L, k, kp, k);    // T <- Bs P        (k x kp)
    mm(P, L, true, T, L, false, V, L, kp, kp, k);    // V <- P^T Bs P    (kp x kp)
    for (int j = warp; j < kp; j += NW)
      for (int i = lane; i < kp; i += 32) V[j * L + i] = (sc.dis[i] * V[j * L + i]) * sc.dis[j];
    __syncthreads();
  }
  if (threadIdx.x == 0) g_k5prof[4] = clock64();
  // ---- eig(T), T = (V + V^T)/2 (kp x kp) ----
  for (int j = warp; j < kp; j += NW)
    for (int i = lane; i < kp; i += 32) S[j * L + i] = (V[j * L + i] + V[i * L + j]) / 2.0;
  __syncthreads();
  const double nrm = fro_norm(S, kp, L, sc.red), tol = 1e-14 * nrm;
  const double off = jacobi_parallel(S, L, V, L, kp, tol, JACOBI_MAX_SWEEPS, sc, nullptr);
  if (off > tol && nrm > 0.0) {
    if (threadIdx.x == 0) { *status = OFRR_ERR_CONVERGENCE; *n_out = 0; if (off_out) *off_out = off; }
    return;
  }
  for (int i = threadIdx.x; i < kp; i += blockDim.x) tau[i] = S[i * L + i];
  __syncthreads();
  if (threadIdx.x == 0) g_k5prof[5] = clock64();
  // ---- back-transform y = W Z  (W = L^-T, or P D^-1/2) -> S, then sort + sign ----
  if (chol) {
    mm(T, L, true, V, L, false, S, L, k, kp, k);     // S <- L^-T Z
  } else {
    for (int j = warp; j < kp; j += NW)
      for (int i = lane; i < k; i += 32) {
        double s = 0.0;
        for (int l = 0; l < kp; ++l) s = fma(P[l * L + i], sc.dis[l] * V[j * L + l], s);
        T[j * L + i] = s;
      }
    __syncthreads();
    for (int j = warp; j < kp; j += NW)
      for (int i = lane; i < k; i += 32) S[j * L + i] = T[j * L + i];
    __syncthreads();
  }
  sorted_desc(tau, S, L, k, kp, values, vectors, k, sc);
  if (threadIdx.x == 0) g_k5prof[6] = clock64();
  if (threadIdx.x == 0) { *status = 0; *n_out = kp; }
}

size_t small_eig_ws(int k) { return (size_t)4 * k * pad_k(k) * sizeof(double) + 1024; }

int small_eig(int mode, const double* A, const double* M, int k, double raw_tol, int raw_sweeps, double* values,
              double* vectors, int* n_out, int* status, double* off_out, int* sweeps_out, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  if (k < 0 || k > MAXK) { ofrr_set_error("small eig: k=%d outside [0, %d]", k, MAXK); return OFRR_ERR_INVALID; }
  if (ws_bytes < small_eig_ws(k)) { ofrr_set_error("small eig: workspace too small"); return OFRR_ERR_INVALID; }
  EigBufs b;
  double* p = (double*)ws;
  const size_t kL = (size_t)k * pad_k(k);
  b.S = p; b.V = p + kL; b.P = p + 2 * kL; b.T = p + 3 * kL;
  const size_t one = kL * sizeof(double);
  const size_t budget = 190 * 1024;
  int nsm = one ? (int)std::min<size_t>(4, budget / one) : 0;
  const size_t shm = (size_t)nsm * one;
  static bool attr = false;
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_small_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, 190 * 1024));
    attr = true;
  }
  k_small_eig<<<1, ET, shm, st>>>(mode, A, M, k, raw_tol, raw_sweeps, values, vectors, n_out, status, off_out,
                                  sweeps_out, b, nsm);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
