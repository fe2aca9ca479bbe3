// small_eig.cu -- K5: fp64 solve of the projected OFRR pencil  B y = lambda M y.
//
// Replaces ofrr/smallsolve.py:34-88 (sym_eig, _sorted_desc, sym_def_gen_eig) and the
// cyclic Jacobi of ofrr/_kernels.pyx:105-161.  One CTA (1024 threads):
//   * Jacobi with the round-robin (tournament) parallel ordering: each round rotates
//     k/2 disjoint (p,q) pairs at once.  Because the pairs partition the index set,
//     the two-sided update J^T S J splits into independent 2x2 blocks
//     S[{pa,qa},{pb,qb}] <- R_a^T S[..] R_b, one block per thread, read/written once
//     per round; V <- V J likewise.  Same rotation formula, skip threshold
//     off/k^2, stopping rule off <= 1e-14 ||S||_F and 30-sweep cap as the reference.
//   * the independence safeguard (keep mu > k eps mu_max), whitening, second
//     eigensolve and back-transform, stable descending sort and the
//     largest-|entry|-positive sign rule, all on device.
// S/V live in shared memory when they fit, otherwise in the (L2-resident) workspace.
#include "common.cuh"
#include <algorithm>

namespace ofrr {

static constexpr int ET = 1024;
static constexpr int MAXK = 512;
static constexpr int JACOBI_MAX_SWEEPS = 30;   // ofrr/smallsolve.py:17

struct EigScratch {
  int p[MAXK / 2], q[MAXK / 2], act[MAXK / 2];
  double c[MAXK / 2], s[MAXK / 2];
  double red[ET / 32];
  double dis[MAXK];
  double vals[MAXK];
  int order[MAXK];
};

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];   // fixed order
    red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

__device__ double off_norm(const double* S, int k, double* red) {
  double v = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
    const int i = e % k, j = e / k;
    if (i != j) v += S[e] * S[e];
  }
  return sqrt(block_sum(v, red));
}

__device__ double fro_norm(const double* S, int k, double* red) {
  double v = 0.0;
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) v += S[e] * S[e];
  return sqrt(block_sum(v, red));
}

// Parallel-order cyclic Jacobi on column-major S (k x k); V <- accumulated rotations.
// Returns the final off-diagonal norm.
__device__ double jacobi_parallel(double* S, double* V, int k, double tol, int max_sweeps, EigScratch& sc,
                                  int* sweeps_out = nullptr) {
  for (int e = threadIdx.x; e < k * k; e += blockDim.x) V[e] = (e % k == e / k) ? 1.0 : 0.0;
  double off = off_norm(S, k, sc.red);
  const int kk = k + (k & 1), np = kk / 2, m = kk - 1;
  int sweeps = 0;
  while (off > tol && sweeps < max_sweeps) {
    const double skip = off / ((double)k * (double)k);
    for (int r = 0; r < m; ++r) {
      if (threadIdx.x < np) {
        const int t = threadIdx.x;
        int a, b;
        if (t == 0) { a = m; b = r % m; }
        else { a = (r + t) % m; b = (r - t + m) % m; }
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        int act = 0;
        if (q < k) {
          const double apq = S[(int64_t)q * k + p];
          if (fabs(apq) > skip) {
            const double app = S[(int64_t)p * k + p], aqq = S[(int64_t)q * k + q];
            const double theta = (aqq - app) / (2.0 * apq);
            const double tt = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(tt * tt + 1.0);
            s = tt * c;
            act = 1;
          }
        }
        sc.p[t] = p; sc.q[t] = q; sc.c[t] = c; sc.s[t] = s; sc.act[t] = act;
      }
      __syncthreads();
      for (int blk = threadIdx.x; blk < np * np; blk += blockDim.x) {
        const int a = blk / np, b = blk % np;
        if (!sc.act[a] && !sc.act[b]) continue;
        const int pa = sc.p[a], qa = sc.q[a], pb = sc.p[b], qb = sc.q[b];
        const bool hqa = qa < k, hqb = qb < k;
        const double x00 = S[(int64_t)pb * k + pa];
        const double x01 = hqb ? S[(int64_t)qb * k + pa] : 0.0;
        const double x10 = hqa ? S[(int64_t)pb * k + qa] : 0.0;
        const double x11 = (hqa && hqb) ? S[(int64_t)qb * k + qa] : 0.0;
        const double ca = sc.c[a], sa = sc.s[a], cb = sc.c[b], sb = sc.s[b];
        // rows (ofrr/_kernels.pyx:131-135): p <- c p - s q ; q <- s p + c q
        const double y00 = ca * x00 - sa * x10, y01 = ca * x01 - sa * x11;
        const double y10 = sa * x00 + ca * x10, y11 = sa * x01 + ca * x11;
        // columns (:136-140)
        double z00 = cb * y00 - sb * y01, z01 = sb * y00 + cb * y01;
        double z10 = cb * y10 - sb * y11, z11 = sb * y10 + cb * y11;
        if (a == b && sc.act[a]) { z01 = 0.0; z10 = 0.0; }   // (:141-142)
        S[(int64_t)pb * k + pa] = z00;
        if (hqb) S[(int64_t)qb * k + pa] = z01;
        if (hqa) S[(int64_t)pb * k + qa] = z10;
        if (hqa && hqb) S[(int64_t)qb * k + qa] = z11;
      }
      for (int e = threadIdx.x; e < k * np; e += blockDim.x) {
        const int i = e / np, a = e % np;
        if (!sc.act[a]) continue;
        const int pa = sc.p[a], qa = sc.q[a];
        const double c = sc.c[a], s = sc.s[a];
        const double vp = V[(int64_t)pa * k + i], vq = V[(int64_t)qa * k + i];
        V[(int64_t)pa * k + i] = c * vp - s * vq;   // (:143-147)
        V[(int64_t)qa * k + i] = s * vp + c * vq;
      }
      __syncthreads();
    }
    off = off_norm(S, k, sc.red);
    ++sweeps;
  }
  if (sweeps_out && threadIdx.x == 0) *sweeps_out = sweeps;
  return off;
}

// ofrr/smallsolve.py:52-61: stable descending sort of vals (length nv) with the columns of
// Vin (k rows, ld k) -> Vout; then the largest-|entry|-positive sign rule.
__device__ void sorted_desc(const double* vals_in, const double* Vin, int rows, int nv, double* vals_out,
                            double* Vout, EigScratch& sc) {
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
  for (int e = threadIdx.x; e < rows * nv; e += blockDim.x) {
    const int r = e % rows, j = e / rows;
    Vout[(int64_t)j * rows + r] = Vin[(int64_t)sc.order[j] * rows + r];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) vals_out[i] = sc.vals[i];
  // sign rule: one warp per column
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = warp; j < nv; j += nw) {
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = lane; r < rows; r += 32) {
      const double a = fabs(Vout[(int64_t)j * rows + r]);
      if (a > best) { best = a; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const bool neg = Vout[(int64_t)j * rows + bi] < 0.0;
    __syncwarp();
    if (neg)
      for (int r = lane; r < rows; r += 32) Vout[(int64_t)j * rows + r] = -Vout[(int64_t)j * rows + r];
  }
  __syncthreads();
}

struct EigBufs { double *S, *V, *P, *T; };

// mode 0: sym_eig(A)      -> values[k], vectors (k x k)            (smallsolve.py:34-49)
// mode 1: raw jacobi_eig  -> values = diag (unsorted), vectors = V  (_kernels.pyx:105-150)
// mode 2: sym_def_gen_eig(B=A, M=Mm)                                 (smallsolve.py:64-88)
__global__ void __launch_bounds__(ET, 1)
    k_small_eig(int mode, const double* __restrict__ A, const double* __restrict__ Mm, int k, double raw_tol,
                int raw_sweeps, double* __restrict__ values, double* __restrict__ vectors, int* __restrict__ n_out,
                int* __restrict__ status, double* __restrict__ off_out, int* __restrict__ sweeps_out, EigBufs gb,
                int s_in_smem, int v_in_smem) {
  extern __shared__ double dsm[];
  __shared__ EigScratch sc;
  double* S = s_in_smem ? dsm : gb.S;
  double* V = v_in_smem ? (s_in_smem ? dsm + (size_t)k * k : dsm) : gb.V;
  double* P = gb.P;
  double* T = gb.T;
  const int kk2 = k * k;
  if (k == 0) {
    if (threadIdx.x == 0) { if (n_out) *n_out = 0; if (status) *status = mode == 2 ? OFRR_ERR_EMPTY_PENCIL : 0; }
    return;
  }

  if (mode == 1) {
    for (int e = threadIdx.x; e < kk2; e += blockDim.x) S[e] = A[e];
    __syncthreads();
    // raw mode counts sweeps like the reference
    double off = jacobi_parallel(S, V, k, raw_tol, raw_sweeps, sc, sweeps_out);
    __syncthreads();
    for (int i = threadIdx.x; i < k; i += blockDim.x) values[i] = S[(int64_t)i * k + i];
    for (int e = threadIdx.x; e < kk2; e += blockDim.x) vectors[e] = V[e];
    if (threadIdx.x == 0) { if (off_out) *off_out = off; if (status) *status = 0; }
    return;
  }

  // ---- eig of (M + M^T)/2  (mode 2)  or  (A + A^T)/2  (mode 0) ----
  const double* src = mode == 2 ? Mm : A;
  for (int e = threadIdx.x; e < kk2; e += blockDim.x) {
    const int i = e % k, j = e / k;
    S[e] = (src[e] + src[(int64_t)i * k + j]) / 2.0;
  }
  __syncthreads();
  double nrm = fro_norm(S, k, sc.red);
  double tol = 1e-14 * nrm;
  double off = jacobi_parallel(S, V, k, tol, JACOBI_MAX_SWEEPS, sc);
  if (off > tol && nrm > 0.0) {
    if (threadIdx.x == 0) { *status = OFRR_ERR_CONVERGENCE; if (n_out) *n_out = 0; if (off_out) *off_out = off; }
    return;
  }
  // diag -> T[0..k) scratch, sort -> values / P
  for (int i = threadIdx.x; i < k; i += blockDim.x) sc.dis[i] = S[(int64_t)i * k + i];
  __syncthreads();
  if (mode == 0) {
    sorted_desc(sc.dis, V, k, k, values, vectors, sc);
    if (threadIdx.x == 0) { *status = 0; if (n_out) *n_out = k; }
    return;
  }
  sorted_desc(sc.dis, V, k, k, sc.dis, P, sc);   // mu (desc) in sc.dis, P = eigenvectors of M
  const double mu_max = sc.dis[0];
  if (!(mu_max > 0.0)) {
    if (threadIdx.x == 0) { *status = OFRR_ERR_EMPTY_PENCIL; *n_out = 0; }
    return;
  }
  // ofrr/smallsolve.py:79: keep = mu > k * eps * mu_max  (a prefix of the sorted values)
  const double thr = (double)k * 2.220446049250313e-16 * mu_max;
  __shared__ int kp_s;
  if (threadIdx.x == 0) {
    int c = 0;
    while (c < k && sc.dis[c] > thr) ++c;
    kp_s = c;
  }
  __syncthreads();
  const int kp = kp_s;
  if (kp == 0) {
    if (threadIdx.x == 0) { *status = OFRR_ERR_EMPTY_PENCIL; *n_out = 0; }
    return;
  }
  for (int i = threadIdx.x; i < kp; i += blockDim.x) sc.dis[i] = 1.0 / sqrt(sc.dis[i]);
  // Bs = (B + B^T)/2 ; T = Bs * P[:, :kp]   (k x kp)
  for (int e = threadIdx.x; e < k * kp; e += blockDim.x) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    for (int l = 0; l < k; ++l) {
      const double b = (A[(int64_t)l * k + i] + A[(int64_t)i * k + l]) / 2.0;
      s += b * P[(int64_t)j * k + l];
    }
    T[e] = s;
  }
  __syncthreads();
  // S = D^-1/2 P^T (Bs P) D^-1/2  (kp x kp), then symmetrized by sym_eig
  for (int e = threadIdx.x; e < kp * kp; e += blockDim.x) {
    const int i = e % kp, j = e / kp;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += P[(int64_t)i * k + l] * T[(int64_t)j * k + l];
    V[e] = (sc.dis[i] * s) * sc.dis[j];   // V used as scratch here
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kp * kp; e += blockDim.x) {
    const int i = e % kp, j = e / kp;
    S[e] = (V[e] + V[(int64_t)i * kp + j]) / 2.0;
  }
  __syncthreads();
  nrm = fro_norm(S, kp, sc.red);
  tol = 1e-14 * nrm;
  off = jacobi_parallel(S, V, kp, tol, JACOBI_MAX_SWEEPS, sc);
  if (off > tol && nrm > 0.0) {
    if (threadIdx.x == 0) { *status = OFRR_ERR_CONVERGENCE; *n_out = 0; if (off_out) *off_out = off; }
    return;
  }
  __shared__ double tau[MAXK];
  for (int i = threadIdx.x; i < kp; i += blockDim.x) tau[i] = S[(int64_t)i * kp + i];
  __syncthreads();
  sorted_desc(tau, V, kp, kp, tau, T, sc);   // T = Z (kp x kp, ld kp)
  // y = P[:, :kp] (D^-1/2 Z)  (k x kp)  -> S scratch (ld k)
  for (int e = threadIdx.x; e < k * kp; e += blockDim.x) {
    const int i = e % k, j = e / k;
    double s = 0.0;
    for (int l = 0; l < kp; ++l) s += P[(int64_t)l * k + i] * (sc.dis[l] * T[(int64_t)j * kp + l]);
    V[e] = s;
  }
  __syncthreads();
  sorted_desc(tau, V, k, kp, values, vectors, sc);
  if (threadIdx.x == 0) { *status = 0; *n_out = kp; }
}

size_t small_eig_ws(int k) { return (size_t)4 * k * k * sizeof(double) + 1024; }

int small_eig(int mode, const double* A, const double* M, int k, double raw_tol, int raw_sweeps, double* values,
              double* vectors, int* n_out, int* status, double* off_out, int* sweeps_out, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  if (k < 0 || k > MAXK) { ofrr_set_error("small eig: k=%d outside [0, %d]", k, MAXK); return OFRR_ERR_INVALID; }
  if (ws_bytes < small_eig_ws(k)) { ofrr_set_error("small eig: workspace too small"); return OFRR_ERR_INVALID; }
  EigBufs b;
  double* p = (double*)ws;
  b.S = p; b.V = p + (size_t)k * k; b.P = p + (size_t)2 * k * k; b.T = p + (size_t)3 * k * k;
  const size_t one = (size_t)k * k * sizeof(double);
  const size_t budget = 180 * 1024;
  int s_sm = one <= budget ? 1 : 0;
  int v_sm = (s_sm ? 2 * one : one) <= budget ? 1 : 0;
  size_t shm = (s_sm ? one : 0) + (v_sm ? one : 0);
  static bool attr = false;
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_small_eig, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  k_small_eig<<<1, ET, shm, st>>>(mode, A, M, k, raw_tol, raw_sweeps, values, vectors, n_out, status, off_out,
                                  sweeps_out, b, s_sm, v_sm);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
