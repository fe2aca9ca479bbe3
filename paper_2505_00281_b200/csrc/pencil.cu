// pencil.cu -- K5 fast path: the projected pencil B y = lambda M y for k <= 160 as a short
// pipeline of small kernels, one working matrix in shared memory per sequential phase and
// the O(k^3) matrix products spread over the GPU.
//
// Same mathematics as the certified Cholesky branch of small_eig.cu (ofrr/smallsolve.py:
// 64-88 when M is certifiably above the safeguard cutoff):
//   k_pc_chol   M = L L^T (right-looking, one barrier per column), X = L^-1 in place
//               (right-looking forward substitution), certificate 1/||X||_F^2 > 4 k eps ||M||_F
//   k_pc_gemm   T = X sym(B) X^T  (two launches)
//   k_pc_tri    T = Q Tri Q^T (Householder, one CTA): the tridiagonal and the reflectors
//   k_pc_eigvec eigenvalues of Tri by multisection on division-free Sturm sequences,
//               eigenvectors Z of Tri by twisted factorisation, W1 = Q Z by applying the
//               reflectors -- a few eigenpairs per CTA, spread over the GPU
//   k_pc_finish Y = X^T W1, descending order + the largest-|entry|-positive sign rule (smallsolve.py:52-61);
//               numerically coincident eigenvalues raise the gate
// Any failure (Cholesky breakdown, certificate not met, eigenvector breakdown) raises a gate
// flag on the device and the general kernel (small_eig.cu: the reference's eig(M)
// whitening + Jacobi fallback) runs instead; with the gate down it returns at once.
#include "common.cuh"
#include <algorithm>

namespace ofrr {

static constexpr int PT = 512;            // threads of the single-CTA phases
static constexpr int PNW = PT / 32;
static constexpr int PK_MAX = 160;        // one k x (k|1) fp64 matrix in shared memory

__device__ __forceinline__ int pc_ld(int k) { return k | 1; }

__device__ unsigned long long g_pcprof[24];   // debug: phase end times (globaltimer ns | SM clock)
__device__ __forceinline__ void pc_mark(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_pcprof[i] = t;
    if (i < 6) g_pcprof[10 + i] = clock64();
  }
}
int pc_profile(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_pcprof, sizeof(g_pcprof)) == cudaSuccess ? 0 : 2;
}

__device__ double pc_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < PNW; ++w) s += red[w];   // fixed order, every thread
  return s;
}

// ---------------------------------------------------------------------------------
// K5a: Cholesky of sym(M) and X = L^-1 (lower, zeros above), certificate -> gate.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(PT, 1)
    k_pc_chol(const double* __restrict__ M, int k, double* __restrict__ Xg, int* __restrict__ gate) {
  extern __shared__ double sm[];
  __shared__ double red[PNW];
  __shared__ double dg[PK_MAX];
  const int ld = pc_ld(k);
  double* S = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double ss = 0.0;
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) {
      const double v = 0.5 * (M[(size_t)j * k + i] + M[(size_t)i * k + j]);
      S[j * ld + i] = v;
      ss = fma(v, v, ss);
    }
  const double mnorm = sqrt(pc_block_sum(ss, red));   // includes a barrier after the loads
  pc_mark(0);
  // ---- right-looking Cholesky, one barrier per column; column j is scaled at the end ----
  bool fail = !(mnorm > 0.0);
  for (int j = 0; j < k && !fail; ++j) {
    const double d = S[j * ld + j];
    if (!(d > 0.0)) { fail = true; break; }        // uniform: every thread read the same d
    const double inv = 1.0 / d;
    for (int c = j + 1 + warp; c < k; c += PNW) {
      const double lc = S[j * ld + c] * inv;
      for (int i = c + lane; i < k; i += 32) S[c * ld + i] -= S[j * ld + i] * lc;
    }
    __syncthreads();
  }
  if (fail) {
    if (threadIdx.x == 0) *gate = 1;
    return;
  }
  pc_mark(1);
  for (int j = threadIdx.x; j < k; j += PT) dg[j] = sqrt(S[j * ld + j]);
  __syncthreads();
  for (int j = warp; j < k; j += PNW)
    for (int i = j + 1 + lane; i < k; i += 32) S[j * ld + i] /= dg[j];
  __syncthreads();
  // ---- X = L^-1 in place: forward substitution on the identity, right-looking --------
  for (int i = 0; i < k; ++i) {
    const double inv = 1.0 / dg[i];
    for (int c = threadIdx.x; c < i; c += PT) S[c * ld + i] *= inv;   // X[i, c] = R[i, c] / L_ii
    if (threadIdx.x == 0) S[i * ld + i] = inv;
    __syncthreads();
    for (int l = i + 1 + warp; l < k; l += PNW) {
      const double lli = S[i * ld + l];                                 // L[l, i]
      for (int c = lane; c < i; c += 32) S[c * ld + l] -= lli * S[c * ld + i];
      __syncwarp();
      if (lane == 0) S[i * ld + l] = -lli * inv;                        // X[l, i] = -L[l,i] X[i,i]
    }
    __syncthreads();
  }
  pc_mark(2);
  double xs = 0.0;
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) {
      const double v = i >= j ? S[j * ld + i] : 0.0;
      Xg[(size_t)j * k + i] = v;
      xs = fma(v, v, xs);
    }
  const double xn2 = pc_block_sum(xs, red);
  // mu_min(M) >= 1 / ||X||_F^2 must clear the reference's cutoff k eps mu_max (<= ||M||_F)
  const bool cert = (1.0 / xn2) > 4.0 * (double)k * 2.220446049250313e-16 * mnorm;
  if (threadIdx.x == 0) *gate = cert ? 0 : 1;
  pc_mark(3);
}

// ---------------------------------------------------------------------------------
// K5a, blocked (64 < k <= 128): the same Cholesky + inverse + certificate on 32 x 32
// blocks, so that the k-step serial chain becomes kb = ceil(k/32) short ones.
//   diagonal block b: one warp, lane r holding row r in registers -- Cholesky with the
//     column broadcast by shuffles, then its triangular inverse Xd_bb (rows finalised in
//     order, each broadcast to the later lanes);
//   panel and trailing update: L_ib = A_ib Xd_bb^T, A_ij -= L_ib L_jb^T, a warp per block;
//   X = L^-1 by block rows: X_ib = -Xd_ii (sum_{b <= m < i} L_im X_mb), all b at once.
// L and X live as lower block triangles in shared memory (10 + 10 blocks, ld 33); the
// matrix is padded with the identity to 32 kb.  Not bitwise the column-by-column kernel
// (different summation order); the certificate and the gate are the same.
// ---------------------------------------------------------------------------------
constexpr int CB_N = 32, CB_LD = 33, CB_SZ = CB_N * CB_LD, CB_KB = 4;
constexpr size_t CB_SMEM = (size_t)2 * (CB_KB * (CB_KB + 1) / 2) * CB_SZ * sizeof(double);
__device__ __forceinline__ int cb_idx(int i, int j) { return (i * (i + 1) / 2 + j) * CB_SZ; }

__device__ __forceinline__ double pc_fast_div(double a, double b);   // below (MUFU seed + Newton)
constexpr int CB_T = 256, CB_NW = CB_T / 32;   // 255 registers per thread: the diagonal warp's rows
__device__ double cb_block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < CB_NW; ++w) s += red[w];   // fixed order, every thread
  return s;
}

__global__ void __launch_bounds__(CB_T, 1)
    k_pc_chol_blk(const double* __restrict__ M, int k, double* __restrict__ Xg, int* __restrict__ gate) {
  extern __shared__ __align__(16) double sm[];
  double* Lr = sm;                                   // lower block triangle: A, then L
  double* Xr = sm + (size_t)(CB_KB * (CB_KB + 1) / 2) * CB_SZ;   // X = L^-1 (diagonal blocks: Xd)
  __shared__ double red[CB_NW];
  __shared__ double sdg[CB_N], srd[CB_N];
  __shared__ int s_fail;
  // this thread's entries (i, c), c <= i < 32, of a diagonal block: e = i (i + 1) / 2 + c
  int pi[3], pc_[3];
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const int e = threadIdx.x + CB_T * q;
    int i = 0;
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    pi[q] = e < CB_N * (CB_N + 1) / 2 ? i : CB_N;            // CB_N: no entry
    pc_[q] = e < CB_N * (CB_N + 1) / 2 ? e - i * (i + 1) / 2 : CB_N;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kb = (k + CB_N - 1) / CB_N;
  // ---- load sym(M) (lower blocks, identity padding) and ||sym(M)||_F --------------------
  double ss = 0.0;
  for (int e = threadIdx.x; e < k * k; e += CB_T) {
    const int i = e % k, j = e / k;
    const double v = 0.5 * (M[(size_t)j * k + i] + M[(size_t)i * k + j]);
    ss = fma(v, v, ss);
  }
  for (int bi = 0; bi < kb; ++bi)
    for (int bj = 0; bj <= bi; ++bj)
      for (int e = threadIdx.x; e < CB_N * CB_N; e += CB_T) {
        const int r = e & 31, c = e >> 5;
        const int gi = bi * CB_N + r, gj = bj * CB_N + c;
        const double v = (gi < k && gj < k) ? 0.5 * (M[(size_t)gj * k + gi] + M[(size_t)gi * k + gj])
                                            : (gi == gj ? 1.0 : 0.0);
        Lr[cb_idx(bi, bj) + c * CB_LD + r] = v;
      }
  if (threadIdx.x == 0) s_fail = 0;
  const double mnorm = sqrt(cb_block_sum(ss, red));   // includes the barrier after the loads
  pc_mark(0);

  // warp-level block product on lane rows: out[c] (row `lane`) += sum_m A(lane, m) B'(m, c)
  // where B'(m, c) = B(c, m) (BT) or B(m, c); A, B blocks in shared memory (ld 33)
  auto row_gemm = [&](double (&out)[CB_N], const double* A, const double* B, bool bt) {
    if (bt) {
#pragma unroll 2
      for (int m = 0; m < CB_N; ++m) {
        const double am = A[m * CB_LD + lane];
#pragma unroll
        for (int c = 0; c < CB_N; ++c) out[c] = fma(am, B[m * CB_LD + c], out[c]);
      }
    } else {
#pragma unroll 2
      for (int m = 0; m < CB_N; ++m) {
        const double am = A[m * CB_LD + lane];
#pragma unroll
        for (int c = 0; c < CB_N; ++c) out[c] = fma(am, B[c * CB_LD + m], out[c]);
      }
    }
  };
  for (int b = 0; b < kb; ++b) {
    // ---- diagonal block: Cholesky + triangular inverse by the whole CTA, thread per
    // lower-triangle entry (up to 3 of the 528); one barrier per step -------------------
    {
      double* Ab = Lr + cb_idx(b, b);
      double* Xb = Xr + cb_idx(b, b);
      // right-looking, columns scaled at the end: A[i][c] -= A[i][j] A[c][j] / A[j][j]
      for (int j = 0; j < CB_N; ++j) {
        const double d = Ab[j * CB_LD + j];
        if (!(d > 0.0)) { if (threadIdx.x == 0) s_fail = 1; break; }   // uniform: same d everywhere
        const double inv = pc_fast_div(1.0, d);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int i = pi[q], c = pc_[q];
          if (c > j) Ab[c * CB_LD + i] -= Ab[j * CB_LD + i] * (Ab[j * CB_LD + c] * inv);
        }
        __syncthreads();
      }
      if (!s_fail) {
        // L[i][j] = A[i][j] / sqrt(A[j][j]); X = L^-1 right-looking: row p final at step p
        // (X[p][c] = (delta_pc - acc[p][c]) / L[p][p]), then acc[i][c] += L[i][p] X[p][c]
        if (threadIdx.x < CB_N) {
          const double dg = sqrt(Ab[threadIdx.x * CB_LD + threadIdx.x]);
          sdg[threadIdx.x] = dg;
          srd[threadIdx.x] = 1.0 / dg;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          const int i = pi[q], c = pc_[q];
          if (i < CB_N) {
            Ab[c * CB_LD + i] = i == c ? sdg[i] : Ab[c * CB_LD + i] * srd[c];
            Xb[c * CB_LD + i] = 0.0;
          }
        }
        __syncthreads();
        for (int pp = 0; pp < CB_N; ++pp) {
#pragma unroll
          for (int q = 0; q < 3; ++q)
            if (pi[q] == pp) Xb[pc_[q] * CB_LD + pp] = ((pc_[q] == pp ? 1.0 : 0.0) - Xb[pc_[q] * CB_LD + pp]) * srd[pp];
          __syncthreads();
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int i = pi[q], c = pc_[q];
            if (i > pp && c <= pp && i < CB_N) Xb[c * CB_LD + i] += Ab[pp * CB_LD + i] * Xb[c * CB_LD + pp];
          }
          __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {                          // zeros above the diagonal
          const int i = pi[q], c = pc_[q];
          if (i < CB_N && i != c) { Ab[i * CB_LD + c] = 0.0; Xb[i * CB_LD + c] = 0.0; }
        }
      }
    }
    __syncthreads();
    if (b == 0) pc_mark(20);
    if (s_fail) break;                                         // uniform
    // ---- panel: L_ib = A_ib Xd_bb^T (each lane rewrites only its own row) --------------
    for (int i = b + 1 + warp; i < kb; i += CB_NW) {
      double out[CB_N];
#pragma unroll
      for (int c = 0; c < CB_N; ++c) out[c] = 0.0;
      double* Ai = Lr + cb_idx(i, b);
      row_gemm(out, Ai, Xr + cb_idx(b, b), true);              // Xd^T(m, c) = Xd(c, m)
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CB_N; ++c) Ai[c * CB_LD + lane] = out[c];
    }
    __syncthreads();
    if (b == 0) pc_mark(21);
    // ---- trailing: A_ij -= L_ib L_jb^T, b < j <= i ------------------------------------
    {
      int pidx = 0;
      for (int i = b + 1; i < kb; ++i)
        for (int j = b + 1; j <= i; ++j, ++pidx) {
          if (pidx % CB_NW != warp) continue;
          double out[CB_N];
          double* Aij = Lr + cb_idx(i, j);
#pragma unroll
          for (int c = 0; c < CB_N; ++c) out[c] = 0.0;
          row_gemm(out, Lr + cb_idx(i, b), Lr + cb_idx(j, b), true);    // L_jb^T(m, c) = L_jb(c, m)
#pragma unroll
          for (int c = 0; c < CB_N; ++c) Aij[c * CB_LD + lane] -= out[c];
        }
    }
    __syncthreads();
  }
  if (s_fail) {
    if (threadIdx.x == 0) *gate = 1;
    return;
  }
  pc_mark(1);
  // ---- X = L^-1 below the diagonal blocks: block row i after block rows < i -------------
  for (int i = 1; i < kb; ++i) {
    for (int b = warp; b < i; b += CB_NW) {
      double t[CB_N];
#pragma unroll
      for (int c = 0; c < CB_N; ++c) t[c] = 0.0;
      for (int m = b; m < i; ++m) row_gemm(t, Lr + cb_idx(i, m), Xr + cb_idx(m, b), false);  // X_mb(m', c)
      double* Xib = Xr + cb_idx(i, b);
#pragma unroll
      for (int c = 0; c < CB_N; ++c) Xib[c * CB_LD + lane] = t[c];          // scratch: T
      __syncwarp();
      double o[CB_N];
#pragma unroll
      for (int c = 0; c < CB_N; ++c) o[c] = 0.0;
      row_gemm(o, Xr + cb_idx(i, i), Xib, false);                            // Xd_ii T
      __syncwarp();
#pragma unroll
      for (int c = 0; c < CB_N; ++c) Xib[c * CB_LD + lane] = -o[c];
    }
    __syncthreads();
  }
  pc_mark(2);
  double xs = 0.0;
  for (int e = threadIdx.x; e < k * k; e += CB_T) {
    const int i = e % k, j = e / k;
    const int bi = i >> 5, bj = j >> 5;
    const double v = i >= j ? Xr[cb_idx(bi, bj) + (j & 31) * CB_LD + (i & 31)] : 0.0;
    Xg[(size_t)j * k + i] = v;
    xs = fma(v, v, xs);
  }
  const double xn2 = cb_block_sum(xs, red);
  // mu_min(M) >= 1 / ||X||_F^2 must clear the reference's cutoff k eps mu_max (<= ||M||_F)
  const bool cert = (1.0 / xn2) > 4.0 * (double)k * 2.220446049250313e-16 * mnorm;
  if (threadIdx.x == 0) *gate = cert ? 0 : 1;
  pc_mark(3);
}

// ---------------------------------------------------------------------------------
// C = op(A) op(B) for k x k column-major operands (ld k); SYMB: B := (B + B^T) / 2.
// 32 x 32 output tile per CTA, 256 threads x 2 x 2 outputs.
// ---------------------------------------------------------------------------------
template <bool TA, bool TB, bool SYMB>
__global__ void __launch_bounds__(256)
    k_pc_gemm(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C, int k,
              const int* __restrict__ gate) {
  if (*gate) return;
  __shared__ double As[32][33], Bs[32][33];
  const int bi = blockIdx.x * 32, bj = blockIdx.y * 32;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int l0 = 0; l0 < k; l0 += 32) {
    for (int e = threadIdx.x; e < 1024; e += 256) {
      const int a = e & 31, b = e >> 5;
      // As[l][i] = op(A)[bi + i, l0 + l]; Bs[l][j] = op(B)[l0 + l, bj + j]
      {
        const int i = bi + a, l = l0 + b;
        As[b][a] = (i < k && l < k) ? (TA ? A[(size_t)i * k + l] : A[(size_t)l * k + i]) : 0.0;
      }
      {
        const int l = l0 + a, j = bj + b;
        double v = 0.0;
        if (l < k && j < k) {
          if (SYMB) v = 0.5 * (B[(size_t)j * k + l] + B[(size_t)l * k + j]);
          else v = TB ? B[(size_t)l * k + j] : B[(size_t)j * k + l];
        }
        Bs[a][b] = v;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      const double a0 = As[l][2 * ty], a1 = As[l][2 * ty + 1];
      const double b0 = Bs[l][2 * tx], b1 = Bs[l][2 * tx + 1];
      acc[0][0] = fma(a0, b0, acc[0][0]);
      acc[0][1] = fma(a0, b1, acc[0][1]);
      acc[1][0] = fma(a1, b0, acc[1][0]);
      acc[1][1] = fma(a1, b1, acc[1][1]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int i = bi + 2 * ty + p, j = bj + 2 * tx + q;
      if (i < k && j < k) C[(size_t)j * k + i] = acc[p][q];
    }
}

// division-free Sturm count (number of eigenvalues of the scaled tridiagonal below x):
// sign changes of the leading principal minors p_i (three-term recurrence), rescaled by a
// power of two after every 8 steps (exponent read from the bits: ilogb is a slow library
// path on the recurrence's critical chain).  The product e2 * p_{i-1} and d_i - x are off
// the dependency chain (one fma per step on it); signs are compared on the raw bits.
__device__ __forceinline__ int pc_sturm(const double* __restrict__ d, const double* __restrict__ e2, int k, double x) {
  double p0 = 1.0, p1 = d[0] - x;
  int cnt = (int)((unsigned)__double2hiint(p1) >> 31);
  int i = 1;
  for (; i + 8 <= k; i += 8) {
    double dx[8], ee[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { dx[u] = d[i + u] - x; ee[u] = e2[i + u - 1]; }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double p2 = fma(dx[u], p1, -ee[u] * p0);
      cnt += (int)((unsigned)(__double2hiint(p2) ^ __double2hiint(p1)) >> 31);
      p0 = p1;
      p1 = p2;
    }
    const int ex = ((__double2hiint(p1) >> 20) & 0x7ff) - 1023;      // biased exponent of p1
    if (ex > 256 || ex < -256) {                                      // (zero/denormal: ex = -1023)
      const int e = ex < -1000 ? 0 : ex;
      const double sc = __hiloint2double((1023 - e) << 20, 0);        // 2^-e, exact
      p0 *= sc;
      p1 *= sc;
    }
  }
  for (; i < k; ++i) {
    const double p2 = fma(d[i] - x, p1, -e2[i - 1] * p0);
    cnt += (int)((unsigned)(__double2hiint(p2) ^ __double2hiint(p1)) >> 31);
    p0 = p1;
    p1 = p2;
  }
  return cnt;
}

__device__ __forceinline__ double pc_fast_div(double a, double b) {
  // a / b to ~1 ulp: MUFU fp64 reciprocal seed and two Newton steps (finite, normal b);
  // a third of the latency of the IEEE division sequence
  const double ab = fabs(b);
  if (ab > 1e-300 && ab < 1e300) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
    r = fma(r, fma(-b, r, 1.0), r);
    r = fma(r, fma(-b, r, 1.0), r);
    return a * r;
  }
  return a / b;
}

// ---------------------------------------------------------------------------------
// K5c: eigen-decomposition of sym(T): lam (ascending), Z (eigenvectors of the tridiagonal,
// column c <-> lam[k-1-c], i.e. descending), Q (k x k) with T = Q Tri Q^T.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(PT, 1)
    k_pc_tri(const double* __restrict__ Tg, int k, double* __restrict__ tri, double* __restrict__ Rg,
             int* __restrict__ gate) {
  if (*gate) return;
  extern __shared__ double sm[];
  __shared__ double red[PNW];
  __shared__ double dd[PK_MAX], ee[PK_MAX], tau[PK_MAX];
  __shared__ double pv[PK_MAX];
  const int ld = pc_ld(k);
  double* S = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) S[j * ld + i] = 0.5 * (Tg[(size_t)j * k + i] + Tg[(size_t)i * k + j]);
  __syncthreads();
  pc_mark(4);
  // ---- 1. Householder tridiagonalisation (reflector j stored in column j, rows > j) ----
  // Group-per-column layout: the CTA is split into groups of tpc adjacent lanes, group g
  // owning column g of S (tpc = 8 / 4 / 2 for k <= 64 / 128 / 160, one column per group).
  // Step j: every group forms p_c = tau S[:, c] . u over its rows (tpc partial sums, an
  // in-group shuffle tree), the leaders fold u_c p_c into a per-warp partial; barrier (A);
  // K = tau/2 u.p in fixed order, then the group applies the rank-2 update to its own
  // column and the group of column j+1 forms the next reflector at once; barrier (B).
  const int tpc = k <= 64 ? 8 : (k <= 128 ? 4 : 2);
  const int grp = threadIdx.x / tpc, sub = threadIdx.x % tpc;
  const unsigned gmask = (tpc == 32 ? 0xffffffffu : (((1u << tpc) - 1u) << (lane & ~(tpc - 1))));
  // the reflector scalars of the next column: formed by the group that owns that column
  __shared__ double s_alpha, s_tau, s_u0, s_x0;
  auto group_sum = [&](double v) {
    for (int o = tpc >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
  };
  auto reflector = [&](int j, double norm2) {                          // group j+1... leader
    const double x0 = S[j * ld + j + 1];
    const double alpha = -copysign(sqrt(norm2), x0);
    const double unorm2 = 2.0 * (norm2 - x0 * alpha);
    const bool skip = !(unorm2 > 0.0) || norm2 == 0.0;
    s_x0 = x0;
    s_alpha = alpha;
    s_tau = skip ? 0.0 : 2.0 / unorm2;
    s_u0 = x0 - alpha;
  };
  if (k > 2 && grp == 0) {
    double s2 = 0.0;
    for (int i = 1 + sub; i < k; i += tpc) s2 = fma(S[i], S[i], s2);
    s2 = group_sum(s2);
    if (sub == 0) reflector(0, s2);
  }
  __syncthreads();
  for (int j = 0; j + 2 < k; ++j) {
    const double tj = s_tau, u0 = s_u0, x0 = s_x0, alpha = s_alpha;
    const bool skip = tj == 0.0;
    const int j1 = j + 1;
    const int c = grp;
    const bool own = c >= j1 && c < k;
    const double* uj = S + j * ld;                                     // u_i = uj[i] (i > j1), u0 at j1
    double pc = 0.0;
    if (!skip) {
      if (own) {
        const double* col = S + c * ld;
        double a0 = 0.0, a1 = 0.0;
        int i = j1 + sub;
        for (; i + tpc < k; i += 2 * tpc) {
          a0 = fma(col[i], i == j1 ? u0 : uj[i], a0);
          a1 = fma(col[i + tpc], uj[i + tpc], a1);
        }
        if (i < k) a0 = fma(col[i], i == j1 ? u0 : uj[i], a0);
        pc = tj * group_sum(a0 + a1);
        if (sub == 0) pv[c] = pc;
      }
      double kp = (own && sub == 0) ? (c == j1 ? u0 : uj[c]) * pc : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kp += __shfl_xor_sync(0xffffffffu, kp, o);
      if (lane == 0) red[warp] = kp;
    }
    if (threadIdx.x == 0) {
      dd[j] = S[j * ld + j];
      ee[j] = skip ? x0 : alpha;
      tau[j] = tj;
    }
    __syncthreads();                                                     // (A)
    if (!skip && own) {
      double ks = 0.0;
      for (int w = 0; w < PNW; ++w) ks += red[w];                        // fixed order
      const double K = 0.5 * tj * ks;
      const double uc = c == j1 ? u0 : uj[c];
      const double qc = pc - K * uc;
      double* col = S + c * ld;
      for (int i = j1 + sub; i < k; i += tpc) {
        const double ui = i == j1 ? u0 : uj[i];
        const double qi = pv[i] - K * ui;
        col[i] = col[i] - (ui * qc + qi * uc);
      }
    }
    if (c == j1 && j1 + 2 < k) {                                         // next column's reflector
      __syncwarp(gmask);
      double s2 = 0.0;
      for (int i = j1 + 1 + sub; i < k; i += tpc) s2 = fma(S[j1 * ld + i], S[j1 * ld + i], s2);
      s2 = group_sum(s2);
      if (sub == 0) reflector(j1, s2);
    }
    if (threadIdx.x == 0 && !skip) S[j * ld + j1] = u0;                 // reflector in place
    __syncthreads();                                                     // (B)
  }
  if (threadIdx.x == 0) {
    if (k >= 2) {
      dd[k - 2] = S[(k - 2) * ld + k - 2];
      ee[k - 2] = S[(k - 2) * ld + k - 1];
      tau[k - 2] = 0.0;
    }
    dd[k - 1] = S[(k - 1) * ld + k - 1];
    ee[k - 1] = 0.0;
    tau[k - 1] = 0.0;
  }
  __syncthreads();
  pc_mark(5);
  // tridiagonal (d, e, tau) and the reflectors (column j, rows > j) to global for K5d
  for (int i = threadIdx.x; i < k; i += PT) {
    tri[i] = dd[i];
    tri[k + i] = ee[i];
    tri[2 * k + i] = tau[i];
  }
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) Rg[(size_t)j * k + i] = i > j ? S[j * ld + i] : 0.0;
}

// ---------------------------------------------------------------------------------
// K5c for k <= 128: the same Householder tridiagonalisation with the matrix held in
// registers (shared memory bandwidth bounds the in-smem version: every step re-reads and
// re-writes the trailing matrix in fp64).  Group g of TPC adjacent lanes owns column g;
// lane `sub` of the group holds the contiguous rows sub*RPT + t (t < RPT).  The step's
// vectors (reflector u, p = tau S u) live in shared memory padded by two doubles per RPT
// rows, so the TPC lanes of a group read them as conflict-free 16-byte vectors.
// Step j: every group forms p_c from its registers, the leaders fold u_c p_c per warp;
// barrier (A); K (a 16-term tree), the rank-2 update in registers as two fmas per entry
// (S -= u (q_c - K u_c) + p u_c), the group of column j+1 accumulating the norm of its
// new column on the way and forming the next reflector at once; barrier (B).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double pc_sum8(const double* r) {
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double v[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) { const double2 x = r2[w]; v[w] = x.x + x.y; }
  return (v[0] + v[1]) + (v[2] + v[3]);
}
__device__ __forceinline__ double pc_sum16(const double* r) {
  const double2* r2 = reinterpret_cast<const double2*>(r);
  double v[8];
#pragma unroll
  for (int w = 0; w < 8; ++w) { const double2 x = r2[w]; v[w] = x.x + x.y; }
  return ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
}

template <int TPC, int RPT, int NT = PT>
__global__ void __launch_bounds__(NT, 1)
    k_pc_tri_reg(const double* __restrict__ Tg, int k, double* __restrict__ tri, double* __restrict__ Rg,
                 int* __restrict__ gate) {
  if (*gate) return;
  constexpr int NW = NT / 32;
  static_assert(NW == 16 || NW == 8, "16 or 8 warp partials");
  constexpr int RP = RPT + 2;                                     // padded chunk
  __shared__ __align__(16) double red[2][NW];
  __shared__ __align__(16) double uv[2][TPC * RP];               // reflector of the step, by parity
  __shared__ __align__(16) double pv[TPC * RP];
  __shared__ double dd[PK_MAX], ee[PK_MAX], tau[PK_MAX];
  __shared__ double s_tau[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = threadIdx.x / TPC, sub = threadIdx.x % TPC;      // my column, my lane in the group
  const unsigned gmask = (TPC == 32 ? 0xffffffffu : (((1u << TPC) - 1u) << (lane & ~(TPC - 1))));
  const int gl0 = lane & ~(TPC - 1);                              // lane of the group's sub 0
  const int r0 = sub * RPT;                                       // my first row
  const bool colok = c < k;
  auto pidx = [](int i) { return i + 2 * (i / RPT); };            // padded index of row i
  double a[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = r0 + t;
    a[t] = (colok && i < k) ? 0.5 * (Tg[(size_t)c * k + i] + Tg[(size_t)i * k + c]) : 0.0;
  }
  for (int i = threadIdx.x; i < TPC * RP; i += NT) {            // rows >= k stay zero
    pv[i] = 0.0;
    uv[0][i] = 0.0;
    uv[1][i] = 0.0;
  }
  __syncthreads();
  auto group_sum = [&](double v) {
#pragma unroll
    for (int o = TPC >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
  };
  // group of column j (after its update): reflector from rows > j -> uv[buf], tau, d_j, e_j.
  // s2 = this lane's sum of squares over rows > j + 1.
  auto make_reflector = [&](int j, int buf, double s2) {
    double x0 = 0.0, djj = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      if (r0 + t == j + 1) x0 = a[t];
      if (r0 + t == j) djj = a[t];
    }
    s2 = group_sum(s2);
    x0 = __shfl_sync(gmask, x0, gl0 + (j + 1) / RPT);
    djj = __shfl_sync(gmask, djj, gl0 + j / RPT);
    const double norm2 = fma(x0, x0, s2);
    const double alpha = -copysign(sqrt(norm2), x0);
    const double unorm2 = 2.0 * (norm2 - x0 * alpha);
    const bool skip = !(unorm2 > 0.0) || norm2 == 0.0;
    const double u0 = x0 - alpha;
    double* ub = uv[buf] + sub * RP;
#pragma unroll
    for (int t = 0; t < RPT; t += 2) {
      const int i = r0 + t;
      double2 w;
      w.x = i > j + 1 ? a[t] : (i == j + 1 ? u0 : 0.0);
      w.y = i + 1 > j + 1 ? a[t + 1] : (i + 1 == j + 1 ? u0 : 0.0);
      *reinterpret_cast<double2*>(ub + t) = w;
      if (i < k) Rg[(size_t)j * k + i] = w.x;                       // reflector j for K5d
      if (i + 1 < k) Rg[(size_t)j * k + i + 1] = w.y;
    }
    if (sub == 0) {
      const double tj = skip ? 0.0 : pc_fast_div(2.0, unorm2);
      s_tau[buf] = tj;
      tau[j] = tj;
      dd[j] = djj;
      ee[j] = skip ? x0 : alpha;
    }
  };
  pc_mark(4);
  if (k > 2 && c == 0) {
    double s2 = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; ++t)
      if (r0 + t > 1 && r0 + t < k) s2 = fma(a[t], a[t], s2);
    make_reflector(0, 0, s2);
  }
  __syncthreads();
#ifdef OFRR_PC_TRI_PROF
  __shared__ unsigned long long s_prof[4];
  if (threadIdx.x < 4) s_prof[threadIdx.x] = 0;
  unsigned long long tp_b = clock64(), tp_a = 0;
#endif
  for (int j = 0; j + 2 < k; ++j) {
    const int buf = j & 1, j1 = j + 1;
    const double tj = s_tau[buf];
    const bool skip = tj == 0.0;
    const bool own = colok && c >= j1;
    const double* ub = uv[buf] + sub * RP;
    double pc = 0.0, uc = 0.0;
    if (!skip) {
      if (own) {
        double s0 = 0.0, s1 = 0.0;                              // u is zero at rows <= j
#pragma unroll
        for (int t = 0; t < RPT; t += 2) {
          const double2 w = *reinterpret_cast<const double2*>(ub + t);
          s0 = fma(a[t], w.x, s0);
          s1 = fma(a[t + 1], w.y, s1);
        }
        pc = tj * group_sum(s0 + s1);
        uc = uv[buf][pidx(c)];
        if (sub == 0) pv[pidx(c)] = pc;
      }
      double kp = (own && sub == 0) ? uc * pc : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kp += __shfl_xor_sync(0xffffffffu, kp, o);
      if (lane == 0) red[buf][warp] = kp;
    }
    __syncthreads();                                                     // (A)
#ifdef OFRR_PC_TRI_PROF
    tp_a = clock64();
    if (threadIdx.x == 0) s_prof[0] += tp_a - tp_b;
#endif
    double s2 = 0.0;                                                     // column j+1's new norm
    if (!skip && own) {
      const double K = 0.5 * tj * (NW == 16 ? pc_sum16(red[buf]) : pc_sum8(red[buf]));
      const double qc = fma(-K, uc, pc) - K * uc;                        // q_c - K u_c
      const double* pb = pv + sub * RP;
#pragma unroll
      for (int t = 0; t < RPT; t += 2) {
        const int i = r0 + t;
        const double2 w = *reinterpret_cast<const double2*>(ub + t);
        const double2 q = *reinterpret_cast<const double2*>(pb + t);
        if (i >= j1) a[t] = fma(-q.x, uc, fma(-w.x, qc, a[t]));
        if (i + 1 >= j1) a[t + 1] = fma(-q.y, uc, fma(-w.y, qc, a[t + 1]));
        if (i > j1 + 1) s2 = fma(a[t], a[t], s2);
        if (i + 1 > j1 + 1) s2 = fma(a[t + 1], a[t + 1], s2);
      }
    } else if (c == j1) {
#pragma unroll
      for (int t = 0; t < RPT; ++t)
        if (r0 + t > j1 + 1) s2 = fma(a[t], a[t], s2);
    }
#ifdef OFRR_PC_TRI_PROF
    const unsigned long long tp_m = clock64();
#endif
    if (c == j1) {
      if (j1 + 2 < k) {
        make_reflector(j1, buf ^ 1, s2);
#ifdef OFRR_PC_TRI_PROF
        if (sub == 0) { s_prof[2] += tp_m - tp_a; s_prof[3] += clock64() - tp_m; }
#endif
      } else if (sub == 0) {                                             // last two: no reflector
        s_tau[buf ^ 1] = 0.0;
      }
    }
    __syncthreads();                                                     // (B)
#ifdef OFRR_PC_TRI_PROF
    tp_b = clock64();
    if (threadIdx.x == 0) s_prof[1] += tp_b - tp_a;
#endif
  }
#ifdef OFRR_PC_TRI_PROF
  if (threadIdx.x < 4) g_pcprof[16 + threadIdx.x] = s_prof[threadIdx.x];
#endif
  // d_{k-2}, e_{k-2}, d_{k-1} from the owners' registers
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = r0 + t;
    if (k >= 2 && c == k - 2 && i == k - 2) dd[k - 2] = a[t];
    if (k >= 2 && c == k - 2 && i == k - 1) ee[k - 2] = a[t];
    if (c == k - 1 && i == k - 1) dd[k - 1] = a[t];
  }
  if (threadIdx.x == 0) {
    if (k >= 2) tau[k - 2] = 0.0;
    ee[k - 1] = 0.0;
    tau[k - 1] = 0.0;
  }
  __syncthreads();
  pc_mark(5);
  for (int i = threadIdx.x; i < k; i += NT) {
    tri[i] = dd[i];
    tri[k + i] = ee[i];
    tri[2 * k + i] = tau[i];
  }
}

// ---------------------------------------------------------------------------------
// K5a for k <= 64: the same Cholesky + inverse + certificate with sym(M) in registers
// (group-per-column layout of k_pc_tri_reg).  Step j: the group of column j forms
// l = column j / sqrt(m_jj) from its registers and publishes it (shared memory, double
// buffered); barrier; every later column takes the rank-1 update in registers, and every
// column c <= j takes step j of its forward substitution L x = e_c with the same published
// column (x_j broadcast by shuffle from the lane holding row j) -- so X = L^-1 is done when
// L is, in the operation order of the column-by-column solve.
// ---------------------------------------------------------------------------------
template <int TPC, int RPT>
__global__ void __launch_bounds__(PT, 1)
    k_pc_chol_reg(const double* __restrict__ M, int k, double* __restrict__ Xg, int* __restrict__ gate,
                  const double* __restrict__ B, double* __restrict__ Tg) {
  constexpr int RP = RPT + 2;
  extern __shared__ double sm[];                                 // L, k x k column-major (ld k); then X
  double* sm2 = sm + (size_t)k * k;                              // sym(B), then G = sym(B) X^T
  __shared__ __align__(16) double lv[2][TPC * RP];
  __shared__ double red[PNW];
  __shared__ double dinv[PK_MAX];
  __shared__ int s_fail;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = threadIdx.x / TPC, sub = threadIdx.x % TPC;
  const unsigned gmask = (TPC == 32 ? 0xffffffffu : (((1u << TPC) - 1u) << (lane & ~(TPC - 1))));
  const int gl0 = lane & ~(TPC - 1);
  const int r0 = sub * RPT;
  const bool colok = c < k;
  double a[RPT];
  double ss = 0.0;
#pragma unroll
  for (int t = 0; t < RPT; ++t) {
    const int i = r0 + t;
    a[t] = (colok && i < k) ? 0.5 * (M[(size_t)c * k + i] + M[(size_t)i * k + c]) : 0.0;
    ss = fma(a[t], a[t], ss);
  }
  if (threadIdx.x == 0) s_fail = 0;
  const double mnorm = sqrt(pc_block_sum(ss, red));             // includes barriers
  pc_mark(0);
  auto group_sum = [&](double v) {
#pragma unroll
    for (int o = TPC >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(gmask, v, o);
    return v;
  };
  // group j: publish l = L[:, j] (rows >= j) to lv[buf], 1 / L_jj to dinv[j]
  auto publish = [&](int j, int buf) {
    double d = 0.0;
#pragma unroll
    for (int t = 0; t < RPT; ++t)
      if (r0 + t == j) d = a[t];
    d = __shfl_sync(gmask, d, gl0 + j / RPT);
    const bool bad = !(d > 0.0);
    const double lj = bad ? 1.0 : sqrt(d);
    const double il = pc_fast_div(1.0, lj);
    double* lb = lv[buf] + sub * RP;
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = r0 + t;
      const double l = i > j ? a[t] * il : (i == j ? lj : 0.0);
      a[t] = l;                                                  // my column now holds L[:, j]
      lb[t] = l;
    }
    if (sub == 0) {
      dinv[j] = il;
      if (bad) s_fail = 1;
    }
  };
  // X = L^-1 alongside: column c of X in registers (x = e_c); step j applies row j of the
  // column solve (x_j *= 1/L_jj, x_i -= L_ij x_j below) with the published column j -- the
  // operation order of a column-by-column forward substitution, without its k serial steps
  double x[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) x[t] = (r0 + t == c) ? 1.0 : 0.0;
  if (c == 0) publish(0, 0);
  __syncthreads();
  for (int j = 0; j + 1 < k; ++j) {
    const int buf = j & 1;
    if (s_fail) break;                                           // uniform (read after a barrier)
    const double* lb = lv[buf] + sub * RP;
    if (colok && c > j) {
      const double lc = lv[buf][c + 2 * (c / RPT)];
#pragma unroll
      for (int t = 0; t < RPT; t += 2) {
        const double2 w = *reinterpret_cast<const double2*>(lb + t);
        a[t] = fma(-w.x, lc, a[t]);
        a[t + 1] = fma(-w.y, lc, a[t + 1]);
      }
    }
    if (c == j + 1) publish(j + 1, buf ^ 1);
    if (colok && c <= j) {                                       // x_j = 0 for columns past j
      const double dj = dinv[j];
      double xj = 0.0;
#pragma unroll
      for (int t = 0; t < RPT; ++t)
        if (r0 + t == j) { x[t] *= dj; xj = x[t]; }
      xj = __shfl_sync(gmask, xj, gl0 + j / RPT);
#pragma unroll
      for (int t = 0; t < RPT; ++t)
        if (r0 + t > j) x[t] = fma(-lb[t], xj, x[t]);
    }
    __syncthreads();
  }
  if (s_fail) {
    if (threadIdx.x == 0) *gate = 1;
    return;
  }
  pc_mark(1);
  double xs = 0.0;
  if (colok) {
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = r0 + t;
      if (i == k - 1) x[t] *= dinv[k - 1];
      a[t] = x[t];
      if (i < k) {
        const double v = i >= c ? x[t] : 0.0;
        Xg[(size_t)c * k + i] = v;
        xs = fma(v, v, xs);
      }
    }
  }
  pc_mark(2);
  const double xn2 = pc_block_sum(xs, red);                      // (barriers: L is dead after)
  // mu_min(M) >= 1 / ||X||_F^2 must clear the reference's cutoff k eps mu_max (<= ||M||_F)
  const bool cert = (1.0 / xn2) > 4.0 * (double)k * 2.220446049250313e-16 * mnorm;
  if (threadIdx.x == 0) *gate = cert ? 0 : 1;
  pc_mark(3);
  if (!Tg || !cert) return;
  // T = X sym(B) X^T here (no GEMM launches): X -> shared (column c from my registers),
  // sym(B) -> shared; G[:, c] = sym(B) X[c, :]^T in registers, G -> shared, T[:, c] = X G[:, c]
  if (colok) {
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = r0 + t;
      if (i < k) sm[(size_t)c * k + i] = i >= c ? a[t] : 0.0;
    }
  }
  for (int e = threadIdx.x; e < k * k; e += PT) {
    const int i = e % k, j = e / k;
    sm2[e] = 0.5 * (B[(size_t)j * k + i] + B[(size_t)i * k + j]);
  }
  __syncthreads();
  double g[RPT];
#pragma unroll
  for (int t = 0; t < RPT; ++t) g[t] = 0.0;
  if (colok) {
    for (int l = 0; l <= c; ++l) {                               // X[c, l] = 0 for l > c
      const double xcl = sm[(size_t)l * k + c];
      const double* bl = sm2 + (size_t)l * k;                    // sym(B)[:, l] = sym(B)[l, :]
#pragma unroll
      for (int t = 0; t < RPT; ++t)
        if (r0 + t < k) g[t] = fma(bl[r0 + t], xcl, g[t]);
    }
  }
  __syncthreads();
  if (colok) {
#pragma unroll
    for (int t = 0; t < RPT; ++t)
      if (r0 + t < k) sm2[(size_t)c * k + r0 + t] = g[t];
  }
  __syncthreads();
  if (colok) {
    const double* gc = sm2 + (size_t)c * k;
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int i = r0 + t;
      if (i >= k) continue;
      double acc = 0.0;
      for (int l = 0; l <= i; ++l) acc = fma(sm[(size_t)l * k + i], gc[l], acc);   // X[i, l], l <= i
      Tg[(size_t)c * k + i] = acc;
    }
  }
}

// ---------------------------------------------------------------------------------
// K5d: eigenpairs of the tridiagonal and their back-transformation, EPB eigenvalues per
// CTA (ascending index m), spread over the GPU:
//   multisection on division-free Sturm counts, one warp per eigenvalue (32 points per
//     round: the interval shrinks 33x), on the power-of-two scaled tridiagonal;
//   twisted factorisation, two lanes per eigenvalue (D+ and D- in parallel, shared memory);
//   W1[:, k-1-m] = Q z_m = H_0 ... H_{k-3} z_m, one warp per eigenvector, the reflectors
//     staged in shared memory by cp.async while the multisection runs.
// Numerically coincident eigenvalues are left to k_pc_finish, which raises the gate (the
// general kernel then runs); a failed eigenvector raises it here.
// ---------------------------------------------------------------------------------
static constexpr int EPT = 256;                       // threads of K5d (8 warps)
__host__ __device__ constexpr int pc_epb(int k) { return k <= 128 ? 8 : 4; }

__global__ void __launch_bounds__(EPT)
    k_pc_eigvec(const double* __restrict__ tri, const double* __restrict__ Rg, int k, double* __restrict__ lam_g,
                double* __restrict__ W1, double* __restrict__ tnrm_g, int* __restrict__ gate) {
  if (*gate) return;
  extern __shared__ double sm[];
  __shared__ double dd[PK_MAX], ee[PK_MAX], tau[PK_MAX], e2[PK_MAX], ds[PK_MAX], e2s[PK_MAX];
  __shared__ double lam[8];
  __shared__ double s_lo, s_hi;
  const int epb = pc_epb(k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* R = sm;                                        // k x k reflectors (ld k)
  double* zb = sm + (size_t)k * k;                       // [epb][k]: D+ then z
  double* dm = zb + (size_t)epb * k;                     // [epb][k]: D-
  const int m0 = blockIdx.x * epb;
  // reflectors -> shared memory, asynchronously (needed only by the back-transformation)
  {
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(R);
    const int nel = k * k;
    for (int e = threadIdx.x; e < nel; e += EPT)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sbase + 8u * (unsigned)e), "l"(Rg + e) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int i = threadIdx.x; i < k; i += EPT) {
    dd[i] = tri[i];
    ee[i] = tri[k + i];
    tau[i] = tri[2 * k + i];
  }
  __syncthreads();
  // Gershgorin bounds (fixed order, warp 0)
  if (warp == 0) {
    double lo = 1e300, hi = -1e300;
    for (int i = lane; i < k; i += 32) {
      const double r = (i > 0 ? fabs(ee[i - 1]) : 0.0) + (i + 1 < k ? fabs(ee[i]) : 0.0);
      lo = fmin(lo, dd[i] - r);
      hi = fmax(hi, dd[i] + r);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) { s_lo = lo; s_hi = hi; }
  }
  __syncthreads();
  const double glo = s_lo, ghi = s_hi;
  const double tnrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
  if (blockIdx.x == 0 && threadIdx.x == 0) *tnrm_g = tnrm;
  const int sx = ilogb(tnrm);
  for (int i = threadIdx.x; i < k; i += EPT) {
    ds[i] = ldexp(dd[i], -sx);
    const double es = ldexp(ee[i], -sx);
    e2s[i] = es * es;
    e2[i] = ee[i] * ee[i];
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double pivmin = fmax(tnrm * 2.2250738585072014e-308 / eps, 2.2250738585072014e-308);
  pc_mark(6);
  // ---- eigenvalues: one warp per eigenvalue, 32-point multisection ----------------------
  if (warp < epb) {
    const int m = m0 + warp;                          // m-th smallest eigenvalue
    if (m < k) {
      const double sn = ldexp(tnrm, -sx);              // in [1, 2)
      const double atol = 2.0 * eps * sn;
      double lo = ldexp(glo, -sx) - (eps * sn + 2.0 * atol), hi = ldexp(ghi, -sx) + (eps * sn + 2.0 * atol);
      const double inv33 = 1.0 / 33.0;
      for (int it = 0; it < 64; ++it) {
        if (!(hi - lo > fmax(atol, 4.0 * eps * fmax(fabs(lo), fabs(hi))))) break;   // warp-uniform
        const double x = lo + (hi - lo) * (double)(lane + 1) * inv33;
        const int c = pc_sturm(ds, e2s, k, x);
        const unsigned bits = __ballot_sync(0xffffffffu, c > m);
        const int f = bits ? __ffs(bits) - 1 : 32;
        const double nlo = f == 0 ? lo : lo + (hi - lo) * (double)f * inv33;
        const double nhi = f == 32 ? hi : lo + (hi - lo) * (double)(f + 1) * inv33;
        lo = nlo;
        hi = nhi;
      }
      if (lane == 0) {
        const double l = ldexp(0.5 * (lo + hi), sx);
        lam[warp] = l;
        lam_g[m] = l;
      }
    }
  }
  __syncthreads();
  pc_mark(7);
  // ---- eigenvectors of the tridiagonal: twisted factorisation, one warp per eigenvalue ----
  // lanes 0 / 1 run the D+ / D- recurrences (serial); the twist index (first minimum of
  // |gamma_i|, ties to the lowest i) is a warp argmin; the vector's entries, products of the
  // ratios from the twist outwards, are a warp suffix / prefix product scan over chunks of
  // TCH rows per lane, and the norm a warp sum.
  {
    constexpr int TCH = (PK_MAX + 31) / 32;
    const int e = warp, m = m0 + e;
    if (e < epb && m < k) {
      const double lm = lam[e];
      double* z = zb + (size_t)e * k;
      double* dmn = dm + (size_t)e * k;
      if (lane == 0) {
        double q = dd[0] - lm;
        if (fabs(q) < pivmin) q = -pivmin;
        z[0] = q;
        for (int i = 1; i < k; ++i) {
          q = (dd[i] - lm) - pc_fast_div(e2[i - 1], q);
          if (fabs(q) < pivmin) q = -pivmin;
          z[i] = q;
        }
      } else if (lane == 1) {
        double q = dd[k - 1] - lm;
        if (fabs(q) < pivmin) q = -pivmin;
        dmn[k - 1] = q;
        for (int i = k - 2; i >= 0; --i) {
          q = (dd[i] - lm) - pc_fast_div(e2[i], q);
          if (fabs(q) < pivmin) q = -pivmin;
          dmn[i] = q;
        }
      }
      __syncwarp();
      double best = 1e300;
      int r = 0;
      for (int i = lane; i < k; i += 32) {
        const double g = fabs(z[i] + dmn[i] - (dd[i] - lm));
        if (g < best) { best = g; r = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int orr = __shfl_xor_sync(0xffffffffu, r, o);
        if (ob < best || (ob == best && orr < r)) { best = ob; r = orr; }
      }
      const int i0 = lane * TCH;
      double lf[TCH], rf[TCH];
      double pl = 1.0, pr = 1.0;
#pragma unroll
      for (int t = TCH - 1; t >= 0; --t) {                       // left: suffix products below r
        const int i = i0 + t;
        const double f = (i < r && i < k) ? -pc_fast_div(ee[i], z[i]) : 1.0;
        pl *= f;
        lf[t] = pl;
      }
#pragma unroll
      for (int t = 0; t < TCH; ++t) {                            // right: prefix products above r
        const int i = i0 + t;
        const double f = (i > r && i < k) ? -pc_fast_div(ee[i - 1], dmn[i]) : 1.0;
        pr *= f;
        rf[t] = pr;
      }
      double sl = pl, sr = pr;                                   // inclusive scans over lanes
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double vl = __shfl_down_sync(0xffffffffu, sl, o);
        const double vr = __shfl_up_sync(0xffffffffu, sr, o);
        if (lane + o < 32) sl *= vl;
        if (lane >= o) sr *= vr;
      }
      double xl = __shfl_down_sync(0xffffffffu, sl, 1), xr = __shfl_up_sync(0xffffffffu, sr, 1);
      if (lane == 31) xl = 1.0;
      if (lane == 0) xr = 1.0;
      double xv[TCH];
      double nrm = 0.0;
#pragma unroll
      for (int t = 0; t < TCH; ++t) {
        const int i = i0 + t;
        xv[t] = i < r ? lf[t] * xl : (i == r ? 1.0 : rf[t] * xr);
        if (i < k) nrm = fma(xv[t], xv[t], nrm);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
      nrm = sqrt(nrm);
      __syncwarp();                                              // z / dmn reads done
      if (!(nrm > 0.0) || !isfinite(nrm)) {
        if (lane == 0) *gate = 1;
      } else {
        const double inv = 1.0 / nrm;
#pragma unroll
        for (int t = 0; t < TCH; ++t)
          if (i0 + t < k) z[i0 + t] = xv[t] * inv;
      }
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  pc_mark(8);
  // ---- back-transformation: W1[:, k-1-m] = H_0 ... H_{k-3} z, one warp per eigenvector ----
  constexpr int RT = (PK_MAX + 31) / 32;
  if (warp < epb && m0 + warp < k) {
    const double* z = zb + (size_t)warp * k;
    double v[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = lane + 32 * t;
      v[t] = i < k ? z[i] : 0.0;
    }
    for (int j = k - 3; j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double* uj = R + (size_t)j * k;          // zero at rows <= j
      double ur[RT];
      double sum = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = lane + 32 * t;
        ur[t] = i < k ? uj[i] : 0.0;
        sum = fma(ur[t], v[t], sum);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const double wc = tj * sum;
#pragma unroll
      for (int t = 0; t < RT; ++t) v[t] = fma(-ur[t], wc, v[t]);
    }
    double* out = W1 + (size_t)(k - 1 - (m0 + warp)) * k;
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = lane + 32 * t;
      if (i < k) out[i] = v[t];
    }
  }
  pc_mark(9);
}

// Y[:, c] = X^T W1[:, c] (X = L^-1 lower triangular: rows l >= i), values (descending) and
// the sign rule on Y's columns (smallsolve.py:52-61), one column per CTA.
__global__ void __launch_bounds__(256)
    k_pc_finish(const double* __restrict__ lam, const double* __restrict__ X, const double* __restrict__ W1, int k,
                double* __restrict__ values, double* __restrict__ vectors, int* __restrict__ n_out,
                int* __restrict__ status, const double* __restrict__ tnrm_g, int* __restrict__ gate) {
  if (*gate) return;
  const int c = blockIdx.x;                  // one column per CTA
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double sb[8];
  __shared__ int si[8];
  __shared__ int s_neg;
  __shared__ double w1[PK_MAX], yc[PK_MAX];
  for (int l = threadIdx.x; l < k; l += blockDim.x) w1[l] = W1[(size_t)c * k + l];
  __syncthreads();
  // warp per output row: y_i = sum_{l >= i} X[l, i] w1[l] (column i of X, coalesced)
  for (int i = warp; i < k; i += blockDim.x / 32) {
    double sacc = 0.0;
    for (int l = i + lane; l < k; l += 32) sacc = fma(X[(size_t)i * k + l], w1[l], sacc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) yc[i] = sacc;
  }
  __syncthreads();
  // numerically coincident eigenvalues (gap <= 1e-9 of the Gershgorin bound): the twisted
  // vectors are not orthogonal there -- every CTA sees the same verdict and leaves the
  // pencil to the general kernel
  {
    const double ctol = 1e-9 * *tnrm_g;
    int clus = 0;
    for (int m = 1 + threadIdx.x; m < k; m += blockDim.x) clus |= (lam[m] - lam[m - 1] <= ctol) ? 1 : 0;
    if (__syncthreads_or(clus)) {
      if (c == 0 && threadIdx.x == 0) *gate = 1;
      return;
    }
  }
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const double a = fabs(yc[r]);
    if (a > best) { best = a; bi = r; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
  }
  if (lane == 0) { sb[warp] = best; si[warp] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = sb[0];
    int ii = si[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (sb[w] > b || (sb[w] == b && si[w] < ii)) { b = sb[w]; ii = si[w]; }
    s_neg = yc[ii] < 0.0;
    values[c] = lam[k - 1 - c];
    if (c == 0) { *n_out = k; *status = 0; }
  }
  __syncthreads();
  const double sg = s_neg ? -1.0 : 1.0;
  for (int r = threadIdx.x; r < k; r += blockDim.x) vectors[(size_t)c * k + r] = sg * yc[r];
}

// ---------------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------------
int pencil_max_k() { return PK_MAX; }
size_t pencil_ws(int k) { return (size_t)7 * k * k * sizeof(double) + (size_t)k * sizeof(double) + 1024; }

// Launches the fast pipeline; leaves *gate = 1 (device) when the general kernel must run.
int pencil_eig(const double* B, const double* M, int k, double* values, double* vectors, int* n_out, int* status,
               void* ws, int* gate, cudaStream_t st) {
  double* p = (double*)ws;
  const size_t kk = (size_t)k * k;
  double* X = p;            // L^-1
  double* T1 = p + kk;      // X sym(B)
  double* T = p + 2 * kk;   // T1 X^T
  double* R = p + 3 * kk;   // reflectors of the tridiagonalisation
  double* tri = p + 4 * kk; // d | e | tau | tnrm (3k + 1 <= kk for k >= 4; else T1, dead by then)
  double* W1 = p + 5 * kk;  // Q Z
  double* lam = p + 7 * kk;
  if (3 * (size_t)k + 1 > kk) tri = T1;
  double* tnrm = tri + 3 * k;
  const size_t shm = (size_t)k * (k | 1) * sizeof(double);
  const size_t shm_e = (kk + 2 * (size_t)pc_epb(k) * k) * sizeof(double);
  static std::atomic<bool> attr{false};   // set once; concurrent callers may both set it (idempotent)
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_chol, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((size_t)PK_MAX * (PK_MAX | 1) * sizeof(double))));
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_tri, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((size_t)PK_MAX * (PK_MAX | 1) * sizeof(double))));
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_chol_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CB_SMEM));
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_chol_reg<8, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((size_t)2 * 64 * 64 * sizeof(double))));
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_eigvec, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(((size_t)PK_MAX * PK_MAX + 2 * pc_epb(PK_MAX) * PK_MAX) * sizeof(double))));
    attr = true;
  }
  const dim3 gg((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
  // register-resident for k <= 64 (k = 64: 61 -> 51 us); at k = 128 the 32-row register
  // blocks make the in-smem kernel faster (100 + 116 us vs 131 + 257 us)
  if (k <= 64) {
    // register Cholesky + inverse + certificate; T on the multi-CTA GEMMs (the in-kernel
    // T = X sym(B) X^T measured 65 us against 28 us for the two launches)
    k_pc_chol_reg<8, 8><<<1, PT, (size_t)2 * k * k * sizeof(double), st>>>(M, k, X, gate, nullptr, nullptr);
    OFRR_CHECK_LAUNCH();
    k_pc_gemm<false, false, true><<<gg, 256, 0, st>>>(X, B, T1, k, gate);
    k_pc_gemm<false, true, false><<<gg, 256, 0, st>>>(T1, X, T, k, gate);
    OFRR_CHECK_LAUNCH();
  } else if (k <= CB_KB * CB_N) {
    k_pc_chol_blk<<<1, CB_T, CB_SMEM, st>>>(M, k, X, gate);
    OFRR_CHECK_LAUNCH();
    k_pc_gemm<false, false, true><<<gg, 256, 0, st>>>(X, B, T1, k, gate);
    k_pc_gemm<false, true, false><<<gg, 256, 0, st>>>(T1, X, T, k, gate);
    OFRR_CHECK_LAUNCH();
  } else {
    k_pc_chol<<<1, PT, shm, st>>>(M, k, X, gate);
    OFRR_CHECK_LAUNCH();
    k_pc_gemm<false, false, true><<<gg, 256, 0, st>>>(X, B, T1, k, gate);
    k_pc_gemm<false, true, false><<<gg, 256, 0, st>>>(T1, X, T, k, gate);
    OFRR_CHECK_LAUNCH();
  }
  if (k <= 64) k_pc_tri_reg<8, 8><<<1, PT, 0, st>>>(T, k, tri, R, gate);   // (<4, 16, 256>: same 2.4K cycles per step)
  else if (k <= 128) k_pc_tri_reg<4, 32><<<1, PT, 0, st>>>(T, k, tri, R, gate);
  else k_pc_tri<<<1, PT, shm, st>>>(T, k, tri, R, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_eigvec<<<(k + pc_epb(k) - 1) / pc_epb(k), EPT, shm_e, st>>>(tri, R, k, lam, W1, tnrm, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_finish<<<k, 256, 0, st>>>(lam, X, W1, k, values, vectors, n_out, status, tnrm, gate);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
