// pencil.cu -- K5 fast path: the projected pencil B y = lambda M y for k <= 160 as a short
// pipeline of small kernels, one working matrix in shared memory per sequential phase and
// the O(k^3) matrix products spread over the GPU.
//
// Same mathematics as the certified Cholesky branch of small_eig.cu (ofrr/smallsolve.py:
// 64-88 when M is certifiably above the safeguard cutoff):
//   k_pc_chol   M = L L^T (right-looking, one barrier per column), X = L^-1 in place
//               (right-looking forward substitution), certificate 1/||X||_F^2 > 4 k eps ||M||_F
//   k_pc_gemm   T = X sym(B) X^T  (two launches)
//   k_pc_tri    T = Q Tri Q^T (Householder), eigenvalues of Tri by multisection on
//               division-free Sturm sequences (4 lanes per eigenvalue), eigenvectors Z of
//               Tri by twisted factorisation (+ Gram-Schmidt inside numerically coincident
//               clusters), Q formed in place from the reflectors
//   k_pc_gemm   Y = X^T (Q Z)  (two launches)
//   k_pc_finish descending order + the largest-|entry|-positive sign rule (smallsolve.py:52-61)
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

__device__ unsigned long long g_pcprof[16];   // debug: phase end times (globaltimer ns)
__device__ __forceinline__ void pc_mark(int i) {
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    g_pcprof[i] = t;
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
// power of two after every 8 steps.  The product e2 * p_{i-1} and d_i - x are off the
// dependency chain (one fma per step on it); signs are compared on the raw bits.
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
    const int ex = ilogb(p1);
    if (ex > 256 || ex < -256) { p0 = ldexp(p0, -ex); p1 = ldexp(p1, -ex); }
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
  // a / b to ~1 ulp via an f32 reciprocal and two Newton steps (finite, normal b)
  const double ab = fabs(b);
  if (ab > 1e-300 && ab < 1e300) {
    double r = (double)__frcp_rn((float)b);
    r = r * fma(-b, r, 2.0);
    r = r * fma(-b, r, 2.0);
    return a * r;
  }
  return a / b;
}

// ---------------------------------------------------------------------------------
// K5c: eigen-decomposition of sym(T): lam (ascending), Z (eigenvectors of the tridiagonal,
// column c <-> lam[k-1-c], i.e. descending), Q (k x k) with T = Q Tri Q^T.
// ---------------------------------------------------------------------------------
__global__ void __launch_bounds__(PT, 1)
    k_pc_tri(const double* __restrict__ Tg, int k, double* __restrict__ lam_g, double* __restrict__ Zg,
             double* __restrict__ Qg, double* __restrict__ wk, int* __restrict__ gate) {
  if (*gate) return;
  extern __shared__ double sm[];
  __shared__ double red[PNW];
  __shared__ double dd[PK_MAX], ee[PK_MAX], tau[PK_MAX], lam[PK_MAX], e2[PK_MAX], ds[PK_MAX], e2s[PK_MAX];
  __shared__ double pv[PK_MAX];
  __shared__ double s_norm2;
  __shared__ int flag;
  const int ld = pc_ld(k);
  double* S = sm;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int quad = threadIdx.x >> 2, ql = threadIdx.x & 3;   // 4 threads per row / column
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) S[j * ld + i] = 0.5 * (Tg[(size_t)j * k + i] + Tg[(size_t)i * k + j]);
  if (threadIdx.x == 0) flag = 1;
  __syncthreads();
  pc_mark(4);
  // ---- 1. Householder tridiagonalisation (reflector j stored in column j, rows > j) ----
  // Column-owner layout: warp w owns the trailing columns c = j+1+w, j+1+w+16, ...; the
  // symmetric matvec p_c = tau S[:, c] . u is a warp dot product over the owner's column,
  // the rank-2 update touches only the owner's columns.  Two barriers per column.
  constexpr int RT = (PK_MAX + 31) / 32;                               // rows per lane
  // the reflector scalars of the next column are formed by warp 0 as soon as that column is
  // final (end of the previous step), off the next step's critical path
  __shared__ double s_alpha, s_tau, s_u0, s_x0;
  auto reflector = [&](int j, double norm2) {                          // lane 0 of warp 0
    const double x0 = S[j * ld + j + 1];
    const double alpha = -copysign(sqrt(norm2), x0);
    const double unorm2 = 2.0 * (norm2 - x0 * alpha);
    const bool skip = !(unorm2 > 0.0) || norm2 == 0.0;
    s_x0 = x0;
    s_alpha = alpha;
    s_tau = skip ? 0.0 : 2.0 / unorm2;
    s_u0 = x0 - alpha;
  };
  if (warp == 0 && k > 2) {
    double s2 = 0.0;
    for (int i = 1 + lane; i < k; i += 32) s2 = fma(S[i], S[i], s2);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) reflector(0, s2);
  }
  __syncthreads();
  for (int j = 0; j + 2 < k; ++j) {
    const double tj = s_tau, u0 = s_u0, x0 = s_x0, alpha = s_alpha;
    const bool skip = tj == 0.0;
    const int j1 = j + 1;
    // u in registers: lane holds u_i for i = j1 + lane + 32 t
    double ur[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = j1 + lane + 32 * t;
      ur[t] = i < k ? (i == j1 ? u0 : S[j * ld + i]) : 0.0;
    }
    if (!skip) {
      double kpart = 0.0;
      for (int c = j1 + warp; c < k; c += PNW) {
        const double* col = S + c * ld;
        double sum = 0.0;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j1 + lane + 32 * t;
          if (i < k) sum = fma(col[i], ur[t], sum);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double pc = tj * sum;
        if (lane == 0) pv[c] = pc;
        kpart = fma(c == j1 ? u0 : S[j * ld + c], pc, kpart);
      }
      if (lane == 0) red[warp] = kpart;
    }
    if (threadIdx.x == 0) {
      dd[j] = S[j * ld + j];
      ee[j] = skip ? x0 : alpha;
      tau[j] = tj;
    }
    __syncthreads();                                                     // (A)
    if (threadIdx.x == 0 && !skip) S[j * ld + j1] = u0;                 // reflector in place
    double s2 = 0.0;
    if (!skip) {
      double ks = lane < PNW ? red[lane] : 0.0;                          // fixed-order tree
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ks += __shfl_xor_sync(0xffffffffu, ks, o);
      const double K = 0.5 * tj * ks;
      double qr[RT];
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = j1 + lane + 32 * t;
        qr[t] = i < k ? pv[i] - K * ur[t] : 0.0;
      }
      for (int c = j1 + warp; c < k; c += PNW) {
        const double uc = c == j1 ? u0 : S[j * ld + c];
        const double qc = pv[c] - K * uc;
        double* col = S + c * ld;
#pragma unroll
        for (int t = 0; t < RT; ++t) {
          const int i = j1 + lane + 32 * t;
          if (i < k) {
            const double nv = col[i] - (ur[t] * qc + qr[t] * uc);
            col[i] = nv;
            if (c == j1 && i > c) s2 = fma(nv, nv, s2);
          }
        }
      }
    } else if (warp == 0) {
      for (int i = j1 + 1 + lane; i < k; i += 32) s2 = fma(S[j1 * ld + i], S[j1 * ld + i], s2);
    }
    if (warp == 0 && j1 + 2 < k) {                                      // next column's reflector
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (lane == 0) reflector(j1, s2);
    }
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
  // ---- 2. eigenvalues: 4-lane multisection on the power-of-two scaled tridiagonal -------
  double glo = 0.0, ghi = 0.0;
  for (int i = 0; i < k; ++i) {
    const double r = (i > 0 ? fabs(ee[i - 1]) : 0.0) + (i + 1 < k ? fabs(ee[i]) : 0.0);
    glo = i == 0 ? dd[i] - r : fmin(glo, dd[i] - r);
    ghi = i == 0 ? dd[i] + r : fmax(ghi, dd[i] + r);
  }
  const double tnrm = fmax(fmax(fabs(glo), fabs(ghi)), 1e-300);
  const int sx = ilogb(tnrm);
  for (int i = threadIdx.x; i < k; i += PT) {
    ds[i] = ldexp(dd[i], -sx);
    const double es = ldexp(ee[i], -sx);
    e2s[i] = es * es;
    e2[i] = ee[i] * ee[i];
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double pivmin = fmax(tnrm * 2.2250738585072014e-308 / eps, 2.2250738585072014e-308);
  {
    const double sn = ldexp(tnrm, -sx);                  // in [1, 2)
    const double atol = 2.0 * eps * sn;
    const double lo0 = ldexp(glo, -sx) - (eps * sn + 2.0 * atol), hi0 = ldexp(ghi, -sx) + (eps * sn + 2.0 * atol);
    const unsigned qshift = (unsigned)(lane & ~3);
    for (int base = 0; base < k; base += PT / 4) {
      const int m = base + quad;                        // m-th smallest eigenvalue
      const bool act = m < k;
      double lo = lo0, hi = hi0;
      for (int it = 0; it < 64; ++it) {
        const bool more = act && hi - lo > fmax(atol, 4.0 * eps * fmax(fabs(lo), fabs(hi)));
        if (!__any_sync(0xffffffffu, more)) break;
        const double x = lo + (hi - lo) * (double)(ql + 1) * 0.2;
        const int c = more ? pc_sturm(ds, e2s, k, x) : 0;
        const unsigned bits = (__ballot_sync(0xffffffffu, more && c > m) >> qshift) & 0xfu;
        if (more) {
          const int f = bits ? __ffs(bits) - 1 : 4;
          const double nlo = f == 0 ? lo : lo + (hi - lo) * (double)f * 0.2;
          const double nhi = f == 4 ? hi : lo + (hi - lo) * (double)(f + 1) * 0.2;
          lo = nlo;
          hi = nhi;
        }
      }
      if (act && ql == 0) lam[m] = ldexp(0.5 * (lo + hi), sx);
    }
  }
  __syncthreads();
  pc_mark(6);
  for (int i = threadIdx.x; i < k; i += PT) lam_g[i] = lam[i];
  // ---- 3. Q = H_0 H_1 ... H_{k-3}, one column per warp, straight to global -------------
  // Column c of Q is H_0 ... H_{k-3} e_c; H_j leaves e_c alone for j >= c, so the warp
  // starts from v = e_c (registers, lane holds rows lane + 32 t) and applies H_{min(c-1,k-3)}
  // down to H_0: v -= tau_j (u_j . v) u_j.  The reflectors stay read-only in S: no barrier.
  for (int c = warp; c < k; c += PNW) {
    double v[RT];
#pragma unroll
    for (int t = 0; t < RT; ++t) v[t] = (lane + 32 * t == c) ? 1.0 : 0.0;
    for (int j = std::min(c - 1, k - 3); j >= 0; --j) {
      const double tj = tau[j];
      if (tj == 0.0) continue;
      const double* uj = S + j * ld;
      double sum = 0.0;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = lane + 32 * t;
        if (i > j && i < k) sum = fma(uj[i], v[t], sum);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const double wc = tj * sum;
#pragma unroll
      for (int t = 0; t < RT; ++t) {
        const int i = lane + 32 * t;
        if (i > j && i < k) v[t] = fma(-uj[i], wc, v[t]);
      }
    }
#pragma unroll
    for (int t = 0; t < RT; ++t) {
      const int i = lane + 32 * t;
      if (i < k) Qg[(size_t)c * k + i] = v[t];
    }
  }
  __syncthreads();
  pc_mark(7);
  // ---- 4. eigenvectors of the tridiagonal: twisted factorisation, one thread each, into
  // the (now free) shared matrix; D- in global scratch -------------------------------------
  double* dminus = wk;                      // [k][k], dminus[i * k + m]
  for (int m = threadIdx.x; m < k; m += PT) {
    const double lm = lam[m];
    double* z = S + (size_t)(k - 1 - m) * ld;   // descending column order; holds D+ first
    double q = dd[0] - lm;
    if (fabs(q) < pivmin) q = -pivmin;
    z[0] = q;
    for (int i = 1; i < k; ++i) {
      q = (dd[i] - lm) - pc_fast_div(e2[i - 1], q);
      if (fabs(q) < pivmin) q = -pivmin;
      z[i] = q;
    }
    q = dd[k - 1] - lm;
    if (fabs(q) < pivmin) q = -pivmin;
    dminus[(size_t)(k - 1) * k + m] = q;
    for (int i = k - 2; i >= 0; --i) {
      q = (dd[i] - lm) - pc_fast_div(e2[i], q);
      if (fabs(q) < pivmin) q = -pivmin;
      dminus[(size_t)i * k + m] = q;
    }
    int r = 0;
    double best = 1e300;
    for (int i = 0; i < k; ++i) {
      const double g = fabs(z[i] + dminus[(size_t)i * k + m] - (dd[i] - lm));
      if (g < best) { best = g; r = i; }
    }
    double xv = 1.0;
    for (int i = r - 1; i >= 0; --i) {
      xv = -pc_fast_div(ee[i], z[i]) * xv;
      z[i] = xv;
    }
    z[r] = 1.0;
    xv = 1.0;
    for (int i = r + 1; i < k; ++i) {
      xv = -pc_fast_div(ee[i - 1], dminus[(size_t)i * k + m]) * xv;
      z[i] = xv;
    }
    double nrm = 0.0;
    for (int i = 0; i < k; ++i) nrm = fma(z[i], z[i], nrm);
    nrm = sqrt(nrm);
    if (!(nrm > 0.0) || !isfinite(nrm)) { flag = 0; continue; }
    const double inv = 1.0 / nrm;
    for (int i = 0; i < k; ++i) z[i] *= inv;
  }
  __syncthreads();
  pc_mark(8);
  // numerically coincident clusters: Gram-Schmidt (twice), one thread per cluster
  const double ctol = 1e-9 * tnrm;
  for (int m0 = threadIdx.x; m0 < k; m0 += PT) {
    if (m0 > 0 && lam[m0] - lam[m0 - 1] <= ctol) continue;
    int m1 = m0 + 1;
    while (m1 < k && lam[m1] - lam[m1 - 1] <= ctol) ++m1;
    for (int m = m0 + 1; m < m1; ++m) {
      double* z = S + (size_t)(k - 1 - m) * ld;
      for (int pass = 0; pass < 2; ++pass)
        for (int mm = m0; mm < m; ++mm) {
          const double* y = S + (size_t)(k - 1 - mm) * ld;
          double dot = 0.0;
          for (int i = 0; i < k; ++i) dot = fma(y[i], z[i], dot);
          for (int i = 0; i < k; ++i) z[i] -= dot * y[i];
        }
      double nrm = 0.0;
      for (int i = 0; i < k; ++i) nrm = fma(z[i], z[i], nrm);
      nrm = sqrt(nrm);
      if (!(nrm > 1e-8)) { flag = 0; continue; }
      for (int i = 0; i < k; ++i) z[i] /= nrm;
    }
  }
  __syncthreads();
  if (!flag) {
    if (threadIdx.x == 0) *gate = 1;
    return;
  }
  for (int j = warp; j < k; j += PNW)
    for (int i = lane; i < k; i += 32) Zg[(size_t)j * k + i] = S[j * ld + i];
  pc_mark(9);
}

// values (descending) and the sign rule on Y's columns (smallsolve.py:52-61).
__global__ void __launch_bounds__(256)
    k_pc_finish(const double* __restrict__ lam, const double* __restrict__ Y, int k, double* __restrict__ values,
                double* __restrict__ vectors, int* __restrict__ n_out, int* __restrict__ status,
                const int* __restrict__ gate) {
  if (*gate) return;
  const int c = blockIdx.x;                  // one column per CTA
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double sb[8];
  __shared__ int si[8];
  __shared__ int s_neg;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const double a = fabs(Y[(size_t)c * k + r]);
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
    s_neg = Y[(size_t)c * k + ii] < 0.0;
    values[c] = lam[k - 1 - c];
    if (c == 0) { *n_out = k; *status = 0; }
  }
  __syncthreads();
  const double sg = s_neg ? -1.0 : 1.0;
  for (int r = threadIdx.x; r < k; r += blockDim.x) vectors[(size_t)c * k + r] = sg * Y[(size_t)c * k + r];
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
  double* Z = p + 3 * kk;
  double* Q = p + 4 * kk;
  double* W1 = p + 5 * kk;  // Q Z
  double* Y = p + 6 * kk;   // X^T W1
  double* lam = p + 7 * kk;
  double* dminus = T1;      // scratch of k_pc_tri (T1 is dead by then)
  const size_t shm = (size_t)k * (k | 1) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_chol, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((size_t)PK_MAX * (PK_MAX | 1) * sizeof(double))));
    OFRR_CUDA_TRY(cudaFuncSetAttribute(k_pc_tri, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)((size_t)PK_MAX * (PK_MAX | 1) * sizeof(double))));
    attr = true;
  }
  const dim3 gg((unsigned)((k + 31) / 32), (unsigned)((k + 31) / 32));
  k_pc_chol<<<1, PT, shm, st>>>(M, k, X, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_gemm<false, false, true><<<gg, 256, 0, st>>>(X, B, T1, k, gate);
  k_pc_gemm<false, true, false><<<gg, 256, 0, st>>>(T1, X, T, k, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_tri<<<1, PT, shm, st>>>(T, k, lam, Z, Q, dminus, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_gemm<false, false, false><<<gg, 256, 0, st>>>(Q, Z, W1, k, gate);
  k_pc_gemm<true, false, false><<<gg, 256, 0, st>>>(X, W1, Y, k, gate);
  OFRR_CHECK_LAUNCH();
  k_pc_finish<<<k, 256, 0, st>>>(lam, Y, k, values, vectors, n_out, status, gate);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
