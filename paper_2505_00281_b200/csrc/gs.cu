// gs.cu -- the classical comparators of SURVEY.md 8(f) rank 4: the Gram-Schmidt basis
// builders that OFRR + Hessenberg replaces (ofrr/basis.py:65-148, orthonormalize,
// _mgs_project, _cgs_project, _mgs_right), on the device.
//
// Element arithmetic follows the reference op for op (ofrr/precision.py:107-185):
//   mixed_dot   products rounded to the compute format, sums in the accumulate format;
//   axpy        t = c(alpha) * x, r = y - t (compute-format roundings), stored rounded;
//   safe_norm2  m = max|x|, u = c(x / m), r = c(sqrt(dot(u, u))), c(m r);
//   normalize   s(c(v / nrm));
//   drop rules  nrm < drop_tol * pre or nrm == 0; MGS-L re-projects once when the norm
//               shrank below sqrt(2)/2 of the pre-projection norm; CGS2 drops a column whose
//               norm keeps shrinking after the second sweep.
// The sums are parallel (per-thread partials, fixed-order block and grid combination), not
// index-ascending: values agree with the reference to the rounding of the accumulate format,
// not bitwise (the Hessenberg kernel, hessenberg.cu, is the bitwise one).
//
// One cooperative kernel per call (grid <= #SMs): each CTA owns a contiguous row block of
// an fp64 working copy (values stay representable in the storage format); every inner
// product is one grid-wide reduction (per-CTA partials, grid.sync, every CTA combines the
// partials in CTA order -> identical scalars and identical control flow everywhere).  MGS-L
// needs one grid reduction per previous column -- the serial latency chain that makes QR
// the bottleneck OFRR removes; CGS/CGS2 batch a column's coefficients into one reduction.
#include "common.cuh"
#include <cooperative_groups.h>
#include <algorithm>

namespace cg = cooperative_groups;

namespace ofrr {

static constexpr int GS_T = 256;
enum GsMethod : int { GS_MGS_LEFT = 0, GS_MGS_RIGHT = 1, GS_CGS = 2, GS_CGS2 = 3 };

struct GsArgs {
  const void* X;
  int64_t n, ldx, ldq;
  int k, sfmt, cfmt, afmt, method, reorth;
  double drop_tol;
  void* Q;
  int* kept;
  int* n_kept;
  double* W;      // n x k working copy (column j at W + j * n)
  double* Qw;     // n x k kept columns (fp64 copies of the stored values)
  double* part;   // [2][G][PW] per-CTA partials (double buffered by reduction parity)
  double* pre;    // [k] MGS-R pre-projection norms
  int PW;         // partial slots per CTA
};

// accumulate-format addition (one rounding per add, as the sequential reference dot)
__device__ __forceinline__ double acc_add(double s, double p, int a) { return a == F64 ? s + p : rnd(s + p, a); }

struct GsCtx {
  const GsArgs& A;
  cg::grid_group grid;
  int64_t r0, r1;
  int parity;
  double* sred;   // [GS_T / 32 * width] block reduction scratch
  __device__ GsCtx(const GsArgs& a, double* s) : A(a), grid(cg::this_grid()), parity(0), sred(s) {
    const int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
    r0 = std::min<int64_t>(a.n, (int64_t)blockIdx.x * per);
    r1 = std::min<int64_t>(a.n, r0 + per);
  }

  // Grid-wide reduction of `w` per-thread values (sum in the accumulate format, or max):
  // returns the combined value of slot `slot` in every thread of every CTA.
  template <bool MAX>
  __device__ void reduce(double* v, int w) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int s = 0; s < w; ++s) {
      double x = v[s];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double y = __shfl_xor_sync(0xffffffffu, x, o);
        x = MAX ? fmax(x, y) : acc_add(x, y, A.afmt);
      }
      if (lane == 0) sred[warp * w + s] = x;
    }
    __syncthreads();
    double* mine = A.part + ((size_t)parity * gridDim.x + blockIdx.x) * A.PW;
    for (int s = threadIdx.x; s < w; s += blockDim.x) {
      double x = sred[s];
      for (int q = 1; q < GS_T / 32; ++q) x = MAX ? fmax(x, sred[q * w + s]) : acc_add(x, sred[q * w + s], A.afmt);
      mine[s] = x;
    }
    grid.sync();
    const double* all = A.part + (size_t)parity * gridDim.x * A.PW;
    for (int s = 0; s < w; ++s) {
      double x = all[s];
      for (unsigned b = 1; b < gridDim.x; ++b) x = MAX ? fmax(x, all[(size_t)b * A.PW + s]) : acc_add(x, all[(size_t)b * A.PW + s], A.afmt);
      v[s] = x;
    }
    parity ^= 1;
    __syncthreads();    // sred reuse
  }

  __device__ double dot(const double* x, const double* y) {
    double s = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) s = acc_add(s, c_mul(x[i], y[i], A.cfmt), A.afmt);
    reduce<false>(&s, 1);
    return s;
  }

  // safe_norm2 (ofrr/precision.py:138-156)
  __device__ double safe_norm2(const double* x) {
    double m = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) m = fmax(m, fabs(x[i]));
    reduce<true>(&m, 1);
    if (m == 0.0) return 0.0;
    const int c = A.cfmt;
    double s = 0.0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
      const double u = rnd(x[i] / m, c);
      s = acc_add(s, c_mul(u, u, c), A.afmt);
    }
    reduce<false>(&s, 1);
    const double r = rnd(sqrt(s), c);
    return rnd(m * r, c);
  }

  // y <- s(c(y - c(c(alpha) x))) on this CTA's rows (ofrr/precision.py:172-180)
  __device__ void axpy(double* y, double alpha, const double* x) {
    const int c = A.cfmt, sf = A.sfmt;
    const double ac = rnd(alpha, c);
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) y[i] = rnd(c_sub(y[i], c_mul(ac, x[i], c), c), sf);
  }

  // CGS sweep: all coefficients against the current v (reductions of up to PW at a time,
  // kept in shared memory), then the updates in column order (ofrr/basis.py:126-130)
  __device__ void cgs_project(double* v, int nq, double* scoef) {
    double part[64];
    for (int q0 = 0; q0 < nq; q0 += A.PW) {
      const int w = std::min(A.PW, nq - q0);
      for (int q = 0; q < w; ++q) part[q] = 0.0;
      for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
        const double vi = v[i];
        for (int q = 0; q < w; ++q) part[q] = acc_add(part[q], c_mul(A.Qw[(size_t)(q0 + q) * A.n + i], vi, A.cfmt), A.afmt);
      }
      reduce<false>(part, w);
      if (threadIdx.x < w) scoef[q0 + threadIdx.x] = part[threadIdx.x];
    }
    __syncthreads();
    for (int q = 0; q < nq; ++q) axpy(v, scoef[q], A.Qw + (size_t)q * A.n);
    __syncthreads();
  }

  __device__ void store_normalized(const double* v, double nrm, int slot) {
    double* q = A.Qw + (size_t)slot * A.n;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) q[i] = rnd(rnd(v[i] / nrm, A.cfmt), A.sfmt);
  }
};

static constexpr int GS_KMAX = 512;

__global__ void __launch_bounds__(GS_T) k_gram_schmidt(GsArgs a) {
  __shared__ double sred[(GS_T / 32) * 64];
  __shared__ double scoef[GS_KMAX];
  __shared__ double spre[GS_KMAX];
  GsCtx ctx(a, sred);
  const int64_t n = a.n;
  const int k = a.k;
  // working copy (values representable in the storage format; read exactly)
  for (int j = 0; j < k; ++j)
    for (int64_t i = ctx.r0 + threadIdx.x; i < ctx.r1; i += blockDim.x)
      a.W[(size_t)j * n + i] = ld_fmt(a.X, (long)((int64_t)j * a.ldx + i), a.sfmt);
  ctx.grid.sync();
  const double thr = 0.70710678118654757;   // REORTH_THRESHOLD = sqrt(2) / 2
  int nk = 0;
  if (a.method == GS_MGS_RIGHT) {
    for (int j = 0; j < k; ++j) {
      const double pj = ctx.safe_norm2(a.W + (size_t)j * n);
      if (threadIdx.x == 0) spre[j] = pj;
    }
    __syncthreads();
    for (int j = 0; j < k; ++j) {
      double* v = a.W + (size_t)j * n;
      const double nrm = ctx.safe_norm2(v);
      if (nrm < a.drop_tol * spre[j] || nrm == 0.0) continue;
      ctx.store_normalized(v, nrm, nk);
      const double* q = a.Qw + (size_t)nk * n;
      if (threadIdx.x == 0 && blockIdx.x == 0) a.kept[j] = 1;
      ++nk;
      // one right-looking sweep: h_i = dot(q, a_i) for every later column at once
      double part[64];
      for (int i0 = j + 1; i0 < k; i0 += a.PW) {
        const int w = std::min(a.PW, k - i0);
        for (int t = 0; t < w; ++t) part[t] = 0.0;
        for (int64_t r = ctx.r0 + threadIdx.x; r < ctx.r1; r += blockDim.x) {
          const double qr = q[r];
          for (int t = 0; t < w; ++t) part[t] = acc_add(part[t], c_mul(qr, a.W[(size_t)(i0 + t) * n + r], a.cfmt), a.afmt);
        }
        ctx.reduce<false>(part, w);
        for (int t = 0; t < w; ++t) ctx.axpy(a.W + (size_t)(i0 + t) * n, part[t], q);
      }
    }
  } else {
    for (int j = 0; j < k; ++j) {
      double* v = a.W + (size_t)j * n;
      const double pre = ctx.safe_norm2(v);
      double nrm;
      if (a.method == GS_MGS_LEFT) {
        for (int q = 0; q < nk; ++q) ctx.axpy(v, ctx.dot(a.Qw + (size_t)q * n, v), a.Qw + (size_t)q * n);
        nrm = ctx.safe_norm2(v);
        if (a.reorth && nrm < thr * pre) {
          for (int q = 0; q < nk; ++q) ctx.axpy(v, ctx.dot(a.Qw + (size_t)q * n, v), a.Qw + (size_t)q * n);
          nrm = ctx.safe_norm2(v);
        }
      } else {
        ctx.cgs_project(v, nk, scoef);
        nrm = ctx.safe_norm2(v);
        if (a.method == GS_CGS2) {
          const double n1 = nrm;
          ctx.cgs_project(v, nk, scoef);
          nrm = ctx.safe_norm2(v);
          if (nrm < thr * n1) continue;     // "twice is enough" failed: numerically dependent
        }
      }
      if (nrm < a.drop_tol * pre || nrm == 0.0) continue;
      ctx.store_normalized(v, nrm, nk);
      if (threadIdx.x == 0 && blockIdx.x == 0) a.kept[j] = 1;
      ++nk;
    }
  }
  ctx.grid.sync();
  // Q (storage format): the kept columns, then zeros (the driver narrows to n_kept)
  for (int j = 0; j < k; ++j)
    for (int64_t i = ctx.r0 + threadIdx.x; i < ctx.r1; i += blockDim.x)
      st_fmt(a.Q, (long)((int64_t)j * a.ldq + i), a.sfmt, j < nk ? a.Qw[(size_t)j * n + i] : 0.0);
  if (threadIdx.x == 0 && blockIdx.x == 0) *a.n_kept = nk;
}

static int gs_grid(int64_t n) {
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  return (int)std::max<int64_t>(1, std::min<int64_t>(sms, (n + 255) / 256));
}

size_t gram_schmidt_ws(int64_t n, int k) {
  const int G = gs_grid(n);
  return (size_t)2 * n * k * sizeof(double) + (size_t)2 * G * 64 * sizeof(double) + (size_t)k * sizeof(double) + 4096;
}

int gram_schmidt(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, int accumulate,
                 double drop_tol, int method, int reorth, void* Q, int64_t ldq, int* kept, int* n_kept, void* ws,
                 size_t ws_bytes, cudaStream_t st) {
  if (n <= 0 || k <= 0 || k > GS_KMAX || method < 0 || method > 3) {
    ofrr_set_error("gram_schmidt: invalid arguments (n %lld, k %d, method %d)", (long long)n, k, method);
    return OFRR_ERR_INVALID;
  }
  if (ws_bytes < gram_schmidt_ws(n, k)) { ofrr_set_error("gram_schmidt: workspace too small"); return OFRR_ERR_INVALID; }
  const int G = gs_grid(n);
  uint8_t* p = (uint8_t*)ws;
  GsArgs a;
  a.X = X; a.n = n; a.ldx = ldx; a.ldq = ldq; a.k = k; a.sfmt = storage; a.cfmt = compute; a.afmt = accumulate;
  a.method = method; a.reorth = reorth; a.drop_tol = drop_tol; a.Q = Q; a.kept = kept; a.n_kept = n_kept;
  a.W = (double*)p; p += (size_t)n * k * sizeof(double);
  a.Qw = (double*)p; p += (size_t)n * k * sizeof(double);
  a.PW = 64;
  a.part = (double*)p; p += (size_t)2 * G * a.PW * sizeof(double);
  a.pre = (double*)p;
  OFRR_CUDA_TRY(cudaMemsetAsync(kept, 0, sizeof(int) * k, st));
  void* args[] = {(void*)&a};
  OFRR_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_gram_schmidt, dim3(G), dim3(GS_T), args, 0, st));
  return OFRR_OK;
}

}  // namespace ofrr
