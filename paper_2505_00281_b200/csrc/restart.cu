// restart.cu -- K6f: the restart step of one outer iteration as one pass over (U, W).
//
// After the pencil, the iteration needs three products with the same k x r eigenvector
// block Y (ofrr/projection.py:86, ofrr/driver.py:109 with A-pass reuse, and the residual
// estimate of the convergence test):
//   Xu  = round(U Y)                the Ritz block (and its fp64 copy U64 when asked),
//   Xw  = round(W Y), colmax        the next power step A (U Y) = (A U) Y = W Y,
//   s_j = sum_i ((W Y)_ij - lambda_j (U Y)_ij)^2   for j < t (K7e's residual estimate),
// which K6 (twice) and K7e computed as three kernels re-reading U, W and Y.  Here each CTA
// forms both products of a 64-row x 64-column tile on the fp64 tensor cores (DMMA m8n8k4)
// from one shared Y slab and finishes all three outputs in its epilogue; per-column sums of
// squares go to part[row block][j] and the fixed-order k_residual_reduce finishes them.
// The products accumulate in the same order as k_ritz_dmma (k slabs of 16, k4 steps
// ascending), so Xu / U64 / Xw equal K6's outputs bit for bit.
#include "common.cuh"
#include <algorithm>
#include <atomic>
#include <type_traits>

namespace ofrr {

int residual_reduce(const double* part, int nblocks, int n, const double* vals, const int* r_dev, double* res,
                    int mode, cudaStream_t st);

namespace {
__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
constexpr int RB_M = 64, RB_N = 64, RB_K = 16, RB_RS = RB_K + 4;   // tile, k slab, smem row stride
constexpr int RB_T = 256;
constexpr int RB_YS = RB_N + 4;                                    // Y row stride (doubles)
constexpr int RB_KMAX = 256;                                       // kp bound of the resident Y block
constexpr size_t rb_smem(int kp) {
  return (size_t)(4 * RB_M * RB_RS + ((kp + RB_K - 1) / RB_K) * RB_K * RB_YS) * sizeof(double);
}

}  // namespace

struct RestartOut {
  void* Xu; int64_t ldxu; int xu_fmt; int* flags_u;             // round(U Y)   (optional)
  double* U64; int64_t ld64;                                    // U Y in fp64   (optional)
  void* Xw; int64_t ldxw; int xw_fmt; int* flags_w; double* colmax;   // round(W Y) + column max (optional)
  const double* vals; int t; double* part;                      // residual sums, columns < t (optional)
};

template <typename TU, typename TW, bool HW>
__global__ void __launch_bounds__(RB_T, 2)
    k_restart_dmma(const TU* __restrict__ U, int64_t ldu, const TW* __restrict__ W, int64_t ldw, int64_t n, int kp,
                   const double* __restrict__ Y, int ldy, const int* __restrict__ r_dev, int r_max, RestartOut o) {
  // Persistent over row tiles: the CTA's 64 columns of Y stay in shared memory for all its
  // tiles, and the U / W slabs stream as one pipeline across tile boundaries (the next tile's
  // first slab is in flight during this tile's last MMAs and its epilogue).
  extern __shared__ __align__(16) double rb_dyn[];
  auto Us = reinterpret_cast<double (*)[RB_M][RB_RS]>(rb_dyn);                          // [stage][row][l]
  auto Ws = reinterpret_cast<double (*)[RB_M][RB_RS]>(rb_dyn + 2 * RB_M * RB_RS);
  double* Yr = rb_dyn + 4 * RB_M * RB_RS;                                               // [l][col], ld RB_YS
  __shared__ double cm[RB_N];
  __shared__ double cs[4][RB_N];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 16, wn = (warp & 1) * 32;     // warp: 16 rows x 32 columns of both products
  const int n0 = blockIdx.y * RB_N;
  const int r = r_dev ? min(r_max, *r_dev) : r_max;
  const int nslab = (kp + RB_K - 1) / RB_K;
  const int nmt = (int)((n + RB_M - 1) / RB_M);
  // Y[:, n0 .. n0 + 64) -> shared memory once (columns >= r and rows >= kp are zero)
  for (int e = tid; e < nslab * RB_K * RB_N; e += RB_T) {
    const int l = e % (nslab * RB_K), c = e / (nslab * RB_K);
    const int gj = n0 + c;
    Yr[l * RB_YS + c] = (gj < r && l < kp) ? Y[(int64_t)gj * ldy + l] : 0.0;
  }
  int m = blockIdx.x;
  if (m >= nmt || n0 >= r_max) return;                       // uniform per CTA
  __syncthreads();

  TU ru[4];
  TW rw[4];
  auto fetch = [&](int mt, int l0) {
    const int64_t m0 = (int64_t)mt * RB_M;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + RB_T * q, rr = e & 63, ll = e >> 6;
      const int64_t gi = m0 + rr;
      const bool ok = gi < n && l0 + ll < kp;
      ru[q] = ok ? U[(int64_t)(l0 + ll) * ldu + gi] : TU();
      if constexpr (HW) rw[q] = ok ? W[(int64_t)(l0 + ll) * ldw + gi] : TW();
    }
  };
  auto stash = [&](int st) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + RB_T * q, rr = e & 63, ll = e >> 6;
      Us[st][rr][ll] = to_d(ru[q]);
      if constexpr (HW) Ws[st][rr][ll] = to_d(rw[q]);
    }
  };
  double au[2][4][2] = {}, aw[2][4][2] = {};
  fetch(m, 0);
  stash(0);
  __syncthreads();
  for (int it = 0;; ++it) {
    const int sl = it % nslab, s = it & 1;
    const bool last = sl + 1 == nslab;
    const int mn = last ? m + (int)gridDim.x : m;
    const bool more = mn < nmt;
    if (more) fetch(mn, last ? 0 : (sl + 1) * RB_K);          // in flight during this slab's MMAs
    const double* ys = Yr + (size_t)sl * RB_K * RB_YS;
#pragma unroll
    for (int kk = 0; kk < RB_K; kk += 4) {
      double a[2], w[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        a[i] = Us[s][wm + 8 * i + g][kk + t4];
        if constexpr (HW) w[i] = Ws[s][wm + 8 * i + g][kk + t4];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = ys[(kk + t4) * RB_YS + wn + 8 * j + g];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma884(au[i][j], a[i], b[j]);
          if constexpr (HW) dmma884(aw[i][j], w[i], b[j]);
        }
    }
    if (more) stash(s ^ 1);                                    // the other stage: last read one slab ago
    if (last) {
      // ---- epilogue of row tile m: thread holds rows wm + 8i + g, columns wn + 8j + 2 t4 + h
      const int64_t m0 = (int64_t)m * RB_M;
      if (tid < RB_N) cm[tid] = 0.0;
      __syncthreads();
      int bad_u = 0, bad_w = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double cmx[2] = {0.0, 0.0}, ss[2] = {0.0, 0.0};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gj = n0 + wn + 8 * j + 2 * t4 + h;
          const double lam = (o.part && gj < o.t && gj < r) ? o.vals[gj] : 0.0;
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int64_t gi = m0 + wm + 8 * i + g;
            if (gi >= n || gj >= r_max) continue;
            const double vu = gj < r ? au[i][j][h] : 0.0;
            const double vw = gj < r ? aw[i][j][h] : 0.0;
            if (o.U64) o.U64[(int64_t)gj * o.ld64 + gi] = vu;
            if (o.Xu) {
              const double xv = rnd(vu, o.xu_fmt);
              if (!isfinite(xv)) bad_u = 1;
              st_fmt(o.Xu, (int64_t)gj * o.ldxu + gi, o.xu_fmt, xv);
            }
            if (o.Xw) {
              const double xv = rnd(vw, o.xw_fmt);
              if (!isfinite(xv)) bad_w = 1;
              st_fmt(o.Xw, (int64_t)gj * o.ldxw + gi, o.xw_fmt, xv);
              cmx[h] = fmax(cmx[h], fabs(xv));
            }
            if (o.part && gj < o.t && gj < r) {
              const double d = vw - lam * vu;
              ss[h] += d * d;
            }
          }
        }
        if (o.colmax) {
#pragma unroll
          for (int h = 0; h < 2; ++h) atomic_max_nonneg(&cm[wn + 8 * j + 2 * t4 + h], cmx[h]);
        }
        if (o.part) {
          // fixed order: the 8 row lanes of the MMA tile by a butterfly, then the 4 row warps
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double v = ss[h];
            v += __shfl_xor_sync(0xffffffffu, v, 4);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            v += __shfl_xor_sync(0xffffffffu, v, 16);
            if (g == 0) cs[warp >> 1][wn + 8 * j + 2 * t4 + h] = v;
          }
        }
      }
      if (bad_u && o.flags_u) atomicOr(o.flags_u, OFRR_FLAG_NONFINITE);
      if (bad_w && o.flags_w) atomicOr(o.flags_w, OFRR_FLAG_NONFINITE);
      __syncthreads();
      if (tid < RB_N) {
        const int gj = n0 + tid;
        if (o.colmax && gj < r_max) atomic_max_nonneg(&o.colmax[gj], cm[tid]);
        if (o.part && gj < o.t)
          o.part[(int64_t)m * o.t + gj] = ((cs[0][tid] + cs[1][tid]) + cs[2][tid]) + cs[3][tid];
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) au[i][j][0] = au[i][j][1] = aw[i][j][0] = aw[i][j][1] = 0.0;
      if (!more) break;
      m = mn;
    }
    __syncthreads();
  }
}

size_t restart_ws(int64_t n, int t) { return t > 0 ? (size_t)((n + RB_M - 1) / RB_M) * (size_t)t * sizeof(double) : 0; }

int restart(const void* U, int64_t ldu, int u_fmt, const void* W, int64_t ldw, int w_fmt, int64_t n, int kp,
            const double* Y, int ldy, const int* r_dev, int r_max, void* Xu, int64_t ldxu, int xu_fmt, int* flags_u,
            double* U64, int64_t ld64, void* Xw, int64_t ldxw, int xw_fmt, int* flags_w, double* colmax,
            const double* vals, int t, double* res, int mode, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n <= 0 || r_max <= 0) return OFRR_OK;
  t = std::min(t, r_max);
  if ((Xw || colmax || t > 0) && !W) { ofrr_set_error("restart: W Y outputs need W"); return OFRR_ERR_INVALID; }
  if (t > 0 && (!vals || !res || ws_bytes < restart_ws(n, t))) {
    ofrr_set_error("restart: residual estimate needs vals, res and a workspace of restart_ws bytes");
    return OFRR_ERR_INVALID;
  }
  if (kp > RB_KMAX) { ofrr_set_error("restart: kp %d above %d", kp, RB_KMAX); return OFRR_ERR_UNSUPPORTED; }
  const int nb = (int)((n + RB_M - 1) / RB_M);
  const int ncb = (r_max + RB_N - 1) / RB_N;
  RestartOut o{Xu, ldxu, xu_fmt, flags_u, U64, ld64, Xw, ldxw, xw_fmt, flags_w, colmax, vals, t,
               t > 0 ? (double*)ws : nullptr};
  const size_t smem = rb_smem(kp);
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  int rc = OFRR_OK;
  auto go = [&](auto tu, auto tw, auto hw) {
    using TU = decltype(tu);
    using TW = decltype(tw);
    constexpr bool HW = decltype(hw)::value;
    auto kern = k_restart_dmma<TU, TW, HW>;
    static std::atomic<bool> attr{false};   // once per instantiation (idempotent if raced)
    if (!attr) {
      if (cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)rb_smem(RB_KMAX)) != cudaSuccess) { rc = OFRR_ERR_CUDA; return; }
      attr = true;
    }
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, RB_T, smem) != cudaSuccess || per_sm < 1)
      per_sm = 1;
    // persistent row tiles: every resident CTA slot of the GPU, split over the column blocks
    const int gx = std::max(1, std::min(nb, per_sm * sms / std::max(ncb, 1)));
    kern<<<dim3((unsigned)gx, (unsigned)ncb), RB_T, smem, st>>>((const TU*)U, ldu, (const TW*)W, ldw, n, kp, Y,
                                                                 ldy, r_dev, r_max, o);
  };
  auto with_w = [&](auto tu) {
    if (!W) go(tu, double(), std::false_type());
    else if (w_fmt == F64) go(tu, double(), std::true_type());
    else if (w_fmt == F32) go(tu, float(), std::true_type());
    else rc = OFRR_ERR_UNSUPPORTED;
  };
  switch (u_fmt) {
    case F64: with_w(double()); break;
    case F32: with_w(float()); break;
    case F16: with_w(__half()); break;
    case BF16: with_w(__nv_bfloat16()); break;
    case FP8: with_w(__nv_fp8_e4m3()); break;
    default: rc = OFRR_ERR_UNSUPPORTED;
  }
  if (rc != OFRR_OK) { ofrr_set_error("restart: formats U %d / W %d unsupported", u_fmt, w_fmt); return rc; }
  OFRR_CHECK_LAUNCH();
  if (t > 0) return residual_reduce((const double*)ws, nb, t, vals, r_dev, res, mode, st);
  return OFRR_OK;
}

}  // namespace ofrr
