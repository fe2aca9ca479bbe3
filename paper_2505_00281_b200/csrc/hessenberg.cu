// hessenberg.cu -- K3: inner-product-free basis by pivot scaling and elimination
// (LU with partial pivoting of the tall-skinny block X, n x k).
//
// Replaces ofrr/basis.py:151-204 (hessenberg_basis, _pivot_row) with the axpy of
// ofrr/precision.py:172-180.  The elementwise arithmetic is the reference's, op for op
// (compute-format products / subtractions / divisions, storage rounding), so the
// pivots, kept mask and Q agree bit for bit with the reference for every policy.
//
// One persistent cooperative kernel, one CTA per SM (grid <= #SMs), each CTA owning a
// contiguous row block (in shared memory when it fits).  Per column j there is exactly
// one grid-wide barrier, split into arrive and wait:
//   after the wait every CTA reduces the published candidates in ascending CTA order
//   (= ascending row order, so ties resolve to the lowest index), scales column j by the
//   pivot and updates column j+1 only; it then publishes its candidate for column j+1
//   (max |X[i,j+1]| over its free rows, and that row's values in columns j+1..k-1 with the
//   pending update applied on the fly) and arrives; the bulk trailing update of columns
//   j+2..k-1 runs between arrive and wait, hidden behind the slowest CTA's arrival.
//   Candidates are double buffered by step parity.
#include "common.cuh"
#include <cooperative_groups.h>
#include <algorithm>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace ofrr {

static constexpr int HT = 256;

struct HessWs {
  unsigned* bar_count;  // grid barrier arrivals
  unsigned* bar_gen;    // grid barrier generation
  double* cand_val;   // [2][G]
  long long* cand_idx;  // [2][G]
  double* cand_row;   // [2][G][k]
  unsigned char* freerow;  // [n]
};

__device__ __forceinline__ void block_argmax(double& v, long long& idx, double* sv, long long* si) {
  // max value; ties -> lowest index; idx < 0 means "no candidate"
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
  if (lane == 0) { sv[warp] = v; si[warp] = idx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < HT / 32; ++w) {
      const double ov = sv[w];
      const long long oi = si[w];
      if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
    }
    sv[0] = v;
    si[0] = idx;
  }
  __syncthreads();
  v = sv[0];
  idx = si[0];
  __syncthreads();
}

template <typename T, int compute>
__global__ void __launch_bounds__(HT)
    k_hessenberg(const T* __restrict__ X, int64_t n, int k, int64_t ldx, T* __restrict__ Xg, int64_t ldg,
                 int storage, int compute_rt, double tol, T* __restrict__ Q, int64_t ldq,
                 int64_t* __restrict__ pivots, int* __restrict__ kept, int* __restrict__ n_kept, HessWs ws,
                 int in_smem) {
  __shared__ double sv[HT / 32];
  __shared__ long long si[HT / 32];
  extern __shared__ double dyn[];
  double* prow = dyn;                                        // pivot row values, k entries

  const int G = gridDim.x, c = blockIdx.x;
  const int64_t rows_per = (n + G - 1) / G;
  const int64_t r0 = std::min<int64_t>(n, (int64_t)c * rows_per);
  const int64_t r1 = std::min<int64_t>(n, r0 + rows_per);
  const int64_t nr = r1 - r0;
  // my working rows: in shared memory when they fit (column-major, ld rows_per), else in
  // the global workspace.  Xw is indexed with global row numbers.
  const int64_t ldw = in_smem ? rows_per : ldg;
  T* Xw = in_smem ? reinterpret_cast<T*>(dyn + k) - r0 : Xg;

  // prologue: private copy of my rows, free flags, candidate for column 0
  for (int j = 0; j < k; ++j)
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) Xw[(int64_t)j * ldw + i] = X[(int64_t)j * ldx + i];
  for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) ws.freerow[i] = 1;
  __syncthreads();

  // split grid barrier: arrive (release) ... independent work ... wait (acquire).  The
  // counters are zeroed before the launch; all CTAs are co-resident (cooperative launch).
  unsigned phase = 0;
  auto arrive = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned old = atomicAdd(ws.bar_count, 1u);
      if (old == (unsigned)G - 1) {
        atomicExch(ws.bar_count, 0u);
        __threadfence();
        atomicAdd(ws.bar_gen, 1u);
      }
    }
    ++phase;
  };
  auto wait = [&]() {
    if (threadIdx.x == 0) {
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(ws.bar_gen) : "memory");
      } while (g < phase);
    }
    __syncthreads();
  };

  // publish my pivot candidate for column jn: max |Xw[i, jn]| over my free rows (lowest
  // index on ties) and that row's values in columns jn..k-1 *after* the current step's
  // elimination.  Columns > jn may still be pending (deferred) in Xw: their values for the
  // candidate row are formed here with exactly the arithmetic of the deferred update.
  auto publish = [&](int jn, int buf, bool pending, int jp, long long rp) {
    double v = -1.0;
    long long idx = -1;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) {
      if (!ws.freerow[i]) continue;
      const double a = fabs(to_d(Xw[(int64_t)jn * ldw + i]));
      if (idx < 0 || a > v) { v = a; idx = i; }   // ascending i per thread: keeps lowest on ties
    }
    block_argmax(v, idx, sv, si);
    if (threadIdx.x == 0) {
      ws.cand_val[buf * G + c] = v;
      ws.cand_idx[buf * G + c] = idx;
    }
    if (idx >= 0) {
      const double vr = pending ? rnd(to_d(Xw[(int64_t)jp * ldw + idx]), compute) : 0.0;
      for (int cc = jn + threadIdx.x; cc < k; cc += HT) {
        double y = to_d(Xw[(int64_t)cc * ldw + idx]);
        if (pending && cc > jn)
          y = rnd(c_sub(rnd(y, compute), c_mul(prow[cc], vr, compute), compute), storage);
        ws.cand_row[((int64_t)buf * G + c) * k + cc] = y;
      }
    }
    (void)rp;
  };

  publish(0, 0, false, 0, -1);
  arrive();
  wait();

  int nk = 0;
  for (int j = 0; j < k; ++j) {
    const int buf = j & 1;
    // reduce the candidates: warp 0, lanes strided over CTAs; max value, ties -> lowest row
    // (CTA row blocks ascend, so the lowest row is the reference's np.argmax choice)
    __shared__ double s_best;
    __shared__ long long s_r;
    __shared__ int s_owner;
    if (threadIdx.x < 32) {
      double bv = -1.0;
      long long bi = -1;
      int bo = -1;
      for (int cc = threadIdx.x; cc < G; cc += 32) {
        const long long oi = __ldcg(&ws.cand_idx[buf * G + cc]);
        const double ov = __ldcg(&ws.cand_val[buf * G + cc]);
        if (oi >= 0 && (bi < 0 || ov > bv)) { bv = ov; bi = oi; bo = cc; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const int oo = __shfl_xor_sync(0xffffffffu, bo, o);
        if (oi >= 0 && (bi < 0 || ov > bv || (ov == bv && oi < bi))) { bv = ov; bi = oi; bo = oo; }
      }
      if (threadIdx.x == 0) { s_best = bv; s_r = bi; s_owner = bo; }
    }
    __syncthreads();
    const double best = s_best;
    const long long r = s_r;
    const int owner = s_owner;
    // ofrr/basis.py:178-180: skip when no free row or |pivot| < tol (NaN pivots skip too)
    const bool skip = (r < 0) || !(best >= tol);
    if (!skip) {
      for (int cc = j + threadIdx.x; cc < k; cc += HT) prow[cc] = __ldcg(&ws.cand_row[((int64_t)buf * G + owner) * k + cc]);
      __syncthreads();
      const double piv = prow[j];
      // ofrr/basis.py:181-187: v = round_s(round_c(v / piv)); v[r] = 1
      for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) {
        const double x = to_d(Xw[(int64_t)j * ldw + i]);
        const double v = (i == r) ? 1.0 : rnd(c_div(x, piv, compute), storage);
        Xw[(int64_t)j * ldw + i] = from_d<T>(v);
        Q[(int64_t)nk * ldq + i] = from_d<T>(v);
      }
      if (r >= r0 && r < r1 && threadIdx.x == 0) ws.freerow[r] = 0;
      if (c == 0 && threadIdx.x == 0) { kept[j] = 1; pivots[nk] = r; }
      // alpha_c = round_c(a[r, c]) for the axpys of ofrr/precision.py:172-180
      for (int cc = j + 1 + threadIdx.x; cc < k; cc += HT) prow[cc] = rnd(prow[cc], compute);
      __syncthreads();
      // ofrr/basis.py:188-190: column j+1 now (the next pivot search needs it) ...
      if (j + 1 < k) {
        for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) {
          const double v = rnd(to_d(Xw[(int64_t)j * ldw + i]), compute);
          T* yp = Xw + (int64_t)(j + 1) * ldw + i;
          *yp = from_d<T>(rnd(c_sub(rnd(to_d(*yp), compute), c_mul(prow[j + 1], v, compute), compute), storage));
        }
        __syncthreads();
        publish(j + 1, buf ^ 1, true, j, r);
        arrive();
        // ... columns j+2.. while the other CTAs catch up (hidden behind the barrier)
        for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) {
          const double v = rnd(to_d(Xw[(int64_t)j * ldw + i]), compute);
          T* yp = Xw + i;
          for (int cc = j + 2; cc < k; ++cc) {
            const double y = to_d(yp[(int64_t)cc * ldw]);
            yp[(int64_t)cc * ldw] = from_d<T>(rnd(c_sub(rnd(y, compute), c_mul(prow[cc], v, compute), compute), storage));
          }
        }
        wait();
      }
      ++nk;
    } else {
      if (c == 0 && threadIdx.x == 0) kept[j] = 0;
      if (j + 1 < k) {
        publish(j + 1, buf ^ 1, false, 0, -1);
        arrive();
        wait();
      }
    }
  }
  // columns nk..k-1 of Q are zero (a caller may project with all k columns speculatively)
  for (int j = nk; j < k; ++j)
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) Q[(int64_t)j * ldq + i] = from_d<T>(0.0);
  if (c == 0 && threadIdx.x == 0) *n_kept = nk;
}

static int hess_grid(int64_t n) {
  int sms = ofrr_device_sm_count(-1);
  if (sms <= 0) sms = 148;
  static int min_rows = -1;
  if (min_rows < 0) {
    const char* e = getenv("OFRR_HESS_MIN_ROWS");   // tuning knob (rows per CTA lower bound)
    min_rows = e ? atoi(e) : 128;
    if (min_rows < 32) min_rows = 32;
  }
  int64_t g = (n + min_rows - 1) / min_rows;
  return (int)std::max<int64_t>(1, std::min<int64_t>(sms, g));
}

size_t hessenberg_ws(int64_t n, int k, int storage) {
  const int G = hess_grid(n);
  size_t b = 0;
  b += 2 * G * sizeof(double);
  b += 2 * G * sizeof(long long);
  b += (size_t)2 * G * k * sizeof(double);
  b += (size_t)n * fmt_bytes(storage) * k;  // working copy
  b += n;
  return b + 4096;
}

template <typename T, int C>
static int launch_hess(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, double tol,
                       void* Q, int64_t ldq, int64_t* pivots, int* kept, int* n_kept, void* ws, cudaStream_t st) {
  const int G = hess_grid(n);
  uint8_t* p = (uint8_t*)ws;
  auto take = [&](size_t bytes) { uint8_t* q = p; p += (bytes + 255) & ~size_t(255); return q; };
  HessWs h;
  h.bar_count = (unsigned*)take(256);
  h.bar_gen = h.bar_count + 32;
  OFRR_CUDA_TRY(cudaMemsetAsync(h.bar_count, 0, 256, st));
  h.cand_val = (double*)take(2 * G * sizeof(double));
  h.cand_idx = (long long*)take(2 * G * sizeof(long long));
  h.cand_row = (double*)take((size_t)2 * G * k * sizeof(double));
  T* Xw = (T*)take((size_t)n * sizeof(T) * k);
  h.freerow = (unsigned char*)take(n);
  const T* Xp = (const T*)X;
  T* Qp = (T*)Q;
  int64_t ldw = n;
  const int64_t rows_per = (n + G - 1) / G;
  const size_t tile = (size_t)rows_per * k * sizeof(T);
  // up to the 227 KB opt-in per CTA (one CTA per SM): C3's fp32 rows (443 x 128) fit
  const size_t smem_max = 226 * 1024;
  int in_smem = (size_t)k * sizeof(double) + tile + 16 <= smem_max ? 1 : 0;
  size_t shmem = (size_t)k * sizeof(double) + (in_smem ? tile + 16 : 0);
  static bool attr = false;
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute((const void*)k_hessenberg<T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_max));
    attr = true;
  }
  void* args[] = {(void*)&Xp, (void*)&n, (void*)&k, (void*)&ldx, (void*)&Xw, (void*)&ldw, (void*)&storage,
                  (void*)&compute, (void*)&tol, (void*)&Qp, (void*)&ldq, (void*)&pivots, (void*)&kept,
                  (void*)&n_kept, (void*)&h, (void*)&in_smem};
  OFRR_CUDA_TRY(cudaMemsetAsync(kept, 0, sizeof(int) * k, st));
  OFRR_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)k_hessenberg<T, C>, dim3(G), dim3(HT), args, shmem, st));
  return OFRR_OK;
}

int hessenberg(const void* X, int64_t n, int k, int64_t ldx, int storage, int compute, double tol, void* Q,
               int64_t ldq, int64_t* pivots, int* kept, int* n_kept, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (ws_bytes < hessenberg_ws(n, k, storage)) { ofrr_set_error("hessenberg: workspace too small"); return OFRR_ERR_INVALID; }
#define HESS(T, C) return launch_hess<T, C>(X, n, k, ldx, storage, compute, tol, Q, ldq, pivots, kept, n_kept, ws, st)
  switch (storage * 8 + compute) {
    case F64 * 8 + F64: HESS(double, F64);
    case F32 * 8 + F32: HESS(float, F32);
    case F32 * 8 + F64: HESS(float, F64);
    case F16 * 8 + F16: HESS(__half, F16);
    case F16 * 8 + F32: HESS(__half, F32);
    case F16 * 8 + F64: HESS(__half, F64);
    case BF16 * 8 + BF16: HESS(__nv_bfloat16, BF16);
    case BF16 * 8 + F32: HESS(__nv_bfloat16, F32);
    case BF16 * 8 + F64: HESS(__nv_bfloat16, F64);
    default:
      ofrr_set_error("hessenberg: storage %d / compute %d unsupported", storage, compute);
      return OFRR_ERR_UNSUPPORTED;
  }
#undef HESS
}

}  // namespace ofrr
