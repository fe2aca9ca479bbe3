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
#include <type_traits>

namespace cg = cooperative_groups;

namespace ofrr {

#ifndef OFRR_HESS_THREADS
#define OFRR_HESS_THREADS 256
#endif
static constexpr int HT = OFRR_HESS_THREADS;

struct HessWs {
  unsigned* bar_count;  // grid barrier arrivals (monotonic)
  unsigned long long* key;  // [k] packed (|pivot| f32 bits, ~row) maxima, non-f64 storage
  double* cand_row;   // [2][G][k]
  unsigned char* freerow;  // [n]
  ulonglong2* slot;   // [2][G] narrow storage: (packed key, (pivot value, next-column value) as f32 bits)
  double2* slot64;    // [2][G][2] F64 storage: (|candidate|, row as bits), (pivot value, next-column value)
};

__device__ __forceinline__ void block_argmax(double& v, long long& idx, double* sv, long long* si) {
  // max value; ties -> lowest index; idx < 0 means "no candidate".  One barrier: every
  // thread folds the per-warp results itself (the caller separates consecutive uses).
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const long long oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
  if (lane == 0) { sv[warp] = v; si[warp] = idx; }
  __syncthreads();
  v = sv[0];
  idx = si[0];
  for (int w = 1; w < HT / 32; ++w) {
    const double ov = sv[w];
    const long long oi = si[w];
    if (oi >= 0 && (idx < 0 || ov > v || (ov == v && oi < idx))) { v = ov; idx = oi; }
  }
}

// The same argmax on integer keys with warp reductions (redux.sync): |v| >= 0 orders like its
// bit pattern, so the maximum is taken on the high then the low word and the lowest row among
// the maxima on the row.  idx < 0 / v < 0: no candidate.  Every thread gets the result.
__device__ __forceinline__ void block_argmax_redux(double& v, long long& idx, unsigned long long* sk2,
                                                   unsigned* sr2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool has = idx >= 0 && v >= 0.0;
  const unsigned long long key = has ? (unsigned long long)__double_as_longlong(v) : 0ull;
  const unsigned row = has ? (unsigned)idx : 0xFFFFFFFFu;
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
  const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
  const unsigned mrow = __reduce_min_sync(0xffffffffu, (hi == mhi && lo == mlo) ? row : 0xFFFFFFFFu);
  if (lane == 0) {
    sk2[warp] = ((unsigned long long)mhi << 32) | mlo;
    sr2[warp] = mrow;
  }
  __syncthreads();
  unsigned long long bk = sk2[0];
  unsigned br = sr2[0];
  for (int w = 1; w < HT / 32; ++w) {
    const unsigned long long k2 = sk2[w];
    const unsigned r2 = sr2[w];
    if (k2 > bk || (k2 == bk && r2 < br)) { bk = k2; br = r2; }
  }
  idx = br == 0xFFFFFFFFu ? -1 : (long long)br;
  v = idx >= 0 ? __longlong_as_double((long long)bk) : -1.0;
}

// Packed candidate key for storage formats narrower than f64: |x| is exact in f32 and its
// bit pattern orders like the value (NaN above inf, as np.argmax picks NaN); the low word
// ~row makes ties resolve to the lowest row.  0 = no candidate.
__device__ __forceinline__ unsigned long long cand_key(float absval, long long row) {
  return ((unsigned long long)__float_as_uint(absval) << 32) | (unsigned)(0xFFFFFFFFu - (unsigned)row);
}
__device__ __forceinline__ unsigned long long block_max_key(unsigned long long key, unsigned long long* sk) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {   // warp max of a 64-bit key: high word, then the low word among the high maxima (redux.sync)
    const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
    const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
    const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
    key = ((unsigned long long)mhi << 32) | mlo;
  }
  if (lane == 0) sk[warp] = key;
  __syncthreads();
  key = sk[0];
  for (int w = 1; w < HT / 32; ++w) key = sk[w] > key ? sk[w] : key;
  return key;
}

// ---- compute-format arithmetic in the narrowest native type -------------------------
// The reference rounds every product / difference / quotient into the compute format and
// every stored value into the storage format (ofrr/precision.py:172-185).  For compute
// formats up to F32 one f32 operation (RN, no contraction) followed by a rounding into the
// compute format is exactly that (f16/bf16 via f32 are exact by the 2p+2 bound); for F64
// compute the same ops run in f64.  Operands are always representable in the compute
// format (storage <= compute), so loading them needs no rounding.
struct f8 { uint8_t x; };    // FP8 e4m3 storage element
template <int C> struct CT { using type = float; };
template <> struct CT<F64> { using type = double; };

template <int C> __device__ __forceinline__ float rcf(float x) {
  if constexpr (C == F16) return __half2float(__float2half_rn(x));
  else if constexpr (C == BF16) return __bfloat162float(__float2bfloat16_rn(x));
  else return x;
}
template <int C> __device__ __forceinline__ typename CT<C>::type cmul(typename CT<C>::type a, typename CT<C>::type b) {
  if constexpr (C == F64) return __dmul_rn(a, b); else return rcf<C>(__fmul_rn(a, b));
}
template <int C> __device__ __forceinline__ typename CT<C>::type csub(typename CT<C>::type a, typename CT<C>::type b) {
  if constexpr (C == F64) return __dsub_rn(a, b); else return rcf<C>(__fsub_rn(a, b));
}
template <int C> __device__ __forceinline__ typename CT<C>::type cdiv(typename CT<C>::type a, typename CT<C>::type b) {
  if constexpr (C == F64) return __ddiv_rn(a, b); else return rcf<C>(__fdiv_rn(a, b));
}
// element (storage) -> compute type, exact
template <int C, typename T> __device__ __forceinline__ typename CT<C>::type ld_c(T y) {
  if constexpr (std::is_same<T, f8>::value) {
    __nv_fp8_e4m3 v; v.__x = y.x; return (typename CT<C>::type)float(v);
  } else if constexpr (std::is_same<T, double>::value) {
    return (typename CT<C>::type)y;   // storage F64 implies compute F64
  } else if constexpr (std::is_same<T, float>::value) {
    return (typename CT<C>::type)y;
  } else if constexpr (std::is_same<T, __half>::value) {
    return (typename CT<C>::type)__half2float(y);
  } else {
    return (typename CT<C>::type)__bfloat162float(y);
  }
}
// compute value -> storage element, rounded into the storage format (common.cuh rnd)
template <typename T, typename V> __device__ __forceinline__ T st_s(V v) {
  if constexpr (std::is_same<T, double>::value) return (double)v;
  else {
    const float f = std::is_same<V, double>::value ? __double2float_rn((double)v) : (float)v;
    if constexpr (std::is_same<T, float>::value) return f;
    else if constexpr (std::is_same<T, __half>::value) return __float2half_rn(f);
    else if constexpr (std::is_same<T, __nv_bfloat16>::value) return __float2bfloat16_rn(f);
    else {
      f8 o;
      const float r = rnd_fp8f(f);
      __nv_fp8_e4m3 q(r);
      if (isinf(r)) q.__x = r > 0 ? 0x7e : 0xfe;
      o.x = q.__x;
      return o;
    }
  }
}
// L2 load (bypasses L1: written by other CTAs during the launch) of any storage element
template <typename T> __device__ __forceinline__ T ldcg_el(const T* p) {
  T r;
  if constexpr (sizeof(T) == 1) { const unsigned char b = __ldcg(reinterpret_cast<const unsigned char*>(p)); memcpy(&r, &b, 1); }
  else if constexpr (sizeof(T) == 2) { const unsigned short b = __ldcg(reinterpret_cast<const unsigned short*>(p)); memcpy(&r, &b, 2); }
  else if constexpr (sizeof(T) == 4) { const unsigned b = __ldcg(reinterpret_cast<const unsigned*>(p)); memcpy(&r, &b, 4); }
  else { const unsigned long long b = __ldcg(reinterpret_cast<const unsigned long long*>(p)); memcpy(&r, &b, 8); }
  return r;
}
template <typename T> __device__ __forceinline__ double el_d(T y) {
  if constexpr (std::is_same<T, f8>::value) { __nv_fp8_e4m3 v; v.__x = y.x; return (double)float(v); }
  else return to_d(y);
}

__device__ unsigned long long g_hessprof[11];   // debug: CTA 0 per-phase time (ns), last launch
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <typename T, int C>
__global__ void __launch_bounds__(HT)
    k_hessenberg(const T* __restrict__ X, int64_t n, int k, int64_t ldx, T* __restrict__ Xg, int64_t ldg,
                 double tol, T* __restrict__ Q, int64_t ldq, int64_t* __restrict__ pivots, int* __restrict__ kept,
                 int* __restrict__ n_kept, HessWs ws, int in_smem, int pb) {
  using CV = typename CT<C>::type;
  __shared__ double sv[HT / 32];
  __shared__ long long si[HT / 32];
  extern __shared__ __align__(16) double dyn[];
  double* prow = dyn;                                        // pivot row values, k entries
  CV* pc = reinterpret_cast<CV*>(dyn + k);                   // alpha_c (compute format), k entries
  // panel mode (pb > 1): the pivot rows of the panel's kept steps (compute format, k each)
  // and their column indices; columns beyond the panel take those steps in one blocked
  // update at the panel's end (each element read and written once per panel)
  CV* PR = reinterpret_cast<CV*>(dyn + 2 * k);
  __shared__ int s_pl[32];                                   // kept steps of the panel
  __shared__ int s_npl;
  __shared__ long long s_prow[32];                           // their pivot rows
  __shared__ int s_pnk[32];                                  // and Q columns

  const int G = gridDim.x, c = blockIdx.x;
  const int64_t rows_per = (n + G - 1) / G;
  const int64_t r0 = std::min<int64_t>(n, (int64_t)c * rows_per);
  const int64_t r1 = std::min<int64_t>(n, r0 + rows_per);
  const int64_t nr = r1 - r0;
  // my working rows: in shared memory when they fit (column-major, ld rows_per), else in
  // the global workspace.  Xw is indexed with global row numbers.
  const int64_t ldw = in_smem ? ((rows_per + 3) & ~(int64_t)3) : ldg;   // 16-byte columns for 4-byte storage
  const size_t pr_dbl = pb > 1 ? ((size_t)(pb * k + pb * pb) * sizeof(CV) + 7) / 8 : 0;   // PR + M, in doubles
  T* Xw = in_smem ? reinterpret_cast<T*>(dyn + 2 * k + pr_dbl) - r0 : Xg;
  // rows in global memory + panels: the current panel's columns are cached in shared
  // memory (col(cc) is a row-indexed pointer to column cc wherever it lives)
  const bool pwc = !in_smem && pb > 1;
  T* Pw = reinterpret_cast<T*>(dyn + 2 * k + pr_dbl);
  int cp0 = -1;
  auto col = [&](int cc) -> T* {
    return (pwc && cc >= cp0 && cc < cp0 + pb) ? Pw + (int64_t)(cc - cp0) * nr - r0 : Xw + (int64_t)cc * ldw;
  };
  auto load_panel = [&](int q0) {   // global -> shared memory (caller syncs before and after)
    const int qe = min(k, q0 + pb);
    constexpr int PU = 8;             // columns in flight per thread (latency-bound otherwise)
    for (int c0 = q0; c0 < qe; c0 += PU)
      for (int64_t i = threadIdx.x; i < nr; i += HT) {
        T v[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) v[u] = c0 + u < qe ? Xw[(int64_t)(c0 + u) * ldw + r0 + i] : T();
#pragma unroll
        for (int u = 0; u < PU; ++u)
          if (c0 + u < qe) Pw[(int64_t)(c0 + u - q0) * nr + i] = v[u];
      }
    cp0 = q0;
  };
  // thread -> (row, column phase) for the trailing updates: two threads per row when the
  // row block is at most half the CTA
  const int tpr = (2 * nr <= HT) ? 2 : 1;
  const int rb = HT / tpr;
  const int trow = threadIdx.x % rb, tcol = threadIdx.x / rb;

  // prologue: private copy of my rows, free flags
  {
    constexpr int PU = 16;            // columns in flight per thread: the copy is latency-bound otherwise
    for (int j0 = 0; j0 < k; j0 += PU)
      for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) {
        T v[PU];
#pragma unroll
        for (int u = 0; u < PU; ++u) v[u] = j0 + u < k ? X[(int64_t)(j0 + u) * ldx + i] : T();
#pragma unroll
        for (int u = 0; u < PU; ++u)
          if (j0 + u < k) Xw[(int64_t)(j0 + u) * ldw + i] = v[u];
      }
  }
  if (in_smem)   // pad rows of the shared-memory tile (computed on by the 16-byte updates, never read)
    for (int j = 0; j < k; ++j)
      for (int64_t i = r1 + threadIdx.x; i < r0 + ldw; i += HT) Xw[(int64_t)j * ldw + i] = T();
  // free rows: this thread's rows are r0 + threadIdx.x + m * HT in every row loop below, so
  // their flags live in a register bit mask (bit m) -- no memory access on the per-column
  // critical path; a global byte array only when a thread owns more than 64 rows
  const bool fmask = rows_per <= (int64_t)64 * HT;
  unsigned long long fm = 0;
  if (fmask) {
    const int64_t mine = nr > threadIdx.x ? (nr - threadIdx.x + HT - 1) / HT : 0;
    fm = mine >= 64 ? ~0ull : ((1ull << mine) - 1ull);
  } else {
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) ws.freerow[i] = 1;
  }
  auto is_free = [&](int64_t i, int m) -> bool { return fmask ? ((fm >> m) & 1ull) : ws.freerow[i]; };
  __syncthreads();
  if (pwc) {
    load_panel(0);
    __syncthreads();
  }

  // split grid barrier: arrive (release) ... independent work ... wait (acquire).  One
  // monotonically increasing arrival counter (zeroed before the launch): barrier number p
  // is complete once it reaches p * G.  All CTAs are co-resident (cooperative launch).
  unsigned phase = 0;
  auto arrive = [&]() {
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ws.bar_count) : "memory");
    }
    ++phase;
  };
  auto wait = [&]() {
    if (threadIdx.x == 0) {
      const unsigned target = phase * (unsigned)G;
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(ws.bar_count) : "memory");
      } while (g < target);
    }
    __syncthreads();
  };

  // Pivot candidates.  Narrow storage: one packed key per column (atomicMax over CTAs).
  // F64 storage: (value, row) per CTA, reduced by every CTA after the barrier.
  constexpr bool KEYED = !std::is_same<T, double>::value;
  __shared__ unsigned long long sk[HT / 32];
  __shared__ unsigned sr2[HT / 32];
  __shared__ float s_v0, s_v1;                               // candidate / pivot: value, next column
  __shared__ double s_d0, s_d1;                              // the same, F64 storage
  // this thread's candidate over its rows i (free rows only) of column jn
  auto local_scan = [&](int jn, double& v, long long& idx, unsigned long long& key) {
    int m = 0;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT, ++m) {
      if (!is_free(i, m)) continue;
      const double a = fabs(el_d(col(jn)[i]));
      if constexpr (KEYED) {
        const unsigned long long kk = cand_key((float)a, i);
        key = kk > key ? kk : key;
      } else {
        if (idx < 0 || a > v) { v = a; idx = i; }   // ascending i per thread: lowest on ties
      }
    }
  };
  // publish the CTA's candidate for column jn and that row's values in columns jn..k-1
  // *after* the current step's elimination.  Columns > jn may still be pending (deferred)
  // in Xw: their values for the candidate row are formed here with exactly the arithmetic
  // of the deferred update.
  // pending beyond the panel: columns >= pe still owe the panel's kept steps s_pl[0..npl)
  // Panels (pb > 1): only the panel's columns [jn, lim) are published -- the columns beyond
  // the panel take the panel's pivot rows at its end (compute_pr), straight from memory.
  auto publish = [&](int jn, int buf, bool pending, int jp, double v, long long idx, unsigned long long key,
                     int pe, int npl, int lim) {
    if constexpr (KEYED) {
      key = block_max_key(key, sk);
      idx = key ? (long long)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull)) : -1;
    } else {
      block_argmax_redux(v, idx, sk, sr2);
    }
    if (idx >= 0) {
      const CV vr = pending ? ld_c<C>(col(jp)[idx]) : CV(0);
      for (int cc = jn + threadIdx.x; cc < lim; cc += HT) {
        T y = col(cc)[idx];            // cc < lim <= pe: a panel column (or no panels)
        if (pending && cc > jn) y = st_s<T>(csub<C>(ld_c<C>(y), cmul<C>(pc[cc], vr)));
        ws.cand_row[((int64_t)buf * G + c) * k + cc] = el_d(y);
        if constexpr (KEYED) {
          if (cc == jn) s_v0 = (float)el_d(y);
          if (cc == jn + 1) s_v1 = (float)el_d(y);
        } else {
          if (cc == jn) s_d0 = el_d(y);
          if (cc == jn + 1) s_d1 = el_d(y);
        }
      }
    }
    if constexpr (!KEYED) {
      // one 32-byte slot per CTA: (|candidate|, row) and the row's pivot and next-column
      // values -- the critical path after the barrier needs no second read of the row
      __syncthreads();
      if (threadIdx.x == 0) {
        __stcg(&ws.slot64[((int64_t)buf * G + c) * 2], make_double2(v, __longlong_as_double(idx)));
        __stcg(&ws.slot64[((int64_t)buf * G + c) * 2 + 1], make_double2(s_d0, jn + 1 < lim ? s_d1 : 0.0));
      }
    }
    if constexpr (KEYED) {
      // one 16-byte slot per CTA: the winner's pivot and next-column values travel with the
      // key, so the critical path after the barrier needs no second read of the row
      __syncthreads();
      if (threadIdx.x == 0) {
        const float v1 = jn + 1 < k ? s_v1 : 0.0f;
        ulonglong2 sv;
        sv.x = idx >= 0 ? key : 0ull;
        sv.y = ((unsigned long long)__float_as_uint(s_v0) << 32) | (unsigned long long)__float_as_uint(v1);
        __stcg(&ws.slot[buf * G + c], sv);
      }
    }
  };
  // panel end, step 1: the panel's pivot rows in the columns beyond it, PR[q][cc] = row
  // s_prow[q] of column cc after the panel's kept steps 0..q-1 -- formed here from memory
  // (columns >= pe are untouched during the panel; the multipliers are the pivot rows'
  // entries of the panel's Q columns), with exactly the arithmetic of the blocked update.
  // Wavefront order: PR[q'] is final once steps 0..q'-1 are in, then step q' goes into every
  // later row at once (independent chains per column).
  auto compute_pr = [&](int pe, int npl) {
    if (npl == 0 || pe >= k) return;
    CV* Mq = reinterpret_cast<CV*>(PR + (size_t)pb * k);     // [npl][npl]: M[q][q'] (q' < q)
    for (int e = threadIdx.x; e < npl * npl; e += HT) {
      const int q = e / npl, q2 = e - q * npl;
      Mq[e] = q2 < q ? ld_c<C>(ldcg_el(&Q[(int64_t)s_pnk[q2] * ldq + s_prow[q]])) : CV(0);
    }
    __syncthreads();
    // rolled loops (a fully unrolled 32 x 32 wavefront runs once per panel end and is
    // instruction-fetch bound); each thread owns columns cc and keeps them in PR itself
    for (int cc = pe + threadIdx.x; cc < k; cc += HT) {
      {                                                        // all the loads in flight at once
        T t32[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) t32[u] = u < npl ? ldcg_el(&Xw[(int64_t)cc * ldw + s_prow[u]]) : T();
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if (u < npl) PR[(size_t)u * k + cc] = ld_c<C>(t32[u]);
      }
      for (int q2 = 0; q2 + 1 < npl; ++q2) {
        const CV a = PR[(size_t)q2 * k + cc];
        for (int q0 = q2 + 1; q0 < npl; q0 += 4) {            // 4 independent rows: loads first
          CV y4[4], m4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = min(q0 + u, npl - 1);
            y4[u] = PR[(size_t)q * k + cc];
            m4[u] = Mq[q * npl + q2];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (q0 + u < npl) PR[(size_t)(q0 + u) * k + cc] = ld_c<C>(st_s<T>(csub<C>(y4[u], cmul<C>(a, m4[u]))));
        }
      }
    }
    __syncthreads();
  };
  // panel end, step 2: columns >= pe take the panel's kept steps, element by element in step
  // order.  Work units (row, 8-column segment), rows fastest (coalesced): each unit holds its
  // row's npl multipliers and 8 trailing elements in registers, the pivot rows broadcast
  // from shared memory; every trailing element is read and written once per panel.
  auto blocked_update = [&](int pe, int npl) {
    if (npl == 0 || pe >= k) return;
    constexpr int QMAX = 32, CB = 8;
    const bool kvec = (k % 4 == 0) && (pb % 4 == 0);   // PR rows and segments 16-byte aligned
    const unsigned nseg = (unsigned)((k - pe + CB - 1) / CB);
    const unsigned nru = (unsigned)nr, units = nru * nseg;
    // the next unit's elements are loaded while this unit computes (software pipeline)
    T yn[CB];
    auto unit_at = [&](unsigned u, int64_t& i, int& c0) {
      const unsigned seg = u / nru;
      i = r0 + (int64_t)(u - seg * nru);
      c0 = pe + (int)seg * CB;
    };
    auto load_unit = [&](unsigned u) {
      int64_t i;
      int c0;
      unit_at(u, i, c0);
      const T* b = Xw + (int64_t)c0 * ldw + i;
#pragma unroll
      for (int v = 0; v < CB; ++v) yn[v] = c0 + v < k ? b[(int64_t)v * ldw] : T();
    };
    if (threadIdx.x < units) load_unit(threadIdx.x);
    // the panel columns' offsets in the panel cache, once per panel end (not per unit)
    int moff[QMAX];
#pragma unroll
    for (int q = 0; q < QMAX; ++q) moff[q] = (pwc && q < npl) ? (s_pl[q] - cp0) * (int)nr : 0;
    for (unsigned u = threadIdx.x; u < units; u += HT) {
      int64_t i;
      int c0;
      unit_at(u, i, c0);
      T y[CB];
#pragma unroll
      for (int v = 0; v < CB; ++v) y[v] = yn[v];
      if (u + HT < units) load_unit(u + HT);
      CV mult[QMAX];
      const int li = (int)(i - r0);
#pragma unroll
      for (int q = 0; q < QMAX; ++q)
        mult[q] = q < npl ? ld_c<C>(pwc ? Pw[moff[q] + li] : col(s_pl[q])[i]) : CV(0);
      T* base = Xw + (int64_t)c0 * ldw + i;
#pragma unroll
      for (int q = 0; q < QMAX; ++q) {
        if (q < npl) {
          const CV* pr = PR + (size_t)q * k + c0;               // may run past row q: unused lanes
          CV pv[CB];
          if (kvec) {                                           // 16-byte broadcasts
#pragma unroll
            for (int v = 0; v < CB; v += 16 / (int)sizeof(CV))
              *reinterpret_cast<uint4*>(&pv[v]) = *reinterpret_cast<const uint4*>(pr + v);
          } else {
#pragma unroll
            for (int v = 0; v < CB; ++v) pv[v] = pr[v];
          }
#pragma unroll
          for (int v = 0; v < CB; ++v) y[v] = st_s<T>(csub<C>(ld_c<C>(y[v]), cmul<C>(pv[v], mult[q])));
        }
      }
#pragma unroll
      for (int v = 0; v < CB; ++v)
        if (c0 + v < k) base[(int64_t)v * ldw] = y[v];
    }
  };

  if (threadIdx.x == 0) s_npl = 0;
  {
    double v = -1.0;
    long long idx = -1;
    unsigned long long key = 0;
    local_scan(0, v, idx, key);
    publish(0, 0, false, 0, v, idx, key, k, 0, pb > 1 ? min(k, pb) : k);
  }
  arrive();
  wait();

  int nk = 0;
  unsigned long long pacc[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, tp = gtime();
  auto mark = [&](int ph) {
    if (c == 0 && threadIdx.x == 0) { const unsigned long long t = gtime(); pacc[ph] += t - tp; tp = t; }
  };
  __shared__ int s_owner;
  for (int j = 0; j < k; ++j) {
    const int buf = j & 1;
    // panel [p0, pe): its columns take every step at once; columns >= pe wait for the
    // panel's end (pb <= 1: one panel, the whole block)
    const int p0 = pb > 1 ? (j / pb) * pb : 0;
    const int pe = pb > 1 ? min(k, p0 + pb) : k;
    double best;
    long long r;
    int owner;
    if constexpr (KEYED) {
      // the G slots (one 16-byte read per thread), max key -> pivot row, its value and the
      // next column's value
      ulonglong2 sv = make_ulonglong2(0ull, 0ull);
      if (threadIdx.x < G) sv = __ldcg(&ws.slot[buf * G + threadIdx.x]);
      const unsigned long long key = block_max_key(threadIdx.x < G ? sv.x : 0ull, sk);
      if (key && sv.x == key && threadIdx.x < G) {
        s_owner = threadIdx.x;
        s_v0 = __uint_as_float((unsigned)(sv.y >> 32));
        s_v1 = __uint_as_float((unsigned)(sv.y & 0xffffffffull));
      }
      __syncthreads();
      r = key ? (long long)(0xFFFFFFFFu - (unsigned)(key & 0xFFFFFFFFull)) : -1;
      best = (double)__uint_as_float((unsigned)(key >> 32));
      owner = r >= 0 ? s_owner : 0;
    } else {
      // every thread reads one CTA's 32-byte slot (one round trip), block argmax: max value,
      // ties -> lowest row (the reference's np.argmax choice); the winner's pivot and
      // next-column values travel in its slot
      double bv = -1.0, d0 = 0.0, d1 = 0.0;
      long long bi = -1;
      if (threadIdx.x < G) {
        const double2 a = __ldcg(&ws.slot64[((int64_t)buf * G + threadIdx.x) * 2]);
        const double2 b = __ldcg(&ws.slot64[((int64_t)buf * G + threadIdx.x) * 2 + 1]);
        bv = a.x;
        bi = __double_as_longlong(a.y);
        d0 = b.x;
        d1 = b.y;
      }
      const long long mine = bi;
      block_argmax_redux(bv, bi, sk, sr2);
      if (threadIdx.x < G && bi >= 0 && mine == bi) {
        s_owner = threadIdx.x;
        s_d0 = d0;
        s_d1 = d1;
      }
      __syncthreads();
      best = bv;
      r = bi;
      owner = r >= 0 ? s_owner : 0;
    }
    // ofrr/basis.py:178-180: skip when no free row or |pivot| < tol (NaN pivots skip too)
    const bool skip = (r < 0) || !(best >= tol);
    mark(0);
    if (!skip) {
      // pivot row (values exact in the storage format); alpha_c = round_c(a[r, c]) is the
      // value itself (storage <= compute)
      // narrow storage: the row's loads are issued now and land in shared memory after the
      // column work below (which needs only the pivot and next-column values of the slot)
      // the row's loads (the panel's columns) are issued now and land in shared memory after
      // the column work below, which needs only the pivot and next-column values of the slot
      double prr[2] = {0.0, 0.0};
#pragma unroll
      for (int t2 = 0; t2 < 2; ++t2) {
        const int cc = j + threadIdx.x + t2 * HT;
        if (cc < pe) prr[t2] = __ldcg(&ws.cand_row[((int64_t)buf * G + owner) * k + cc]);
      }
      for (int cc = j + threadIdx.x + 2 * HT; cc < pe; cc += HT) {   // pe > 2 HT + j: rare
        const double a = __ldcg(&ws.cand_row[((int64_t)buf * G + owner) * k + cc]);
        prow[cc] = a;
        pc[cc] = (CV)a;
      }
      if (r >= r0 && r < r1) {
        if (!fmask) {
          if (threadIdx.x == 0) ws.freerow[r] = 0;
        } else if ((r - r0) % HT == threadIdx.x) {
          fm &= ~(1ull << (int)((r - r0) / HT));
        }
      }
      if (c == 0 && threadIdx.x == 0) { kept[j] = 1; pivots[nk] = r; }
      __syncthreads();
      if (pb > 1 && pe < k && threadIdx.x == 0) {            // this step, owed by columns >= pe
        s_pl[s_npl] = j;
        s_prow[s_npl] = r;
        s_pnk[s_npl] = nk;
        s_npl = s_npl + 1;
      }
      mark(1);
      const CV piv = KEYED ? (CV)s_v0 : (CV)s_d0;
      const CV a1 = j + 1 < pe ? (KEYED ? (CV)s_v1 : (CV)s_d1) : CV(0);
      // ofrr/basis.py:181-187: v = round_s(round_c(v / piv)); v[r] = 1; then (188-190,
      // precision.py:172-180) column j+1 at once -- the next pivot search needs it -- and
      // this thread's candidate for it
      double cv = -1.0;
      long long cidx = -1;
      unsigned long long ckey = 0;
      int m = 0;
      for (int64_t i = r0 + threadIdx.x; i < r1; i += HT, ++m) {
        const T v = (i == r) ? st_s<T>(CV(1)) : st_s<T>(cdiv<C>(ld_c<C>(col(j)[i]), piv));
        col(j)[i] = v;
        Q[(int64_t)nk * ldq + i] = v;
        if (j + 1 < pe) {
          T* yp = col(j + 1) + i;
          const T y = st_s<T>(csub<C>(ld_c<C>(*yp), cmul<C>(a1, ld_c<C>(v))));
          *yp = y;
          if (i != r && is_free(i, m)) {
            const double a = fabs(el_d(y));
            if constexpr (KEYED) {
              const unsigned long long kk = cand_key((float)a, i);
              ckey = kk > ckey ? kk : ckey;
            } else {
              if (cidx < 0 || a > cv) { cv = a; cidx = i; }
            }
          }
        }
      }
      mark(10);
#pragma unroll
      for (int t2 = 0; t2 < 2; ++t2) {
        const int cc = j + threadIdx.x + t2 * HT;
        if (cc < pe) { prow[cc] = prr[t2]; pc[cc] = (CV)prr[t2]; }
      }
      mark(2);
      if (j + 1 < pe) {
        __syncthreads();                                       // s_pl / s_npl visible
        publish(j + 1, buf ^ 1, true, j, cv, cidx, ckey, pe, pb > 1 ? s_npl : 0, pe);
        arrive();
        mark(3);
        // ... columns j+2.. while the other CTAs catch up (hidden behind the barrier).
        bool vec_done = false;
        if constexpr (sizeof(T) == 4) {
          if (in_smem) {
            // 4-byte storage in shared memory: four consecutive rows per 16-byte access (the
            // columns are 16-byte aligned, ldw % 4 == 0; the pad rows past r1 compute garbage
            // nobody reads), threads spread over (row quad, column phase), two columns in flight
            const int ngr = (int)((nr + 3) >> 2);
            const bool wide = ngr >= HT;
            const int P = wide ? 1 : HT / max(ngr, 1);
            const int ph = wide ? 0 : threadIdx.x / max(ngr, 1);
            if (ngr > 0 && ph < P) {
              for (int g = wide ? threadIdx.x : threadIdx.x % ngr; g < ngr; g += wide ? HT : ngr) {
                float* base = reinterpret_cast<float*>(Xw + r0) + 4 * g;
                const float4 vq = *reinterpret_cast<const float4*>(base + (int64_t)j * ldw);
                const CV v0 = ld_c<C>(vq.x), v1 = ld_c<C>(vq.y), v2 = ld_c<C>(vq.z), v3 = ld_c<C>(vq.w);
                auto upd = [&](float4 y, CV a) {
                  y.x = st_s<T>(csub<C>(ld_c<C>(y.x), cmul<C>(a, v0)));
                  y.y = st_s<T>(csub<C>(ld_c<C>(y.y), cmul<C>(a, v1)));
                  y.z = st_s<T>(csub<C>(ld_c<C>(y.z), cmul<C>(a, v2)));
                  y.w = st_s<T>(csub<C>(ld_c<C>(y.w), cmul<C>(a, v3)));
                  return y;
                };
                // U columns in flight per thread (all loads before the stores)
                constexpr int U = 4;
                int cc = j + 2 + ph;
                for (; cc + (U - 1) * P < pe; cc += U * P) {
                  float4* pp[U];
                  float4 y[U];
                  CV a[U];
#pragma unroll
                  for (int u = 0; u < U; ++u) {
                    pp[u] = reinterpret_cast<float4*>(base + (int64_t)(cc + u * P) * ldw);
                    y[u] = *pp[u];
                    a[u] = pc[cc + u * P];
                  }
#pragma unroll
                  for (int u = 0; u < U; ++u) *pp[u] = upd(y[u], a[u]);
                }
                for (; cc < pe; cc += P) {
                  float4* p0 = reinterpret_cast<float4*>(base + (int64_t)cc * ldw);
                  *p0 = upd(*p0, pc[cc]);
                }
              }
            }
            vec_done = true;
          }
        }
        // Two rows x two columns per iteration, all loads before the stores (ILP).
        for (int64_t i0 = r0 + trow; !vec_done && i0 < r1; i0 += 2 * rb) {
          const bool h1 = i0 + rb < r1;
          const CV v0 = ld_c<C>(col(j)[i0]);
          const CV v1 = h1 ? ld_c<C>(col(j)[i0 + rb]) : CV(0);
          T* p = col(j + 2 + tcol) + i0;
          const int64_t st1 = (int64_t)tpr * (pwc ? nr : ldw);   // panel columns only
          int cc = j + 2 + tcol;
          for (; cc + tpr < pe; cc += 2 * tpr, p += 2 * st1) {
            const CV a0 = pc[cc], a1 = pc[cc + tpr];
            const CV y00 = ld_c<C>(p[0]), y01 = ld_c<C>(p[st1]);
            const CV y10 = h1 ? ld_c<C>(p[rb]) : CV(0), y11 = h1 ? ld_c<C>(p[st1 + rb]) : CV(0);
            p[0] = st_s<T>(csub<C>(y00, cmul<C>(a0, v0)));
            p[st1] = st_s<T>(csub<C>(y01, cmul<C>(a1, v0)));
            if (h1) {
              p[rb] = st_s<T>(csub<C>(y10, cmul<C>(a0, v1)));
              p[st1 + rb] = st_s<T>(csub<C>(y11, cmul<C>(a1, v1)));
            }
          }
          if (cc < pe) {
            const CV a0 = pc[cc];
            const CV y00 = ld_c<C>(p[0]);
            const CV y10 = h1 ? ld_c<C>(p[rb]) : CV(0);
            p[0] = st_s<T>(csub<C>(y00, cmul<C>(a0, v0)));
            if (h1) p[rb] = st_s<T>(csub<C>(y10, cmul<C>(a0, v1)));
          }
        }
        __syncthreads();
        mark(4);
        wait();
        mark(5);
      } else if (pe < k) {
        // the panel's last column: columns >= pe take its kept steps, then column pe's search
        __syncthreads();
        compute_pr(pe, s_npl);
        mark(6);
        blocked_update(pe, s_npl);
        __syncthreads();
        if (threadIdx.x == 0) s_npl = 0;                       // next panel (read after the barrier)
        mark(7);
        if (pwc) {
          load_panel(pe);
          __syncthreads();
        }
        mark(8);
        double v = -1.0;
        long long idx = -1;
        unsigned long long key = 0;
        local_scan(pe, v, idx, key);
        publish(pe, buf ^ 1, false, 0, v, idx, key, k, 0, min(k, pe + pb));
        arrive();
        wait();
        mark(9);
      }
      ++nk;
    } else {
      if (c == 0 && threadIdx.x == 0) kept[j] = 0;
      if (j + 1 < k) {
        __syncthreads();
        const bool pend = j + 1 == pe;                         // panel end: blocked update first
        if (pend) {
          compute_pr(pe, s_npl);
          blocked_update(pe, s_npl);
          __syncthreads();
          if (threadIdx.x == 0) s_npl = 0;
          if (pwc) {
            load_panel(pe);
            __syncthreads();
          }
        }
        double v = -1.0;
        long long idx = -1;
        unsigned long long key = 0;
        local_scan(j + 1, v, idx, key);
        publish(j + 1, buf ^ 1, false, 0, v, idx, key, pend ? k : pe, pend ? 0 : (pb > 1 ? s_npl : 0),
                pb > 1 ? (pend ? min(k, pe + pb) : pe) : k);
        arrive();
        wait();
      }
    }
  }
  // columns nk..k-1 of Q are zero (a caller may project with all k columns speculatively)
  for (int j = nk; j < k; ++j)
    for (int64_t i = r0 + threadIdx.x; i < r1; i += HT) Q[(int64_t)j * ldq + i] = st_s<T>(CV(0));
  if (c == 0 && threadIdx.x == 0) {
    *n_kept = nk;
    for (int i = 0; i < 11; ++i) g_hessprof[i] = pacc[i];
  }
}

int hess_profile(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_hessprof, sizeof(g_hessprof)) == cudaSuccess ? 0 : 2;
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

// test/tuning knobs (ofrr_debug_hess_mode): rows in global memory even when they fit in
// shared memory; the panel width of the global-memory mode (-1: default)
static int g_hess_force_global = 0;
static int g_hess_pb = -2;
int hess_mode(int force_global, int pb) {
  g_hess_force_global = force_global;
  g_hess_pb = pb;
  return 0;
}

size_t hessenberg_ws(int64_t n, int k, int storage) {
  const int G = hess_grid(n);
  size_t b = 256 + (size_t)k * 8 + 256;
  b += (size_t)2 * G * 32 + 256;           // F64 slots
  b += (size_t)2 * G * k * sizeof(double);
  b += (size_t)2 * G * 16 + 256;            // slots
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
  h.key = (unsigned long long*)take((size_t)k * 8);
  OFRR_CUDA_TRY(cudaMemsetAsync(h.bar_count, 0, 256 + ((size_t)k * 8 + 255) / 256 * 256, st));
  h.slot64 = (double2*)take((size_t)2 * G * 32);
  h.cand_row = (double*)take((size_t)2 * G * k * sizeof(double));
  h.slot = (ulonglong2*)take((size_t)2 * G * 16);
  T* Xw = (T*)take((size_t)n * sizeof(T) * k);
  h.freerow = (unsigned char*)take(n);
  const T* Xp = (const T*)X;
  T* Qp = (T*)Q;
  int64_t ldw = n;
  const int64_t rows_per = (n + G - 1) / G;
  const size_t tile = (size_t)((rows_per + 3) & ~(int64_t)3) * k * sizeof(T);   // kernel: ldw % 4 == 0
  // up to the 227 KB opt-in per CTA (one CTA per SM): C3's fp32 rows (443 x 128) fit
  const size_t smem_max = 226 * 1024;
  // rows in shared memory: no panels (the per-step trailing update hides behind the grid
  // barrier).  Rows in global memory: panels of pb (32) columns cached in shared memory, the
  // columns beyond the panel updated once per panel (OFRR_HESS_PANEL overrides pb, <= 32)
  if (g_hess_pb == -2) { const char* e = getenv("OFRR_HESS_PANEL"); g_hess_pb = e ? atoi(e) : -1; }
  const int pb_env = g_hess_pb;
  auto pr_bytes = [&](int b) { return b > 1 ? (((size_t)(b * k + b * b) * sizeof(typename CT<C>::type) + 7) / 8) * 8 : 0; };
  const size_t base = (size_t)2 * k * sizeof(double);
  int in_smem = (base + tile + 16 <= smem_max && !g_hess_force_global) ? 1 : 0;
  int pb = 1;
  size_t shmem = base + (in_smem ? tile + 16 : 0);
  if (!in_smem) {
    for (int b = pb_env >= 1 ? std::min(pb_env, 32) : 32; b > 1; b /= 2) {
      const size_t need = base + pr_bytes(b) + (size_t)rows_per * b * sizeof(T) + 16;
      if (need <= smem_max) { pb = b; shmem = need; break; }
    }
  }
  static std::atomic<bool> attr{false};   // set once; concurrent callers may both set it (idempotent)
  if (!attr) {
    OFRR_CUDA_TRY(cudaFuncSetAttribute((const void*)k_hessenberg<T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem_max));
    attr = true;
  }
  (void)storage; (void)compute;
  void* args[] = {(void*)&Xp, (void*)&n, (void*)&k, (void*)&ldx, (void*)&Xw, (void*)&ldw, (void*)&tol,
                  (void*)&Qp, (void*)&ldq, (void*)&pivots, (void*)&kept, (void*)&n_kept, (void*)&h,
                  (void*)&in_smem, (void*)&pb};
  // kept[j] is written for every column by the kernel (kept or skipped): no clearing node
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
    case FP8 * 8 + F16: HESS(f8, F16);
    case FP8 * 8 + BF16: HESS(f8, BF16);
    case FP8 * 8 + F32: HESS(f8, F32);
    case FP8 * 8 + F64: HESS(f8, F64);
    default:
      ofrr_set_error("hessenberg: storage %d / compute %d unsupported", storage, compute);
      return OFRR_ERR_UNSUPPORTED;
  }
#undef HESS
}

}  // namespace ofrr
