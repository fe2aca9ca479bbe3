// upload.cu -- symmetric operator upload: only one triangle of A crosses PCIe.
//
// The eigen path (ofrr/driver.py:84-111) is defined for symmetric A, and a caller that
// holds A on the host pays ~55 GB/s of PCIe for it -- the end-to-end solve at C3 is
// dominated by the 8 GiB host->device copy.  Like LAPACK's dsyev(uplo), the caller may
// declare which triangle of its row-major array is authoritative; the other triangle is
// never read.  Row block b of the triangle (rows [r0, r1), columns [r0, n) for 'U') goes
// over as one 2-D copy on the caller's stream; as soon as it lands, a mirror kernel on a
// side stream fills the transposed strip of the other triangle (columns [r0, r1), rows
// below the diagonal) from it, overlapping the next block's copy.  Bits are copied, not
// converted: the host array is already in the operator's storage format.
#include "common.cuh"
#include <algorithm>
#include <vector>

namespace ofrr {

// One 32 x 32 tile of the mirror.  UPPER: for j in [a0, a1) and i > j, A[i][j] = A[j][i]
// (source rows j in the strip, already uploaded).  !UPPER: A[j][i] = A[i][j] for the same
// (i, j) -- the lower triangle is the source and the strip is a row strip of the upper one.
template <typename E, bool UPPER>
__global__ void __launch_bounds__(256) k_mirror_strip(E* __restrict__ A, int64_t lda, int64_t n, int64_t a0,
                                                      int64_t a1) {
  __shared__ E tile[32][33];
  const int64_t j0 = a0 + (int64_t)blockIdx.x * 32;      // strip index (column of the lower triangle)
  const int64_t i0 = a0 + (int64_t)blockIdx.y * 32;      // other index (row of the lower triangle)
  if (i0 + 31 <= j0 || j0 >= a1) return;                 // tile entirely on or above the diagonal
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  // read the source tile: entries (j, i) = (j0 + y, i0 + x) of the upper triangle (UPPER), or
  // (i, j) = (i0 + y, j0 + x) of the lower one -- coalesced along x either way
  for (int y = ty; y < 32; y += 8) {
    if (UPPER) {
      const int64_t j = j0 + y, i = i0 + tx;
      if (j < a1 && i < n && i > j) tile[y][tx] = A[j * lda + i];
    } else {
      const int64_t i = i0 + y, j = j0 + tx;
      if (j < a1 && i < n && i > j) tile[y][tx] = A[i * lda + j];
    }
  }
  __syncthreads();
  for (int y = ty; y < 32; y += 8) {
    if (UPPER) {
      const int64_t i = i0 + y, j = j0 + tx;              // destination (i, j), i > j
      if (j < a1 && i < n && i > j) A[i * lda + j] = tile[tx][y];
    } else {
      const int64_t j = j0 + y, i = i0 + tx;              // destination (j, i), i > j
      if (j < a1 && i < n && i > j) A[j * lda + i] = tile[tx][y];
    }
  }
}

template <typename E>
static int mirror_strip(void* A, int64_t lda, int64_t n, int64_t a0, int64_t a1, bool upper, cudaStream_t st) {
  const dim3 grid((unsigned)((a1 - a0 + 31) / 32), (unsigned)((n - a0 + 31) / 32));
  if (upper) k_mirror_strip<E, true><<<grid, 256, 0, st>>>((E*)A, lda, n, a0, a1);
  else k_mirror_strip<E, false><<<grid, 256, 0, st>>>((E*)A, lda, n, a0, a1);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

int upload_sym(const void* host, int64_t ld_host, void* A, int64_t lda, int64_t n, int fmt, int uplo,
               int64_t block_rows, long long* bytes, cudaStream_t st) {
  if (!host || !A || n < 0 || ld_host < n || lda < n || (uplo != 0 && uplo != 1) || fmt < 0 || fmt > FP8) {
    ofrr_set_error("upload_sym: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  if (bytes) *bytes = 0;
  if (n == 0) return OFRR_OK;
  const int64_t es = fmt_bytes(fmt);
  const int64_t br = std::max<int64_t>(32, ((block_rows > 0 ? block_rows : 2048) + 31) / 32 * 32);
  const bool upper = uplo == 0;
  cudaStream_t ms;
  OFRR_CUDA_TRY(cudaStreamCreateWithFlags(&ms, cudaStreamNonBlocking));
  cudaEvent_t start;
  OFRR_CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  // the side stream starts after everything already queued on the caller's stream
  OFRR_CUDA_TRY(cudaEventRecord(start, st));
  OFRR_CUDA_TRY(cudaStreamWaitEvent(ms, start, 0));
  const int64_t nb = (n + br - 1) / br;
  std::vector<cudaEvent_t> ev((size_t)nb);
  long long moved = 0;
  int rc = OFRR_OK;
  // 'U': blocks in ascending order (strip b's sources are rows of block b); 'L': descending
  // (the upper part of rows [r0, r1) mirrors rows below r1, which arrive first)
  for (int64_t s = 0; s < nb && rc == OFRR_OK; ++s) {
    const int64_t b = upper ? s : nb - 1 - s;
    const int64_t r0 = b * br, r1 = std::min(n, r0 + br);
    const int64_t c0 = upper ? r0 : 0, c1 = upper ? n : r1;
    const char* src = (const char*)host + (r0 * ld_host + c0) * es;
    char* dst = (char*)A + (r0 * lda + c0) * es;
    if (cudaMemcpy2DAsync(dst, (size_t)(lda * es), src, (size_t)(ld_host * es), (size_t)((c1 - c0) * es),
                          (size_t)(r1 - r0), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[(size_t)b], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev[(size_t)b], st) != cudaSuccess || cudaStreamWaitEvent(ms, ev[(size_t)b], 0) != cudaSuccess) {
      ofrr_set_error("upload_sym: copy of row block %lld failed: %s", (long long)b,
                     cudaGetErrorString(cudaGetLastError()));
      rc = OFRR_ERR_CUDA;
      break;
    }
    moved += (long long)((c1 - c0) * es * (r1 - r0));
    switch (es) {
      case 1: rc = mirror_strip<uint8_t>(A, lda, n, r0, r1, upper, ms); break;
      case 2: rc = mirror_strip<uint16_t>(A, lda, n, r0, r1, upper, ms); break;
      case 4: rc = mirror_strip<uint32_t>(A, lda, n, r0, r1, upper, ms); break;
      default: rc = mirror_strip<uint64_t>(A, lda, n, r0, r1, upper, ms); break;
    }
  }
  // join: the caller's stream continues once the last strip is mirrored
  cudaEvent_t done;
  if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess) {
    cudaEventRecord(done, ms);
    cudaStreamWaitEvent(st, done, 0);
    cudaEventDestroy(done);
  } else if (rc == OFRR_OK) {
    rc = OFRR_ERR_CUDA;
  }
  for (auto& e : ev)
    if (e) cudaEventDestroy(e);
  cudaEventDestroy(start);
  cudaStreamDestroy(ms);   // released once its queued work completes
  if (bytes) *bytes = moved;
  return rc;
}

}  // namespace ofrr
