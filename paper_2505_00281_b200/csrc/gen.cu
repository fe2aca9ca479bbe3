// gen.cu -- K8b: the reference's seeded Gaussian-kernel test matrices evaluated on the device
// (the experiment harness's inputs; ofrr/matrix.py:97-113).
//
//   A_ij = f * (exp(-d2_ij / (2 l^2)) + s [square, i == j]),
//   d2_ij = max((|x_i|^2 + |y_j|^2) - 2 (x_i . y_j), 0)
//
// in FP64 with the reference's operation order: |x|^2 = x0 x0 + x1 x1 (numpy's two-term sum),
// x_i . y_j = fma(x1, y1, x0 y0) (the k = 2 BLAS dot of `x @ y.T`), the exponent argument
// (-d2) / ((2 l) l).  exp is CUDA's double exp (<= 1 ulp from the host's), then one rounding
// into the output format.  One thread per entry; row-major output (the operator layout).
#include "common.cuh"

namespace ofrr {

__global__ void __launch_bounds__(256)
    k_gaussian_kernel(const double* __restrict__ px, int64_t n, const double* __restrict__ py, int64_t m, double f,
                      double l, double s, void* __restrict__ out, int64_t ld, int fmt) {
  const int64_t j = (int64_t)blockIdx.x * 64 + (threadIdx.x & 63);
  const int64_t i = (int64_t)blockIdx.y * 4 + (threadIdx.x >> 6);
  if (i >= n || j >= m) return;
  const bool square = py == nullptr;
  const double* y = square ? px : py;
  const double x0 = px[2 * i], x1 = px[2 * i + 1];
  const double y0 = y[2 * j], y1 = y[2 * j + 1];
  const double sx = __dadd_rn(__dmul_rn(x0, x0), __dmul_rn(x1, x1));
  const double sy = __dadd_rn(__dmul_rn(y0, y0), __dmul_rn(y1, y1));
  const double dot = fma(x1, y1, __dmul_rn(x0, y0));
  double d2 = __dsub_rn(__dadd_rn(sx, sy), __dmul_rn(2.0, dot));
  d2 = d2 > 0.0 ? d2 : 0.0;
  const double t = __dmul_rn(__dmul_rn(2.0, l), l);
  double a = exp(__ddiv_rn(-d2, t));
  if (square && i == j) a = __dadd_rn(a, s);
  a = __dmul_rn(a, f);
  st_fmt(out, (long)(i * ld + j), fmt, rnd(a, fmt));
}

int gaussian_kernel(const double* px, int64_t n, const double* py, int64_t m, double f, double l, double s,
                    void* out, int64_t ld, int fmt, cudaStream_t st) {
  if (n <= 0 || m <= 0 || !px || !out || ld < m) {
    ofrr_set_error("gaussian_kernel: invalid arguments");
    return OFRR_ERR_INVALID;
  }
  const dim3 grid((unsigned)((m + 63) / 64), (unsigned)((n + 3) / 4));
  k_gaussian_kernel<<<grid, 256, 0, st>>>(px, n, py, m, f, l, s, out, ld, fmt);
  OFRR_CHECK_LAUNCH();
  return OFRR_OK;
}

}  // namespace ofrr
