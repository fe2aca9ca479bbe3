/*
 * ofrr_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU checker, never shipped).
 *
 * Plain-C restatement of the reference's compiled reduction kernels
 * (/root/reference/pkg/src/ofrr/_kernels.pyx, /root/reference/pkg/src/ofrr/halfround.h),
 * extended with the two formats the B200 path adds (bfloat16, fp8-e4m3).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Format codes follow ofrr/precision.py:20-25 (F16=0, F32=1, F64=2) and extend
 * them with BF16=3 and FP8_E4M3=4.
 *
 * Semantics (ofrr/_kernels.pyx:34-47): every product is rounded to the compute
 * format and accumulated index-ascending, rounding after every add into the
 * accumulate format.  All data travels as float64 holding format-representable
 * values.  Rounding a double to binary16 / bfloat16 goes through binary32 first,
 * which is exact by the 2p+2 double-rounding bound (ofrr/halfround.h:4-9).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

enum { F16 = 0, F32 = 1, F64 = 2, BF16 = 3, FP8E4M3 = 4 };

static inline double rnd_f32(double x) { return (double)(float)x; }   /* halfround.h:98 */

static inline double rnd_f16(double x) {                                /* halfround.h:17-20 */
    float f = (float)x;
    _Float16 h = (_Float16)f;            /* IEEE RNE, overflow -> inf, subnormals kept */
    return (double)(float)h;
}

static inline double rnd_bf16(double x) {
    float f = (float)x;
    uint32_t b;
    memcpy(&b, &f, 4);
    if ((b & 0x7f800000u) == 0x7f800000u) return (double)f;   /* inf / nan propagate */
    uint32_t lsb = (b >> 16) & 1u;
    b += 0x7fffu + lsb;                                         /* RNE on the low 16 bits */
    b &= 0xffff0000u;                                           /* overflow lands on inf */
    memcpy(&f, &b, 4);
    return (double)f;
}

/* e4m3 ("fn": no infinities): p=4, emin=-6, max finite 448.  Out-of-range values
 * become +-inf here so that the overflow diagnostic fires exactly as the
 * reference's binary16 overflow does (ofrr/precision.py:90-104). */
static inline double rnd_fp8e4m3(double x) {
    if (x == 0.0 || isnan(x) || isinf(x)) return x;
    double mag = fabs(x);
    int e;
    frexp(mag, &e);
    int q = e - 4;
    if (q < -6 - 4 + 1) q = -6 - 4 + 1;
    double r = ldexp(nearbyint(ldexp(mag, -q)), q);
    if (r > 448.0) r = INFINITY;
    return x < 0 ? -r : r;
}

static inline double rnd(double x, int code) {                          /* _kernels.pyx:26-31 */
    switch (code) {
    case F64: return x;
    case F32: return rnd_f32(x);
    case F16: return rnd_f16(x);
    case BF16: return rnd_bf16(x);
    default: return rnd_fp8e4m3(x);
    }
}

void oracle_round(const double* x, double* y, long n, int code) {
    for (long i = 0; i < n; ++i) y[i] = rnd(x[i], code);
}

/* _kernels.pyx:34-47 */
static double dot(const double* x, long incx, const double* y, long incy, long n,
                  int compute, int accumulate) {
    double acc = 0.0;
    if (compute == F64 && accumulate == F64) {
        for (long i = 0; i < n; ++i) acc = acc + x[i * incx] * y[i * incy];
        return acc;
    }
    for (long i = 0; i < n; ++i) {
        double p = rnd(x[i * incx] * y[i * incy], compute);
        acc = rnd(acc + p, accumulate);
    }
    return acc;
}

double oracle_dot_mixed(const double* x, const double* y, long n, int compute, int accumulate) {
    if (n == 0) return 0.0;
    return dot(x, 1, y, 1, n, compute, accumulate);
}

/*
 * _kernels.pyx:60-84.  C (m x n, column-major, ldc = m) = A (m x k, element (i,l) at
 * a[i*ars + l*acs]) times B (k x n, element (l,j) at b[l*brs + j*bcs]).
 * The loop is reordered (i outer, l middle, j inner) so the compiler vectorises
 * across output columns; every output entry still sees the identical
 * index-ascending sequence of rounded products and rounded adds.
 */
void oracle_gemm_mixed(const double* a, long ars, long acs, const double* b, long brs, long bcs,
                       long m, long k, long n, int compute, int accumulate, int out_fmt,
                       double* c) {
    if (m == 0 || n == 0) return;
    if (k == 0) { memset(c, 0, sizeof(double) * m * n); return; }
    double* acc = (double*)malloc(sizeof(double) * n);
    double* brow = (double*)malloc(sizeof(double) * n);
    for (long i = 0; i < m; ++i) {
        for (long j = 0; j < n; ++j) acc[j] = 0.0;
        const double* ai = a + i * ars;
        if (compute == F64 && accumulate == F64) {
            for (long l = 0; l < k; ++l) {
                double av = ai[l * acs];
                const double* bl = b + l * brs;
                for (long j = 0; j < n; ++j) acc[j] = acc[j] + av * bl[j * bcs];
            }
        } else if (compute == F32 && accumulate == F32) {
            for (long l = 0; l < k; ++l) {
                double av = ai[l * acs];
                const double* bl = b + l * brs;
                for (long j = 0; j < n; ++j) brow[j] = bl[j * bcs];
                for (long j = 0; j < n; ++j)
                    acc[j] = (double)(float)(acc[j] + (double)(float)(av * brow[j]));
            }
        } else {
            for (long l = 0; l < k; ++l) {
                double av = ai[l * acs];
                const double* bl = b + l * brs;
                for (long j = 0; j < n; ++j)
                    acc[j] = rnd(acc[j] + rnd(av * bl[j * bcs], compute), accumulate);
            }
        }
        for (long j = 0; j < n; ++j) c[i + j * m] = rnd(acc[j], out_fmt);
    }
    free(acc);
    free(brow);
}

/* _kernels.pyx:153-161 */
static double off_norm(const double* a, long n) {
    double ss = 0.0;
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < n; ++j)
            if (i != j) ss += a[i * n + j] * a[i * n + j];
    return sqrt(ss);
}

/*
 * _kernels.pyx:105-150: cyclic row-wise Jacobi on a C-order n x n copy `a`
 * (overwritten), eigenvectors into `v` (C-order, v[i*n+p] = V[i,p]).
 * Returns sweeps; *off_out receives the final off-diagonal norm.
 */
int oracle_jacobi_eig(double* a, double* v, long n, int max_sweeps, double tol, double* off_out) {
    for (long i = 0; i < n; ++i)
        for (long j = 0; j < n; ++j) v[i * n + j] = (i == j) ? 1.0 : 0.0;
    double off = off_norm(a, n);
    int sweeps = 0;
    while (off > tol && sweeps < max_sweeps) {
        double skip = off / (double)(n * n);
        for (long p = 0; p < n - 1; ++p) {
            for (long q = p + 1; q < n; ++q) {
                double apq = a[p * n + q];
                if (fabs(apq) <= skip) continue;
                double app = a[p * n + p], aqq = a[q * n + q];
                double theta = (aqq - app) / (2.0 * apq);
                double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                double c = 1.0 / sqrt(t * t + 1.0);
                double s = t * c;
                for (long i = 0; i < n; ++i) {
                    double tp = a[p * n + i], tq = a[q * n + i];
                    a[p * n + i] = c * tp - s * tq;
                    a[q * n + i] = s * tp + c * tq;
                }
                for (long i = 0; i < n; ++i) {
                    double tp = a[i * n + p], tq = a[i * n + q];
                    a[i * n + p] = c * tp - s * tq;
                    a[i * n + q] = s * tp + c * tq;
                }
                a[p * n + q] = 0.0;
                a[q * n + p] = 0.0;
                for (long i = 0; i < n; ++i) {
                    double tp = v[i * n + p], tq = v[i * n + q];
                    v[i * n + p] = c * tp - s * tq;
                    v[i * n + q] = s * tp + c * tq;
                }
            }
        }
        off = off_norm(a, n);
        sweeps += 1;
    }
    *off_out = off;
    return sweeps;
}

/*
 * ofrr/basis.py:151-196 (hessenberg_basis, right-looking layout; the reference
 * test tests/test_basis.py:92-98 pins left == right bitwise) with the axpy of
 * ofrr/precision.py:172-180 and the pivot rule of ofrr/basis.py:199-204.
 * x: n x k column-major (overwritten with the working block).
 * q: n x k column-major output, kept columns compacted to the front.
 * pivots[k], kept[k] (0/1).  Returns the number of kept columns.
 */
long oracle_hessenberg(double* x, long n, long k, int storage, int compute, double tol,
                       double* q, long* pivots, int* kept) {
    unsigned char* freerow = (unsigned char*)malloc(n);
    memset(freerow, 1, n);
    long nk = 0;
    for (long j = 0; j < k; ++j) {
        double* v = x + j * n;
        kept[j] = 0;
        long r = -1;
        double best = -1.0;
        for (long i = 0; i < n; ++i)
            if (freerow[i] && fabs(v[i]) > best) { best = fabs(v[i]); r = i; }
        if (r < 0 || fabs(v[r]) < tol) continue;
        double piv = v[r];
        for (long i = 0; i < n; ++i) v[i] = rnd(rnd(v[i] / piv, compute), storage);
        v[r] = 1.0;
        kept[j] = 1;
        freerow[r] = 0;
        pivots[nk] = r;
        memcpy(q + nk * n, v, sizeof(double) * n);
        nk++;
        for (long c = j + 1; c < k; ++c) {
            double* y = x + c * n;
            double alpha = rnd(y[r], compute);
            for (long i = 0; i < n; ++i) {
                double t = rnd(alpha * rnd(v[i], compute), compute);
                y[i] = rnd(rnd(rnd(y[i], compute) - t, compute), storage);
            }
        }
    }
    free(freerow);
    return nk;
}
