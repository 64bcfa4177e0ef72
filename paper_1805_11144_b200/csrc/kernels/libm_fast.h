/* libm_fast.h — the reduced Taylor polynomials of the speculative LIF-range
 * evaluation (x in [-1/16, 0)), shared verbatim by the device (libm.cuh) and
 * the table generator (csrc/tools/gen_libm_tables.c), which records every
 * input whose rounded polynomial value differs from glibc's so that the
 * device's fix-up finds it in the table.  Plain C; IEEE double fma on both
 * sides gives identical results.  The coefficients are lists so the device
 * can keep them in constant memory (DFMA reads a constant-bank operand
 * directly instead of materialising each double immediate). */
#pragma once

#ifdef __CUDACC__
#define NENG_FAST_FN static __host__ __device__ __forceinline__
#else
#include <math.h>
#define NENG_FAST_FN static inline
#endif

/* x + x^2 sum_{k=2..7} x^(k-2)/k!   (truncation error < 1e-13 relative on [-1/16, 0)) */
#define NENG_EXPM1_FAST_N 6
#define NENG_EXPM1_FAST_C                                                                              \
    {1.9841269841269841e-04, 1.3888888888888889e-03, 8.3333333333333332e-03, 4.1666666666666664e-02, \
     1.6666666666666666e-01, 0.5}

/* x + x^2 sum_{k=2..9} (-1)^(k+1) x^(k-2)/k   (relative error < 3e-11 on [-1/16, 0)) */
#define NENG_LOG1P_FAST_N 8
#define NENG_LOG1P_FAST_C \
    {1.0 / 9.0, -1.0 / 8.0, 1.0 / 7.0, -1.0 / 6.0, 1.0 / 5.0, -1.0 / 4.0, 1.0 / 3.0, -0.5}

/* x + x^2 P(x), P(x) = sum_k c[n-1-k] x^k by Horner from the highest coefficient. */
NENG_FAST_FN double neng_poly_fast(double x, const double* c, int n) {
    double p = c[0];
#ifdef __CUDACC__
#pragma unroll
#endif
    for (int k = 1; k < n; ++k) p = fma(p, x, c[k]);
    return fma(x * x, p, x);
}

#ifndef __CUDACC__
static const double neng_expm1_fast_c[NENG_EXPM1_FAST_N] = NENG_EXPM1_FAST_C;
static const double neng_log1p_fast_c[NENG_LOG1P_FAST_N] = NENG_LOG1P_FAST_C;
static inline double neng_expm1_fast(double x) { return neng_poly_fast(x, neng_expm1_fast_c, NENG_EXPM1_FAST_N); }
static inline double neng_log1p_fast(double x) { return neng_poly_fast(x, neng_log1p_fast_c, NENG_LOG1P_FAST_N); }
#endif
