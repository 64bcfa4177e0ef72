/* libm_fast.h — the reduced Taylor polynomials of the speculative LIF-range
 * evaluation (x in [-1/16, 0)), shared verbatim by the device (libm.cuh) and
 * the table generator (csrc/tools/gen_libm_tables.c), which records every
 * input whose rounded polynomial value differs from glibc's so that the
 * device's fix-up finds it in the table.  Plain C; IEEE double fma on both
 * sides gives identical results. */
#pragma once

#ifdef __CUDACC__
#define NENG_FAST_FN static __host__ __device__ __forceinline__
#else
#include <math.h>
#define NENG_FAST_FN static inline
#endif

/* x + x^2 sum_{k=2..7} x^(k-2)/k!   (relative error < 1e-13 on [-1/16, 0)) */
NENG_FAST_FN double neng_expm1_fast(double x) {
    double p = 1.9841269841269841e-04;
    p = fma(p, x, 1.3888888888888889e-03);
    p = fma(p, x, 8.3333333333333332e-03);
    p = fma(p, x, 4.1666666666666664e-02);
    p = fma(p, x, 1.6666666666666666e-01);
    p = fma(p, x, 0.5);
    return fma(x * x, p, x);
}

/* x + x^2 sum_{k=2..9} (-1)^(k+1) x^(k-2)/k   (relative error < 3e-11 on [-1/16, 0)) */
NENG_FAST_FN double neng_log1p_fast(double x) {
    double p = 1.0 / 9.0;
    p = fma(p, x, -1.0 / 8.0);
    p = fma(p, x, 1.0 / 7.0);
    p = fma(p, x, -1.0 / 6.0);
    p = fma(p, x, 1.0 / 5.0);
    p = fma(p, x, -1.0 / 4.0);
    p = fma(p, x, 1.0 / 3.0);
    p = fma(p, x, -0.5);
    return fma(x * x, p, x);
}
