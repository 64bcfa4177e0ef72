// libm.cuh — device expm1f / log1pf that return exactly what the host's glibc
// returns (the reference's EngineCore<float> calls them in lif_spike_step,
// neuron_math.hpp:62,67, and lif_rate_t, :15).
//
// r = (float)f((double)x) is correctly rounded except where f(x) lies within
// a double ulp of a float midpoint; glibc's float code is ~0.53 ulp accurate
// and rounds one ulp away from r on a calibrated set of inputs, every one of
// which lies close to a rounding midpoint.  Those inputs and glibc's results
// live in open-addressing hash tables (Fibonacci hash, linear probing) built
// from data/libm_tables.bin, and the table is consulted only when the double
// result is within the calibrated distance of a midpoint (per 2^18-key region
// on the LIF range x in [-1/16, 0), where ~3% of calls qualify).  On that range
// f is a short Taylor polynomial in double (a few double ulps, far inside the
// 0.01-ulp margin); tests/test_libm_parity.py sweeps every float, device vs
// host, bit for bit.
#pragma once

#include "libm_fast.h"
#include "program.hpp"

namespace nengb {

__device__ __forceinline__ float probe_slots(const unsigned long long* slots, uint32_t mask, int shift,
                                             uint32_t key, float fallback) {
    uint32_t i = (key * 0x9E3779B1u) >> shift;
    for (;;) {
        unsigned long long s = __ldg(slots + i);
        if (s == 0ull) return fallback;
        if (static_cast<uint32_t>(s >> 32) == key) return __uint_as_float(static_cast<uint32_t>(s));
        i = (i + 1u) & mask;
    }
}

/// True when y is within (0.5 - from) float ulps of a float rounding midpoint.
__device__ __forceinline__ bool near_midpoint(double y, float from) {
    const float lo = __double2float_rd(y), hi = __double2float_ru(y);
    if (lo == hi) return false;  // y is a float: t = 0
    const double gap = static_cast<double>(hi) - static_cast<double>(lo);
    const double mid = 0.5 * (static_cast<double>(lo) + static_cast<double>(hi));
    return fabs(y - mid) <= (0.5 - static_cast<double>(from)) * gap;
}

/// Horner tail P(x) with f(x) = x + x^2 P(x) for x in [-1/16, 0):
///   log1p: sum_{k=2..16} (-1)^(k+1) x^(k-2)/k     expm1: sum_{k=2..10} x^(k-2)/k!
/// expm1's sequence is log1p's with leading zero coefficients, so one code
/// path serves both (fma(0, x, c) == c exactly).
__device__ __forceinline__ double small_f(double x, bool is_log) {
    double p = is_log ? -1.0 / 16.0 : 0.0;
    p = fma(p, x, is_log ? 1.0 / 15.0 : 0.0);
    p = fma(p, x, is_log ? -1.0 / 14.0 : 0.0);
    p = fma(p, x, is_log ? 1.0 / 13.0 : 0.0);
    p = fma(p, x, is_log ? -1.0 / 12.0 : 0.0);
    p = fma(p, x, is_log ? 1.0 / 11.0 : 0.0);
    p = fma(p, x, is_log ? -1.0 / 10.0 : 2.7557319223985893e-07);
    p = fma(p, x, is_log ? 1.0 / 9.0 : 2.7557319223985888e-06);
    p = fma(p, x, is_log ? -1.0 / 8.0 : 2.4801587301587302e-05);
    p = fma(p, x, is_log ? 1.0 / 7.0 : 1.9841269841269841e-04);
    p = fma(p, x, is_log ? -1.0 / 6.0 : 1.3888888888888889e-03);
    p = fma(p, x, is_log ? 1.0 / 5.0 : 8.3333333333333332e-03);
    p = fma(p, x, is_log ? -1.0 / 4.0 : 4.1666666666666664e-02);
    p = fma(p, x, is_log ? 1.0 / 3.0 : 1.6666666666666666e-01);
    p = fma(p, x, is_log ? -0.5 : 0.5);
    return fma(x * x, p, x);
}

// Out-of-range fallbacks stay out of line so the hot loops keep their registers.
static __device__ __noinline__ double expm1_wide(double x) { return expm1(x); }
static __device__ __noinline__ double log1p_wide(double x) { return log1p(x); }

__device__ __forceinline__ bool lif_range(float x) { return x >= -0.0625f && x < 0.0f; }

__device__ __forceinline__ float region_from(const LibmHash& h, uint32_t key) {
    return __ldg(h.region_from + ((key - 0x80000000u) >> h.region_shift));
}

// ---- the fast screen on the LIF range ----------------------------------
// Reduced Taylor polynomials (libm_fast.h), relative error < 3e-11 on
// [-1/16, 0): far below the screening window, so a value outside the window
// rounds exactly as the true value does (and as glibc does: every glibc
// exception lies inside).  Inside the window the rounded polynomial value is
// glibc's unless the input is in the table: the generator records every
// LIF-range input where the two differ, exceptions or not.
static __constant__ double kExpm1FastC[NENG_EXPM1_FAST_N] = NENG_EXPM1_FAST_C;
static __constant__ double kLog1pFastC[NENG_LOG1P_FAST_N] = NENG_LOG1P_FAST_C;
__device__ __forceinline__ double expm1_fast(double x) { return neng_poly_fast(x, kExpm1FastC, NENG_EXPM1_FAST_N); }
__device__ __forceinline__ double log1p_fast(double x) { return neng_poly_fast(x, kLog1pFastC, NENG_LOG1P_FAST_N); }

/// True when y lies within `win` x 2^-29 float ulps of a float rounding
/// midpoint (the low 29 mantissa bits of a double are the position between
/// two consecutive floats of its binade).  Results in the float-denormal
/// range are always reported (the exact path handles them).
__device__ __forceinline__ bool in_window(double y, uint32_t win) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(y));
    if (((u >> 52) & 0x7FFull) < 897ull) return true;  // |y| < 2^-126
    const uint32_t low = static_cast<uint32_t>(u) & 0x1FFFFFFFu;
    const uint32_t d = low > 0x10000000u ? low - 0x10000000u : 0x10000000u - low;
    return d <= win;
}

__device__ __forceinline__ uint32_t region_win(const LibmHash& h, uint32_t key) {
    return __ldg(h.region_win + ((key - 0x80000000u) >> h.region_shift));
}

/// Speculative evaluation on the LIF range: the value glibc returns unless
/// `doubtful` (then resolve exactly with glibc_expm1f / glibc_log1pf).
struct Spec {
    float r;
    bool doubtful;
};
__device__ __forceinline__ Spec spec_expm1(float x, const LibmTables& t) {
    const double y = expm1_fast(static_cast<double>(x));
    return {static_cast<float>(y), in_window(y, region_win(t.t[0], __float_as_uint(x)))};
}
__device__ __forceinline__ Spec spec_log1p(float x, const LibmTables& t) {
    const double y = log1p_fast(static_cast<double>(x));
    return {static_cast<float>(y), in_window(y, region_win(t.t[1], __float_as_uint(x)))};
}
__device__ __forceinline__ Spec spec_lif(float x, bool is_log, const LibmTables& t) {
    return is_log ? spec_log1p(x, t) : spec_expm1(x, t);
}

/// glibc expm1f.
__device__ __forceinline__ float glibc_expm1f(float x, const LibmTables& t) {
    if (x == 0.0f) return x;  // expm1(+-0) = +-0 exactly
    const uint32_t k = __float_as_uint(x);
    if (lif_range(x)) {
        const Spec s = spec_expm1(x, t);
        if (!s.doubtful) return s.r;
        const double y = small_f(static_cast<double>(x), false);
        const float r = static_cast<float>(y);
        return near_midpoint(y, region_from(t.t[0], k))
                   ? probe_slots(t.t[0].hot_slots, t.t[0].hot_mask, t.t[0].hot_shift, k, r)
                   : r;
    }
    const double y = expm1_wide(static_cast<double>(x));
    const float r = static_cast<float>(y);
    if (k >= 0x80000001u && k <= 0xC2D00000u && near_midpoint(y, t.t[0].lookup_from))
        return probe_slots(t.t[0].slots, t.t[0].mask, t.t[0].shift, k, r);
    return r;  // x < -104: both give -1; NaN: NaN; x > 0 never produced by the LIF step
}

/// glibc log1pf over the whole float line.
__device__ __forceinline__ float glibc_log1pf(float x, const LibmTables& t) {
    if (x == 0.0f) return x;
    const uint32_t k = __float_as_uint(x);
    if (lif_range(x)) {
        const Spec s = spec_log1p(x, t);
        if (!s.doubtful) return s.r;
        const double y = small_f(static_cast<double>(x), true);
        const float r = static_cast<float>(y);
        return near_midpoint(y, region_from(t.t[1], k))
                   ? probe_slots(t.t[1].hot_slots, t.t[1].hot_mask, t.t[1].hot_shift, k, r)
                   : r;
    }
    const double y = log1p_wide(static_cast<double>(x));
    const float r = static_cast<float>(y);
    if (k >= 0x80000001u && k <= 0xBF800000u) {
        if (near_midpoint(y, t.t[1].lookup_from)) return probe_slots(t.t[1].slots, t.t[1].mask, t.t[1].shift, k, r);
    } else if (k >= 0x00000001u && k <= 0x7F7FFFFFu) {
        if (near_midpoint(y, t.t[2].lookup_from)) return probe_slots(t.t[2].slots, t.t[2].mask, t.t[2].shift, k, r);
    }
    return r;  // x < -1: NaN; -1: -inf; +inf: +inf; NaN: NaN
}

/// Whether key is listed in the LIF-range table (an exception, or an input
/// where the speculative polynomial rounds differently from glibc).
/// The block filter: false means key is certainly not in the LIF-range table.
__device__ __forceinline__ bool hot_maybe(const LibmHash& h, uint32_t key) {
    const uint32_t k = key - 0x80000001u;  // key in the LIF range (callers check)
    return (__ldg(h.hot_filter + (k >> 11)) >> ((k >> 6) & 31u)) & 1u;
}

__device__ __forceinline__ bool hot_listed(const LibmHash& h, uint32_t key) {
    uint32_t i = (key * 0x9E3779B1u) >> h.hot_shift;
    for (;;) {
        const unsigned long long s = __ldg(h.hot_slots + i);
        if (s == 0ull) return false;
        if (static_cast<uint32_t>(s >> 32) == key) return true;
        i = (i + 1u) & h.hot_mask;
    }
}

/// The fused kernel's resolution of a value (fused.cu, A2 fix-up): on the LIF
/// range the speculation stands unless it is doubtful AND x is table-listed,
/// then the exact path decides.  Equal to glibc for every float (exhaustive test).
__device__ __forceinline__ float glibc_spec_resolved(float x, bool is_log, const LibmTables& t) {
    if (lif_range(x)) {
        const Spec s = spec_lif(x, is_log, t);
        if (!s.doubtful || !hot_maybe(t.t[is_log ? 1 : 0], __float_as_uint(x)) ||
            !hot_listed(t.t[is_log ? 1 : 0], __float_as_uint(x)))
            return s.r;
    }
    return is_log ? glibc_log1pf(x, t) : glibc_expm1f(x, t);
}

/// lif_spike_step<float> (neuron_math.hpp:55-77), operation for operation.
/// No FMA contraction anywhere (built with -fmad=false).
__device__ __forceinline__ float lif_spike_step(float j, float& voltage, float& refractory, float dt, float tau_rc,
                                                float tau_ref, float amplitude, const LibmTables& t, float em_dt) {
    float delta = dt - refractory;
    if (delta < 0.0f) delta = 0.0f;
    if (delta > dt) delta = dt;
    // delta == dt (not refractory): the same argument -dt / tau_rc every step, so em_dt
    // (the host's glibc expm1f of it) is the value expm1f returns here
    float v = voltage - (j - voltage) * (delta == dt ? em_dt : glibc_expm1f(-delta / tau_rc, t));
    if (v < 0.0f) v = 0.0f;
    float out;
    if (v > 1.0f) {
        float since_spike = -tau_rc * glibc_log1pf(-(v - 1.0f) / (j - 1.0f), t);
        out = amplitude / dt;
        voltage = 0.0f;
        refractory = tau_ref - since_spike;
    } else {
        out = 0.0f;
        voltage = v;
        refractory = refractory > dt ? refractory - dt : 0.0f;
    }
    return out;
}

/// amplitude * lif_rate_t<float>(j, tau_rc, tau_ref)  (neuron_math.hpp:12-16)
__device__ __forceinline__ float lif_rate_out(float j, float tau_rc, float tau_ref, float amplitude,
                                              const LibmTables& t) {
    float rate = j <= 1.0f ? 0.0f : 1.0f / (tau_ref + tau_rc * glibc_log1pf(1.0f / (j - 1.0f), t));
    return amplitude * rate;
}

/// relu_rate<float> (neuron_math.hpp:22-25)
__device__ __forceinline__ float relu_out(float j, float amplitude) { return j > 0.0f ? amplitude * j : 0.0f; }

}  // namespace nengb
