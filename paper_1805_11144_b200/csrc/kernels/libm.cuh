// libm.cuh — device expm1f / log1pf that return exactly what the host's glibc
// returns (the reference's EngineCore<float> calls them in lif_spike_step,
// neuron_math.hpp:62,67, and lif_rate_t, :15).
//
// r = (float)f((double)x) is correctly rounded except where x lies within a
// double ulp of a float midpoint; glibc's float code is one ulp off r for a
// calibrated set of inputs.  Those inputs and glibc's results live in three
// open-addressing hash tables (Fibonacci hash, linear probing) built from
// data/libm_tables.bin at engine creation.  One probe (one 32-B sector) on a
// hit or a miss in the common case.
#pragma once

#include "program.hpp"

namespace nengb {

__device__ __forceinline__ float libm_lookup(const LibmHash& h, uint32_t key, float fallback) {
    uint32_t i = (key * 0x9E3779B1u) >> h.shift;
    for (;;) {
        unsigned long long s = __ldg(h.slots + i);
        if (s == 0ull) return fallback;
        if (static_cast<uint32_t>(s >> 32) == key) return __uint_as_float(static_cast<uint32_t>(s));
        i = (i + 1u) & h.mask;
    }
}

/// glibc expm1f for the inputs the LIF step produces (x = -delta/tau_rc <= 0).
__device__ __forceinline__ float glibc_expm1f(float x, const LibmTables& t) {
    if (x == 0.0f) return x;  // expm1(+-0) = +-0 exactly
    float r = static_cast<float>(expm1(static_cast<double>(x)));
    uint32_t k = __float_as_uint(x);
    if (k >= 0x80000001u && k <= 0xC2D00000u) return libm_lookup(t.t[0], k, r);
    return r;  // x < -104: both give -1; NaN: NaN
}

/// glibc log1pf over the whole float line.
__device__ __forceinline__ float glibc_log1pf(float x, const LibmTables& t) {
    if (x == 0.0f) return x;
    float r = static_cast<float>(log1p(static_cast<double>(x)));
    uint32_t k = __float_as_uint(x);
    if (k >= 0x80000001u && k <= 0xBF800000u) return libm_lookup(t.t[1], k, r);
    if (k >= 0x00000001u && k <= 0x7F7FFFFFu) return libm_lookup(t.t[2], k, r);
    return r;  // x < -1: NaN; +inf: +inf; NaN: NaN
}

/// lif_spike_step<float> (neuron_math.hpp:55-77), operation for operation.
/// No FMA contraction anywhere (built with -fmad=false).
__device__ __forceinline__ float lif_spike_step(float j, float& voltage, float& refractory, float dt, float tau_rc,
                                                float tau_ref, float amplitude, const LibmTables& t) {
    float delta = dt - refractory;
    if (delta < 0.0f) delta = 0.0f;
    if (delta > dt) delta = dt;
    float v = voltage - (j - voltage) * glibc_expm1f(-delta / tau_rc, t);
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
