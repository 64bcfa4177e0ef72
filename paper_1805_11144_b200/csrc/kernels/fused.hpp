// fused.hpp — descriptors of the fused ensemble pipeline (host + device).
//
// A recognised ensemble network is advanced with two phases per step and one
// grid barrier after each (fused.cu):
//   A  per (ensemble, 32-column batch tile):
//        in   = Reset payload + sum of incoming filtered values, plan order
//        J    = bias + E.in (sequential in j);  LIF step on v, r;  spikes as bits
//        xhat = Reset payload + sum over spiking i of D[r,i]*(amp/dt), i ascending
//   B  per (connection, batch column):
//        acc  = Reset payload + T.src (sequential);  state = filt = a*state + b*acc
// J, out, in and acc never touch HBM except on the last step of a call (so the
// arena holds the reference's full state at every call boundary).
#pragma once

#include <cstdint>

#include "program.hpp"

namespace nengb {

struct FEns {
    int64_t in_base, j_base, out_base, v_base, r_base, xhat_base;  // per-batch: element e, copy b at base + e*B + b
    int64_t enc_base, dec_base;                                    // shared: E [n][d], D [dx][n] row-major
    int32_t n, d, dx;                                              // neurons, input dims, decoded dims
    int32_t n_pad;                                                 // n rounded up to 4 (bulk-copy granularity)
    int32_t inc_begin, inc_count;                                  // incoming connections (plan order)
    int32_t in_init_off, xhat_init_off;                            // Reset payloads in `values`
    int64_t bias_off;        // Reset(J) payload, n_pad floats (16-B aligned)
    int64_t epad_off;        // encoders [n][DMAX], rows zero padded (16-B aligned)
    int64_t dec_scaled_off;  // fp32(D[r,i]) * fp32(amp/dt), transposed [n][dx] — the DotInc term of a spike
    int32_t dec_bytes;       // n*dx*4 rounded up to 16 (bulk-copy size)
    float dt, tau_rc, tau_ref, amplitude;
    float amp_dt;  // amplitude / dt (the spike value, exec: amplitude / dt)
    float em_dt;   // glibc expm1f(-dt / tau_rc): the refractory-free step
    double inv_tau_rc;  // 1 / (double)tau_rc
};

struct FConn {
    int64_t src_base;  // xhat of an ensemble or a fed node signal (per-batch)
    int64_t t_base;    // shared T [dd][ds]
    int64_t tpad_off;  // T rows zero padded to DMAX in `values` (16-B aligned)
    int64_t acc_base, filt_base, state_base;
    int32_t dd, ds;
    int32_t src_feed;  // feed slot index when the source is a fed node (read from the staged feeds), else -1
    int32_t acc_init_off;
    int32_t probe_filt, probe_state;  // probe indices capturing filt / state, -1 none
    float a, b;                       // lowpass coefficients (f32 of the f64 values)
};

struct FProbe {  // capture of a value not written in phase B
    int64_t base;  // arena base of the signal
    int32_t dim, per_batch;
    int32_t index;      // probe index (ring slot)
    int32_t feed_slot;  // >= 0: a fed node's signal (captured from the staged feeds when present)
};

struct FFeed {
    int64_t base;  // arena base of the fed signal
    int32_t dim, copies;
    int32_t slot;
};

struct FusedProgram {
    float* arena = nullptr;
    const float* values = nullptr;
    const FEns* ens = nullptr;
    const FConn* conns = nullptr;
    const int64_t* incoming = nullptr;  // per ensemble, plan order: arena base of each incoming filter state
    const FProbe* probes = nullptr;     // xhat / feed / other-phase-A-final captures
    const FFeed* feeds = nullptr;
    int32_t n_ens = 0, n_conn = 0, n_probes = 0, n_feeds = 0;
    int32_t batch = 1, btiles = 1, nmax = 0, nwords = 0;
    int32_t has_time = 0, time_probe_step = -1, time_probe_time = -1;
    int32_t stage_dec = 0;    // decoder products staged into shared memory (when they fit)
    int32_t pmax_floats = 0;  // max over ensembles of n*dx rounded up to 4
    int64_t step_base = 0, time_base = 0;
    float dt = 0.f;
    LibmTables libm;
    // per call
    const float* feed_data = nullptr;
    const int64_t* feed_off = nullptr;  // per slot
    const int32_t* feed_present = nullptr;
    float* ring = nullptr;
    const int64_t* ring_off = nullptr;  // per probe
    int32_t call_steps = 0;
    // optional section timers (NENG_FUSED_PROFILE=1): per-CTA ns summed over CTAs
    unsigned long long* prof = nullptr;
    int32_t* work = nullptr;  // two phase-A unit counters (step parity), zero at launch
};

enum FusedSection { FS_FEED, FS_A1, FS_A2, FS_FIX, FS_A3, FS_A4, FS_BAR1, FS_B, FS_BAR2, FS_COUNT };

}  // namespace nengb
