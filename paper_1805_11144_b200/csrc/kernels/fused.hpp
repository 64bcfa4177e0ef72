// fused.hpp — descriptors of the fused ensemble pipeline (host + device).
//
// A recognised ensemble network advances with ONE grid barrier per step
// (fused.cu).  A unit is (ensemble, group of 32-column batch tiles); each warp
// of the CTA owns one tile (and a slice of the neurons when a unit has fewer
// tiles than warps).  For step k a unit
//   1. applies the step k-1 update of every connection INTO its ensemble
//      (destination side):  acc = Reset payload + T.src(k-1);
//      state = filt = a*state + b*acc           (exec.cpp:226-240, 267-284)
//      and sums in = Reset payload + filt_c in plan-group order (exec.cpp:189-210);
//   2. sweeps its neurons: J = bias + E.in (sequential in j), lif_spike_step;
//      neurons whose step needs a transcendental (a spike: log1p; leaving the
//      refractory period: expm1) leave the sweep through warp queues and are
//      resolved 32 at a time;
//   3. decodes xhat = Reset payload + sum over spiking i (ascending) of
//      D[r,i]*(amp/dt) into the step-parity buffer xbuf[k & 1] (xbuf[k % 3]
//      when stepping barrier-free, see FusedProgram::dataflow).
// The update of step k-1 for connections without a destination ensemble, the
// probe captures of step k-1 and the clock run at the start of step k; the
// launch's last step is completed by an epilogue after a final barrier.
//
// Ensemble sharding (one engine per GPU): a shard owns a contiguous range of
// ensembles and the connections into them; its units write xhat rows
// [rank * stride, ...) of the parity buffer, which the host all-gathers
// between per-step launches (first_update / epilogue select the pieces).
// J, out, in, acc and filt reach the arena on a call's last step only, so the
// arena holds the reference's full state at every call boundary.
#pragma once

#include <cstdint>

#include "program.hpp"

namespace nengb {

struct FEns {
    int64_t in_base, j_base, out_base, v_base, r_base, xhat_base;  // per-batch: element e, copy b at base + e*B + b
    int32_t n, d, dx;                                              // neurons, input dims, decoded dims
    int32_t n_pad;                                                 // n rounded up to 4 (bulk-copy granularity)
    int32_t inc_begin, inc_count;                                  // incoming connections (plan order) in `incoming`
    int32_t in_init_off, xhat_init_off;                            // Reset payloads in `values`
    int32_t xb_row;          // first row of this ensemble's xhat in the parity buffers
    int64_t bias_off;        // Reset(J) payload, n_pad floats (16-B aligned)
    int64_t epad_off;        // encoders [n (even) / 2][DMAX][2] (neuron pairs interleaved), rows zero padded (16-B aligned)
    int64_t dec_scaled_off;  // fp32(D[r,i]) * fp32(amp/dt), transposed [n][dx] — the DotInc term of a spike
    int32_t dec_bytes;       // n*dx*4 rounded up to 16 (bulk-copy size)
    float dt, tau_rc, tau_ref, amplitude;
    float amp_dt;  // amplitude / dt (the spike value, exec: amplitude / dt)
    float em_dt;   // glibc expm1f(-dt / tau_rc): the refractory-free step
    double inv_tau_rc;  // 1 / (double)tau_rc
    // barrier-free stepping (FusedProgram::dataflow): index ranges into deps / ens_orph / xprobes
    int32_t dep_begin, dep_count;    // (ensemble << 1) | lag: wait for done >= t - lag
    int32_t orph_begin, orph_count;  // destination-less connections this ensemble feeds
    int32_t xp_begin, xp_count;      // captures of this ensemble's xhat
    int32_t sc_begin, sc_count;      // captures of its neuron state: (FStateCap kind, probe index) pairs in scaps
};

/// Probes on an ensemble's own per-neuron signals, captured by the unit that
/// steps it (capture_probes, exec.cpp:328-338): the spike output, the voltage
/// and refractory state after the step, and the input current J.
enum FStateCap : int32_t { SC_OUT = 0, SC_VOLTAGE = 1, SC_REFRACTORY = 2, SC_J = 3 };

struct FConn {
    int64_t src_base;  // arena base of the source signal (an ensemble's xhat or a fed node)
    int64_t tpad_off;  // T rows zero padded to DMAX in `values` (16-B aligned)
    int64_t acc_base, filt_base, state_base;
    int32_t dd, ds;
    int32_t src_xb;    // first parity-buffer row of the source ensemble's xhat, or -1
    int32_t src_ens;   // the source ensemble (global index), or -1
    int32_t src_feed;  // feed slot index when the source is a fed node, else -1
    int32_t acc_init_off;
    int32_t probe_filt, probe_state;  // probe indices capturing filt / state, -1 none
    float a, b;                       // lowpass coefficients (f32 of the f64 values)
};

struct FProbe {  // capture of a value the units produce (xhat) or a fed node
    int64_t base;  // arena base of the signal
    int32_t dim, per_batch;
    int32_t index;      // probe index (ring slot)
    int32_t feed_slot;  // >= 0: a fed node's signal (captured from the staged feeds when present)
    int32_t xb_row;     // >= 0: an ensemble's xhat (captured from the parity buffer)
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
    const int32_t* incoming = nullptr;  // per ensemble, plan order: connection indices
    const int32_t* orphans = nullptr;   // connections with no destination ensemble (updated by shard 0)
    const int32_t* my_conns = nullptr;  // connections this shard updates: into its ensembles (+ orphans on shard 0)
    const FProbe* probes = nullptr;
    const FFeed* feeds = nullptr;
    float* xbuf = nullptr;  // two parity buffers of xrows rows x B
    int32_t n_ens = 0, n_conn = 0, n_orphans = 0, n_probes = 0, n_feeds = 0, n_my_conns = 0;
    int32_t ens_lo = 0, ens_hi = 0;  // this shard's ensembles (all of them unsharded)
    int32_t xrows = 0;
    int32_t batch = 1, btiles = 1, nmax = 0;
    int32_t tu = 8, slices = 1, groups = 1;  // tiles per unit, warps per tile, units per ensemble
    int32_t has_time = 0, time_probe_step = -1, time_probe_time = -1;
    int32_t stage_dec = 0;    // decoder products staged into shared memory (when they fit)
    int32_t small_words = 0;  // fused_small_kernel: spike words, sum over ensembles of B * ceil(n / 32)
    int32_t small_pfloats = 0;  // fused_small_kernel: decoder products staged in shared memory (sum n*dx), or 0
    int32_t pmax_floats = 0;  // max over ensembles of n*dx rounded up to 4
    int64_t step_base = 0, time_base = 0;
    float dt = 0.f;
    uint64_t neg_zero2 = 0x8000000080000000ull;  // (-0, -0): the addend of an exact paired product (fused.cu)
    LibmTables libm;
    // per call
    const float* feed_data = nullptr;
    const int64_t* feed_off = nullptr;  // per slot
    const int32_t* feed_present = nullptr;
    float* ring = nullptr;
    const int64_t* ring_off = nullptr;  // per probe
    int32_t call_steps = 0;
    int32_t first_update = 0;  // apply the step k_begin-1 connection updates at k_begin (stepped / sharded runs)
    int32_t epilogue = 1;      // complete the launch's last step (connection updates, captures, clock)
    // optional section timers (NENG_FUSED_PROFILE=1): per-CTA ns summed over CTAs
    unsigned long long* prof = nullptr;
    int32_t* work = nullptr;  // two unit counters (step parity), zero at launch
    // barrier-free stepping (unsharded runs): unit (e, g) of step t waits for
    // done[s, g] >= t of its sources and itself and done[d, g] >= t - 1 of its
    // destinations (xbuf is triple-buffered: slot k % 3), then publishes
    // done[e, g] = t + 1.  Units are claimed in `order` (a permutation that keeps
    // a unit's sources away from the end of the previous step), so there is no
    // grid barrier and no end-of-step tail; one barrier before the epilogue.
    int32_t dataflow = 0;
    int32_t* done = nullptr;            // per unit (local index), zero at launch
    const int32_t* order = nullptr;     // claim position -> unit
    const int32_t* deps = nullptr;      // FEns::dep_*
    const int32_t* ens_orph = nullptr;  // FEns::orph_*
    const int32_t* xprobes = nullptr;   // FEns::xp_*: indices into probes
    const int32_t* scaps = nullptr;     // FEns::sc_*: (FStateCap, probe index) pairs
    const int32_t* free_orph = nullptr;   // destination-less connections from fed / constant sources
    int32_t n_free_orph = 0;
    const int32_t* dest_conns = nullptr;  // connections into an ensemble (the epilogue's)
    int32_t n_dest_conns = 0;
    // fault localisation (builds with -DNENG_FUSED_TRACE, run with NENG_FUSED_TRACE=1): per warp
    // (checkpoint, value) pairs in host-mapped memory, readable after the context has faulted
    int32_t* trace = nullptr;
};

enum FusedSection { FS_DEFER, FS_IN, FS_SWEEP, FS_QUEUE, FS_FIX, FS_DECODE, FS_BAR, FS_EPI, FS_COUNT };

}  // namespace nengb
