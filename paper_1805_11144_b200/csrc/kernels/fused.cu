// fused.cu — the fused ensemble pipeline: one persistent cooperative kernel
// advancing K timesteps with ONE grid barrier per step (see fused.hpp).
//
// Unit = (ensemble, group of tu 32-column batch tiles), claimed dynamically by
// CTAs; each warp owns one tile (lane = batch column) and, when a unit has
// fewer tiles than warps, a slice of the neurons.
//   * encoders, biases and (when they fit) decoder spike products are staged
//     into shared memory by bulk copies (cp.async.bulk + mbarrier) issued at
//     unit start, overlapping the connection updates;
//   * the connection updates of step k-1 run on the destination side, so the
//     filter state is read and written once per step and the only cross-CTA
//     data is xhat, double-buffered by step parity;
//   * the neuron sweep streams v/r coalesced ([row][B] arena layout, 128 B per
//     warp access, evict-first) and does the common LIF step inline; the two
//     transcendental branches (log1p at a spike, expm1 on the step a neuron
//     leaves its refractory period — each taken by ~25% of neuron-updates on
//     the config-4 network) leave through warp-aggregated shared-memory queues
//     (ballot + popc, no atomics) and are evaluated 32 at a time, one per lane,
//     so their cost follows the spike rate instead of P(any lane of 32);
//   * transcendentals use a double Taylor polynomial whose rounding is glibc's
//     except inside a calibrated window next to float rounding midpoints; a
//     doubtful value goes to a third queue that resolves it exactly (table
//     probes) and patches v, r and the spike bit;
//   * spikes are ballot words (bit = column); the decoder transposes 32x32 bit
//     blocks with shuffles and walks each column's set bits in ascending neuron
//     order, adding the precomputed products fp32(D[r,i]) * fp32(amp/dt).
// Zero padding (encoder rows and transforms to DMAX) and skipping non-spiking
// neurons are exact: a running sum that starts at +0 is never -0, and
// x + (+-0) == x for every x, so the extra +0 terms change no bit.
//
// Every other floating-point operation is the reference's, in its order:
//   in   : Reset payload, then += filtered_c for c in plan-group order (exec.cpp:189-210)
//   J    : bias + (0 + E[i,0]in0 + E[i,1]in1 + ...)                      (exec.cpp:226-240)
//   LIF  : lif_spike_step<float>                                         (neuron_math.hpp:55-77)
//   xhat : payload + (0 + sum_i D[r,i]*out[i])                            (exec.cpp:226-240)
//   acc  : payload + (0 + sum_j T[r,j]*src[j]);  f = a*state + b*acc      (exec.cpp:267-284)
#include <algorithm>
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "fused.hpp"
#include "libm.cuh"

namespace cg = cooperative_groups;

namespace nengb {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;   // neuron rows per prefetch round (pairs inside)
constexpr int kMinBlocks = 3;  // CTAs per SM the register budget is sized for
#ifndef NENG_L2_AHEAD
#define NENG_L2_AHEAD 24
#endif
constexpr int kL2Ahead = NENG_L2_AHEAD;  // rows of v/r pulled into L2 ahead of the round being computed
constexpr uint32_t kFull = 0xffffffffu;


__device__ __forceinline__ void grid_sync(cg::grid_group& g) {
    if (gridDim.x == 1)
        __syncthreads();
    else
        g.sync();
}

// ---- bulk copy + mbarrier (sm_90+ async proxy) -------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}
/// ld.shared.f32 at a 32-bit shared-window address (no generic-to-shared conversion).
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
/// Pull `bytes` (multiple of 16, 16-B aligned) of global memory into L2 (TMA prefetch).
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(p), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
#ifdef NENG_FUSED_TRACE
#define FTRACE(cp, val)                                                                             \
    do {                                                                                           \
        if (p.trace && (threadIdx.x & 31) == 0) {                                                  \
            volatile int32_t* t_ = p.trace + 2 * (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)); \
            t_[0] = (cp);                                                                          \
            t_[1] = (val);                                                                         \
            __threadfence_system();                                                                \
        }                                                                                          \
    } while (0)
#else
#define FTRACE(cp, val) \
    do {                \
    } while (0)
#endif

// Paired fp32 arithmetic.  ptxas contracts mul.rn.f32x2 feeding add.rn.f32x2
// into FFMA2 (one rounding) even under -fmad=false, so a paired product is
// formed as fma(a, b, -0) — exactly the rounded product (x + -0 == x for every
// x, -0 included) — with the -0 pair from the kernel parameters, which ptxas
// cannot fold away (tests/test_abi.py checks every FFMA2's addend in the SASS).
__device__ __forceinline__ uint64_t pk2(float a, float b) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float2 unpk2(uint64_t v) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
    return r;
}
__device__ __forceinline__ uint64_t mul2_exact(uint64_t a, uint64_t b, uint64_t neg_zero2) {
    uint64_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(neg_zero2));
    return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

/// Encoder element (i, j) in the pair-interleaved layout [i / 2][DMAX][2].
template <int DMAX>
__device__ __forceinline__ float enc_at(const float* E, int i, int j) {
    return E[(i >> 1) * 2 * DMAX + j * 2 + (i & 1)];
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- optional section timers (PROF instantiation; thread 0 of each CTA) ----
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
template <bool PROF>
struct Ticker {
    unsigned long long acc[PROF ? FS_COUNT : 1];
    unsigned long long t;
    __device__ __forceinline__ void start() {
        if constexpr (PROF) {
            for (int s = 0; s < FS_COUNT; ++s) acc[s] = 0;
            t = gtime();
        }
    }
    __device__ __forceinline__ void tick(int section) {
        if constexpr (PROF) {
            if (threadIdx.x == 0) {
                const unsigned long long now = gtime();
                acc[section] += now - t;
                t = now;
            }
        }
    }
    __device__ __forceinline__ void flush(unsigned long long* out) {
        if constexpr (PROF) {
            if (threadIdx.x == 0)
                for (int s = 0; s < FS_COUNT; ++s) atomicAdd(out + s, acc[s]);
        }
    }
};

/// A queued neuron step (exception queues, see run_unit): key = neuron << 5 | lane.
///   exit queue  (the step leaving the refractory period): a, b, c = the step's v, r, J
///   spike queue (a spike; v = 0 is already stored):       a, b    = the pre-reset voltage, J
struct __align__(16) QEnt {
    uint32_t key;
    float a, b, c;
};
constexpr int kQ = 64;  // per-warp queue capacity: <= 31 pending + 32 from a row (drained at >= 32)

struct Smem {
    uint64_t* bar;
    uint64_t* bar2;  // the decoder products' copy into the encoder region (when not staged up front)
    int* cur;      // the CTA's current unit
    float* E;      // nmax x DMAX (zero padded)
    float* bias;   // nmax
    float* P;      // decoder products [n][dx] (when p.stage_dec)
    float* in;     // tu x DMAX x 32 (aliases the queues: read into registers before the sweep)
    uint32_t* words;  // tu x nmax: spike ballot of neuron i in tile slot t (bit = lane)
    float* ring;      // kWarps x [2 stages][v, r][kUnroll rows][32]
    QEnt* qe;         // kWarps x kQ exit-queue entries
    QEnt* qs;         // kWarps x kQ spike-queue entries
};

constexpr int kRingFloats = 2 * 2 * kUnroll * 32;  // per warp
// The rings of the CTA's warps are interleaved: row `row` of stage `st` of array
// `arr` (v = 0, r = 1) is line (arr * 2 + st) * kUnroll + row of kRowB bytes,
// warp w's 32 columns at w * 128; a lane's address is then base + threadIdx.x * 4
// plus a row offset (nothing warp-dependent to keep live across the sweep).
constexpr uint32_t kRowB = kWarps * 32 * 4;
constexpr size_t kQueueBytes = 2 * sizeof(QEnt) * kQ * kWarps;

/// Bytes of the region shared by the input staging `in` and the queues.
template <int DMAX>
__host__ __device__ __forceinline__ size_t inq_bytes(const FusedProgram& p) {
    const size_t in = static_cast<size_t>(p.tu) * DMAX * 32 * 4;
    return in > kQueueBytes ? in : kQueueBytes;
}

template <int DMAX>
__device__ Smem carve(uint32_t* base, const FusedProgram& p) {
    Smem S;
    char* at = reinterpret_cast<char*>(base);
    S.bar = reinterpret_cast<uint64_t*>(at);
    S.cur = reinterpret_cast<int*>(at + 8);
    S.bar2 = reinterpret_cast<uint64_t*>(at + 16);
    at += 128;
    S.ring = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(kWarps) * kRingFloats * 4;
    S.qe = reinterpret_cast<QEnt*>(at);
    S.qs = S.qe + kQ * kWarps;
    S.in = reinterpret_cast<float*>(at);
    at += inq_bytes<DMAX>(p);
    S.E = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.nmax) * DMAX * 4;
    S.bias = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.nmax) * 4;
    S.P = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.stage_dec ? p.pmax_floats : 0) * 4;
    S.words = reinterpret_cast<uint32_t*>(at);
    at += static_cast<size_t>(p.tu) * p.nmax * 4;
    return S;
}

template <int DMAX>
__host__ __device__ size_t smem_bytes(const FusedProgram& p) {
    return 128 + static_cast<size_t>(kWarps) * kRingFloats * 4 + inq_bytes<DMAX>(p) +
           static_cast<size_t>(p.nmax) * DMAX * 4 + static_cast<size_t>(p.nmax) * 4 +
           static_cast<size_t>(p.stage_dec ? p.pmax_floats : 0) * 4 + static_cast<size_t>(p.tu) * p.nmax * 4;
}

/// The batch width: BT when the kernel is specialised for it (row strides then
/// fold into load/store immediates), else the program's.
template <int BT>
__device__ __forceinline__ int batch_of(const FusedProgram& p) {
    if constexpr (BT > 0)
        return BT;
    else
        return p.batch;
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// No L2::cache_hint operand on cp.async: for some kernel shapes (the BT = 0
// instances) ptxas 12.9 encodes the hinted LDGSTS with its 64-bit memory
// descriptor in an odd uniform register (desc[UR1]), which faults at run time
// with "illegal instruction"; tests/test_abi.py scans the SASS for it.
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4_s(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}

/// The speculative LIF-range evaluation of libm.cuh (expm1_fast / log1p_fast)
/// with the per-region screen read from the byte table (8 KB, L1-resident):
/// doubtful when |low29 - 2^28| >> 21 <= w8 (a superset of the exact window,
/// so every value the exact screen flags is flagged here too), when the result
/// is a float denormal, or when x is outside the LIF range [-1/16, 0).
__device__ __forceinline__ Spec spec_any(float x, bool is_log, const uint8_t* w8, uint32_t shift) {
    const uint32_t k = __float_as_uint(x) - 0x80000001u;  // x in [-1/16, 0) <=> k <= 0x3D7FFFFF
    const bool inr = k <= 0x3D7FFFFFu;
    const double y = is_log ? log1p_fast(static_cast<double>(x)) : expm1_fast(static_cast<double>(x));
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(y));
    const uint32_t hi = static_cast<uint32_t>(u >> 32), lo = static_cast<uint32_t>(u);
    const bool den = (hi & 0x7FF00000u) < (897u << 20);  // |y| < 2^-126: float-denormal result
    const uint32_t d = static_cast<uint32_t>(abs(static_cast<int>(lo & 0x1FFFFFFFu) - 0x10000000));
    const uint32_t w = __ldg(w8 + (min(k + 1u, 0x3D800000u) >> shift));
    return {static_cast<float>(y), !inr || den || (d >> 21) <= w};
}

/// glibc's value of expm1f / log1pf (is_log) at x on the LIF range, without the
/// slow paths: the rounded polynomial unless it is doubtful and x is listed in
/// the bucketed table (then the table value).  Returns false when only the
/// exact path can decide (x outside the LIF range, or a full bucket).  The
/// table pointers come from the kernel parameters (constant bank), so nothing
/// of this stays live in registers across the sweep.
__device__ __forceinline__ bool glibc_fast(float x, bool is_log, const LibmTables& lt, float* out) {
    const LibmHash& h = lt.t[is_log ? 1 : 0];
    const Spec sp = spec_any(x, is_log, h.region_w8, h.region_shift);
    *out = sp.r;
    if (!sp.doubtful) return true;
    const uint32_t ka = __float_as_uint(x);
    if (ka - 0x80000001u > 0x3D7FFFFFu) return false;  // outside the LIF range
    const uint32_t bi = (ka * 0x9E3779B1u) >> h.bucket_shift;
    const uint4 bk = __ldg(h.hot_buckets + bi);
    const int j = bk.x == ka ? 0 : bk.y == ka ? 1 : bk.z == ka ? 2 : bk.w == ka ? 3 : -1;
    if (j < 0) return !(bk.x && bk.y && bk.z && bk.w);  // not listed (its home bucket has room)
    *out = __uint_as_float(__ldg(h.bucket_results + bi * 4 + j));  // listed: glibc's value
    return true;
}

/// glibc expm1f / log1pf for any float (out of line and rare: arguments outside
/// the LIF range and full buckets; tests/test_libm_parity.py sweeps every float).
__device__ __noinline__ float glibc_exact(float x, bool is_log, const LibmTables* lt) {
    return glibc_spec_resolved(x, is_log, *lt);
}

__device__ __forceinline__ float glibc_value(float x, bool is_log, const FusedProgram& p) {
    float y;
    return glibc_fast(x, is_log, p.libm, &y) ? y : glibc_exact(x, is_log, &p.libm);
}

/// Speculative glibc value (libm.cuh): the rounded polynomial, and whether it
/// may differ from glibc's (then the lane's step is recomputed by a doubt batch).
__device__ __forceinline__ float glibc_spec(float x, bool is_log, const FusedProgram& p, bool& doubtful) {
    const LibmHash& h = p.libm.t[is_log ? 1 : 0];
    const Spec sp = spec_any(x, is_log, h.region_w8, h.region_shift);
    doubtful = doubtful || sp.doubtful;
    return sp.r;
}

/// lif_spike_step<float> (neuron_math.hpp:55-77) of one lane from its step's
/// v, r, J; F(x, is_log) evaluates expm1f / log1pf.  Returns whether it spiked.
template <typename F>
__device__ __forceinline__ bool lif_step(float J, float& v, float& r, float dt, float em_dt, double inv_tau_rc,
                                         float tau_rc, float tau_ref, F&& f) {
    float delta = dt - r;
    if (delta < 0.0f) delta = 0.0f;
    if (delta > dt) delta = dt;
    float em;
    if (delta == dt) {
        em = em_dt;  // expm1f(-dt / tau_rc): the host's glibc value
    } else if (delta == 0.0f) {
        em = -0.0f;  // expm1f(-0)
    } else {
        // == -delta / tau_rc in IEEE float: the double product is within 2^-52 of the quotient,
        // and a quotient of floats is never within 2^-49 of a float midpoint unless on it,
        // which needs a power-of-two divisor (then the product is exact)
        em = f(static_cast<float>(static_cast<double>(-delta) * inv_tau_rc), false);
    }
    float vn = v - (J - v) * em;
    if (vn < 0.0f) vn = 0.0f;
    if (vn > 1.0f) {
        const float since = -tau_rc * f(-(vn - 1.0f) / (J - 1.0f), true);
        v = 0.0f;
        r = tau_ref - since;
        return true;
    }
    v = vn;
    r = r > dt ? r - dt : 0.0f;
    return false;
}

/// The exception queue's batch (lane l takes entry l of q[0, cnt)): the whole
/// step of a neuron whose step needs a transcendental — it leaves the
/// refractory period (0 < delta < dt, or NaN: expm1f) or it spikes (log1pf) —
/// recomputed from its v, r, J with the speculative values.  v, r and the spike
/// bit are written; a lane whose value was doubtful joins the doubt queue and
/// is recomputed exactly by doubt_batch.  Returns the new doubt count.
template <int BT>
__device__ __forceinline__ int exc_batch(const FusedProgram& p, const FEns* ep, float* vcol, int64_t rdelta,
                                         const QEnt* q, int cnt, QEnt* qd, int nd, uint32_t* words) {
    const int lane = threadIdx.x & 31;
    const bool on = lane < cnt;
    const QEnt x = on ? q[lane] : QEnt{0u, 0.0f, 0.0f, 0.0f};  // idle lanes: delta = dt, no spike
    float v = x.a, r = x.b;
    bool doubtful = false;
    const bool spike = lif_step(x.c, v, r, __ldg(&ep->dt), __ldg(&ep->em_dt), __ldg(&ep->inv_tau_rc),
                                __ldg(&ep->tau_rc), __ldg(&ep->tau_ref),
                                [&](float a, bool is_log) { return glibc_spec(a, is_log, p, doubtful); });
    const uint32_t i = x.key >> 5, col = x.key & 31u;
    if (on) {
        float* vp = vcol + static_cast<int64_t>(i) * (BT > 0 ? BT : p.batch) + col;
        vp[0] = v;
        vp[rdelta] = r;
        if (spike) atomicOr(words + i, 1u << col);  // exit lanes' bits are 0; spiking lanes' already set
    }
    const bool d = on && doubtful;
    const uint32_t m = __ballot_sync(kFull, d);
    if (d) qd[nd + __popc(m & lanemask_lt())] = x;
#ifdef NENG_FUSED_CHECKS
    if (nd + __popc(m) > kQ) {
        printf("fused check: doubt queue overflow %d\n", nd + __popc(m));
        __trap();
    }
#endif
    return nd + __popc(m);
}

/// The doubt queue's batch: the step recomputed with glibc's exact values
/// (bucketed table, else the exact path); v, r and the spike bit rewritten.
template <int BT>
__device__ __forceinline__ void doubt_batch(const FusedProgram& p, const FEns* ep, float* vcol, int64_t rdelta,
                                            const QEnt* q, int cnt, uint32_t* words) {
    const int lane = threadIdx.x & 31;
    if (lane >= cnt) return;
    const QEnt x = q[lane];
    float v = x.a, r = x.b;
    const bool spike = lif_step(x.c, v, r, __ldg(&ep->dt), __ldg(&ep->em_dt), __ldg(&ep->inv_tau_rc),
                                __ldg(&ep->tau_rc), __ldg(&ep->tau_ref),
                                [&](float a, bool is_log) { return glibc_value(a, is_log, p); });
    const uint32_t i = x.key >> 5, col = x.key & 31u;
    float* vp = vcol + static_cast<int64_t>(i) * (BT > 0 ? BT : p.batch) + col;
    vp[0] = v;
    vp[rdelta] = r;
    if (spike)
        atomicOr(words + i, 1u << col);
    else
        atomicAnd(words + i, ~(1u << col));
}

// ---- connections ----------------------------------------------------------

/// The xhat buffer slot of step k: parity (two slots) with a barrier per step,
/// k % 3 when stepping barrier-free (a slot is rewritten only after the
/// destinations that read it have finished the step after).
__device__ __forceinline__ int64_t xslot(const FusedProgram& p, int k) {
    return p.dataflow ? k % 3 : k & 1;
}

/// Step-kk update of connection cn for batch column b, rows [r_lo, r_hi):
/// acc = payload + T.src(kk) (sequential in j); f = a*state + b*acc; state = f.
/// Returns f in f_out[r].  last: also write acc and filt to the arena.
template <int DMAX, int BT>
__device__ __forceinline__ void conn_rows(const FusedProgram& p, const FConn& cn_g, int kk, int b, int r_lo, int r_hi,
                                          bool valid, bool last, float* f_out) {
    const FConn cn = cn_g;  // a private copy: the fields stay in registers across the arena stores
    const int B = batch_of<BT>(p);
    float* A = p.arena;
    const float* src;
    if (cn.src_xb >= 0)
        src = p.xbuf + (xslot(p, kk) * p.xrows + cn.src_xb) * B + b;
    else if (cn.src_feed >= 0 && p.feed_present[cn.src_feed])
        src = p.feed_data + p.feed_off[cn.src_feed] + static_cast<int64_t>(kk) * cn.ds * B + b;
    else
        src = A + cn.src_base + b;
    float x[DMAX], s0[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = (valid && j < cn.ds) ? src[static_cast<int64_t>(j) * B] : 0.0f;
    float* st = A + cn.state_base + b;
#pragma unroll
    for (int r = 0; r < DMAX; ++r) s0[r] = (valid && r >= r_lo && r < r_hi) ? st[static_cast<int64_t>(r) * B] : 0.0f;
    const float4* Tm = reinterpret_cast<const float4*>(p.values + cn.tpad_off);
    const bool extra = last || cn.probe_filt >= 0 || cn.probe_state >= 0;
#pragma unroll
    for (int r = 0; r < DMAX; ++r) {
        if (r < r_lo || r >= r_hi) continue;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < DMAX / 4; ++q) {
            const float4 w = __ldg(Tm + r * (DMAX / 4) + q);
            acc = acc + w.x * x[4 * q];
            acc = acc + w.y * x[4 * q + 1];
            acc = acc + w.z * x[4 * q + 2];
            acc = acc + w.w * x[4 * q + 3];
        }
        const float accv = __ldg(p.values + cn.acc_init_off + r) + acc;
        const float f = cn.a * s0[r] + cn.b * accv;  // lowpass_step (neuron_math.hpp:39-42)
        f_out[r] = f;
        if (valid) st[static_cast<int64_t>(r) * B] = f;
        if (valid && extra) {  // the call's last step, probe captures (uniform: one branch per row)
            if (last) {
                A[cn.acc_base + static_cast<int64_t>(r) * B + b] = accv;
                A[cn.filt_base + static_cast<int64_t>(r) * B + b] = f;
            }
            if (cn.probe_filt >= 0)
                p.ring[p.ring_off[cn.probe_filt] + (static_cast<int64_t>(kk) * cn.dd + r) * B + b] = f;
            if (cn.probe_state >= 0)
                p.ring[p.ring_off[cn.probe_state] + (static_cast<int64_t>(kk) * cn.dd + r) * B + b] = f;
        }
    }
}

/// Work of step kk that is not owned by a unit, strided over threads
/// [tid, nthreads): connection updates (all connections in the epilogue,
/// destination-less ones otherwise), probe captures (captures: 0 none, 1 all,
/// 2 all but xhat, which barrier-free units capture themselves) and the clock.
template <int DMAX, int BT>
__device__ void step_work(const FusedProgram& p, int kk, const int* list, int nc, int captures, bool last, int64_t tid,
                          int64_t nthreads) {
    const int B = batch_of<BT>(p);
    const int64_t items = static_cast<int64_t>(nc) * B;
    for (int64_t it = tid; it < items; it += nthreads) {
        const int q = static_cast<int>(it / B);
        const int b = static_cast<int>(it - static_cast<int64_t>(q) * B);
        const int c = __ldg(list + q);
        float f[DMAX];
        conn_rows<DMAX, BT>(p, p.conns[c], kk, b, 0, p.conns[c].dd, true, last, f);
    }
    if (!captures) return;
    for (int q = 0; q < p.n_probes; ++q) {
        const FProbe& pr = p.probes[q];
        if (captures == 2 && pr.xb_row >= 0) continue;
        const int64_t n = static_cast<int64_t>(pr.dim) * B;
        float* dst = p.ring + p.ring_off[pr.index] + static_cast<int64_t>(kk) * pr.dim * B;
        const bool fed = pr.feed_slot >= 0 && p.feed_present[pr.feed_slot];
        for (int64_t i = tid; i < n; i += nthreads) {
            const int64_t d = i / B;
            const int bb = static_cast<int>(i - d * B);
            float val;
            if (pr.xb_row >= 0)
                val = p.xbuf[(xslot(p, kk) * p.xrows + pr.xb_row + d) * B + bb];
            else if (fed)
                val = p.feed_data[p.feed_off[pr.feed_slot] + static_cast<int64_t>(kk) * pr.dim * B + d * B +
                                  (pr.per_batch ? bb : 0)];
            else
                val = p.arena[pr.base + (pr.per_batch ? d * B + bb : d)];
            dst[i] = val;
        }
    }
    if (p.has_time && tid == 0) {  // TimeUpdate (exec.cpp:300-309)
        const float next = p.arena[p.step_base] + 1.0f;
        p.arena[p.step_base] = next;
        p.arena[p.time_base] = next * p.dt;
        if (p.time_probe_step >= 0)
            for (int bb = 0; bb < B; ++bb) p.ring[p.ring_off[p.time_probe_step] + static_cast<int64_t>(kk) * B + bb] = next;
        if (p.time_probe_time >= 0)
            for (int bb = 0; bb < B; ++bb)
                p.ring[p.ring_off[p.time_probe_time] + static_cast<int64_t>(kk) * B + bb] = next * p.dt;
    }
}

template <int DMAX, int BT>
__device__ void grid_step_work(const FusedProgram& p, int kk, const int* list, int nc, int captures, bool last) {
    step_work<DMAX, BT>(p, kk, list, nc, captures, last, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                        static_cast<int64_t>(gridDim.x) * blockDim.x);
}

/// write_feeds (exec.cpp:313-326) of step k into the arena, strided over
/// threads: only the call's last step's values survive (connections read fed
/// sources from the feed block).
template <int BT>
__device__ void write_feeds(const FusedProgram& p, int k, int64_t tid, int64_t nthreads) {
    const int B = batch_of<BT>(p);
    for (int f = 0; f < p.n_feeds; ++f) {
        if (!p.feed_present[f]) continue;
        const FFeed& fd = p.feeds[f];
        const float* src = p.feed_data + p.feed_off[f] + static_cast<int64_t>(k) * fd.dim * B;
        const int64_t n = static_cast<int64_t>(fd.dim) * fd.copies;
        for (int64_t i = tid; i < n; i += nthreads) {
            const int64_t d = i / fd.copies;
            const int bb = static_cast<int>(i - d * fd.copies);
            p.arena[fd.base + d * (fd.copies > 1 ? B : 1) + bb] = src[d * B + bb];
        }
    }
}

// ---- bit transpose --------------------------------------------------------

/// Lane r holds row r of a 32x32 bit matrix (bit c = M[r][c]); returns column
/// `lane` (bit r = M[r][lane]).  Recursive block swap, five shuffle rounds.
__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    constexpr uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int j = 16 >> s;
        const uint32_t m = masks[s];
        const uint32_t y = __shfl_xor_sync(kFull, x, j);
        x = (lane & j) ? ((x & ~m) | ((y >> j) & m)) : ((x & m) | ((y << j) & ~m));
    }
    return x;
}

// ---- the unit ---------------------------------------------------------------

// ---- barrier-free stepping (FusedProgram::dataflow) ---------------------------

__device__ __forceinline__ int ld_acquire(const int* f) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(int* f, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

/// Thread 0 waits until unit (ensemble ei, group g) may run step t of the
/// launch: its sources and itself have finished step t-1, its destinations
/// step t-2.  (The caller's __syncthreads publishes the result to the CTA.)
__device__ __forceinline__ void df_wait(const FusedProgram& p, int ei, int g, int t) {
    if (threadIdx.x != 0) return;
    const int begin = p.ens[ei].dep_begin, cnt = p.ens[ei].dep_count;
    for (int i = 0; i < cnt; ++i) {
        const int d = __ldg(p.deps + begin + i);
        const int need = t - (d & 1);
        const int* f = p.done + static_cast<int64_t>((d >> 1) - p.ens_lo) * p.groups + g;
        while (need > 0 && ld_acquire(f) < need) __nanosleep(32);
    }
    __threadfence();
}

/// Destination-less connections fed by ensemble ei: step-k update for the
/// unit's batch columns, after its decode.
template <int DMAX, int BT>
__device__ void df_orphans(const FusedProgram& p, int ei, int g, int k, bool last) {
    const FEns& e = p.ens[ei];
    const int B = batch_of<BT>(p);
    const int c0 = g * p.tu * 32, cols = min(B, c0 + p.tu * 32) - c0;
    const int items = e.orph_count * cols;
    for (int it = threadIdx.x; it < items; it += blockDim.x) {
        const int q = it / cols;
        const int c = __ldg(p.ens_orph + e.orph_begin + q);
        float f[DMAX];
        conn_rows<DMAX, BT>(p, p.conns[c], k, c0 + it - q * cols, 0, p.conns[c].dd, true, last, f);
    }
}

/// The decode of one-tile units (B <= 32: the 8 warps are neuron slices of one
/// tile): the slices compact each column's spiking neurons into an ascending index
/// list (in the ring and queue regions, free after the sweep), then a thread per
/// (column, row) chains the products over its column's list — all 8 warps decode
/// instead of 2, and the sum keeps the ascending neuron order.  Out of line (once per unit): its registers stay out
/// of the sweep's allocation.  Returns false (nothing written) when a column's list
/// would not fit; the caller then runs the row-split decode.
template <int DMAX, int BT>
__device__ __noinline__ bool decode_listed(const FusedProgram& p, int ei, int k, bool last, float* ring, int lbytes,
                                           const float* P, const uint32_t* words, int slice, bool valid, int b) {
    const FEns& e = p.ens[ei];
    const int B = batch_of<BT>(p);
    const int lane = threadIdx.x & 31;
    float* A = p.arena;
    const int nw = (e.n + 31) >> 5;
    // the ring and queue regions (contiguous, free after the sweep): counts, lengths, lists
    uint16_t* cntw = reinterpret_cast<uint16_t*>(ring);       // [word][column] spike counts
    int* stot = reinterpret_cast<int*>(ring) + nw * 16;       // [column] list lengths
    uint16_t* list = reinterpret_cast<uint16_t*>(stot + 32);  // [position][column] (columns interleaved)
    const int cap = (lbytes - (nw * 64 + 128)) / 64;          // uint16 entries per column
    for (int w = slice; w < nw; w += kWarps) {
        const int i = w * 32 + lane;
        uint32_t bits = transpose32(i < e.n ? words[i] : 0u, lane);
        if (!valid) bits = 0u;
        cntw[w * 32 + lane] = static_cast<uint16_t>(__popc(bits));
    }
    __syncthreads();
    int tot = 0;
    for (int w = 0; w < nw; ++w) tot += cntw[w * 32 + lane];
    if (__any_sync(kFull, tot > cap)) return false;  // the same in every warp: CTA-uniform
    if (slice == 0) stot[lane] = tot;
    for (int w = slice; w < nw; w += kWarps) {
        int pos = 0;
        for (int q = 0; q < w; ++q) pos += cntw[q * 32 + lane];
        const int i = w * 32 + lane;
        uint32_t bits = transpose32(i < e.n ? words[i] : 0u, lane);
        if (!valid) bits = 0u;
        while (bits) {
            list[pos++ * 32 + lane] = static_cast<uint16_t>(w * 32 + __ffs(bits) - 1);
            bits &= bits - 1u;
        }
    }
    __syncthreads();
    // a thread per (column, row): the rows of one column sit in consecutive lanes, so the
    // products P[i][r] of one neuron are consecutive words (no bank conflicts)
    const int dx = e.dx;
    for (int it = threadIdx.x; it < 32 * dx; it += blockDim.x) {
        const int col = it / dx, r = it - col * dx;
        const int n = stot[col];
        const uint16_t* lc = list + col;
        float acc = 0.0f;
        int q = 0;
        for (; q + 8 <= n; q += 8) {
            float t[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) t[u] = P[static_cast<int>(lc[(q + u) * 32]) * dx + r];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = acc + t[u];
        }
        for (; q < n; ++q) acc = acc + P[static_cast<int>(lc[q * 32]) * dx + r];
        const int bc = b - lane + col;  // this tile's column col
        if ((BT > 0 && BT % 32 == 0) || bc < B) {
            const float xv = __ldg(p.values + e.xhat_init_off + r) + acc;
            p.xbuf[(xslot(p, k) * p.xrows + e.xb_row + r) * B + bc] = xv;
            if (last) A[e.xhat_base + static_cast<int64_t>(r) * B + bc] = xv;
            for (int c = 0; p.dataflow && c < e.xp_count; ++c) {  // barrier-free xhat captures
                const FProbe& pr = p.probes[__ldg(p.xprobes + e.xp_begin + c)];
                p.ring[p.ring_off[pr.index] + (static_cast<int64_t>(k) * pr.dim + r) * B + bc] = xv;
            }
        }
    }
    return true;
}

template <int DMAX, int BT, bool PROF>
__device__ void run_unit(const FusedProgram& p, int u, int k, bool do_update, bool last, const Smem& S,
                         uint32_t parity, Ticker<PROF>& tk, int df_pos, int df_t) {
    const int B = batch_of<BT>(p);
    const int ul = u / p.groups;
    const int g = u - ul * p.groups;
    const int ei = p.ens_lo + ul;
    const FEns e = p.ens[ei];  // a private copy: fields stay in registers across the arena stores
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tslot = warp / p.slices, slice = warp - tslot * p.slices;
    const int tile = g * p.tu + tslot;
    const int b0 = tile * 32;
    const bool active = tslot < p.tu && b0 < B;  // warp-uniform
    const int b = b0 + lane;
    const bool valid = active && ((BT > 0 && BT % 32 == 0) || b < B);
    float* A = p.arena;
    FTRACE(1, u);

    // stage encoders, biases and decoder products (async; overlaps the connection updates)
    if (threadIdx.x == 0) {
        fence_proxy_async_smem();  // prior generic accesses of the staging buffers are ordered first
        const uint32_t eb = static_cast<uint32_t>((e.n + 1) & ~1) * DMAX * 4, bb = static_cast<uint32_t>(e.n_pad) * 4;
        const uint32_t pb = p.stage_dec ? static_cast<uint32_t>(e.dec_bytes) : 0u;
        mbar_expect_tx(S.bar, eb + bb + pb);
        bulk_g2s(S.E, p.values + e.epad_off, eb, S.bar);
        bulk_g2s(S.bias, p.values + e.bias_off, bb, S.bar);
        if (pb) bulk_g2s(S.P, p.values + e.dec_scaled_off, pb, S.bar);
    }
    // L2 prefetch of the unit's first HBM reads (overlapping the dependency wait and the
    // connection updates): the incoming connections' filter-state rows and the first
    // kL2Ahead rows of v and r (the sweep prefetches the rest ahead of itself).  Only
    // when the unit spans every column (the rows are then contiguous).
    if (warp == 0 && p.groups == 1 && p.tu * 32 >= B && (B & 3) == 0) {
        if (lane < e.inc_count) {
            const FConn& cn = p.conns[__ldg(p.incoming + e.inc_begin + lane)];
            prefetch_l2_bulk(A + cn.state_base, static_cast<uint32_t>(cn.dd * B) * 4u);
        } else if (lane >= 30) {
            prefetch_l2_bulk(A + (lane == 30 ? e.v_base : e.r_base), static_cast<uint32_t>(min(kL2Ahead, e.n) * B) * 4u);
        }
    }
    if (df_pos >= 0) {  // barrier-free schedule: wait for the dependencies (overlaps the staging copies)
        df_wait(p, ei, g, df_t);
        __syncthreads();
        tk.tick(FS_BAR);
        if (df_pos == 0) {  // the step's work owned by no unit (serialised: order[0] waits for itself)
            if (last) write_feeds<BT>(p, k, threadIdx.x, blockDim.x);
            step_work<DMAX, BT>(p, k, p.free_orph, p.n_free_orph, 2, last, threadIdx.x, blockDim.x);
            tk.tick(FS_DEFER);
        }
    }

    // 1. connection updates of step k-1 (destination side) and the input sum, plan order
    FTRACE(2, k);
    float* sin = S.in + tslot * DMAX * 32;
    if (active) {
        const int rper = (e.d + p.slices - 1) / p.slices;
        const int r_lo = slice * rper, r_hi = min(e.d, r_lo + rper);
        float in[DMAX];
#pragma unroll
        for (int r = 0; r < DMAX; ++r) in[r] = (r >= r_lo && r < r_hi) ? __ldg(p.values + e.in_init_off + r) : 0.0f;
        for (int q = 0; q < e.inc_count; ++q) {
            const FConn& cn = p.conns[__ldg(p.incoming + e.inc_begin + q)];
            float f[DMAX];
#ifdef NENG_FUSED_CHECKS
            // checked builds: the barrier-free schedule's claim on the source's step k-1 xhat —
            // the source unit has finished step k-1 (done >= t) and has not yet finished step
            // k+2, which rewrites slot (k-1) % 3 (done <= t + 2)
            if (df_pos >= 0 && do_update && cn.src_ens >= 0 && lane == 0) {
                const int seen = ld_acquire(p.done + static_cast<int64_t>(cn.src_ens - p.ens_lo) * p.groups + g);
                if (seen < df_t || seen > df_t + 2) {
                    printf("fused check: unit %d step %d reads ensemble %d's xhat at done=%d\n", u, k, cn.src_ens, seen);
                    __trap();
                }
            }
#endif
            if (do_update) {
                conn_rows<DMAX, BT>(p, cn, k - 1, b, r_lo, r_hi, valid, false, f);
            } else {
#pragma unroll
                for (int r = 0; r < DMAX; ++r)
                    f[r] = (valid && r >= r_lo && r < r_hi) ? A[cn.state_base + static_cast<int64_t>(r) * B + b] : 0.0f;
            }
#pragma unroll
            for (int r = 0; r < DMAX; ++r)
                if (r >= r_lo && r < r_hi) in[r] = in[r] + f[r];
        }
#pragma unroll
        for (int r = 0; r < DMAX; ++r) {
            if (r >= r_lo && r < r_hi) {
                sin[r * 32 + lane] = in[r];
                if (last && valid) A[e.in_base + static_cast<int64_t>(r) * B + b] = in[r];
            } else if (slice == 0 && r >= e.d) {
                sin[r * 32 + lane] = 0.0f;  // padding rows hold +0
            }
        }
    }
    if (p.slices > 1)
        __syncthreads();
    else
        __syncwarp();
    tk.tick(FS_IN);

    float x[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = active ? sin[j * 32 + lane] : 0.0f;
    __syncthreads();  // every warp holds its inputs in registers: the queues reuse `in`
    FTRACE(4, 0);
    mbar_wait(S.bar, parity);
    FTRACE(5, 0);

    // 2. neuron sweep over this warp's slice
    const int nper = ((e.n + p.slices - 1) / p.slices + 31) & ~31;
    const int n0 = min(e.n, slice * nper), n1 = min(e.n, n0 + nper);
    uint32_t* words = S.words + tslot * p.nmax;
    if (active && n0 < n1) {
        const float dt = e.dt, em_dt = e.em_dt;
        const float2 dt2 = make_float2(dt, dt), ndt2 = make_float2(-dt, -dt);
        // addresses inside the sweep derive from vst (row i, this lane's column): a
        // separate row-0 pointer would be one more 64-bit value live across the loop
        const uint32_t ring_base = smem_addr(S.ring);
        const bool vec = (B & 3) == 0;
        float* vst = A + e.v_base + b0 + static_cast<int64_t>(n0) * B + lane;  // row i of this lane
        const int64_t rdelta = e.r_base - e.v_base;
        // the lane's share of the ring copies (addresses recomputed per round: fewer live
        // registers).  vec (B % 4 == 0): 16 B, columns lc..lc+3 of row lr of each 4-row
        // round; else 4 B (its own column) of every row
        auto ring_issue = [&](int st, int r0, const float* rowp) {  // rowp: row r0, this lane's column
            const int lr = vec ? (lane >> 3) : 0, lc = vec ? (lane & 7) * 4 : lane;
            if (b0 + lc < B) {
                const float* src = rowp + static_cast<int64_t>(lr) * B + (lc - lane);
                const uint32_t dst = ring_base + (st * kUnroll + lr) * kRowB + warp * 128 + lc * 4;
                if (vec) {
                    if (r0 + lr < n1) {
                        cp_async16_s(dst, src);
                        cp_async16_s(dst + 2 * kUnroll * kRowB, src + rdelta);
                    }
                } else {
#pragma unroll
                    for (int rr = 0; rr < kUnroll; ++rr)
                        if (r0 + rr < n1) {
                            cp_async4_s(dst + rr * kRowB, src + static_cast<int64_t>(rr) * B);
                            cp_async4_s(dst + rr * kRowB + 2 * kUnroll * kRowB, src + static_cast<int64_t>(rr) * B + rdelta);
                        }
                }
            }
            cp_async_commit();
        };
        FTRACE(50, n0);
        ring_issue(0, n0, vst);
        FTRACE(51, n1);
        const bool lv = (BT > 0 && BT % 32 == 0) ? true : valid;  // inside the sweep the tile is active
        const FEns* ep = p.ens + ei;
        const uint32_t lt_mask = lanemask_lt();
        // exception queues: the two branches of lif_spike_step that need a
        // transcendental leave the sweep and are evaluated 32 lanes at a time
        QEnt* qe = S.qe + warp * kQ;  // exceptions: leaving the refractory period (expm1f) or spiking (log1pf)
        QEnt* qd = S.qs + warp * kQ;  // doubtful speculative values: recomputed exactly
        int ne = 0, nd = 0;           // warp-uniform counts
        const uint32_t ring_a = ring_base + threadIdx.x * 4u;  // this lane's column of the ring
        const float* sE = S.E + n0 * DMAX;
        const float* sbias = S.bias + n0;
        for (int i = n0; i < n1; i += 2, vst += 2 * B, sE += 2 * DMAX, sbias += 2) {
            const int rel = i - n0;
            if ((rel & (kUnroll - 1)) == 0) {
                const int st = (rel / kUnroll) & 1;
                __syncwarp();  // every lane's reads of the stage being refilled are done
                FTRACE(52, i);
                ring_issue(st ^ 1, i + kUnroll, vst + kUnroll * B);
                FTRACE(53, i);
                cp_async_wait1();
                __syncwarp();
                FTRACE(54, i);
                // L2 prefetch kL2Ahead rows ahead.  When the unit spans every column the
                // rows are contiguous: lane 0 of the unit's first tile pulls kUnroll whole
                // rows of v and of r with two bulk prefetches; otherwise lanes 0..2*kUnroll-1
                // pull their tile's segments of the kUnroll v and r rows.
                const int pi = i + kL2Ahead;
                if (pi < n1) {
                    if (p.groups == 1 && p.tu * 32 >= B && vec) {
                        if (threadIdx.x == 0) {  // warp 0 owns tile slot 0
                            const uint32_t nb = static_cast<uint32_t>(min(kUnroll, n1 - pi) * B) * 4u;
                            const float* pv = vst + kL2Ahead * B;  // thread 0: tile 0, column 0
                            prefetch_l2_bulk(pv, nb);
                            prefetch_l2_bulk(pv + rdelta, nb);
                        }
                    } else if (lane < 2 * kUnroll && pi + (lane & (kUnroll - 1)) < n1) {
                        const float* pa = vst - lane + static_cast<int64_t>(kL2Ahead + (lane & (kUnroll - 1))) * B +
                                          (lane < kUnroll ? 0 : rdelta);
                        if (vec)
                            prefetch_l2_bulk(pa, static_cast<uint32_t>(min(32, B - b0)) * 4u);
                        else
                            prefetch_l2_line(pa);
                    }
                }
            }
            const uint32_t sv = ring_a + static_cast<uint32_t>(rel & (2 * kUnroll - 1)) * kRowB;
            FTRACE(6, i);
            const float2 v2 = make_float2(lds_f32(sv), lds_f32(sv + kRowB));
            const float2 r2 = make_float2(lds_f32(sv + 2 * kUnroll * kRowB), lds_f32(sv + 2 * kUnroll * kRowB + kRowB));
            // DotInc(E, in, J) for neurons i, i+1: acc from +0, j ascending, then J = bias + acc;
            // the two neurons' sums side by side (encoders pair-interleaved: [j][i, i+1])
            float acc[2];
            {
                const float4* er = reinterpret_cast<const float4*>(sE);
                uint64_t a2 = 0;  // (+0, +0)
#pragma unroll
                for (int q = 0; q < DMAX / 2; ++q) {
                    const float4 w = er[q];
                    a2 = add2(a2, mul2_exact(pk2(w.x, w.y), pk2(x[2 * q], x[2 * q]), p.neg_zero2));
                    a2 = add2(a2, mul2_exact(pk2(w.z, w.w), pk2(x[2 * q + 1], x[2 * q + 1]), p.neg_zero2));
                }
                const float2 a = unpk2(a2);
                acc[0] = a.x;
                acc[1] = a.y;
            }
            const float2 J2 = __fadd2_rn(*reinterpret_cast<const float2*>(sbias), make_float2(acc[0], acc[1]));
            const float2 dl2 = __fadd2_rn(dt2, make_float2(-r2.x, -r2.y));  // dt - r
            const float2 rr2 = __fadd2_rn(r2, ndt2);                        // r - dt
            // lif_spike_step<float> (neuron_math.hpp:55-77) for the lanes that need
            // no transcendental: delta = dt (em = expm1f(-dt/tau_rc), the host's
            // glibc value) or delta = 0 (em = expm1f(-0) = -0).  A lane with
            // 0 < delta < dt (or NaN) goes to the exit queue; a spiking lane stores
            // v = 0 and goes to the spike queue for its refractory time.
            const float2 d2 = __fadd2_rn(J2, make_float2(-v2.x, -v2.y));  // J - v
            bool ex[2];
            float t[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float delta = h ? dl2.y : dl2.x;
                const bool ge = delta >= dt, le = delta <= 0.0f;
                ex[h] = !ge && !le;
                t[h] = __fmul_rn(h ? d2.y : d2.x, ge ? em_dt : -0.0f);  // scalar products between paired sums
            }
            const float2 vn2 = __fadd2_rn(v2, make_float2(-t[0], -t[1]));
            const bool two = i + 1 < n1;  // warp-uniform
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const bool row = lv && (h == 0 || two);
                const float J = h ? J2.y : J2.x;
                float vn = h ? vn2.y : vn2.x;
                if (vn < 0.0f) vn = 0.0f;
                const bool spike = !ex[h] && vn > 1.0f;
                const float rh = h ? r2.y : r2.x;
                if (row) {  // queued lanes store placeholders their batch overwrites
#ifdef NENG_ROW_STORE_NORMAL
                    vst[h * B] = spike ? 0.0f : vn;
                    vst[h * B + rdelta] = rh > dt ? (h ? rr2.y : rr2.x) : 0.0f;
#else
                    __stcs(vst + h * B, spike ? 0.0f : vn);
                    __stcs(vst + h * B + rdelta, rh > dt ? (h ? rr2.y : rr2.x) : 0.0f);
#endif
                }
                const uint32_t key = (static_cast<uint32_t>(i + h) << 5) | lane;
                const uint32_t word = __ballot_sync(kFull, row && spike);
                if (lane == 0 && (h == 0 || two)) words[i + h] = word;
                const bool xq = row && (ex[h] || spike);
                const uint32_t me = __ballot_sync(kFull, xq);
                if (xq) qe[ne + __popc(me & lt_mask)] = QEnt{key, h ? v2.y : v2.x, rh, J};
                ne += __popc(me);
#ifdef NENG_FUSED_CHECKS
                if (ne > kQ || nd > kQ) {
                    printf("fused check: queue overflow ne=%d nd=%d\n", ne, nd);
                    __trap();
                }
#endif
                // warp-uniform drains; a row adds <= 32 entries, so ne < 32 before a row
                if (ne >= 32) {
                    ne -= 32;
                    __syncwarp();
                    tk.tick(FS_SWEEP);
                    FTRACE(9, ne);
                    float* vcol = vst - static_cast<int64_t>(i) * B - lane;  // row 0, column b0
                    nd = exc_batch<BT>(p, ep, vcol, rdelta, qe + ne, 32, qd, nd, words);
                    FTRACE(10, nd);
                    if (nd >= 32) {
                        nd -= 32;
                        __syncwarp();
                        doubt_batch<BT>(p, ep, vcol, rdelta, qd + nd, 32, words);
                    }
                    __syncwarp();
                    tk.tick(FS_FIX);
                }
            }
        }
        __syncwarp();
        FTRACE(11, ne);
        float* vrow0 = A + __ldg(&ep->v_base) + b0;  // row 0, column b0 of this tile (reloaded: not live in the loop)
        if (ne > 0) nd = exc_batch<BT>(p, ep, vrow0, rdelta, qe, ne, qd, nd, words);
        while (nd > 0) {  // <= 63 entries
            __syncwarp();
            const int c = min(nd, 32);
            nd -= c;
            doubt_batch<BT>(p, ep, vrow0, rdelta, qd + nd, c, words);
        }
        __syncwarp();
        FTRACE(12, 0);
        // probes on the ensemble's own neuron signals (capture_probes, exec.cpp:328-338):
        // read back after the queues have written v, r and the spike bits
        for (int c = 0; c < e.sc_count; ++c) {
            const int2 cap = __ldg(reinterpret_cast<const int2*>(p.scaps) + e.sc_begin + c);
            float* dst = p.ring + p.ring_off[cap.y] + static_cast<int64_t>(k) * e.n * B + b;
            for (int i = n0; valid && i < n1; ++i) {
                float val;
                if (cap.x == SC_OUT) {
                    val = (words[i] >> lane) & 1u ? e.amp_dt : 0.0f;
                } else if (cap.x == SC_VOLTAGE || cap.x == SC_REFRACTORY) {
                    val = vrow0[static_cast<int64_t>(i) * B + lane + (cap.x == SC_REFRACTORY ? rdelta : 0)];
                } else {
                    float a = 0.0f;
#pragma unroll
                    for (int j = 0; j < DMAX; ++j) a = a + enc_at<DMAX>(S.E, i, j) * x[j];
                    val = S.bias[i] + a;
                }
                dst[static_cast<int64_t>(i) * B] = val;
            }
        }
        // the call's last step leaves J in the arena (DotInc(E, in, J) as above, once)
        if (last && valid) {
            for (int i = n0; i < n1; ++i) {
                float a = 0.0f;
#pragma unroll
                for (int j = 0; j < DMAX; ++j) a = a + enc_at<DMAX>(S.E, i, j) * x[j];
                A[e.j_base + static_cast<int64_t>(i) * B + b] = S.bias[i] + a;
            }
        }
    }
    tk.tick(FS_SWEEP);
    // the decoder products replace the encoders in shared memory once every warp
    // is past its sweep (they are the same size or smaller: dx <= DMAX)
    const bool p_late = !p.stage_dec;
    if (p.slices > 1 || p_late)
        __syncthreads();
    else
        __syncwarp();
    if (p_late) {
        if (threadIdx.x == 0) {
            fence_proxy_async_smem();  // the sweep's reads of the encoders are ordered first
            mbar_expect_tx(S.bar2, static_cast<uint32_t>(e.dec_bytes));
            bulk_g2s(S.E, p.values + e.dec_scaled_off, static_cast<uint32_t>(e.dec_bytes), S.bar2);
        }
        mbar_wait(S.bar2, parity);
    }

    // 3. decode: rows [r0, r0 + R) of this warp's tile over all neurons, ascending
    FTRACE(13, 0);
    // One-tile units (B <= 32: the 8 warps are neuron slices of one tile): the slices
    // compact each column's spiking neurons into an ascending index list, then every
    // thread chains (column, row) items over the lists — all 8 warps decode instead of 2
    const bool listed = active && p.tu == 1 && p.slices == kWarps &&
                        decode_listed<DMAX, BT>(p, ei, k, last, S.ring,
                                                static_cast<int>(kWarps * kRingFloats * 4 + inq_bytes<DMAX>(p)),
                                                p.stage_dec ? S.P : S.E, words, slice, valid, b);
    if (active && !listed) {
        const int dx = e.dx;
        int R = (dx + p.slices - 1) / p.slices;
        if ((dx & 3) == 0) R = (R + 3) & ~3;
        const int r0 = slice * R;
        if (r0 < dx) {
            const int rn = min(R, dx - r0);
            const float* Pb = (p.stage_dec ? S.P : S.E) + r0;
            const bool vec = (dx & 3) == 0 && (rn & 3) == 0;
            float a[DMAX];
#pragma unroll
            for (int q = 0; q < DMAX; ++q) a[q] = 0.0f;
            const int nw = (e.n + 31) >> 5;
            for (int w = 0; w < nw; ++w) {
                const int i = w * 32 + lane;
                uint32_t bits = transpose32(i < e.n ? words[i] : 0u, lane);
                if (!valid) bits = 0u;
                while (bits) {
                    const int c = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const float* pr = Pb + static_cast<int64_t>(w * 32 + c) * dx;
                    if (vec) {
#pragma unroll
                        for (int q = 0; q < DMAX / 4; ++q) {
                            if (4 * q < rn) {
                                const float4 t4 = *reinterpret_cast<const float4*>(pr + 4 * q);
                                a[4 * q] = a[4 * q] + t4.x;
                                a[4 * q + 1] = a[4 * q + 1] + t4.y;
                                a[4 * q + 2] = a[4 * q + 2] + t4.z;
                                a[4 * q + 3] = a[4 * q + 3] + t4.w;
                            }
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < DMAX; ++q)
                            if (q < rn) a[q] = a[q] + pr[q];
                    }
                }
            }
            if (valid) {
                float* xo = p.xbuf + (xslot(p, k) * p.xrows + e.xb_row + r0) * B + b;
#pragma unroll
                for (int q = 0; q < DMAX; ++q) {
                    if (q < rn) {
                        const float xv = __ldg(p.values + e.xhat_init_off + r0 + q) + a[q];
                        xo[static_cast<int64_t>(q) * B] = xv;
                        if (last) A[e.xhat_base + static_cast<int64_t>(r0 + q) * B + b] = xv;
                        a[q] = xv;
                    }
                }
                // barrier-free stepping captures xhat probes here (else grid_step_work does)
                for (int c = 0; p.dataflow && c < e.xp_count; ++c) {
                    const FProbe& pr = p.probes[__ldg(p.xprobes + e.xp_begin + c)];
                    float* dst = p.ring + p.ring_off[pr.index] + (static_cast<int64_t>(k) * pr.dim + r0) * B + b;
#pragma unroll
                    for (int q = 0; q < DMAX; ++q)
                        if (q < rn) dst[static_cast<int64_t>(q) * B] = a[q];
                }
            }
        }
    }
    // out = amp/dt on a spike (the call's last step only reaches the arena)
    if (active && last && valid) {
        const int nper = ((e.n + p.slices - 1) / p.slices + 31) & ~31;
        const int n0 = min(e.n, slice * nper), n1 = min(e.n, n0 + nper);
        for (int i = n0; i < n1; ++i)
            A[e.out_base + static_cast<int64_t>(i) * B + b] = (words[i] >> lane) & 1u ? e.amp_dt : 0.0f;
    }
    tk.tick(FS_DECODE);
    FTRACE(14, 0);
    if (df_pos >= 0) {  // barrier-free schedule: destination-less connections, then publish the step
        __syncthreads();
        if (e.orph_count) {
            df_orphans<DMAX, BT>(p, ei, g, k, last);
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            __threadfence();
            st_release(p.done + u, df_t + 1);
        }
    }
}

template <int DMAX, int BT, bool PROF, bool DF>
__global__ void __launch_bounds__(kThreads, kMinBlocks) fused_run_kernel(const __grid_constant__ FusedProgram p, int k_begin, int k_end) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) uint32_t smem[];
    const Smem S = carve<DMAX>(smem, p);
#ifdef NENG_FUSED_CHECKS
    {
        uint32_t dyn;
        asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        if (threadIdx.x == 0 && smem_bytes<DMAX>(p) > dyn) {
            printf("fused check: carve needs %llu of %u bytes\n", (unsigned long long)smem_bytes<DMAX>(p), dyn);
            __trap();
        }
    }
#endif
    if (threadIdx.x == 0) {
        mbar_init(S.bar);
        mbar_init(S.bar2);
    }
    __syncthreads();
    uint32_t parity = 0;
    const int B = batch_of<BT>(p);
    const int units = (p.ens_hi - p.ens_lo) * p.groups;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    Ticker<PROF> tk;
    tk.start();

    if constexpr (!DF) {
        // one grid barrier per step: the units of step k are claimed from work[k & 1]
        for (int k = k_begin; k < k_end; ++k) {
            const bool last = k == p.call_steps - 1;
            if (gtid == 0) p.work[(k + 1) & 1] = 0;  // last used by step k-1; next used by step k+1
            if (last) write_feeds<BT>(p, k, gtid, gthreads);
            const bool upd = k > k_begin || p.first_update;
            if (upd) grid_step_work<DMAX, BT>(p, k - 1, p.orphans, p.n_orphans, 1, false);
            tk.tick(FS_DEFER);
            int* work = p.work + (k & 1);
            for (;;) {
                if (threadIdx.x == 0) *S.cur = atomicAdd(work, 1);
                __syncthreads();
                const int u = *S.cur;
                __syncthreads();  // every thread has read cur before thread 0 claims again
                tk.tick(FS_QUEUE);  // (profile: the unit barrier and claim)
                if (u >= units) break;  // uniform
                run_unit<DMAX, BT, PROF>(p, u, k, upd, last, S, parity, tk, -1, 0);
                parity ^= 1u;
                __syncthreads();  // staging buffers, words and queues are reused by the next unit
            }
            grid_sync(grid);
            tk.tick(FS_BAR);
        }
        // epilogue: connection updates, captures and clock of the launch's last step
        if (p.epilogue)
            grid_step_work<DMAX, BT>(p, k_end - 1, p.my_conns, p.n_my_conns, 1, k_end - 1 == p.call_steps - 1);
    } else {
        // barrier-free: position gi = t * units + pos of one launch-wide claim
        // counter runs unit order[pos] of step k_begin + t once its
        // dependencies are done; the only grid barrier precedes the epilogue
        const int total = units * (k_end - k_begin);
        for (;;) {
            if (threadIdx.x == 0) *S.cur = atomicAdd(p.work, 1);
            __syncthreads();
            const int gi = *S.cur;
            __syncthreads();  // every thread has read cur before thread 0 claims again
            tk.tick(FS_QUEUE);
            if (gi >= total) break;  // uniform
            const int t = gi / units, pos = gi - t * units;
            const int u = __ldg(p.order + pos);
            const int k = k_begin + t;
            run_unit<DMAX, BT, PROF>(p, u, k, t > 0 || p.first_update, k == p.call_steps - 1, S, parity, tk, pos, t);
            parity ^= 1u;
            __syncthreads();  // staging buffers, words and queues are reused by the next unit
        }
        grid_sync(grid);
        tk.tick(FS_BAR);
        // epilogue: the step k_end-1 updates of connections into ensembles (the
        // units captured their xhat and updated their destination-less connections)
        if (p.epilogue)
            grid_step_work<DMAX, BT>(p, k_end - 1, p.dest_conns, p.n_dest_conns, 0, k_end - 1 == p.call_steps - 1);
    }
    tk.tick(FS_EPI);
    tk.flush(p.prof);
}

// ---- the small-program step ---------------------------------------------------

constexpr int kSmallThreads = 512;

/// Programs too small to fill the GPU (config 0: one 800-neuron ensemble at
/// batch 1) run on ONE CTA, phase by phase with block barriers, and with lanes
/// over (ensemble, neuron, column) items instead of batch columns: the step's
/// dependency chain, not the GPU's width, is the cost.  Per step k:
///   deferred work of step k-1 (destination-less connections, captures, clock);
///   connection updates of step k-1 into every ensemble, one (connection, row,
///   column) per item (conn_rows: the sequential T.src sum and lowpass_step);
///   input sums in plan order (Copy increments, exec.cpp:189-210) into the arena;
///   the neuron sweep (DotInc(E, in, J) sequential in j, lif_spike_step<float>
///   with glibc's expm1f / log1pf), spike bits into shared-memory words;
///   the decode, one (ensemble, row, column) per item: payload + the spiking
///   neurons' products fp32(D[r,i]) * fp32(amp/dt) in ascending i.
/// Every sum keeps the reference's order, so results are the fused kernel's
/// (and EngineCore<float>'s) bit for bit.
/// Step-kk updates of the connections list[0, nc), one (connection, row, column) per item.
template <int DMAX>
__device__ void small_conn_rows(const FusedProgram& p, int kk, const int* list, int nc, bool last) {
    const int B = p.batch;
    const int64_t items = static_cast<int64_t>(nc) * DMAX * B;
    for (int64_t it = threadIdx.x; it < items; it += blockDim.x) {
        const int q = static_cast<int>(it / (DMAX * B));
        const int r = static_cast<int>((it / B) % DMAX), b = static_cast<int>(it % B);
        const FConn& cn = p.conns[__ldg(list + q)];
        if (r >= cn.dd) continue;
        float f[DMAX];
        conn_rows<DMAX, 0>(p, cn, kk, b, r, r + 1, true, last, f);
    }
}

template <int DMAX>
__global__ void __launch_bounds__(kSmallThreads) fused_small_kernel(const __grid_constant__ FusedProgram p, int k_begin,
                                                                     int k_end) {
    extern __shared__ uint32_t swords[];
    const int B = p.batch;
    const int tid = threadIdx.x, nt = blockDim.x;
    float* A = p.arena;
    // the decoder products of every ensemble, staged once per launch when they fit
    // (p.small_pfloats > 0; ensembles in order, each n*dx floats from dec_scaled_off)
    float* sP = reinterpret_cast<float*>(swords + p.small_words);
    int* scnt = reinterpret_cast<int*>(sP + p.small_pfloats);  // [B] spike counts (decode)
    int* sidx = scnt + B;                                      // [B][nmax] spiking neurons (decode)
    if (p.small_pfloats > 0) {
        int at = 0;
        for (int ei = 0; ei < p.n_ens; ++ei) {
            const int n = p.ens[ei].n * p.ens[ei].dx;
            const float* src = p.values + p.ens[ei].dec_scaled_off;
            for (int q = tid; q < n; q += nt) sP[at + q] = __ldg(src + q);
            at += n;
        }
        __syncthreads();
    }
    unsigned long long t0 = 0, sec[FS_COUNT] = {};  // NENG_FUSED_PROFILE: ns per phase (thread 0)
    auto tick = [&](int s) {
        if (p.prof && tid == 0) {
            const unsigned long long t = gtime();
            if (t0) sec[s] += t - t0;
            t0 = t;
        }
    };
    tick(FS_EPI);
    for (int k = k_begin; k < k_end; ++k) {
        const bool last = k == p.call_steps - 1;
        const bool upd = k > k_begin || p.first_update;
        if (last) write_feeds<0>(p, k, tid, nt);
        if (upd) {  // step k-1's destination-less connections (row-parallel), captures and clock
            small_conn_rows<DMAX>(p, k - 1, p.orphans, p.n_orphans, false);
            step_work<DMAX, 0>(p, k - 1, nullptr, 0, 1, false, tid, nt);
        }
        for (int w = tid; w < p.small_words; w += nt) swords[w] = 0u;
        __syncthreads();
        tick(FS_DEFER);
        if (upd) {  // connection updates of step k-1 into the ensembles
            small_conn_rows<DMAX>(p, k - 1, p.dest_conns, p.n_dest_conns, false);
            __syncthreads();
        }
        for (int ei = 0; ei < p.n_ens; ++ei) {  // input sums: payload, then the filtered values in plan order
            const FEns& e = p.ens[ei];
            for (int it = tid; it < e.d * B; it += nt) {
                const int r = it / B, b = it - (it / B) * B;
                float in = __ldg(p.values + e.in_init_off + r);
                for (int q = 0; q < e.inc_count; ++q) {
                    const FConn& cn = p.conns[__ldg(p.incoming + e.inc_begin + q)];
                    in = in + A[cn.state_base + static_cast<int64_t>(r) * B + b];
                }
                A[e.in_base + static_cast<int64_t>(r) * B + b] = in;
            }
        }
        __syncthreads();
        tick(FS_IN);
        int wofs = 0;
        for (int ei = 0; ei < p.n_ens; ++ei) {  // the neuron sweep
            const FEns e = p.ens[ei];  // a private copy: fields stay in registers across the arena stores
            const int nw = (e.n + 31) >> 5;
            const float* E = p.values + e.epad_off;
            for (int it = tid; it < e.n * B; it += nt) {
                const int i = it / B, b = it - (it / B) * B;
                float x[DMAX], w[DMAX];
#pragma unroll
                for (int j = 0; j < DMAX; ++j) {
                    x[j] = j < e.d ? A[e.in_base + static_cast<int64_t>(j) * B + b] : 0.0f;
                    w[j] = j < e.d ? __ldg(E + (i >> 1) * 2 * DMAX + j * 2 + (i & 1)) : 0.0f;
                }
                float acc = 0.0f;
#pragma unroll
                for (int j = 0; j < DMAX; ++j)
                    if (j < e.d) acc = acc + w[j] * x[j];
                const float J = __ldg(p.values + e.bias_off + i) + acc;
                const int64_t o = static_cast<int64_t>(i) * B + b;
                float v = A[e.v_base + o], r = A[e.r_base + o];
                const bool spike = lif_step(J, v, r, e.dt, e.em_dt, e.inv_tau_rc, e.tau_rc, e.tau_ref,
                                            [&](float a, bool is_log) { return glibc_value(a, is_log, p); });
                A[e.v_base + o] = v;
                A[e.r_base + o] = r;
                if (spike) atomicOr(swords + wofs + b * nw + (i >> 5), 1u << (i & 31));
                if (last) {
                    A[e.j_base + o] = J;
                    A[e.out_base + o] = spike ? e.amp_dt : 0.0f;
                }
                for (int c = 0; c < e.sc_count; ++c) {  // captures of the ensemble's own neuron signals
                    const int2 cap = __ldg(reinterpret_cast<const int2*>(p.scaps) + e.sc_begin + c);
                    const float val = cap.x == SC_OUT ? (spike ? e.amp_dt : 0.0f)
                                      : cap.x == SC_VOLTAGE ? v
                                      : cap.x == SC_REFRACTORY ? r
                                                               : J;
                    p.ring[p.ring_off[cap.y] + static_cast<int64_t>(k) * e.n * B + o] = val;
                }
            }
            wofs += nw * B;
        }
        __syncthreads();
        tick(FS_SWEEP);
        wofs = 0;
        int pofs = 0;
        for (int ei = 0; ei < p.n_ens; ++ei) {  // the decode
            const FEns e = p.ens[ei];
            const int nw = (e.n + 31) >> 5;
            const float* P = p.small_pfloats > 0 ? sP + pofs : p.values + e.dec_scaled_off;
            pofs += e.n * e.dx;
            // 1. the spiking neurons of every column, ascending, compacted into sidx[b][0, cnt_b)
            //    (a thread per (word, column): its rank is the popcount of the words before)
            for (int it = tid; it < nw * B; it += nt) {
                const int b = it / nw, w = it - b * nw;
                const uint32_t* cw = swords + wofs + b * nw;
                int pos = 0;
                for (int q = 0; q < w; ++q) pos += __popc(cw[q]);
                uint32_t bits = cw[w];
                int* out = sidx + b * e.n;
                if (w == nw - 1) scnt[b] = pos + __popc(bits);
                while (bits) {
                    out[pos++] = w * 32 + __ffs(bits) - 1;
                    bits &= bits - 1u;
                }
            }
            __syncthreads();
            // 2. a thread per (row, column): payload + the products of those neurons in order,
            //    eight indices and eight products in flight ahead of the dependent adds
            for (int it = tid; it < e.dx * B; it += nt) {
                const int r = it / B, b = it - (it / B) * B;
                const int cnt = scnt[b];
                const int* ix = sidx + b * e.n;
                const float* Pr = P + r;
                float a = 0.0f;
                int q = 0;
                for (; q + 8 <= cnt; q += 8) {
                    float t[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) t[u] = Pr[ix[q + u] * e.dx];
#pragma unroll
                    for (int u = 0; u < 8; ++u) a = a + t[u];
                }
                for (; q < cnt; ++q) a = a + Pr[ix[q] * e.dx];
                const float xv = __ldg(p.values + e.xhat_init_off + r) + a;
                p.xbuf[(xslot(p, k) * p.xrows + e.xb_row + r) * B + b] = xv;
                if (last) A[e.xhat_base + static_cast<int64_t>(r) * B + b] = xv;
            }
            __syncthreads();  // sidx / scnt are reused by the next ensemble
            wofs += nw * B;
        }
        __syncthreads();
        tick(FS_DECODE);
    }
    if (p.epilogue) {  // connection updates, captures and clock of the launch's last step
        small_conn_rows<DMAX>(p, k_end - 1, p.my_conns, p.n_my_conns, k_end - 1 == p.call_steps - 1);
        step_work<DMAX, 0>(p, k_end - 1, nullptr, 0, 1, k_end - 1 == p.call_steps - 1, tid, nt);
    }
    tick(FS_EPI);
    if (p.prof && tid == 0)
        for (int s2 = 0; s2 < FS_COUNT; ++s2) atomicAdd(p.prof + s2, sec[s2]);
}

template <int DMAX>
cudaError_t launch_small(const FusedProgram& p, int k0, int k1, cudaStream_t stream) {
    const size_t sm = (static_cast<size_t>(p.small_words) + p.small_pfloats + p.batch + static_cast<size_t>(p.nmax) * p.batch) * 4;
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fused_small_kernel<DMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    fused_small_kernel<DMAX><<<1, kSmallThreads, sm, stream>>>(p, k0, k1);
    return cudaGetLastError();
}

template <int DMAX, int BT, bool PROF, bool DF>
cudaError_t launch_k(const FusedProgram& p, int grid, int k0, int k1, cudaStream_t stream) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fused_run_kernel<DMAX, BT, PROF, DF>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    FusedProgram prog = p;
    void* args[] = {&prog, &k0, &k1};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_run_kernel<DMAX, BT, PROF, DF>), dim3(grid),
                                       dim3(kThreads), args, sm, stream);
}

template <int DMAX, int BT, bool PROF>
cudaError_t launch_t(const FusedProgram& p, int grid, int k0, int k1, cudaStream_t stream) {
    return p.dataflow ? launch_k<DMAX, BT, PROF, true>(p, grid, k0, k1, stream)
                      : launch_k<DMAX, BT, PROF, false>(p, grid, k0, k1, stream);
}

template <int DMAX, int BT, bool PROF, bool DF>
int per_sm_k(size_t sm) {
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(fused_run_kernel<DMAX, BT, PROF, DF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, fused_run_kernel<DMAX, BT, PROF, DF>, kThreads, sm);
    return n;
}

template <int DMAX, int BT>
int max_grid_t(const FusedProgram& p, int device) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 227 * 1024) return 0;
    const int per_sm = std::min(std::min(per_sm_k<DMAX, BT, false, false>(sm), per_sm_k<DMAX, BT, true, false>(sm)),
                                std::min(per_sm_k<DMAX, BT, false, true>(sm), per_sm_k<DMAX, BT, true, true>(sm)));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

// Batch widths with a stride-specialised kernel (others run the runtime-stride one).
#ifdef NENG_FUSED_DEBUG_BUILD  // quick experiment builds: DMAX 8, the bench's batch width and the generic one
#define NENG_FUSED_BATCHES(X) X(256)
#else
#define NENG_FUSED_BATCHES(X) X(32) X(256)
#endif

template <int DMAX, bool PROF>
cudaError_t launch_d(const FusedProgram& p, int grid, int k0, int k1, cudaStream_t stream) {
#define NENG_CASE(BB) \
    if (p.batch == BB) return launch_t<DMAX, BB, PROF>(p, grid, k0, k1, stream);
    NENG_FUSED_BATCHES(NENG_CASE)
#undef NENG_CASE
    return launch_t<DMAX, 0, PROF>(p, grid, k0, k1, stream);
}

template <int DMAX>
int max_grid_d(const FusedProgram& p, int device) {
#define NENG_CASE(BB) \
    if (p.batch == BB) return max_grid_t<DMAX, BB>(p, device);
    NENG_FUSED_BATCHES(NENG_CASE)
#undef NENG_CASE
    return max_grid_t<DMAX, 0>(p, device);
}

}  // namespace

int fused_dmax_for(int d) { return d <= 8 ? 8 : d <= 16 ? 16 : d <= 32 ? 32 : 0; }

size_t fused_smem_bytes(const FusedProgram& p, int dmax) {
    switch (dmax) {
        case 8: return smem_bytes<8>(p);
        case 16: return smem_bytes<16>(p);
        case 32: return smem_bytes<32>(p);
    }
    return 0;
}

cudaError_t launch_fused(const FusedProgram& p, int dmax, int grid, int k0, int k1, cudaStream_t stream) {
    const bool prof = p.prof != nullptr;
    switch (dmax) {
#ifdef NENG_FUSED_DEBUG_BUILD
        case 8: return prof ? cudaErrorNotSupported : launch_d<8, false>(p, grid, k0, k1, stream);
#else
        case 8: return prof ? launch_d<8, true>(p, grid, k0, k1, stream) : launch_d<8, false>(p, grid, k0, k1, stream);
        case 16: return prof ? launch_d<16, true>(p, grid, k0, k1, stream) : launch_d<16, false>(p, grid, k0, k1, stream);
        case 32: return prof ? launch_d<32, true>(p, grid, k0, k1, stream) : launch_d<32, false>(p, grid, k0, k1, stream);
#endif
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_fused_small(const FusedProgram& p, int dmax, int k0, int k1, cudaStream_t stream) {
    FusedProgram q = p;
    q.dataflow = 0;  // parity xhat slots: the step's phases are ordered by block barriers
    switch (dmax) {
        case 8: return launch_small<8>(q, k0, k1, stream);
#ifndef NENG_FUSED_DEBUG_BUILD
        case 16: return launch_small<16>(q, k0, k1, stream);
        case 32: return launch_small<32>(q, k0, k1, stream);
#endif
    }
    return cudaErrorInvalidValue;
}

int fused_max_grid(const FusedProgram& p, int dmax, int device) {
    switch (dmax) {
        case 8: return max_grid_d<8>(p, device);
#ifndef NENG_FUSED_DEBUG_BUILD
        case 16: return max_grid_d<16>(p, device);
        case 32: return max_grid_d<32>(p, device);
#endif
    }
    return 0;
}

}  // namespace nengb
