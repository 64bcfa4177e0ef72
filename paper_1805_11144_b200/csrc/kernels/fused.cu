// fused.cu — the fused ensemble pipeline: one persistent cooperative kernel
// advancing K timesteps, two grid barriers per step (see fused.hpp).
//
// Phase A unit = (ensemble, 32-column batch tile), claimed dynamically;
// lane = batch column, warp = a contiguous range of neurons:
//   * the ensemble's zero-padded encoder rows, biases and (when they fit)
//     decoder products are staged into shared memory by TMA bulk copies
//     (cp.async.bulk + mbarrier) issued at unit start, overlapping the input sums;
//   * the input vector of each column lives in DMAX registers for the unit;
//   * v/r stream coalesced (arena layout [row][B]: 128 B per warp access) with
//     evict-first hints and one round of software prefetch;
//   * the two transcendental branches of the LIF step (expm1 for the step a
//     neuron leaves its refractory period, log1p for the spike time) are
//     evaluated inline from a double Taylor polynomial — the value glibc
//     returns except on calibrated exceptions, all of which lie next to a
//     float rounding midpoint.  A result in that window is used speculatively
//     and its neuron is queued; after the sweep one parallel pass recomputes
//     the queued neurons exactly (with table probes) and patches v, r and the
//     spike bit.  No probe latency sits inside the sweep.
//   * spikes leave the LIF as ballot words, are bit-transposed with ballots,
//     and the decoder walks only set bits in ascending neuron order.
// Zero padding (encoder rows to DMAX, transforms to DMAX) and skipping
// non-spiking neurons are exact: a running sum that starts at +0 is never -0,
// and x + (+-0) == x for every x, so the extra +0 terms change no bit.
//
// Every other floating-point operation is the reference's, in its order:
//   in   : Reset payload, then += filtered_c for c in plan-group order (exec.cpp:189-210)
//   J    : bias + (0 + E[i,0]in0 + E[i,1]in1 + ...)                      (exec.cpp:226-240)
//   LIF  : lif_spike_step<float>                                         (neuron_math.hpp:55-77)
//   xhat : payload + (0 + sum_i D[r,i]*out[i])                            (exec.cpp:226-240)
//   acc  : payload + (0 + sum_j T[r,j]*src[j]);  f = a*state + b*acc      (exec.cpp:267-284)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "fused.hpp"
#include "libm.cuh"

namespace cg = cooperative_groups;

namespace nengb {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;
constexpr int kFixCap = 1024;  // per-CTA fix-up entries (overflow is resolved inline, exactly)

__device__ __forceinline__ void grid_sync(cg::grid_group& g) {
    if (gridDim.x == 1)
        __syncthreads();
    else
        g.sync();
}

// ---- TMA bulk copy + mbarrier (sm_90+ async proxy) -------------------------
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
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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

struct FixEntry {
    int32_t key;  // neuron << 5 | lane
    float v, r, J;
};

struct Smem {
    uint64_t* bar;
    float* E;      // nmax x DMAX (zero padded)
    float* bias;   // nmax
    float* P;      // decoder products [n][dx] (when p.stage_dec)
    float* in;     // DMAX x 32
    uint32_t* words;
    uint32_t* col;
    FixEntry* fix;  // kFixCap
    int* nfix;
    int* next_unit;
};

/// lif_spike_step<float> resolved exactly (table probes as needed); returns
/// whether the neuron spiked.
__device__ __forceinline__ bool lif_exact(float J, float& v, float& r, float dt, float tau_rc, float tau_ref,
                                          const LibmTables& t) {
    float delta = dt - r;
    if (delta < 0.0f) delta = 0.0f;
    if (delta > dt) delta = dt;
    float vn = v - (J - v) * glibc_expm1f(-delta / tau_rc, t);
    if (vn < 0.0f) vn = 0.0f;
    if (vn > 1.0f) {
        const float since = -tau_rc * glibc_log1pf(-(vn - 1.0f) / (J - 1.0f), t);
        v = 0.0f;
        r = tau_ref - since;
        return true;
    }
    v = vn;
    r = r > dt ? r - dt : 0.0f;
    return false;
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

template <int DMAX, int BT, bool PROF>
__device__ void phase_a_unit(const FusedProgram& p, int unit, bool last, const Smem& S, uint32_t parity,
                             Ticker<PROF>& tk) {
    const int B = batch_of<BT>(p);
    const int t = unit / p.btiles;
    const int b0 = (unit - t * p.btiles) * 32;
    const FEns& e = p.ens[t];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = b0 + lane;
    const bool valid = (BT > 0 && BT % 32 == 0) || b < B;
    float* A = p.arena;

    // stage encoders, biases and decoder products (async; overlaps A1)
    if (threadIdx.x == 0) {
        fence_proxy_async_smem();  // prior generic accesses of the staging buffers are ordered first
        const uint32_t eb = static_cast<uint32_t>((e.n + 1) & ~1) * DMAX * 4, bb = static_cast<uint32_t>(e.n_pad) * 4;
        const uint32_t pb = p.stage_dec ? static_cast<uint32_t>(e.dec_bytes) : 0u;
        mbar_expect_tx(S.bar, eb + bb + pb);
        bulk_g2s(S.E, p.values + e.epad_off, eb, S.bar);
        bulk_g2s(S.bias, p.values + e.bias_off, bb, S.bar);
        if (pb) bulk_g2s(S.P, p.values + e.dec_scaled_off, pb, S.bar);
        *S.nfix = 0;
    }

    // A1: in[j] = payload[j] (+ filtered_c[j] for each incoming c, in plan order)
    for (int idx = threadIdx.x; idx < DMAX * 32; idx += kThreads) {
        const int j = idx >> 5;
        float acc = 0.0f;
        if (j < e.d) {
            acc = __ldg(p.values + e.in_init_off + j);
            if (valid) {
                const float* col = A + static_cast<int64_t>(j) * B + b;
                const int64_t* src = p.incoming + e.inc_begin;
                int q = 0;
                for (; q + 4 <= e.inc_count; q += 4) {  // four loads in flight, summed in order
                    const float f0 = col[__ldg(src + q)], f1 = col[__ldg(src + q + 1)];
                    const float f2 = col[__ldg(src + q + 2)], f3 = col[__ldg(src + q + 3)];
                    acc = acc + f0;
                    acc = acc + f1;
                    acc = acc + f2;
                    acc = acc + f3;
                }
                for (; q < e.inc_count; ++q) acc = acc + col[__ldg(src + q)];
                if (last) A[e.in_base + static_cast<int64_t>(j) * B + b] = acc;
            }
        }
        S.in[j * 32 + lane] = acc;  // padding rows hold +0
    }
    __syncthreads();

    float x[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = S.in[j * 32 + lane];
    mbar_wait(S.bar, parity);
    tk.tick(FS_A1);

    // A2: encoder + lif_spike_step<float> (neuron_math.hpp:55-77), speculative transcendentals.
    // Neurons go in pairs through the paired fp32 pipe (FADD2/FMUL2: two IEEE
    // round-to-nearest operations per instruction, bit-identical to scalar ones);
    // the rarely taken transcendental branches stay scalar.
    const float dt = e.dt, tau_rc = e.tau_rc, tau_ref = e.tau_ref, amp_dt = e.amp_dt, em_dt = e.em_dt;
    const int npw = ((e.n + kWarps - 1) / kWarps + kUnroll - 1) / kUnroll * kUnroll;
    const int nbeg = warp * npw, nend = min(e.n, nbeg + npw);
    float* vp = A + e.v_base + b + static_cast<int64_t>(nbeg) * B;  // row i0 of the current round
    float* rp = A + e.r_base + b + static_cast<int64_t>(nbeg) * B;
    const float2 dt2 = make_float2(dt, dt), ndt2 = make_float2(-dt, -dt);
    float vnx[kUnroll], rnx[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
        vnx[u] = rnx[u] = 0.f;
        if (nbeg + u < nend && valid) {
            vnx[u] = __ldcs(vp + u * B);
            rnx[u] = __ldcs(rp + u * B);
        }
    }
    for (int i0 = nbeg; i0 < nend; i0 += kUnroll, vp += kUnroll * B, rp += kUnroll * B) {
        float v[kUnroll], r[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            v[u] = vnx[u];
            r[u] = rnx[u];
            vnx[u] = rnx[u] = 0.f;
            if (i0 + kUnroll + u < nend && valid) {  // prefetch the next round
                vnx[u] = __ldcs(vp + (kUnroll + u) * B);
                rnx[u] = __ldcs(rp + (kUnroll + u) * B);
            }
        }
#pragma unroll
        for (int k = 0; k < kUnroll / 2; ++k) {
            const int i = i0 + 2 * k;
            if (i >= nend) break;  // warp-uniform
            // DotInc(E, in, J) for neurons i, i+1: acc from +0, j ascending, then J = bias + acc.
            // Products two dims at a time (FMUL2), sums scalar and in order.  A
            // paired product must never feed a paired sum: ptxas contracts
            // FMUL2 -> FADD2 into FFMA2 even for .rn (tests/test_abi.py checks the SASS).
            float acc[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const float4* er = reinterpret_cast<const float4*>(S.E + (i + h) * DMAX);
                float a = 0.0f;
#pragma unroll
                for (int q = 0; q < DMAX / 4; ++q) {
                    const float4 w = er[q];
                    const float2 m0 = __fmul2_rn(make_float2(w.x, w.y), make_float2(x[4 * q], x[4 * q + 1]));
                    const float2 m1 = __fmul2_rn(make_float2(w.z, w.w), make_float2(x[4 * q + 2], x[4 * q + 3]));
                    a = a + m0.x;
                    a = a + m0.y;
                    a = a + m1.x;
                    a = a + m1.y;
                }
                acc[h] = a;
            }
            const float2 J2 = __fadd2_rn(*reinterpret_cast<const float2*>(S.bias + i), make_float2(acc[0], acc[1]));
            const float2 v2 = make_float2(v[2 * k], v[2 * k + 1]), r2 = make_float2(r[2 * k], r[2 * k + 1]);
            const float2 dl2 = __fadd2_rn(dt2, make_float2(-r2.x, -r2.y));  // dt - r
            const float2 rr2 = __fadd2_rn(r2, ndt2);                        // r - dt
            float em[2];
            bool doubt[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float delta = h ? dl2.y : dl2.x;
                if (delta < 0.0f) delta = 0.0f;
                if (delta > dt) delta = dt;
                // expm1(-delta/tau_rc): delta == dt -> the host glibc value; delta == +0 -> expm1(-0) = -0
                em[h] = delta == dt ? em_dt : -0.0f;
                doubt[h] = false;
                if (valid && delta != dt && delta != 0.0f) {
                    // == -delta / tau_rc in IEEE float: the double product is within 2^-52 of the quotient,
                    // and a quotient of floats is never within 2^-49 of a float midpoint unless on it,
                    // which needs a power-of-two divisor (then the product is exact)
                    const float xa = static_cast<float>(static_cast<double>(-delta) * e.inv_tau_rc);
                    if (lif_range(xa)) {
                        const Spec s = spec_lif(xa, false, p.libm);
                        em[h] = s.r;
                        doubt[h] = s.doubtful;
                    } else {
                        em[h] = glibc_expm1f(xa, p.libm);
                    }
                }
            }
            // v - (J - v) * em: scalar products between the paired sums (see above)
            const float2 d2 = __fadd2_rn(J2, make_float2(-v2.x, -v2.y));
            const float t0 = __fmul_rn(d2.x, em[0]), t1 = __fmul_rn(d2.y, em[1]);
            const float2 vn2 = __fadd2_rn(v2, make_float2(-t0, -t1));
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h && i + 1 >= nend) break;  // warp-uniform
                const float J = h ? J2.y : J2.x, vh = h ? v2.y : v2.x, rh = h ? r2.y : r2.x;
                float vn = h ? vn2.y : vn2.x;
                if (vn < 0.0f) vn = 0.0f;
                const bool spike = valid && vn > 1.0f;
                bool dbt = doubt[h];
                float vo, ro;
                if (spike) {
                    const float xl = -(vn - 1.0f) / (J - 1.0f);
                    float lg;
                    if (lif_range(xl)) {
                        const Spec s = spec_lif(xl, true, p.libm);
                        lg = s.r;
                        dbt = dbt || s.doubtful;
                    } else {
                        lg = glibc_log1pf(xl, p.libm);
                    }
                    const float since = -tau_rc * lg;
                    vo = 0.0f;
                    ro = tau_ref - since;
                } else {
                    vo = vn;
                    ro = rh > dt ? (h ? rr2.y : rr2.x) : 0.0f;
                }
                bool spike_final = spike;
                if (dbt) {  // queue the neuron for exact resolution from its original inputs
                    const int slot = atomicAdd(S.nfix, 1);
                    if (slot < kFixCap) {
                        S.fix[slot] = {((i + h) << 5) | lane, vh, rh, J};
                    } else {  // queue full: resolve right here
                        float ve = vh, re = rh;
                        spike_final = lif_exact(J, ve, re, dt, tau_rc, tau_ref, p.libm);
                        vo = ve;
                        ro = re;
                    }
                }
                const uint32_t word = __ballot_sync(0xffffffffu, spike_final);
                if (valid) {
                    __stcs(vp + (2 * k + h) * B, vo);
                    __stcs(rp + (2 * k + h) * B, ro);
                    if (last) {
                        A[e.j_base + static_cast<int64_t>(i + h) * B + b] = J;
                        A[e.out_base + static_cast<int64_t>(i + h) * B + b] = spike_final ? amp_dt : 0.0f;
                    }
                }
                if (lane == 0) S.words[i + h] = word;
            }
        }
    }
    __syncthreads();
    tk.tick(FS_A2);

    // A2': exact resolution of the queued neurons (all threads, probes overlap)
    const int nfix = min(*S.nfix, kFixCap);
    // Stage 1 re-derives the speculative arguments and probes the tables for
    // both at once; only a real glibc exception (~0.6% of queued neurons)
    // triggers the exact recomputation and the patch.
    for (int f = threadIdx.x; f < nfix; f += kThreads) {
        const FixEntry fe = S.fix[f];
        const int i = fe.key >> 5, l = fe.key & 31;
        float delta = dt - fe.r;
        if (delta < 0.0f) delta = 0.0f;
        if (delta > dt) delta = dt;
        const float xe = -delta / tau_rc;
        const bool pe = delta != dt && delta != 0.0f && lif_range(xe);
        float em = delta == dt ? em_dt : -0.0f;
        bool de = false;
        if (delta != dt && delta != 0.0f) {
            if (pe) {
                const Spec s = spec_lif(xe, false, p.libm);
                em = s.r;
                de = s.doubtful;
            } else {
                em = glibc_expm1f(xe, p.libm);
            }
        }
        float vn = fe.v - (fe.J - fe.v) * em;
        if (vn < 0.0f) vn = 0.0f;
        const float xl = -(vn - 1.0f) / (fe.J - 1.0f);
        const bool dl = vn > 1.0f && lif_range(xl) && spec_lif(xl, true, p.libm).doubtful;
        const LibmHash &h0 = p.libm.t[0], &h1 = p.libm.t[1];
        const uint32_t ke = __float_as_uint(xe), kl = __float_as_uint(xl);
        uint32_t ie = (ke * 0x9E3779B1u) >> h0.hot_shift, il = (kl * 0x9E3779B1u) >> h1.hot_shift;
        unsigned long long se = de ? __ldg(h0.hot_slots + ie) : 0ull;  // both first probes in flight
        unsigned long long sl = dl ? __ldg(h1.hot_slots + il) : 0ull;
        while (se != 0ull && static_cast<uint32_t>(se >> 32) != ke) {
            ie = (ie + 1u) & h0.hot_mask;
            se = __ldg(h0.hot_slots + ie);
        }
        while (sl != 0ull && static_cast<uint32_t>(sl >> 32) != kl) {
            il = (il + 1u) & h1.hot_mask;
            sl = __ldg(h1.hot_slots + il);
        }
        if (se == 0ull && sl == 0ull) continue;  // neither value is an exception: the speculation stands
        float ve = fe.v, re = fe.r;
        const bool spk = lif_exact(fe.J, ve, re, dt, tau_rc, tau_ref, p.libm);
        const int64_t o = static_cast<int64_t>(i) * B + b0 + l;
        A[e.v_base + o] = ve;
        A[e.r_base + o] = re;
        if (last) A[e.out_base + o] = spk ? amp_dt : 0.0f;
        if (spk != static_cast<bool>((S.words[i] >> l) & 1u)) atomicXor(S.words + i, 1u << l);
    }
    __syncthreads();
    tk.tick(FS_FIX);

    // A3: transpose neuron words (bit = column) into column words (bit = neuron)
    const int nw = (e.n + 31) >> 5;
    for (int w = warp; w < nw; w += kWarps) {
        const int i = w * 32 + lane;
        const uint32_t mine = i < e.n ? S.words[i] : 0u;
#pragma unroll 8
        for (int c = 0; c < 32; ++c) {
            const uint32_t bits = __ballot_sync(0xffffffffu, (mine >> c) & 1u);
            if (lane == c) S.col[c * p.nwords + w] = bits;
        }
    }
    __syncthreads();
    tk.tick(FS_A3);

    // A4: decoders over the spiking neurons of each column, ascending i; the
    // terms are the precomputed products fp32(D[r,i]) * fp32(amp/dt), stored
    // transposed ([n][dx]).  Staged and dx % 4 == 0: lane = column, one warp
    // per 4 decoded rows, one LDS.128 and four independent sums per spike.
    if (p.stage_dec && (e.dx & 3) == 0) {
        const int stride4 = e.dx >> 2;
        const uint32_t* cw = S.col + lane * p.nwords;
        for (int g = warp; g < stride4; g += kWarps) {
            const float4* P4 = reinterpret_cast<const float4*>(S.P) + g;
            float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
            for (int w = 0; w < nw; ++w) {
                uint32_t bits = cw[w];
                while (bits) {
                    const int i1 = w * 32 + __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const float4 t = P4[i1 * stride4];
                    a0 = a0 + t.x;
                    a1 = a1 + t.y;
                    a2 = a2 + t.z;
                    a3 = a3 + t.w;
                }
            }
            if (valid) {
                const float* init = p.values + e.xhat_init_off + 4 * g;
                float* xo = A + e.xhat_base + static_cast<int64_t>(4 * g) * B + b;
                xo[0] = __ldg(init) + a0;
                xo[B] = __ldg(init + 1) + a1;
                xo[2 * B] = __ldg(init + 2) + a2;
                xo[3 * B] = __ldg(init + 3) + a3;
            }
        }
        __syncthreads();
        tk.tick(FS_A4);
        return;
    }
    // general layout: lanes are (column, row) with the row fastest, so the
    // rows of one column walk the same spike list together
    const int rd = e.dx <= 1 ? 1 : 1 << (32 - __clz(e.dx - 1));  // rows per column group (pow2 <= 32)
    for (int idx = threadIdx.x; idx < 32 * rd; idx += kThreads) {
        const int l = idx / rd, rrow = idx - l * rd, bb = b0 + l;
        const bool act = bb < B && rrow < e.dx;
        const float* pc = (p.stage_dec ? S.P : p.values + e.dec_scaled_off) + rrow;
        float acc = 0.0f;
        const uint32_t* cw = S.col + l * p.nwords;
        for (int w = 0; w < nw; ++w) {
            uint32_t bits = cw[w];
            const float* pw = pc + static_cast<int64_t>(w) * 32 * e.dx;
            while (bits) {
                const int i1 = __ffs(bits) - 1;
                bits &= bits - 1u;
                if (bits) {
                    const int i2 = __ffs(bits) - 1;
                    bits &= bits - 1u;
                    const float t1 = act ? pw[i1 * e.dx] : 0.f, t2 = act ? pw[i2 * e.dx] : 0.f;
                    acc = acc + t1;
                    acc = acc + t2;
                } else {
                    acc = acc + (act ? pw[i1 * e.dx] : 0.f);
                }
            }
        }
        if (act) A[e.xhat_base + static_cast<int64_t>(rrow) * B + bb] = __ldg(p.values + e.xhat_init_off + rrow) + acc;
    }
    __syncthreads();
    tk.tick(FS_A4);
}

template <int DMAX, int BT>
__device__ __forceinline__ void phase_b_item(const FusedProgram& p, int c, int b, bool last, int ks) {
    const int B = batch_of<BT>(p);
    const FConn& cn = p.conns[c];
    float* A = p.arena;
    float x[DMAX];
    // a fed source is read straight from the staged feed block of step ks
    // (write_feeds precedes every reader, exec.cpp:353-356); the arena copy
    // of fed nodes is refreshed on a call's last step only
    const float* src = (cn.src_feed >= 0 && p.feed_present[cn.src_feed])
                           ? p.feed_data + p.feed_off[cn.src_feed] + static_cast<int64_t>(ks) * cn.ds * B + b
                           : A + cn.src_base + b;
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = j < cn.ds ? src[j * B] : 0.0f;
    const float4* T = reinterpret_cast<const float4*>(p.values + cn.tpad_off);
    float* st = A + cn.state_base + b;
    float s0[DMAX];  // every state load in flight before the arithmetic
#pragma unroll
    for (int r = 0; r < DMAX; ++r) s0[r] = r < cn.dd ? st[r * B] : 0.0f;
#pragma unroll
    for (int r = 0; r < DMAX; ++r) {
        if (r >= cn.dd) break;
        float acc = 0.0f;
#pragma unroll
        for (int q = 0; q < DMAX / 4; ++q) {
            const float4 w = __ldg(T + r * (DMAX / 4) + q);
            acc = acc + w.x * x[4 * q];
            acc = acc + w.y * x[4 * q + 1];
            acc = acc + w.z * x[4 * q + 2];
            acc = acc + w.w * x[4 * q + 3];
        }
        const float accv = __ldg(p.values + cn.acc_init_off + r) + acc;
        const float f = cn.a * s0[r] + cn.b * accv;  // lowpass_step (neuron_math.hpp:39-42)
        st[r * B] = f;
        if (last) {
            A[cn.acc_base + static_cast<int64_t>(r) * B + b] = accv;
            A[cn.filt_base + static_cast<int64_t>(r) * B + b] = f;
        }
        if (cn.probe_filt >= 0)
            p.ring[p.ring_off[cn.probe_filt] + (static_cast<int64_t>(ks) * cn.dd + r) * B + b] = f;
        if (cn.probe_state >= 0)
            p.ring[p.ring_off[cn.probe_state] + (static_cast<int64_t>(ks) * cn.dd + r) * B + b] = f;
    }
}

template <int DMAX>
__device__ Smem carve(uint32_t* base, const FusedProgram& p) {
    Smem S;
    char* at = reinterpret_cast<char*>(base);
    S.bar = reinterpret_cast<uint64_t*>(at);
    S.nfix = reinterpret_cast<int*>(at + 8);
    S.next_unit = reinterpret_cast<int*>(at + 12);
    at += 128;
    S.E = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.nmax) * DMAX * 4;
    S.bias = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.nmax) * 4;
    S.P = reinterpret_cast<float*>(at);
    at += static_cast<size_t>(p.stage_dec ? p.pmax_floats : 0) * 4;
    S.in = reinterpret_cast<float*>(at);
    at += DMAX * 32 * 4;
    S.words = reinterpret_cast<uint32_t*>(at);
    at += static_cast<size_t>(p.nmax) * 4;
    S.col = reinterpret_cast<uint32_t*>(at);
    at += static_cast<size_t>(32) * p.nwords * 4;
    S.fix = reinterpret_cast<FixEntry*>(at);
    return S;
}

template <int DMAX>
size_t smem_bytes(const FusedProgram& p) {
    return 128 + static_cast<size_t>(p.nmax) * DMAX * 4 + static_cast<size_t>(p.nmax) * 4 +
           static_cast<size_t>(p.stage_dec ? p.pmax_floats : 0) * 4 + DMAX * 32 * 4 +
           static_cast<size_t>(p.nmax) * 4 + static_cast<size_t>(32) * p.nwords * 4 + sizeof(FixEntry) * kFixCap;
}

template <int DMAX, int BT, bool PROF>
__global__ void __launch_bounds__(kThreads, 3) fused_run_kernel(FusedProgram p, int k_begin, int k_end) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) uint32_t smem[];
    const Smem S = carve<DMAX>(smem, p);
    if (threadIdx.x == 0) mbar_init(S.bar);
    __syncthreads();
    uint32_t parity = 0;
    const int B = batch_of<BT>(p);
    const int units = p.n_ens * p.btiles;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    Ticker<PROF> tk;
    tk.start();

    for (int k = k_begin; k < k_end; ++k) {
        const bool last = k == p.call_steps - 1;
        // write_feeds (exec.cpp:313-326) into the arena: only the last step's
        // values survive a call, and phase B reads fed sources from the feed block
        for (int f = 0; last && f < p.n_feeds; ++f) {
            if (!p.feed_present[f]) continue;
            const FFeed& fd = p.feeds[f];
            const float* src = p.feed_data + p.feed_off[f] + static_cast<int64_t>(k) * fd.dim * B;
            const int64_t n = static_cast<int64_t>(fd.dim) * fd.copies;
            for (int64_t i = gtid; i < n; i += gthreads) {
                const int64_t d = i / fd.copies;
                const int bb = static_cast<int>(i - d * fd.copies);
                p.arena[fd.base + d * (fd.copies > 1 ? B : 1) + bb] = src[d * B + bb];
            }
        }
        tk.tick(FS_FEED);
        // phase A: units claimed dynamically (counter k & 1, reset a step ahead)
        int* work = p.work + (k & 1);
        for (;;) {
            if (threadIdx.x == 0) *S.next_unit = atomicAdd(work, 1);
            __syncthreads();
            const int u = *S.next_unit;
            if (u >= units) break;  // uniform; the next write of next_unit follows a barrier inside the unit
            phase_a_unit<DMAX, BT, PROF>(p, u, last, S, parity, tk);
            parity ^= 1u;
        }
        grid_sync(grid);
        tk.tick(FS_BAR1);
        if (gtid == 0) p.work[(k + 1) & 1] = 0;  // last used by step k-1; next used by step k+1
        // phase B: connections (item = column-fastest, so a warp shares one
        // connection when B % 32 == 0), then time and captures of phase-A values
        const int64_t items = static_cast<int64_t>(p.n_conn) * B;
        for (int64_t it = gtid; it < items; it += gthreads) {
            const int c = static_cast<int>(it / B);
            phase_b_item<DMAX, BT>(p, c, static_cast<int>(it - static_cast<int64_t>(c) * B), last, k);
        }
        for (int q = 0; q < p.n_probes; ++q) {
            const FProbe& pr = p.probes[q];
            const int64_t n = static_cast<int64_t>(pr.dim) * B;
            float* dst = p.ring + p.ring_off[pr.index] + static_cast<int64_t>(k) * pr.dim * B;
            const bool fed = pr.feed_slot >= 0 && p.feed_present[pr.feed_slot];
            const float* fsrc = fed ? p.feed_data + p.feed_off[pr.feed_slot] + static_cast<int64_t>(k) * pr.dim * B
                                    : nullptr;
            for (int64_t i = gtid; i < n; i += gthreads) {
                const int64_t d = i / B;
                const int bb = static_cast<int>(i - d * B);
                dst[i] = fed ? fsrc[d * B + (pr.per_batch ? bb : 0)] : p.arena[pr.base + (pr.per_batch ? d * B + bb : d)];
            }
        }
        if (p.has_time && gtid == 0) {  // TimeUpdate (exec.cpp:300-309)
            const float next = p.arena[p.step_base] + 1.0f;
            p.arena[p.step_base] = next;
            p.arena[p.time_base] = next * p.dt;
            if (p.time_probe_step >= 0)
                for (int bb = 0; bb < B; ++bb) p.ring[p.ring_off[p.time_probe_step] + static_cast<int64_t>(k) * B + bb] = next;
            if (p.time_probe_time >= 0)
                for (int bb = 0; bb < B; ++bb)
                    p.ring[p.ring_off[p.time_probe_time] + static_cast<int64_t>(k) * B + bb] = next * p.dt;
        }
        tk.tick(FS_B);
        grid_sync(grid);
        tk.tick(FS_BAR2);
    }
    tk.flush(p.prof);
}

template <int DMAX, int BT, bool PROF>
cudaError_t launch_t(const FusedProgram& p, int grid, int k0, int k1, cudaStream_t stream) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fused_run_kernel<DMAX, BT, PROF>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    FusedProgram prog = p;
    void* args[] = {&prog, &k0, &k1};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_run_kernel<DMAX, BT, PROF>), dim3(grid),
                                       dim3(kThreads), args, sm, stream);
}

template <int DMAX, int BT>
int max_grid_t(const FusedProgram& p, int device) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 227 * 1024) return 0;
    if (sm > 48 * 1024) {
        cudaFuncSetAttribute(fused_run_kernel<DMAX, BT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
        cudaFuncSetAttribute(fused_run_kernel<DMAX, BT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sm));
    }
    int per_sm = 0, per_sm_prof = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_run_kernel<DMAX, BT, false>, kThreads, sm);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_prof, fused_run_kernel<DMAX, BT, true>, kThreads, sm);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (per_sm < per_sm_prof ? per_sm : per_sm_prof) * sms;
}

// Batch widths with a stride-specialised kernel (others run the runtime-stride one).
#define NENG_FUSED_BATCHES(X) X(32) X(256)

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

cudaError_t launch_fused(const FusedProgram& p, int dmax, int grid, int k0, int k1, cudaStream_t stream) {
    const bool prof = p.prof != nullptr;
    switch (dmax) {
        case 8: return prof ? launch_d<8, true>(p, grid, k0, k1, stream) : launch_d<8, false>(p, grid, k0, k1, stream);
        case 16: return prof ? launch_d<16, true>(p, grid, k0, k1, stream) : launch_d<16, false>(p, grid, k0, k1, stream);
        case 32: return prof ? launch_d<32, true>(p, grid, k0, k1, stream) : launch_d<32, false>(p, grid, k0, k1, stream);
    }
    return cudaErrorInvalidValue;
}

int fused_max_grid(const FusedProgram& p, int dmax, int device) {
    switch (dmax) {
        case 8: return max_grid_d<8>(p, device);
        case 16: return max_grid_d<16>(p, device);
        case 32: return max_grid_d<32>(p, device);
    }
    return 0;
}

}  // namespace nengb
