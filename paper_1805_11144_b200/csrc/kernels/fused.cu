// fused.cu — the fused ensemble pipeline: one persistent cooperative kernel
// advancing K timesteps, two grid barriers per step (see fused.hpp).
//
// Phase A maps lane = batch column, warp = neuron: the ensemble's input
// vector sits in 8-16 registers per lane for the whole unit, encoder rows
// and biases are warp-uniform loads, and v/r stream coalesced
// (arena layout [row][B], 128 B per warp access, evict-first hints since
// they are 2 GB at config 4 and never reused within a step).  Spikes leave
// the LIF as ballot words per neuron, are bit-transposed with ballots to
// per-column words, and the decoder walks only the set bits in ascending
// neuron order: skipping out[i] == 0 is exact for finite decoders because a
// running sum that starts at +0 never becomes -0 and x + (+-0) == x.
//
// Every floating-point operation is the reference's, in its order:
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

__device__ __forceinline__ void grid_sync(cg::grid_group& g) {
    if (gridDim.x == 1)
        __syncthreads();
    else
        g.sync();
}

template <int DMAX>
__device__ void phase_a_unit(const FusedProgram& p, int unit, bool last, float* s_in, uint32_t* s_words,
                             uint32_t* s_col) {
    const int B = p.batch;
    const int t = unit / p.btiles;
    const int b0 = (unit - t * p.btiles) * 32;
    const FEns& e = p.ens[t];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int b = b0 + lane;
    const bool valid = b < B;
    float* A = p.arena;

    // A1: in[j] = payload[j] (+ filtered_c[j] for each incoming c, in plan order)
    for (int idx = threadIdx.x; idx < e.d * 32; idx += kThreads) {
        const int j = idx >> 5;
        float acc = __ldg(p.values + e.in_init_off + j);
        if (valid) {
            for (int q = 0; q < e.inc_count; ++q) {
                const FConn& c = p.conns[__ldg(p.incoming + e.inc_begin + q)];
                acc = acc + A[c.state_base + static_cast<int64_t>(j) * B + b];
            }
            if (last) A[e.in_base + static_cast<int64_t>(j) * B + b] = acc;
        }
        s_in[j * 32 + lane] = acc;
    }
    __syncthreads();

    float x[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = j < e.d ? s_in[j * 32 + lane] : 0.0f;

    // A2: encoder + LIF, one neuron per warp iteration, kUnroll neurons in flight
    const float dt = e.dt, tau_rc = e.tau_rc, tau_ref = e.tau_ref, amp = e.amplitude, amp_dt = e.amp_dt;
    const float em_dt = e.em_dt;
    for (int i0 = warp; i0 < e.n; i0 += kWarps * kUnroll) {
        float vv[kUnroll], rr[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = i0 + u * kWarps;
            vv[u] = 0.f;
            rr[u] = 0.f;
            if (i < e.n && valid) {
                vv[u] = __ldcs(A + e.v_base + static_cast<int64_t>(i) * B + b);
                rr[u] = __ldcs(A + e.r_base + static_cast<int64_t>(i) * B + b);
            }
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const int i = i0 + u * kWarps;
            if (i >= e.n) break;
            const float* erow = A + e.enc_base + static_cast<int64_t>(i) * e.d;
            float acc = 0.0f;
#pragma unroll
            for (int j = 0; j < DMAX; ++j)
                if (j < e.d) acc = acc + __ldg(erow + j) * x[j];
            const float J = __ldg(p.values + e.bias_off + i) + acc;
            // lif_spike_step<float> (neuron_math.hpp:55-77)
            float v = vv[u], r = rr[u];
            float delta = dt - r;
            if (delta < 0.0f) delta = 0.0f;
            if (delta > dt) delta = dt;
            const float em = delta == dt ? em_dt : glibc_expm1f(-delta / tau_rc, p.libm);
            float vn = v - (J - v) * em;
            if (vn < 0.0f) vn = 0.0f;
            const bool spike = vn > 1.0f;
            float out;
            if (spike) {
                const float since = -tau_rc * glibc_log1pf(-(vn - 1.0f) / (J - 1.0f), p.libm);
                out = amp_dt;
                v = 0.0f;
                r = tau_ref - since;
            } else {
                out = 0.0f;
                v = vn;
                r = r > dt ? r - dt : 0.0f;
            }
            const uint32_t word = __ballot_sync(0xffffffffu, spike && valid);
            if (valid) {
                __stcs(A + e.v_base + static_cast<int64_t>(i) * B + b, v);
                __stcs(A + e.r_base + static_cast<int64_t>(i) * B + b, r);
                if (last) {
                    A[e.j_base + static_cast<int64_t>(i) * B + b] = J;
                    A[e.out_base + static_cast<int64_t>(i) * B + b] = out;
                }
            }
            if (lane == 0) s_words[i] = word;
        }
    }
    (void)amp;
    __syncthreads();

    // A3: transpose neuron words (bit = column) into column words (bit = neuron)
    const int nw = (e.n + 31) >> 5;
    for (int w = warp; w < nw; w += kWarps) {
        const int i = w * 32 + lane;
        const uint32_t mine = i < e.n ? s_words[i] : 0u;
#pragma unroll 4
        for (int col = 0; col < 32; ++col) {
            const uint32_t bits = __ballot_sync(0xffffffffu, (mine >> col) & 1u);
            if (lane == col) s_col[col * p.nwords + w] = bits;
        }
    }
    __syncthreads();

    // A4: decoders over the spiking neurons of each column, ascending i
    for (int idx = threadIdx.x; idx < e.dx * 32; idx += kThreads) {
        const int rrow = idx >> 5, l = idx & 31, bb = b0 + l;
        if (bb >= B) continue;
        const float* drow = A + e.dec_base + static_cast<int64_t>(rrow) * e.n;
        float acc = 0.0f;
        for (int w = 0; w < nw; ++w) {
            uint32_t bits = s_col[l * p.nwords + w];
            while (bits) {
                const int bit = __ffs(bits) - 1;
                acc = acc + __ldg(drow + w * 32 + bit) * amp_dt;
                bits &= bits - 1u;
            }
        }
        A[e.xhat_base + static_cast<int64_t>(rrow) * B + bb] = __ldg(p.values + e.xhat_init_off + rrow) + acc;
    }
    __syncthreads();
}

template <int DMAX>
__device__ void phase_b_item(const FusedProgram& p, int64_t item, bool last, int ks) {
    const int B = p.batch;
    const int c = static_cast<int>(item / B);
    const int b = static_cast<int>(item - static_cast<int64_t>(c) * B);
    const FConn& cn = p.conns[c];
    float* A = p.arena;
    float x[DMAX];
#pragma unroll
    for (int j = 0; j < DMAX; ++j) x[j] = j < cn.ds ? A[cn.src_base + static_cast<int64_t>(j) * B + b] : 0.0f;
    for (int r = 0; r < cn.dd; ++r) {
        const float* trow = A + cn.t_base + static_cast<int64_t>(r) * cn.ds;
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < DMAX; ++j)
            if (j < cn.ds) acc = acc + __ldg(trow + j) * x[j];
        const float accv = __ldg(p.values + cn.acc_init_off + r) + acc;
        const int64_t o = static_cast<int64_t>(r) * B + b;
        const float f = cn.a * A[cn.state_base + o] + cn.b * accv;  // lowpass_step
        A[cn.state_base + o] = f;
        if (last) {
            A[cn.acc_base + o] = accv;
            A[cn.filt_base + o] = f;
        }
        if (cn.probe_filt >= 0)
            p.ring[p.ring_off[cn.probe_filt] + (static_cast<int64_t>(ks) * cn.dd + r) * B + b] = f;
        if (cn.probe_state >= 0)
            p.ring[p.ring_off[cn.probe_state] + (static_cast<int64_t>(ks) * cn.dd + r) * B + b] = f;
    }
}

template <int DMAX>
__global__ void __launch_bounds__(kThreads) fused_run_kernel(FusedProgram p, int k_begin, int k_end) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ uint32_t smem[];
    float* s_in = reinterpret_cast<float*>(smem);
    uint32_t* s_words = smem + DMAX * 32;
    uint32_t* s_col = s_words + p.nmax;
    const int B = p.batch;
    const int units = p.n_ens * p.btiles;
    const int64_t gthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t gtid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;

    for (int k = k_begin; k < k_end; ++k) {
        const bool last = k == p.call_steps - 1;
        // write_feeds (exec.cpp:313-326)
        for (int f = 0; f < p.n_feeds; ++f) {
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
        // phase A
        for (int u = blockIdx.x; u < units; u += gridDim.x) phase_a_unit<DMAX>(p, u, last, s_in, s_words, s_col);
        grid_sync(grid);
        // phase B: connections, time, captures of phase-A-final values
        const int64_t items = static_cast<int64_t>(p.n_conn) * B;
        for (int64_t it = gtid; it < items; it += gthreads) phase_b_item<DMAX>(p, it, last, k);
        for (int q = 0; q < p.n_probes; ++q) {
            const FProbe& pr = p.probes[q];
            const int64_t n = static_cast<int64_t>(pr.dim) * B;
            float* dst = p.ring + p.ring_off[pr.index] + static_cast<int64_t>(k) * pr.dim * B;
            for (int64_t i = gtid; i < n; i += gthreads) {
                const int64_t d = i / B;
                const int bb = static_cast<int>(i - d * B);
                dst[i] = p.arena[pr.base + (pr.per_batch ? d * B + bb : d)];
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
        grid_sync(grid);
    }
}

template <int DMAX>
size_t smem_bytes(const FusedProgram& p) {
    return sizeof(float) * DMAX * 32 + sizeof(uint32_t) * (p.nmax + 32 * p.nwords);
}

template <int DMAX>
cudaError_t launch_t(const FusedProgram& p, int grid, int k0, int k1, cudaStream_t stream) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(fused_run_kernel<DMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    FusedProgram prog = p;
    void* args[] = {&prog, &k0, &k1};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_run_kernel<DMAX>), dim3(grid), dim3(kThreads),
                                       args, sm, stream);
}

template <int DMAX>
int max_grid_t(const FusedProgram& p, int device) {
    size_t sm = smem_bytes<DMAX>(p);
    if (sm > 48 * 1024)
        cudaFuncSetAttribute(fused_run_kernel<DMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fused_run_kernel<DMAX>, kThreads, sm);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

}  // namespace

int fused_dmax_for(int d) { return d <= 8 ? 8 : d <= 16 ? 16 : d <= 32 ? 32 : 0; }

cudaError_t launch_fused(const FusedProgram& p, int dmax, int grid, int k0, int k1, cudaStream_t stream) {
    switch (dmax) {
        case 8: return launch_t<8>(p, grid, k0, k1, stream);
        case 16: return launch_t<16>(p, grid, k0, k1, stream);
        case 32: return launch_t<32>(p, grid, k0, k1, stream);
    }
    return cudaErrorInvalidValue;
}

int fused_max_grid(const FusedProgram& p, int dmax, int device) {
    switch (dmax) {
        case 8: return max_grid_t<8>(p, device);
        case 16: return max_grid_t<16>(p, device);
        case 32: return max_grid_t<32>(p, device);
    }
    return 0;
}

}  // namespace nengb
