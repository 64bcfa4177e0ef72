// generic.cu — the persistent cooperative interpreter: advances K timesteps
// per launch over ANY planned model, one pass per plan group with a grid
// barrier between dependent passes (the reference's run loop, exec.cpp:340-366,
// with each Instr's `for b < copies: exec(ins, b)` flattened into one parallel
// pass over (member, element, batch copy)).
//
// Exactness argument: members of a group never overlap in writes and never
// read what another member of the same group writes (every write/read pair on
// overlapping rows is a dependency edge, ir.cpp:351-360, and validate_plan
// puts edge endpoints in different groups, passes.cpp:279-305), so any
// parallel order inside a pass is exact.  Two cases are not data-parallel and
// run in the reference's loop order instead:
//   GF_SERIAL_ALL  a member whose written operand overlaps another operand of
//                  the same member at a different offset (e.g. Copy(s[0:3] ->
//                  s[1:4], inc) cascades); one thread, exact reference loops.
//   GF_SERIAL_B    a per-batch group that writes shared storage: copies b run
//                  in order, elements in parallel within each b.
// Every float operation is the reference's (no FMA: -fmad=false; IEEE div).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "libm.cuh"
#include "neng_gpu.h"
#include "program.hpp"

namespace cg = cooperative_groups;

namespace nengb {

__device__ __forceinline__ float* at(const GenericProgram& p, const DArg& a, int64_t e, int b) {
    return p.arena + a.base + e * a.es + static_cast<int64_t>(b) * a.bs;
}

// One work item of a data-parallel group. local indexes the member's
// per-copy work (element, row, or (row, col) for PES).
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}

/// SMALL: the arena is in shared memory (generic_small_kernel).
template <bool SMALL = false>
__device__ __forceinline__ void exec_item(const GenericProgram& p, const DGroup& g, const DMember& m,
                                          int64_t local, int b) {
    switch (g.kind) {
        case 0: {  // Reset (exec.cpp:179-188)
            *at(p, m.a[0], local, b) = p.values[m.value_at + local];
            break;
        }
        case 1: {  // Copy (exec.cpp:189-210)
            float s = *at(p, m.a[0], local, b);
            float* d = at(p, m.a[1], local, b);
            if (g.flags & GF_INC)
                *d = *d + s;
            else
                *d = s;
            break;
        }
        case 2: {  // ElementwiseInc (exec.cpp:211-225)
            float a = (m.flags & MF_SCALAR_A) ? *at(p, m.a[0], 0, b) : *at(p, m.a[0], local, b);
            float x = *at(p, m.a[1], local, b);
            float* y = at(p, m.a[2], local, b);
            *y = *y + a * x;
            break;
        }
        case 3: {  // DotInc (exec.cpp:226-240): acc = 0; acc += A[r,k]*x[k] in k order; y[r] += acc
            const int64_t n = m.a[1].elems;
            const float* arow = at(p, m.a[0], local * n, b);
            const int32_t aes = m.a[0].es;
            const float* x = at(p, m.a[1], 0, b);
            const int32_t xes = m.a[1].es;
            float acc = 0.0f;
            if (!SMALL && (m.flags & MF_SKIP_ZERO_X)) {  // x[k] first; A[r,k] only for the nonzero terms
                {
#pragma unroll 8
                    for (int64_t k = 0; k < n; ++k) {
                        const float xk = x[k * xes];
                        if (xk != 0.0f) acc = acc + arow[k * aes] * xk;
                    }
                }
            } else if constexpr (SMALL) {  // shared-memory loads, issued ahead of the (sequential) sum
                const uint32_t ar = static_cast<uint32_t>(__cvta_generic_to_shared(arow));
                const uint32_t xr = static_cast<uint32_t>(__cvta_generic_to_shared(x));
                const uint32_t as = 4u * static_cast<uint32_t>(aes), xs = 4u * static_cast<uint32_t>(xes);
                const uint32_t n32 = static_cast<uint32_t>(n);
                uint32_t k = 0;
                for (; k + 8 <= n32; k += 8) {
                    float av[8], xv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        av[u] = lds_f32(ar + (k + u) * as);
                        xv[u] = lds_f32(xr + (k + u) * xs);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = acc + av[u] * xv[u];
                }
                for (; k < n32; ++k) acc = acc + lds_f32(ar + k * as) * lds_f32(xr + k * xs);
            } else {
#pragma unroll 8
                for (int64_t k = 0; k < n; ++k) acc = acc + arow[k * aes] * x[k * xes];
            }
            float* y = at(p, m.a[2], local, b);
            *y = *y + acc;
            break;
        }
        case 4: {  // SimNeurons (exec.cpp:241-266)
            float j = *at(p, m.a[0], local, b);
            float* out = at(p, m.a[1], local, b);
            if (g.neuron == NENG_NEURON_LIF) {
                float* vp = at(p, m.a[2], local, b);
                float* rp = at(p, m.a[3], local, b);
                float v = *vp, r = *rp;
                float o = lif_spike_step(j, v, r, g.dt, g.tau_rc, g.tau_ref, g.amplitude, p.libm, g.em_dt);
                *out = o;  // write order of exec.cpp:252-254 (last write wins on aliasing)
                *vp = v;
                *rp = r;
            } else if (g.neuron == NENG_NEURON_LIF_RATE) {
                *out = lif_rate_out(j, g.tau_rc, g.tau_ref, g.amplitude, p.libm);
            } else {
                *out = relu_out(j, g.amplitude);
            }
            break;
        }
        case 5: {  // SimProcess (exec.cpp:267-284)
            float in = *at(p, m.a[0], local, b);
            float* out = at(p, m.a[1], local, b);
            if (g.flags & GF_HAS_STATE) {
                float* st = at(p, m.a[2], local, b);
                float f = g.tau_a * *st + g.tau_b * in;  // lowpass_step
                *st = f;
                *out = f;
            } else {
                *out = in;
            }
            break;
        }
        case 6: {  // SimPES (exec.cpp:285-299): w[r,k] -= (scale*err[r]) * act[k]
            const int64_t n = m.a[0].elems;
            int64_t r = local / n, k = local - r * n;
            float row_scale = m.pes_scale * *at(p, m.a[1], r, b);
            float* w = at(p, m.a[2], local, b);
            *w = *w - row_scale * *at(p, m.a[0], k, b);
            break;
        }
        case 7: {  // TimeUpdate (exec.cpp:300-309)
            float* step = at(p, m.a[0], 0, b);
            float* time = at(p, m.a[1], 0, b);
            float next = *step + 1.0f;
            *step = next;
            *time = next * g.dt;
            break;
        }
    }
}

// DotInc on a 32-row x 64-column (batch) output tile of one member, by the
// whole CTA: A [M][K] shared row-major, x [K][B] and y [M][B] per-batch.  Each
// output keeps the reference's sum (acc = +0; acc += A[r,k]*x[k] for k
// ascending, each product and sum rounded; y += acc); A and x are staged
// through shared memory 32 k at a time.  Padding rows/columns hold +0, and a
// running sum from +0 is never -0, so the zero terms change nothing.
constexpr int kDTM = 32, kDTN = 64, kDTK = 32;  // 2 rows x 4 columns per thread
__device__ void dense_dot_tile(const GenericProgram& p, const DMember& m, int row0, int col0) {
    __shared__ float As[kDTK][kDTM + 4];
    __shared__ __align__(16) float Xs[kDTK][kDTN];
    const int B = p.batch;
    const int64_t M = m.a[2].elems, K = m.a[1].elems;
    const float* A = p.arena + m.a[0].base;
    const float* X = p.arena + m.a[1].base;
    float* Y = p.arena + m.a[2].base;
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    float acc[2][4];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.0f;
    for (int64_t k0 = 0; k0 < K; k0 += kDTK) {
#pragma unroll
        for (int i = 0; i < (kDTM * kDTK) / 256; ++i) {
            const int idx = threadIdx.x + i * 256;
            const int r = idx / kDTK, kk = idx - r * kDTK;
            const int64_t gr = row0 + r, gk = k0 + kk;
            As[kk][r] = (gr < M && gk < K) ? A[gr * K + gk] : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < (kDTN * kDTK) / 256; ++i) {
            const int idx = threadIdx.x + i * 256;
            const int kk = idx / kDTN, c = idx - kk * kDTN;
            const int64_t gk = k0 + kk;
            const int gc = col0 + c;
            Xs[kk][c] = (gk < K && gc < B) ? X[gk * B + gc] : 0.0f;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < kDTK; ++kk) {
            const float4 xv = *reinterpret_cast<const float4*>(&Xs[kk][tx * 4]);
            const float xs[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const float a = As[kk][ty * 2 + i];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = acc[i][j] + a * xs[j];
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int64_t r = row0 + ty * 2 + i;
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = col0 + tx * 4 + j;
            if (c < B) Y[r * B + c] = Y[r * B + c] + acc[i][j];
        }
    }
}

/// One DotInc output row by a whole warp, for a constant all-finite A
/// (MF_SKIP_ZERO_X): lanes form the products of 32 consecutive k at a time
/// (each rounded, as the reference's), and the nonzero ones are added to the
/// running sum in ascending k — the reference's sum without its zero terms,
/// which change nothing (see MF_SKIP_ZERO_X).  The sequential chain is as long
/// as the number of spikes instead of the row length.
__device__ __forceinline__ void warp_dot_sparse(const GenericProgram& p, const DMember& m, int64_t local, int b,
                                                int lane) {
    const int64_t n = m.a[1].elems;
    const float* arow = at(p, m.a[0], local * n, b);
    const float* x = at(p, m.a[1], 0, b);
    const int32_t aes = m.a[0].es, xes = m.a[1].es;
    float acc = 0.0f;
    for (int64_t k0 = 0; k0 < n; k0 += 32) {
        const int64_t k = k0 + lane;
        const float xv = k < n ? x[k * xes] : 0.0f;
        const bool nz = xv != 0.0f;
        const float pv = nz ? arow[k * aes] * xv : 0.0f;
        uint32_t bits = __ballot_sync(0xffffffffu, nz);
        while (bits) {
            const int c = __ffs(bits) - 1;
            bits &= bits - 1u;
            acc = acc + __shfl_sync(0xffffffffu, pv, c);
        }
    }
    if (lane == 0) {
        float* y = at(p, m.a[2], local, b);
        *y = *y + acc;
    }
}

// Reference loop order for one member and one copy b (GF_SERIAL_ALL).
__device__ void exec_member_serial(const GenericProgram& p, const DGroup& g, const DMember& m, int b) {
    switch (g.kind) {
        case 1: {  // Copy: inc cascades forward; plain copy is std::copy == memmove
            const int64_t n = m.a[0].elems;
            if (g.flags & GF_INC) {
                for (int64_t i = 0; i < n; ++i) {
                    float s = *at(p, m.a[0], i, b);
                    float* d = at(p, m.a[1], i, b);
                    *d = *d + s;
                }
            } else if (m.a[1].base > m.a[0].base) {
                for (int64_t i = n - 1; i >= 0; --i) *at(p, m.a[1], i, b) = *at(p, m.a[0], i, b);
            } else {
                for (int64_t i = 0; i < n; ++i) *at(p, m.a[1], i, b) = *at(p, m.a[0], i, b);
            }
            break;
        }
        case 2: {  // ElementwiseInc: scalar read once before the loop
            const int64_t n = m.a[1].elems;
            if (m.flags & MF_SCALAR_A) {
                float s = *at(p, m.a[0], 0, b);
                for (int64_t i = 0; i < n; ++i) {
                    float* y = at(p, m.a[2], i, b);
                    *y = *y + s * *at(p, m.a[1], i, b);
                }
            } else {
                for (int64_t i = 0; i < n; ++i) {
                    float* y = at(p, m.a[2], i, b);
                    *y = *y + *at(p, m.a[0], i, b) * *at(p, m.a[1], i, b);
                }
            }
            break;
        }
        case 5: {  // SimProcess
            const int64_t n = m.a[0].elems;
            if (g.flags & GF_HAS_STATE) {
                for (int64_t i = 0; i < n; ++i) {
                    float* st = at(p, m.a[2], i, b);
                    float f = g.tau_a * *st + g.tau_b * *at(p, m.a[0], i, b);
                    *st = f;
                    *at(p, m.a[1], i, b) = f;
                }
            } else if (m.a[1].base > m.a[0].base) {
                for (int64_t i = n - 1; i >= 0; --i) *at(p, m.a[1], i, b) = *at(p, m.a[0], i, b);
            } else {
                for (int64_t i = 0; i < n; ++i) *at(p, m.a[1], i, b) = *at(p, m.a[0], i, b);
            }
            break;
        }
        default: {  // element-sequential kinds: one item after another, in order
            int64_t items = m.items;
            for (int64_t i = 0; i < items; ++i) exec_item(p, g, m, i, b);
            break;
        }
    }
}

__device__ __forceinline__ void grid_sync(cg::grid_group& grid) {
    if (gridDim.x == 1)
        __syncthreads();
    else
        grid.sync();
}

/// The step loop of the interpreter.  SMALL: one CTA whose arena is in shared
/// memory (generic_small_kernel); the plain groups' tiles then run side by
/// side, one 256-thread slice per tile, instead of one after another.
template <bool SMALL>
__device__ __forceinline__ void generic_steps(const GenericProgram& p, cg::grid_group& grid, int k_begin, int k_end,
                                              int call_k0) {
    const int B = p.batch;
    for (int k = k_begin; k < k_end; ++k) {
        const int ks = k - call_k0;  // step index within this run() call
        // write_feeds (exec.cpp:313-326): per-batch slots take row b, shared slots row 0
        const int g_end = p.g_end < 0 ? p.n_groups : p.g_end;
        unsigned long long prof_t = p.prof ? clock64() : 0ull;
        if (p.any_feed && p.g_begin == 0) {
            for (int f = 0; f < p.n_feeds; ++f) {
                const DFeed& fd = p.feeds[f];
                if (!fd.present) continue;
                const int64_t n = static_cast<int64_t>(fd.dim) * fd.copies;
                const float* src = p.feed_data + fd.data_off + static_cast<int64_t>(ks) * fd.dim * B;
                for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
                    int64_t d = i / fd.copies;
                    int b = static_cast<int>(i - d * fd.copies);
                    *at(p, fd.dst, d, b) = src[d * B + b];
                }
            }
            grid_sync(grid);
        }
        for (int gi = p.g_begin; gi < g_end; ++gi) {
            const DGroup g = p.groups[gi];
            if (g.flags & GF_SERIAL_ALL) {
                if (blockIdx.x == 0 && threadIdx.x == 0)
                    for (int b = 0; b < g.copies; ++b)
                        for (int mi = 0; mi < g.n_members; ++mi)
                            exec_member_serial(p, g, p.members[g.member_begin + mi], b);
            } else if (g.flags & GF_SERIAL_B) {
                if (blockIdx.x == 0)
                    for (int b = 0; b < g.copies; ++b) {
                        for (int t = 0; t < g.n_tiles; ++t) {
                            const DTile tl = p.tiles[g.tile_begin + t];
                            const DMember& m = p.members[tl.member];
                            for (int j = threadIdx.x; j < tl.count; j += blockDim.x) {
                                const int i = tl.start + j;
                                if (i % g.copies == b) exec_item(p, g, m, i / g.copies, b);
                            }
                        }
                        __syncthreads();
                    }
            } else if (g.flags & GF_DENSE) {
                for (int t = blockIdx.x; t < g.n_tiles; t += gridDim.x) {
                    const DTile tl = p.tiles[g.tile_begin + t];
                    dense_dot_tile(p, p.members[tl.member], tl.start, tl.count);
                }
            } else if (SMALL && g.n_tiles == 1 && p.tiles[g.tile_begin].count <= 32) {
                // a few long items (a decoder's 16 sequential 800-term sums): one per warp, lane 0 —
                // lanes of one warp reading different rows of a row-major matrix at the same
                // column hit one shared-memory bank; separate warps do not conflict
                const DTile tl = p.tiles[g.tile_begin];
                const int j = threadIdx.x >> 5, lane = threadIdx.x & 31;
                if (j < tl.count) {
                    const int i = tl.start + j;
                    const int local = i / g.copies;
                    const DMember& m = p.members[tl.member];
                    if (g.kind == 3 && (m.flags & MF_SKIP_ZERO_X))
                        warp_dot_sparse(p, m, local, i - local * g.copies, lane);
                    else if (lane == 0)
                        exec_item<SMALL>(p, g, m, local, i - local * g.copies);
                }
            } else {
                const int t0 = SMALL ? threadIdx.x / kTile : blockIdx.x;
                const int ts = SMALL ? blockDim.x / kTile : gridDim.x;
                const int j0 = SMALL ? threadIdx.x % kTile : threadIdx.x;
                const int js = SMALL ? kTile : blockDim.x;
                for (int t = t0; t < g.n_tiles; t += ts) {
                    const DTile tl = p.tiles[g.tile_begin + t];
                    const DMember& m = p.members[tl.member];
                    for (int j = j0; j < tl.count; j += js) {
                        const int i = tl.start + j;  // < 2^30 (engine.cpp)
                        const int local = i / g.copies;
                        exec_item<SMALL>(p, g, m, local, i - local * g.copies);
                    }
                }
            }
            if (g.flags & GF_BARRIER) grid_sync(grid);
            if (p.prof && blockIdx.x == 0 && threadIdx.x == 0) {
                const unsigned long long now = clock64();
                p.prof[gi] += now - prof_t;
                prof_t = now;
            }
        }
        // capture_probes (exec.cpp:328-338): shared probes read copy 0
        if (p.n_probes && g_end == p.n_groups) {
            for (int q = 0; q < p.n_probes; ++q) {
                const DProbe& pr = p.probes[q];
                const int64_t n = static_cast<int64_t>(pr.dim) * B;
                float* dst = p.ring + pr.ring_off + static_cast<int64_t>(ks) * pr.dim * B;
                for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
                    int64_t d = i / B;
                    int b = static_cast<int>(i - d * B);
                    dst[i] = *at(p, pr.src, d, pr.per_batch ? b : 0);
                }
            }
            grid_sync(grid);
        }
    }
}

__global__ void __launch_bounds__(kTile) generic_run_kernel(GenericProgram p, int k_begin, int k_end,
                                                            int call_k0) {
    cg::grid_group grid = cg::this_grid();
    generic_steps<false>(p, grid, k_begin, k_end, call_k0);
}

constexpr int kSmallThreads = 4 * kTile;

/// Programs whose whole arena fits in shared memory (config 0: one 800-neuron
/// ensemble, ~170 KB): one CTA copies the arena in, runs the launch's steps on
/// it (every operand access a shared-memory access instead of an L2 round trip
/// after the previous group's stores), and copies it back.
__global__ void __launch_bounds__(kSmallThreads) generic_small_kernel(GenericProgram p, int k_begin, int k_end,
                                                                      int call_k0, int64_t arena_floats) {
    // shared: the program's group / member / tile descriptors (copied once: every group's
    // decode is then a shared-memory read), then the arena
    extern __shared__ __align__(16) float sarena[];
    cg::grid_group grid = cg::this_grid();
    DMember* smem_members = reinterpret_cast<DMember*>(sarena);
    DGroup* smem_groups = reinterpret_cast<DGroup*>(smem_members + p.n_members);
    DTile* smem_tiles = reinterpret_cast<DTile*>(smem_groups + p.n_groups);
    const size_t desc_bytes = (p.n_members * sizeof(DMember) + p.n_groups * sizeof(DGroup) +
                               p.n_tiles * sizeof(DTile) + 15) & ~size_t{15};
    float* arena = reinterpret_cast<float*>(reinterpret_cast<char*>(sarena) + desc_bytes);
    for (int i = threadIdx.x; i < p.n_members; i += blockDim.x) smem_members[i] = p.members[i];
    for (int i = threadIdx.x; i < p.n_groups; i += blockDim.x) smem_groups[i] = p.groups[i];
    for (int i = threadIdx.x; i < p.n_tiles; i += blockDim.x) smem_tiles[i] = p.tiles[i];
    float* garena = p.arena;
    for (int64_t i = threadIdx.x; i < arena_floats; i += blockDim.x) arena[i] = garena[i];
    __syncthreads();
    GenericProgram q = p;
    q.arena = arena;
    q.members = smem_members;
    q.groups = smem_groups;
    q.tiles = smem_tiles;
    generic_steps<true>(q, grid, k_begin, k_end, call_k0);
    __syncthreads();
    for (int64_t i = threadIdx.x; i < arena_floats; i += blockDim.x) garena[i] = arena[i];
}

/// Shared-memory bytes of the small variant for a program (descriptors + arena).
size_t generic_small_smem_bytes(const GenericProgram& p, int64_t arena_floats) {
    const size_t desc = (p.n_members * sizeof(DMember) + p.n_groups * sizeof(DGroup) + p.n_tiles * sizeof(DTile) +
                         15) & ~size_t{15};
    return desc + static_cast<size_t>(arena_floats) * sizeof(float);
}

// reset (exec.cpp:164-174): broadcast the pristine image to every copy
__global__ void reset_kernel(float* arena, const float* pristine, const int64_t* base, const int64_t* pbase,
                             const int64_t* span, const int32_t* per_batch, int nbuf, int B) {
    for (int bi = blockIdx.y; bi < nbuf; bi += gridDim.y) {
        const int copies = per_batch[bi] ? B : 1;
        const int64_t n = span[bi] * copies;
        for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            int64_t e = i / copies;
            arena[base[bi] + i] = pristine[pbase[bi] + e];
        }
    }
}

// [probe][n_steps][dim][B] -> [probe][B][n_steps][dim] (ProbeOutput's Tensor3 order)
__global__ void probe_transpose_kernel(const float* ring, float* out, const int64_t* off, const int32_t* dims,
                                       int nprobes, int steps, int B) {
    for (int q = blockIdx.y; q < nprobes; q += gridDim.y) {
        const int dim = dims[q];
        const int64_t n = static_cast<int64_t>(steps) * dim * B;
        for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
            // i indexes the output: ((b * steps) + s) * dim + d
            int64_t d = i % dim;
            int64_t s = (i / dim) % steps;
            int64_t b = i / (static_cast<int64_t>(dim) * steps);
            out[off[q] + i] = ring[off[q] + (s * dim + d) * B + b];
        }
    }
}

// Build the libm parity hash: insert (key, result) pairs, linear probing.
__global__ void libm_hash_build_kernel(unsigned long long* slots, uint32_t mask, int shift, const uint32_t* keys,
                                       const uint32_t* results, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t key = keys[i];
        unsigned long long v = (static_cast<unsigned long long>(key) << 32) | results[i];
        uint32_t s = (key * 0x9E3779B1u) >> shift;
        for (;;) {
            unsigned long long prev = atomicCAS(slots + s, 0ull, v);
            if (prev == 0ull || prev == v) break;
            s = (s + 1u) & mask;
        }
    }
}

// Device-side evaluation of the parity functions over a key range (tests).
__global__ void libm_eval_kernel(int func, uint32_t lo, int64_t n, uint32_t* out, LibmTables t) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float x = __uint_as_float(static_cast<uint32_t>(lo + i));
        // 0/1: expm1f/log1pf; 2/3: the same through the fused kernel's speculate-and-resolve path
        float r = func == 0   ? glibc_expm1f(x, t)
                  : func == 1 ? glibc_log1pf(x, t)
                              : glibc_spec_resolved(x, func == 3, t);
        out[i] = __float_as_uint(r);
    }
}

// ---- host launchers --------------------------------------------------------

/// Shared memory the small (arena-in-shared-memory) variant can use (next to the
/// dense tiles' 12.5 KB of static shared memory).
size_t generic_small_arena_limit() { return 212 * 1024; }

cudaError_t launch_generic(const GenericProgram& p, int grid, int k_begin, int k_end, int call_k0,
                           cudaStream_t stream, int64_t small_arena_floats) {
    GenericProgram prog = p;
    void* args[] = {&prog, &k_begin, &k_end, &call_k0};
    if (small_arena_floats > 0) {
        const size_t bytes = generic_small_smem_bytes(p, small_arena_floats);
        static size_t attr = 0;
        if (bytes > attr) {
            cudaError_t e = cudaFuncSetAttribute(generic_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(bytes));
            if (e != cudaSuccess) return e;
            attr = bytes;
        }
        generic_small_kernel<<<1, kSmallThreads, bytes, stream>>>(prog, k_begin, k_end, call_k0, small_arena_floats);
        return cudaGetLastError();
    }
    if (grid <= 1) {
        generic_run_kernel<<<1, kTile, 0, stream>>>(prog, k_begin, k_end, call_k0);
        return cudaGetLastError();
    }
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(generic_run_kernel), dim3(grid), dim3(kTile), args, 0,
                                       stream);
}

int generic_max_coresident_blocks(int device) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, generic_run_kernel, kTile, 0);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

// feed staging: per present slot, [B][steps*dim] (the host's Tensor3 order,
// narrowed to f32) -> [steps*dim][B] (the device order), 32x32 tiles through
// smem; offs holds nslots input offsets then nslots output offsets
__global__ void feed_transpose_kernel(const float* in, float* out, const int64_t* offs, const int32_t* cols, int nslots,
                                      int B) {
    __shared__ float tile[32][33];
    for (int s = blockIdx.z; s < nslots; s += gridDim.z) {
        const int C = cols[s];  // steps * dim of this block
        const float* src = in + offs[s];           // [B][C]
        float* dst = out + offs[nslots + s];       // [C][B]
        for (int cb = blockIdx.x * 32; cb < C; cb += gridDim.x * 32)
            for (int bb = blockIdx.y * 32; bb < B; bb += gridDim.y * 32) {
                for (int r = threadIdx.y; r < 32; r += blockDim.y) {
                    const int b = bb + r, c = cb + threadIdx.x;
                    tile[r][threadIdx.x] = (b < B && c < C) ? src[static_cast<int64_t>(b) * C + c] : 0.0f;
                }
                __syncthreads();
                for (int r = threadIdx.y; r < 32; r += blockDim.y) {
                    const int c = cb + r, b = bb + threadIdx.x;
                    if (b < B && c < C) dst[static_cast<int64_t>(c) * B + b] = tile[threadIdx.x][r];
                }
                __syncthreads();
            }
    }
}

cudaError_t launch_feed_transpose(const float* in, float* out, const int64_t* offs, const int32_t* cols, int nslots,
                                  int max_cols, int B, cudaStream_t stream) {
    if (nslots == 0) return cudaSuccess;
    dim3 grid((max_cols + 31) / 32 < 64 ? (max_cols + 31) / 32 : 64, (B + 31) / 32 < 16 ? (B + 31) / 32 : 16,
              nslots < 1024 ? nslots : 1024);
    feed_transpose_kernel<<<grid, dim3(32, 8), 0, stream>>>(in, out, offs, cols, nslots, B);
    return cudaGetLastError();
}

/// Fed-node projections (FProj) for steps [k0, k1) of an n_steps call: projection q
/// is the block [n_steps][dd][B] at out + dd_prefix * n_steps * B (a feed-slot layout).
__global__ void feed_projection_kernel(const FProj* proj, int nproj, const float* weights, const float* feed_data,
                                       const int64_t* feed_off, const int32_t* present, const float* arena,
                                       float* out, int n_steps, int k0, int k1, int B) {
    const int q = blockIdx.y;
    if (q >= nproj) return;
    const FProj P = proj[q];
    const int64_t n = static_cast<int64_t>(k1 - k0) * P.dd * B;
    const bool fed = present[P.slot] != 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(i % B);
        const int64_t kr = i / B;
        const int r = static_cast<int>(kr % P.dd);
        const int k = k0 + static_cast<int>(kr / P.dd);
        const float* T = weights + P.t_off + static_cast<int64_t>(r) * P.ds;
        float acc = 0.0f;
        if (fed) {
            const float* u = feed_data + feed_off[P.slot] + static_cast<int64_t>(k) * P.ds * B + b;
            for (int j = 0; j < P.ds; ++j) acc = acc + T[j] * u[static_cast<int64_t>(j) * B];
        } else {
            const float* u = arena + P.node_base + (P.copies > 1 ? b : 0);
            for (int j = 0; j < P.ds; ++j) acc = acc + T[j] * u[static_cast<int64_t>(j) * P.copies];
        }
        out[static_cast<int64_t>(P.dd_prefix) * n_steps * B + (static_cast<int64_t>(k) * P.dd + r) * B + b] = acc;
    }
}

cudaError_t launch_feed_projection(const FProj* proj, int nproj, const float* weights, const float* feed_data,
                                   const int64_t* feed_off, const int32_t* present, const float* arena, float* out,
                                   int n_steps, int k0, int k1, int B, cudaStream_t stream) {
    if (nproj == 0 || k1 <= k0) return cudaSuccess;
    dim3 grid(64, nproj);
    feed_projection_kernel<<<grid, 256, 0, stream>>>(proj, nproj, weights, feed_data, feed_off, present, arena, out,
                                                     n_steps, k0, k1, B);
    return cudaGetLastError();
}

cudaError_t launch_reset(float* arena, const float* pristine, const int64_t* base, const int64_t* pbase,
                         const int64_t* span, const int32_t* per_batch, int nbuf, int B, cudaStream_t stream) {
    if (nbuf == 0) return cudaSuccess;
    dim3 grid(64, nbuf < 1024 ? nbuf : 1024);
    reset_kernel<<<grid, 256, 0, stream>>>(arena, pristine, base, pbase, span, per_batch, nbuf, B);
    return cudaGetLastError();
}

cudaError_t launch_probe_transpose(const float* ring, float* out, const int64_t* off, const int32_t* dims,
                                   int nprobes, int steps, int B, cudaStream_t stream) {
    if (nprobes == 0) return cudaSuccess;
    dim3 grid(128, nprobes < 1024 ? nprobes : 1024);
    probe_transpose_kernel<<<grid, 256, 0, stream>>>(ring, out, off, dims, nprobes, steps, B);
    return cudaGetLastError();
}

cudaError_t launch_libm_hash_build(unsigned long long* slots, uint32_t mask, int shift, const uint32_t* keys,
                                   const uint32_t* results, int64_t n, cudaStream_t stream) {
    if (n == 0) return cudaSuccess;
    libm_hash_build_kernel<<<1184, 256, 0, stream>>>(slots, mask, shift, keys, results, n);
    return cudaGetLastError();
}

cudaError_t launch_libm_eval(int func, uint32_t lo, int64_t n, uint32_t* out, const LibmTables& t,
                             cudaStream_t stream) {
    libm_eval_kernel<<<1184, 256, 0, stream>>>(func, lo, n, out, t);
    return cudaGetLastError();
}

}  // namespace nengb
