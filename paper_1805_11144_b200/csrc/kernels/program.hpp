// program.hpp — device program descriptors shared by the host compiler
// (csrc/host/engine.cpp) and the CUDA kernels.  Plain PODs only.
//
// Device layout of every base buffer (BufferDesc, passes.hpp:63-70):
//   shared    : float[span]                 element e at  base + e
//   per-batch : float[span][B] (batch inner) element e, copy b at base + e*B + b
// so an operand resolves to DArg{base, es, bs}: addr(e, b) = arena + base + e*es + b*bs
// (es = B, bs = 1 per-batch; es = 1, bs = 0 shared).  This is the reference's
// resolve() (exec.cpp:18-25) with its [b][span] copies transposed so a warp's
// 32 lanes read 32 consecutive batch copies of one element.
#pragma once

#include <cstdint>

#include <vector_types.h>  // uint4

namespace nengb {

/// A fed-node connection wider than the fused pipeline's rows (ds > 32): its
/// DotInc sum y = +0 + sum_j T[r,j]*u[j] (j ascending, rounded products and
/// sums) is computed ahead of the fused kernel for the launch's steps, and the
/// connection then reads y through an identity transform (exact: a running sum
/// from +0 is never -0, so adding the zero terms leaves y unchanged).
struct FProj {
    int64_t t_off;      // T [dd][ds] f32 in the projection weights
    int64_t node_base;  // arena base of the fed node's signal (read when its feed is absent)
    int32_t slot;       // the fed node's feed slot
    int32_t dd, ds;
    int32_t copies;     // B when the node is per-batch, else 1
    int32_t dd_prefix;  // sum of dd over the earlier projections: output rows [dd_prefix, +dd) of [step][rows][B]
    int32_t pad_;
};

struct DArg {
    int64_t base = 0;  // arena offset (floats) of element 0
    int64_t elems = 0; // rows * elements-per-row of the operand
    int32_t es = 1;    // element stride
    int32_t bs = 0;    // batch stride
};

enum : int32_t {
    GF_INC = 1,         // Copy: increment
    GF_PER_BATCH = 2,   // run once per batch copy (exec.cpp:122-125)
    GF_SERIAL_B = 4,    // per-batch group that writes shared storage: b copies in order
    GF_SERIAL_ALL = 8,  // a member aliases itself with an offset: reference loop order, one thread
    GF_HAS_STATE = 16,  // SimProcess with a state operand (tau > 0)
    GF_BARRIER = 32,    // grid barrier after this group
    GF_DENSE = 64,      // DotInc with shared row-major A, per-batch x and y: CTA tiles (DTile = member, row0, col0)
};

// MF_SKIP_ZERO_X: a DotInc whose A is a constant, all-finite signal skips the terms with
// x[k] == 0 — exact: A[r,k] * (+-0) is +-0 and the running sum, started at +0, is never
// -0, so adding it changes nothing (spike vectors are mostly zeros)
enum : int32_t { MF_SCALAR_A = 1, MF_SKIP_ZERO_X = 2 };

struct DMember {
    DArg a[4];
    int64_t value_at = 0;   // Reset payload offset
    int64_t items = 0;      // work items per batch copy
    float pes_scale = 0.f;  // (T)(rate*dt/n), SimPES (exec.cpp:291-292)
    int32_t flags = 0;
};

struct DGroup {
    int32_t kind = 0, flags = 0, neuron = 0;
    int32_t member_begin = 0, n_members = 0;
    int32_t tile_begin = 0, n_tiles = 0;
    int32_t copies = 1;
    float dt = 0.f, tau_a = 0.f, tau_b = 0.f, tau_rc = 0.f, tau_ref = 0.f, amplitude = 0.f;
    float em_dt = 0.f;  // LIF: glibc expm1f(-dt / tau_rc) from the host (the step of a non-refractory neuron)
};

// A tile is up to kTileItems consecutive work items of one member; item index
// i = local * copies + b (batch innermost for coalescing).
constexpr int kTile = 256;        // threads per CTA of the interpreter
constexpr int kTileItems = 1024;  // light work items per tile (4 per thread: the descriptor loads are amortised)
struct DTile {
    int32_t member = 0, start = 0, count = 0;
};

struct DFeed {
    DArg dst;
    int32_t dim = 0, copies = 1;
    int64_t data_off = 0;  // offset of this slot's [n_steps][dim][B] block in the call's feed buffer
    int32_t present = 0;
};

struct DProbe {
    DArg src;
    int32_t dim = 0, per_batch = 0;
    int64_t ring_off = 0;  // offset of this probe's [n_steps][dim][B] block in the call's ring
};

// glibc-parity tables for expm1f / log1pf (see csrc/tools/gen_libm_tables.c)
struct LibmHash {
    const unsigned long long* slots = nullptr;  // (key << 32) | result bits; 0 = empty
    uint32_t mask = 0;
    int32_t shift = 32;
    float lookup_from = 0.f;      // probe only when the result is >= this many ulps from the rounded float
    float lookup_from_hot = 0.f;  // the same bound restricted to x in [-1/16, 0) (the LIF range)
    // the x in [-1/16, 0) subset as its own small (L2-resident) table
    const unsigned long long* hot_slots = nullptr;
    uint32_t hot_mask = 0;
    int32_t hot_shift = 32;
    // per-region bounds on [-1/16, 0): region = (key - 0x80000000) >> region_shift
    const float* region_from = nullptr;
    const uint32_t* region_win = nullptr;  // screening half-window per region, units of 2^-29 float ulp
    const uint8_t* region_w8 = nullptr;    // region_win >> 21 (floor): the byte screen (d >> 21) <= w8 is a superset
    // one bit per 64 consecutive LIF-range keys: set when the block holds a
    // hot-table key (2 MB, L2-resident); a clear bit answers "not listed"
    // without probing the hash table
    const uint32_t* hot_filter = nullptr;
    // the same LIF-range key set as 4-key buckets (one 16-B load answers "listed?"
    // unless the bucket is full): bucket = (key * 0x9E3779B1) >> bucket_shift,
    // linear probing over buckets, empty key 0
    const uint4* hot_buckets = nullptr;
    const uint32_t* bucket_results = nullptr;  // glibc's result bits, parallel to the bucket slots
    uint32_t bucket_mask = 0;
    int32_t bucket_shift = 32;
    uint32_t region_shift = 31;
    uint32_t n_regions = 0;
};
struct LibmTables {
    LibmHash t[3];  // 0: expm1f [-104,0)  1: log1pf [-1,0)  2: log1pf (0,inf)
};

struct GenericProgram {
    float* arena = nullptr;
    const DGroup* groups = nullptr;
    const DMember* members = nullptr;
    const DTile* tiles = nullptr;
    const float* values = nullptr;
    const DFeed* feeds = nullptr;
    const DProbe* probes = nullptr;
    int32_t n_groups = 0, n_feeds = 0, n_probes = 0, batch = 1;
    int32_t n_members = 0, n_tiles = 0;  // descriptor counts (the shared-memory variant copies them)
    int32_t g_begin = 0, g_end = -1;  // plan groups this launch runs (-1: to the end); feeds with
                                      // the first group, probe captures with the last
    int32_t any_feed = 0;
    LibmTables libm;
    // per call
    const float* feed_data = nullptr;
    float* ring = nullptr;
    int32_t call_steps = 0;
    unsigned long long* prof = nullptr;  // NENG_GENERIC_PROFILE: per group, clock cycles (CTA 0, summed over steps)
};

}  // namespace nengb
