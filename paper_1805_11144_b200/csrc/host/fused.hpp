// fused.hpp — the fused ensemble pipeline (see fused_compile.cpp).
#pragma once

#include <memory>
#include <string>

#include <cuda_runtime.h>

#include "../kernels/program.hpp"

namespace nengb {

class Engine;

/// A compiled fused program: recognises the ensemble/connection structure of
/// the planned model and advances whole steps with one grid barrier each.
struct FusedPlan {
    virtual ~FusedPlan() = default;
    int sched = 0;  // NENG_SCHED_* bits of the launches since the last begin()
    /// Advance n_steps; feed data [slot][n][dim][B] f32 (slots absent -> null
    /// entries), probe ring [probe][n][dim][B].  Returns kernel launches.
    virtual int64_t run(int n_steps, const float* d_feed_data, const int64_t* feed_off, const int* present,
                        float* d_ring, const int64_t* ring_off, cudaStream_t stream) = 0;
    /// Write every signal the fused kernel keeps on-chip back to the arena so
    /// the arena holds the reference's state (read_signal, mode switches).
    virtual void materialize(cudaStream_t stream) = 0;
    /// Re-derive fused-private state from the arena (after reset).
    virtual void load_from_arena(cudaStream_t stream) = 0;
    virtual std::string describe() const = 0;
    // stepped calls: per-call tables, then one launch per step (flags:
    // NENG_STEP_FIRST_UPDATE / NENG_STEP_EPILOGUE; k == n_steps: epilogue only)
    virtual void begin(int n_steps, const float* d_feed_data, const int64_t* feed_off, const int* present,
                       float* d_ring, const int64_t* ring_off, cudaStream_t stream) = 0;
    virtual void step(int k, int flags, cudaStream_t stream) = 0;
    // steps [k0, k1) of the open call in one launch (same flags as step)
    virtual void launch(int k0, int k1, int flags, cudaStream_t stream) = 0;
    // steps [k0, k1) of the open call as one run()-style launch (epilogue
    // included, barrier-free when the engine owns its xhat buffer)
    virtual void launch_chunk(int k0, int k1, cudaStream_t stream) = 0;
    virtual void xhat_layout(int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf) const = 0;
    virtual void set_xhat_buffer(float* d_buf) = 0;
};

/// Returns nullptr (and a reason) when the model is not an ensemble network
/// the fused pipeline reproduces exactly.
std::unique_ptr<FusedPlan> try_compile_fused(Engine& e, std::string* why);

}  // namespace nengb
