// engine.hpp — the B200 engine behind include/neng_gpu.h.  Mirrors
// neng::EngineCore<float> (proj/include/nengine/exec.hpp:18-120): it owns the
// planned model, compiles it once into a device program and device storage,
// and steps it with persistent kernels.
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../kernels/program.hpp"
#include "../kernels/tc_dot.hpp"
#include "host_ir.hpp"

namespace nengb {

struct FusedPlan;  // fused ensemble pipeline (fused.hpp)

// Device buffer that frees itself.
struct DevMem {
    void* p = nullptr;
    size_t bytes = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    void ensure(size_t n);  // grow-only
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

struct PinnedMem {
    void* p = nullptr;
    size_t bytes = 0;
    PinnedMem() = default;
    PinnedMem(const PinnedMem&) = delete;
    PinnedMem& operator=(const PinnedMem&) = delete;
    ~PinnedMem() {
        if (p) cudaFreeHost(p);
    }
    void ensure(size_t n);
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

void cuda_check(cudaError_t e, const char* what);

/// Singleton per device: glibc-parity hash tables for expm1f/log1pf.
const LibmTables& libm_tables(int device);

class Engine {
  public:
    Engine(PlannedModel planned, int batch, int unroll, const neng_device_cfg* cfg);
    ~Engine();

    void run(int n_steps, int n_feeds, const neng_feed* feeds, double* probes_out);
    void run_device(int n_steps, const float* const* d_feeds, float* const* d_probes, cudaStream_t stream);
    // stepped calls (sharded runs), see neng_gpu_call_begin
    void call_begin(int n_steps, const float* const* d_feeds, float* const* d_probes, cudaStream_t stream);
    void call_step(int k, int flags);
    void call_end();
    void shard_layout(int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf) const;
    void set_xhat_buffer(float* d_buf);
    int shard_rank() const { return shard_rank_; }
    int shard_count() const { return shard_count_; }
    void reset();
    std::vector<double> read_signal(int sig, int batch_index) const;
    // probe export of the last run() (export.hpp:17-30): NENG1 bytes / CSV text
    int64_t probe_dump_bytes() const;
    void probe_dump(char* out, int64_t capacity) const;
    std::string probe_csv(double dt) const;
    int buffer_storage(int buffer) const;
    void synchronize();

    int batch() const { return batch_; }
    int unroll() const { return unroll_; }
    int steps_completed() const { return steps_done_; }
    int mode() const { return mode_; }
    int requested_mode() const { return requested_mode_; }
    int64_t last_launches() const { return last_launches_; }
    int last_schedule() const;
    const PlannedModel& planned() const { return pm_; }
    int num_probes() const { return static_cast<int>(pm_.model.probes.size()); }
    int probe_dim(int i) const { return static_cast<int>(pm_.model.signals[pm_.model.probes[i].signal].size()); }

    std::string last_error;

    // layout (public for the fused compiler)
    struct BufLayout {
        int64_t epr = 1, span = 0, base = 0;
        int per_batch = 0;
    };
    DArg resolve(const SignalRef& r) const;
    DArg resolve_full(int sig) const;
    const std::vector<BufLayout>& layout() const { return bufs_; }
    float* arena() const { return arena_.as<float>(); }
    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    int steps_per_launch() const { return steps_per_launch_; }

  private:
    void compile();
    void compile_generic();
    void validate_feeds(int n_feeds, const neng_feed* feeds, int n_steps) const;
    void launch_steps(int n_steps, const float* d_feed_data, const std::vector<int>& present, float* d_ring,
                      cudaStream_t stream);
    void device_call_args(int n_steps, const float* const* d_feeds, float* const* d_probes, const float** base,
                          std::vector<int>* present, float** ring) const;
    void call_offsets(int n_steps, const std::vector<int>& present, std::vector<int64_t>* feed_off,
                      std::vector<int64_t>* ring_off) const;

    PlannedModel pm_;
    int batch_, unroll_, steps_done_ = 0;
    int device_ = 0, mode_ = NENG_MODE_GENERIC, requested_mode_ = NENG_MODE_AUTO, steps_per_launch_ = 0;
    int shard_rank_ = 0, shard_count_ = 1;
    int precision_ = NENG_PRECISION_STRICT_FP32;
    // dense DotInc groups run on the tcgen05 tensor cores (precision_ TF32 / BF16X3, tc_dot.cu)
    struct TcGroup {
        int group;
        std::vector<TcDotDesc> dots;  // one per member: Y[M][B] += A[M][K] X[K][B]
        std::vector<std::unique_ptr<DevMem>> scratch;  // BF16X3 split buffers
    };
    std::vector<TcGroup> tc_groups_;
    int64_t small_arena_floats_ = 0;
    std::vector<int32_t> prof_kinds_;  // group kinds (NENG_GENERIC_PROFILE)  // > 0: one CTA runs the interpreter with the arena in shared memory
    void run_tc_dots(const TcGroup& g, cudaStream_t stream);
    int call_steps_ = 0;  // steps of the open stepped call (0: none)
    cudaStream_t call_stream_ = nullptr;
    cudaStream_t stream_ = nullptr;
    int64_t last_launches_ = 0;
    int last_run_steps_ = 0;  // steps of the last run() whose probes sit in probe_stage_ ([probe][B][step][dim] f32)

    std::vector<BufLayout> bufs_;
    DevMem arena_, pristine_, reset_meta_;
    int64_t arena_floats_ = 0;

    // generic program
    GenericProgram prog_;
    DevMem d_groups_, d_members_, d_tiles_, d_values_, d_feeds_, d_probes_;
    std::vector<DFeed> feeds_;
    std::vector<DProbe> probes_;
    int grid_ = 1;
    bool needs_libm_ = false;

    std::unique_ptr<FusedPlan> fused_;

    // per-call scratch
    DevMem feed_buf_, feed_raw_, feed_meta_, ring_, probe_out_, probe_meta_;
    cudaEvent_t feed_events_[2] = {nullptr, nullptr};  // staging-buffer reuse (pipelined host feeds)
    cudaEvent_t xpose_events_[2] = {nullptr, nullptr};  // device raw-buffer reuse (transpose done)
    cudaStream_t copy_stream_ = nullptr;                 // feed H2D copies overlap the kernels
    PinnedMem feed_stage_, probe_stage_, feed_meta_host_;
};

}  // namespace nengb
