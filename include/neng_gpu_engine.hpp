// neng_gpu_engine.hpp — neng::gpu::GpuEngine, the B200 drop-in for the
// reference's neng::EngineCore<float> (proj/include/nengine/exec.hpp:18-120).
//
// Header-only C++ over the C ABI in neng_gpu.h.  It is meant to be compiled
// inside the reference's tree (it includes <nengine/exec.hpp> for the model,
// feed and probe types) and linked against libneng_gpu.so; INTEGRATION.md
// shows the two lines a maintainer adds.  The member surface is
// EngineCore<float>'s, so code written against the CPU engine compiles
// against this one unchanged:
//
//   EngineCore<float>                                   GpuEngine
//   EngineCore(PlannedModel, int batch, int unroll)     same   (exec.cpp:10-16)
//   ProbeOutput run(int n_steps, const FeedData&)       same   (exec.cpp:340-366)
//   void reset()                                        same   (exec.cpp:164-174)
//   batch() / unroll() / steps_completed() / planned()  same   (exec.hpp:36-39)
//   StorageMode buffer_storage(int buffer)              same   (exec.hpp:41-43)
//   std::vector<double> read_signal(SignalId, int)      same   (exec.cpp:368-377)
//   write_probe_binary/csv(path, run(...))              write_probe_binary/csv(path[, dt])
//                                                       of the last run (export.hpp:17-25)
//
// Errors come back as the reference's own exception types (ir.hpp:15-25):
// the C status codes map 1:1 onto StructuralError / BuildError / RunError;
// device failures throw std::runtime_error.  Feeds are validated by the
// reference's own inline validate_feeds (model.hpp:62-83) before crossing
// the ABI, so its messages are the reference's verbatim.
#pragma once

#include <cstddef>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "neng_gpu.h"
#include "nengine/exec.hpp"

namespace neng::gpu {

class GpuEngine {
  public:
    /// EngineCore(PlannedModel planned, int batch = 1, int unroll = 1): takes
    /// ownership of the planned model, compiles it for the device.  `cfg`
    /// selects the CUDA device and executor (defaults: device 0, automatic).
    explicit GpuEngine(PlannedModel planned, int batch = 1, int unroll = 1, const neng_device_cfg* cfg = nullptr)
        : planned_(std::move(planned)) {
        flatten();
        neng_engine* e = nullptr;
        const neng_status s = neng_gpu_create(&view_, batch, unroll, cfg, &e);
        check(s, neng_last_error());
        engine_.reset(e);
    }

    GpuEngine(const GpuEngine&) = delete;
    GpuEngine& operator=(const GpuEngine&) = delete;
    GpuEngine(GpuEngine&&) noexcept = default;
    GpuEngine& operator=(GpuEngine&&) noexcept = default;

    /// Advance n_steps; feeds are indexed by step within this call; state and
    /// clock persist across calls.  Probe traces come back as f64
    /// [batch][n_steps][dim], as the reference's.
    ProbeOutput run(int n_steps, const FeedData& feeds = {}) {
        if (n_steps <= 0) throw RunError("n_steps must be positive");
        validate_feeds(planned_.model, feeds, n_steps, batch());
        std::vector<neng_feed> fv;
        fv.reserve(feeds.size());
        for (const auto& [node, t] : feeds) fv.push_back({node, t.batch, t.steps, t.dim, t.data.data()});
        ProbeOutput out;
        std::vector<std::pair<ProbeKey, int>> layout;
        size_t total = 0;
        const int np = neng_gpu_num_probes(engine_.get());
        for (int i = 0; i < np; ++i) {
            int32_t key = 0, dim = 0;
            check(neng_gpu_probe_info(engine_.get(), i, &key, &dim));
            layout.emplace_back(key, dim);
            total += static_cast<size_t>(batch()) * n_steps * dim;
        }
        std::vector<double> flat(total > 0 ? total : 1);
        check(neng_gpu_run(engine_.get(), n_steps, static_cast<int32_t>(fv.size()), fv.data(), flat.data()));
        size_t at = 0;
        for (const auto& [key, dim] : layout) {
            Tensor3 t(batch(), n_steps, dim);
            std::copy(flat.begin() + static_cast<std::ptrdiff_t>(at),
                      flat.begin() + static_cast<std::ptrdiff_t>(at + t.data.size()), t.data.begin());
            at += t.data.size();
            out.insert_or_assign(key, std::move(t));  // a key bound twice: the last binding wins, as capture_probes
        }
        return out;
    }

    /// Restore every buffer to its initial image and rewind the clock.
    void reset() { check(neng_gpu_reset(engine_.get())); }

    int batch() const { return neng_gpu_batch(engine_.get()); }
    int unroll() const { return neng_gpu_unroll(engine_.get()); }
    int steps_completed() const { return neng_gpu_steps_completed(engine_.get()); }
    const PlannedModel& planned() const { return planned_; }

    StorageMode buffer_storage(int buffer) const {
        int32_t mode = 0;
        check(neng_gpu_buffer_storage(engine_.get(), buffer, &mode));
        return mode == NENG_STORAGE_PER_BATCH ? StorageMode::PerBatch : StorageMode::Shared;
    }

    /// Current values of one signal for one batch entry (RunError on a bad id
    /// or batch index, with the reference's messages).
    std::vector<double> read_signal(SignalId sig, int batch_index = 0) const {
        int64_t n = 0;
        check(neng_gpu_read_signal(engine_.get(), sig, batch_index, nullptr, 0, &n));
        std::vector<double> out(static_cast<size_t>(n));
        check(neng_gpu_read_signal(engine_.get(), sig, batch_index, out.data(), n, &n));
        return out;
    }

    /// NENG_MODE_FUSED or NENG_MODE_GENERIC: which executor the model compiled to.
    int mode() const { return neng_gpu_mode(engine_.get()); }

    /// write_probe_binary / write_probe_csv (export.hpp:17-25) of the traces the
    /// last run() returned, written from the engine's own probe block: the same
    /// bytes as neng::write_probe_binary(path, run(...)) / write_probe_csv.
    void write_probe_binary(const std::string& path) const {
        check(neng_gpu_write_probe_binary(engine_.get(), path.c_str()));
    }
    void write_probe_csv(const std::string& path, double dt) const {
        check(neng_gpu_write_probe_csv(engine_.get(), path.c_str(), dt));
    }
    std::vector<char> probe_dump() const {
        int64_t n = 0;
        check(neng_gpu_probe_dump_size(engine_.get(), &n));
        std::vector<char> out(static_cast<size_t>(n));
        check(neng_gpu_probe_dump(engine_.get(), out.data(), n));
        return out;
    }

  private:
    struct Destroy {
        void operator()(neng_engine* e) const { neng_gpu_destroy(e); }
    };

    void check(neng_status s) const { check(s, neng_gpu_last_error(engine_.get())); }
    static void check(neng_status s, const char* msg) {
        const std::string m = msg ? msg : "";
        switch (s) {
            case NENG_OK: return;
            case NENG_STRUCTURAL_ERROR: throw StructuralError(m);
            case NENG_BUILD_ERROR: throw BuildError(m);
            case NENG_RUN_ERROR: throw RunError(m);
            case NENG_OUT_OF_MEMORY: throw std::bad_alloc();
            default: throw std::runtime_error("neng_gpu: " + m);
        }
    }

    /// POD view of planned_ (borrowed pointers into it; planned_ never moves
    /// its vectors after construction).
    void flatten() {
        const BuiltModel& m = planned_.model;
        sig_.resize(m.signals.size());
        for (size_t i = 0; i < m.signals.size(); ++i) {
            const Signal& s = m.signals[i];
            sig_[i] = {s.id,
                       static_cast<int32_t>(s.shape.size()),
                       s.shape.data(),
                       s.elem == Elem::f32 ? NENG_ELEM_F32 : NENG_ELEM_F64,
                       static_cast<int64_t>(s.initial.size()),
                       s.initial.data(),
                       s.constant,
                       s.minibatched,
                       s.trainable,
                       s.label.c_str()};
        }
        ops_.resize(m.operators.size());
        refs_.resize(m.operators.size());
        for (size_t i = 0; i < m.operators.size(); ++i) {
            const Operator& o = m.operators[i];
            refs_[i].clear();
            for (const SignalRef& r : o.operands) refs_[i].push_back({r.signal, r.start, r.stop});
            neng_operator& d = ops_[i];
            d = neng_operator{};
            d.id = o.id;
            d.kind = static_cast<int32_t>(o.kind);
            d.n_operands = static_cast<int32_t>(refs_[i].size());
            d.operands = refs_[i].data();
            d.n_value = static_cast<int64_t>(o.value.size());
            d.value = o.value.data();
            d.inc = o.inc;
            d.neuron_kind = static_cast<int32_t>(o.neuron.kind);
            d.tau_rc = o.neuron.tau_rc;
            d.tau_ref = o.neuron.tau_ref;
            d.amplitude = o.neuron.amplitude;
            d.tau = o.tau;
            d.learning_rate = o.learning_rate;
            d.dt = o.dt;
        }
        probes_.clear();
        for (const ProbeRegistration& p : m.probes) probes_.push_back({p.key, p.signal, p.label.c_str()});
        slots_.clear();
        for (const FeedSlot& f : m.feed_slots)
            slots_.push_back({f.node_id, f.signal, f.dim, f.has_default, f.label.c_str()});
        goff_.assign(1, 0);
        gmem_.clear();
        for (const OpGroup& g : planned_.plan) {
            gmem_.insert(gmem_.end(), g.members.begin(), g.members.end());
            goff_.push_back(static_cast<int32_t>(gmem_.size()));
        }
        bufs_.resize(planned_.buffers.buffers.size());
        for (size_t i = 0; i < bufs_.size(); ++i) {
            const BufferDesc& b = planned_.buffers.buffers[i];
            bufs_[i] = {static_cast<int32_t>(b.trailing.size()),
                        b.trailing.data(),
                        b.elem == Elem::f32 ? NENG_ELEM_F32 : NENG_ELEM_F64,
                        b.minibatched,
                        b.trainable,
                        b.rows,
                        static_cast<int32_t>(b.order.size()),
                        b.order.data()};
        }
        view_.model = {static_cast<int32_t>(sig_.size()),    sig_.data(),   static_cast<int32_t>(ops_.size()),
                       ops_.data(),
                       static_cast<int32_t>(probes_.size()), probes_.data(), static_cast<int32_t>(slots_.size()),
                       slots_.data(),                        m.dt};
        view_.n_groups = static_cast<int32_t>(planned_.plan.size());
        view_.group_offsets = goff_.data();
        view_.group_members = gmem_.data();
        view_.buffer_of = planned_.buffers.buffer_of.data();
        view_.row_offset = planned_.buffers.row_offset.data();
        view_.n_buffers = static_cast<int32_t>(bufs_.size());
        view_.buffers = bufs_.data();
    }

    PlannedModel planned_;
    std::vector<neng_signal> sig_;
    std::vector<neng_operator> ops_;
    std::vector<std::vector<neng_ref>> refs_;
    std::vector<neng_probe> probes_;
    std::vector<neng_feed_slot> slots_;
    std::vector<int32_t> goff_, gmem_;
    std::vector<neng_buffer_desc> bufs_;
    neng_planned_model view_{};
    std::unique_ptr<neng_engine, Destroy> engine_;
};

}  // namespace neng::gpu
