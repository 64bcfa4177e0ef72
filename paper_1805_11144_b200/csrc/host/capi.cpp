// capi.cpp — the extern "C" surface of include/neng_gpu.h.  Every entry point
// catches C++ exceptions and maps them 1:1 onto status codes (the reference's
// StructuralError/BuildError/RunError, ir.hpp:15-25) with the message kept in
// a thread-local (neng_last_error) and on the engine (neng_gpu_last_error).
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "engine.hpp"
#include "neng_gpu.h"

namespace {

thread_local std::string g_last_error;

template <class F>
neng_status guarded(nengb::Engine* e, F&& f) {
    auto fail = [&](neng_status s, const char* msg) {
        g_last_error = msg;
        if (e) e->last_error = msg;
        return s;
    };
    try {
        f();
        return NENG_OK;
    } catch (const nengb::StructuralError& x) {
        return fail(NENG_STRUCTURAL_ERROR, x.what());
    } catch (const nengb::BuildError& x) {
        return fail(NENG_BUILD_ERROR, x.what());
    } catch (const nengb::RunError& x) {
        return fail(NENG_RUN_ERROR, x.what());
    } catch (const nengb::CudaError& x) {
        return fail(NENG_CUDA_ERROR, x.what());
    } catch (const nengb::InvalidArgument& x) {
        return fail(NENG_INVALID_ARGUMENT, x.what());
    } catch (const std::bad_alloc&) {
        return fail(NENG_OUT_OF_MEMORY, "out of memory");
    } catch (const std::exception& x) {
        return fail(NENG_INVALID_ARGUMENT, x.what());
    }
}

}  // namespace

struct neng_engine {
    nengb::Engine impl;
    template <class... A>
    explicit neng_engine(A&&... a) : impl(std::forward<A>(a)...) {}
};

extern "C" {

neng_status neng_gpu_create(const neng_planned_model* planned, int32_t batch, int32_t unroll,
                            const neng_device_cfg* cfg, neng_engine** out) {
    return guarded(nullptr, [&] {
        if (!planned || !out) throw nengb::InvalidArgument("neng_gpu_create: null argument");
        *out = nullptr;
        nengb::PlannedModel pm = nengb::planned_from_view(*planned);
        *out = new neng_engine(std::move(pm), batch, unroll, cfg);
    });
}

void neng_gpu_destroy(neng_engine* e) { delete e; }

neng_status neng_gpu_run(neng_engine* e, int32_t n_steps, int32_t n_feeds, const neng_feed* feeds,
                         double* probes_out) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.run(n_steps, n_feeds, feeds, probes_out); });
}

neng_status neng_gpu_run_device(neng_engine* e, int32_t n_steps, const float* const* d_feeds,
                                float* const* d_probes, void* stream) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] {
        e->impl.run_device(n_steps, d_feeds, d_probes, static_cast<cudaStream_t>(stream));
    });
}

neng_status neng_gpu_call_begin(neng_engine* e, int32_t n_steps, const float* const* d_feeds, float* const* d_probes,
                                void* stream) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] {
        e->impl.call_begin(n_steps, d_feeds, d_probes, static_cast<cudaStream_t>(stream));
    });
}

neng_status neng_gpu_call_step(neng_engine* e, int32_t k, int32_t flags) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.call_step(k, flags); });
}

neng_status neng_gpu_call_end(neng_engine* e) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.call_end(); });
}

neng_status neng_gpu_shard_layout(const neng_engine* e, int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(const_cast<nengb::Engine*>(&e->impl), [&] {
        e->impl.shard_layout(xbuf_floats, rank_floats, xbuf);
    });
}

neng_status neng_gpu_set_xhat_buffer(neng_engine* e, float* d_buf) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.set_xhat_buffer(d_buf); });
}

neng_status neng_gpu_synchronize(neng_engine* e) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.synchronize(); });
}

neng_status neng_gpu_reset(neng_engine* e) {
    if (!e) return NENG_INVALID_ARGUMENT;
    return guarded(&e->impl, [&] { e->impl.reset(); });
}

neng_status neng_gpu_probe_dump_size(const neng_engine* e, int64_t* bytes) {
    if (!e || !bytes) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] { *bytes = e->impl.probe_dump_bytes(); });
}

neng_status neng_gpu_probe_dump(const neng_engine* e, void* out, int64_t capacity) {
    if (!e || !out) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] { e->impl.probe_dump(static_cast<char*>(out), capacity); });
}

neng_status neng_gpu_write_probe_binary(const neng_engine* e, const char* path) {
    if (!e || !path) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] {
        std::vector<char> buf(static_cast<size_t>(e->impl.probe_dump_bytes()));
        e->impl.probe_dump(buf.data(), static_cast<int64_t>(buf.size()));
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw nengb::RunError(std::string("cannot open '") + path + "' for writing");
        const size_t n = std::fwrite(buf.data(), 1, buf.size(), f);
        if (std::fclose(f) != 0 || n != buf.size()) throw nengb::RunError(std::string("failed writing '") + path + "'");
    });
}

neng_status neng_gpu_write_probe_csv(const neng_engine* e, const char* path, double dt) {
    if (!e || !path) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] {
        const std::string text = e->impl.probe_csv(dt);
        std::FILE* f = std::fopen(path, "wb");
        if (!f) throw nengb::RunError(std::string("cannot open '") + path + "' for writing");
        const size_t n = std::fwrite(text.data(), 1, text.size(), f);
        if (std::fclose(f) != 0 || n != text.size()) throw nengb::RunError(std::string("failed writing '") + path + "'");
    });
}

neng_status neng_gpu_read_signal(const neng_engine* e, int32_t signal, int32_t batch_index, double* out,
                                 int64_t capacity, int64_t* n_out) {
    if (!e) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] {
        std::vector<double> v = e->impl.read_signal(signal, batch_index);
        if (n_out) *n_out = static_cast<int64_t>(v.size());
        if (out) {
            if (capacity < static_cast<int64_t>(v.size()))
                throw nengb::InvalidArgument("read_signal: output capacity too small");
            std::memcpy(out, v.data(), v.size() * sizeof(double));
        }
    });
}

neng_status neng_gpu_buffer_storage(const neng_engine* e, int32_t buffer, int32_t* mode_out) {
    if (!e || !mode_out) return NENG_INVALID_ARGUMENT;
    auto* ee = const_cast<neng_engine*>(e);
    return guarded(&ee->impl, [&] { *mode_out = e->impl.buffer_storage(buffer); });
}

int32_t neng_gpu_batch(const neng_engine* e) { return e ? e->impl.batch() : 0; }
int32_t neng_gpu_unroll(const neng_engine* e) { return e ? e->impl.unroll() : 0; }
int32_t neng_gpu_steps_completed(const neng_engine* e) { return e ? e->impl.steps_completed() : 0; }
int32_t neng_gpu_num_probes(const neng_engine* e) { return e ? e->impl.num_probes() : 0; }
int32_t neng_gpu_mode(const neng_engine* e) { return e ? e->impl.mode() : 0; }
int64_t neng_gpu_last_launch_count(const neng_engine* e) { return e ? e->impl.last_launches() : 0; }
int32_t neng_gpu_last_schedule(const neng_engine* e) { return e ? e->impl.last_schedule() : 0; }

neng_status neng_gpu_probe_info(const neng_engine* e, int32_t i, int32_t* key, int32_t* dim) {
    if (!e || i < 0 || i >= e->impl.num_probes()) return NENG_INVALID_ARGUMENT;
    if (key) *key = e->impl.planned().model.probes[i].key;
    if (dim) *dim = e->impl.probe_dim(i);
    return NENG_OK;
}

neng_status neng_gpu_tc_dot(int32_t mode, int32_t m, int32_t k, int32_t n, const float* a, const float* x,
                            float* y, int32_t reps, double* ms_out) {
    return guarded(nullptr, [&] {
        if (!a || !x || !y || m < 1 || k < 1 || n < 1 || reps < 1)
            throw nengb::InvalidArgument("neng_gpu_tc_dot: bad argument");
        if (mode != NENG_PRECISION_TF32 && mode != NENG_PRECISION_BF16X3)
            throw nengb::InvalidArgument("neng_gpu_tc_dot: mode must be TF32 or BF16X3");
        const int tm = mode == NENG_PRECISION_TF32 ? nengb::TC_TF32 : nengb::TC_BF16X3;
        auto check = [](cudaError_t e, const char* what) { nengb::cuda_check(e, what); };
        const size_t ab = size_t(m) * k * 4, xb = size_t(k) * n * 4, yb = size_t(m) * n * 4;
        nengb::DevMem da, dx, dy, dy0, scr;
        da.ensure(ab);
        dx.ensure(xb);
        dy.ensure(yb);
        dy0.ensure(yb);
        if (tm == nengb::TC_BF16X3) scr.ensure(nengb::tc_dot_scratch_bytes(m, k, n));
        check(cudaMemcpy(da.p, a, ab, cudaMemcpyHostToDevice), "tc_dot H2D");
        check(cudaMemcpy(dx.p, x, xb, cudaMemcpyHostToDevice), "tc_dot H2D");
        check(cudaMemcpy(dy0.p, y, yb, cudaMemcpyHostToDevice), "tc_dot H2D");
        nengb::TcDotDesc d;
        const char* why = nengb::tc_dot_prepare(&d, da.as<float>(), dx.as<float>(), dy.as<float>(), m, k, n, n, n, tm,
                                                scr.p);
        if (*why) throw nengb::InvalidArgument(std::string("neng_gpu_tc_dot: ") + why);
        check(nengb::tc_dot_split_a(d, nullptr), "tc_dot split");
        cudaEvent_t e0, e1;
        check(cudaEventCreate(&e0), "event");
        check(cudaEventCreate(&e1), "event");
        // the result: one launch on the caller's Y
        check(cudaMemcpy(dy.p, dy0.p, yb, cudaMemcpyDeviceToDevice), "tc_dot restore");
        check(nengb::tc_dot_launch(d, nullptr), "tc_dot launch");
        check(cudaMemcpy(y, dy.p, yb, cudaMemcpyDeviceToHost), "tc_dot D2H");
        // the time: `reps` launches back to back (Y accumulates; its values are not returned)
        check(cudaEventRecord(e0, nullptr), "event");
        for (int r = 0; r < reps; ++r) check(nengb::tc_dot_launch(d, nullptr), "tc_dot launch");
        check(cudaEventRecord(e1, nullptr), "event");
        check(cudaEventSynchronize(e1), "tc_dot run");
        float ms = 0.0f;
        check(cudaEventElapsedTime(&ms, e0, e1), "event");
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (ms_out) *ms_out = ms / reps;
    });
}

const char* neng_gpu_last_error(const neng_engine* e) { return e ? e->impl.last_error.c_str() : ""; }
const char* neng_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
