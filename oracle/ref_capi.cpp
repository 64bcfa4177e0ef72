// oracle/ref_capi.cpp — TEST INFRASTRUCTURE ONLY (see oracle/README.md).
//
// A thin C API over the reference's own, unmodified sources
// (/root/reference/proj/src/{ir,passes,exec,reference}.cpp), compiled by
// oracle/Makefile into oracle/_ref/libneng_ref.so.  Only tests/, the smoke
// check and bench.py's cpu_baseline / --impl reference legs load it.  It lets
// Python drive:
//   * run_passes            (passes.cpp:663-694)      -> nref_run_passes
//   * EngineCore<float|double> (exec.cpp:10-380)      -> nref_engine_*
//   * run_reference (f64 interpreter, reference.cpp:194-226) -> nref_run_reference
//   * validate_operators + build_dependency_graph + toposort_schedule
//     (ir.cpp:310-317, 396-488)                        -> nref_validate / nref_toposort
// Models cross as the same POD views the product ABI uses (include/neng_gpu.h).
#include <algorithm>
#include <chrono>
#include <random>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "neng_gpu.h"
#include "nengine/exec.hpp"
#include "nengine/export.hpp"
#include "nengine/ir.hpp"
#include "nengine/passes.hpp"
#include "nengine/reference.hpp"

namespace {

thread_local std::string g_err;

neng_status fail(neng_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

template <class F>
neng_status guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return NENG_OK;
    } catch (const neng::StructuralError& e) {
        return fail(NENG_STRUCTURAL_ERROR, e.what());
    } catch (const neng::BuildError& e) {
        return fail(NENG_BUILD_ERROR, e.what());
    } catch (const neng::RunError& e) {
        return fail(NENG_RUN_ERROR, e.what());
    } catch (const std::bad_alloc&) {
        return fail(NENG_OUT_OF_MEMORY, "out of host memory");
    } catch (const std::exception& e) {
        return fail(NENG_INVALID_ARGUMENT, e.what());
    }
}

neng::BuiltModel to_model(const neng_built_model* v) {
    neng::BuiltModel m;
    m.dt = v->dt;
    m.signals.resize(v->n_signals);
    for (int i = 0; i < v->n_signals; ++i) {
        const neng_signal& s = v->signals[i];
        neng::Signal& d = m.signals[i];
        d.id = s.id;
        d.label = s.label ? s.label : "";
        d.shape.assign(s.shape, s.shape + s.ndim);
        d.elem = s.elem == NENG_ELEM_F32 ? neng::Elem::f32 : neng::Elem::f64;
        if (s.n_initial > 0) d.initial.assign(s.initial, s.initial + s.n_initial);
        d.constant = s.constant != 0;
        d.minibatched = s.minibatched != 0;
        d.trainable = s.trainable != 0;
    }
    m.operators.resize(v->n_operators);
    for (int i = 0; i < v->n_operators; ++i) {
        const neng_operator& o = v->operators[i];
        neng::Operator& d = m.operators[i];
        d.id = o.id;
        d.kind = static_cast<neng::OpKind>(o.kind);
        for (int k = 0; k < o.n_operands; ++k)
            d.operands.push_back({o.operands[k].signal, o.operands[k].start, o.operands[k].stop});
        if (o.n_value > 0) d.value.assign(o.value, o.value + o.n_value);
        d.inc = o.inc != 0;
        d.neuron.kind = static_cast<neng::NeuronKind>(o.neuron_kind);
        d.neuron.tau_rc = o.tau_rc;
        d.neuron.tau_ref = o.tau_ref;
        d.neuron.amplitude = o.amplitude;
        d.tau = o.tau;
        d.learning_rate = o.learning_rate;
        d.dt = o.dt;
    }
    for (int i = 0; i < v->n_probes; ++i)
        m.probes.push_back({v->probes[i].key, v->probes[i].signal,
                            v->probes[i].label ? v->probes[i].label : ""});
    for (int i = 0; i < v->n_feed_slots; ++i) {
        const neng_feed_slot& f = v->feed_slots[i];
        m.feed_slots.push_back({f.node_id, f.signal, f.dim, f.has_default != 0,
                                f.label ? f.label : ""});
    }
    return m;
}

neng::FeedData to_feeds(int n, const neng_feed* feeds) {
    neng::FeedData out;
    for (int i = 0; i < n; ++i) {
        const neng_feed& f = feeds[i];
        neng::Tensor3 t(f.batch, f.steps, f.dim);
        std::memcpy(t.data.data(), f.data, sizeof(double) * t.data.size());
        out.emplace(f.node_id, std::move(t));
    }
    return out;
}

void write_probes(const neng::BuiltModel& m, const neng::ProbeOutput& out, double* dst) {
    size_t at = 0;
    for (const neng::ProbeRegistration& p : m.probes) {
        const neng::Tensor3& t = out.at(p.key);
        std::memcpy(dst + at, t.data.data(), sizeof(double) * t.data.size());
        at += t.data.size();
    }
}

}  // namespace

// ---------------------------------------------------------------------------
// Planned model holder: owns a neng::PlannedModel and a flattened POD view.
struct nref_planned {
    neng::PlannedModel pm;
    // flattened view storage
    std::vector<neng_signal> sig;
    std::vector<neng_operator> ops;
    std::vector<std::vector<neng_ref>> refs;
    std::vector<neng_probe> probes;
    std::vector<neng_feed_slot> slots;
    std::vector<int32_t> goff, gmem;
    std::vector<neng_buffer_desc> bufs;
    neng_planned_model view{};

    void flatten() {
        const neng::BuiltModel& m = pm.model;
        sig.resize(m.signals.size());
        for (size_t i = 0; i < m.signals.size(); ++i) {
            const neng::Signal& s = m.signals[i];
            neng_signal& d = sig[i];
            d.id = s.id;
            d.ndim = static_cast<int32_t>(s.shape.size());
            d.shape = s.shape.data();
            d.elem = s.elem == neng::Elem::f32 ? NENG_ELEM_F32 : NENG_ELEM_F64;
            d.n_initial = static_cast<int64_t>(s.initial.size());
            d.initial = s.initial.data();
            d.constant = s.constant;
            d.minibatched = s.minibatched;
            d.trainable = s.trainable;
            d.label = s.label.c_str();
        }
        ops.resize(m.operators.size());
        refs.resize(m.operators.size());
        for (size_t i = 0; i < m.operators.size(); ++i) {
            const neng::Operator& o = m.operators[i];
            neng_operator& d = ops[i];
            std::memset(&d, 0, sizeof d);
            d.id = o.id;
            d.kind = static_cast<int32_t>(o.kind);
            refs[i].clear();
            for (const neng::SignalRef& r : o.operands) refs[i].push_back({r.signal, r.start, r.stop});
            d.n_operands = static_cast<int32_t>(refs[i].size());
            d.operands = refs[i].data();
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
        probes.clear();
        for (const auto& p : m.probes) probes.push_back({p.key, p.signal, p.label.c_str()});
        slots.clear();
        for (const auto& f : m.feed_slots)
            slots.push_back({f.node_id, f.signal, f.dim, f.has_default, f.label.c_str()});
        goff.assign(1, 0);
        gmem.clear();
        for (const neng::OpGroup& g : pm.plan) {
            gmem.insert(gmem.end(), g.members.begin(), g.members.end());
            goff.push_back(static_cast<int32_t>(gmem.size()));
        }
        bufs.resize(pm.buffers.buffers.size());
        for (size_t i = 0; i < bufs.size(); ++i) {
            const neng::BufferDesc& b = pm.buffers.buffers[i];
            bufs[i] = {static_cast<int32_t>(b.trailing.size()), b.trailing.data(),
                       b.elem == neng::Elem::f32 ? NENG_ELEM_F32 : NENG_ELEM_F64,
                       b.minibatched, b.trainable, b.rows,
                       static_cast<int32_t>(b.order.size()), b.order.data()};
        }
        view.model = {static_cast<int32_t>(sig.size()), sig.data(),
                      static_cast<int32_t>(ops.size()), ops.data(),
                      static_cast<int32_t>(probes.size()), probes.data(),
                      static_cast<int32_t>(slots.size()), slots.data(), m.dt};
        view.n_groups = static_cast<int32_t>(pm.plan.size());
        view.group_offsets = goff.data();
        view.group_members = gmem.data();
        view.buffer_of = pm.buffers.buffer_of.data();
        view.row_offset = pm.buffers.row_offset.data();
        view.n_buffers = static_cast<int32_t>(bufs.size());
        view.buffers = bufs.data();
    }
};

struct nref_engine {
    std::unique_ptr<neng::EngineCore<float>> f32;
    std::unique_ptr<neng::EngineCore<double>> f64;
    neng::ProbeOutput last;  // the last run's traces (for the export checks)
};

extern "C" {

const char* nref_last_error(void) { return g_err.c_str(); }

neng_status nref_validate(const neng_built_model* m) {
    return guarded([&] {
        neng::BuiltModel model = to_model(m);
        neng::validate_operators(model.signals, model.operators);
        neng::build_dependency_graph(model.signals, model.operators);
    });
}

/// toposort_schedule over the model's dependency graph (ir.cpp:465-488);
/// order_out receives n_operators ids.
neng_status nref_toposort(const neng_built_model* m, int32_t* order_out) {
    return guarded([&] {
        neng::BuiltModel model = to_model(m);
        neng::DependencyGraph g = neng::build_dependency_graph(model.signals, model.operators);
        std::vector<neng::OpId> order = neng::toposort_schedule(g);
        std::copy(order.begin(), order.end(), order_out);
    });
}

/// Dependency edges as (from_id, to_id) pairs (ir.cpp:396-463). Call with
/// pairs == NULL to get the count.
neng_status nref_dependency_edges(const neng_built_model* m, int64_t* n_edges, int32_t* pairs) {
    return guarded([&] {
        neng::BuiltModel model = to_model(m);
        neng::DependencyGraph g = neng::build_dependency_graph(model.signals, model.operators);
        int64_t n = 0;
        for (size_t i = 0; i < g.succ.size(); ++i)
            for (int j : g.succ[i]) {
                if (pairs) {
                    pairs[2 * n] = g.op_ids[i];
                    pairs[2 * n + 1] = g.op_ids[j];
                }
                ++n;
            }
        *n_edges = n;
    });
}

/// run_passes (passes.cpp:663-694). planner: 0 greedy, 1 tree, 2 transitive closure.
neng_status nref_run_passes(const neng_built_model* m, int32_t merge, int32_t simplify,
                            int32_t planner, int32_t tree_depth, int32_t sort,
                            nref_planned** out) {
    return guarded([&] {
        neng::PipelineConfig cfg;
        cfg.merge = merge != 0;
        cfg.simplify = simplify != 0;
        cfg.planner = static_cast<neng::Planner>(planner);
        cfg.tree_depth = tree_depth;
        cfg.sort = sort != 0;
        auto p = std::make_unique<nref_planned>();
        p->pm = neng::run_passes(to_model(m), cfg);
        p->flatten();
        *out = p.release();
    });
}

/// Build a PlannedModel directly from a view (model + plan + buffers),
/// bypassing the planner. Read blocks and stats are left empty: EngineCore
/// consumes neither (exec.cpp:41-162).
neng_status nref_planned_from_view(const neng_planned_model* v, nref_planned** out) {
    return guarded([&] {
        auto p = std::make_unique<nref_planned>();
        p->pm.model = to_model(&v->model);
        for (int g = 0; g < v->n_groups; ++g) {
            neng::OpGroup og;
            og.members.assign(v->group_members + v->group_offsets[g],
                              v->group_members + v->group_offsets[g + 1]);
            p->pm.plan.push_back(std::move(og));
        }
        int ns = v->model.n_signals;
        p->pm.buffers.buffer_of.assign(v->buffer_of, v->buffer_of + ns);
        p->pm.buffers.row_offset.assign(v->row_offset, v->row_offset + ns);
        for (int b = 0; b < v->n_buffers; ++b) {
            const neng_buffer_desc& d = v->buffers[b];
            neng::BufferDesc bd;
            bd.trailing.assign(d.trailing, d.trailing + d.n_trailing);
            bd.elem = d.elem == NENG_ELEM_F32 ? neng::Elem::f32 : neng::Elem::f64;
            bd.minibatched = d.minibatched != 0;
            bd.trainable = d.trainable != 0;
            bd.rows = d.rows;
            bd.order.assign(d.order, d.order + d.n_order);
            p->pm.buffers.buffers.push_back(std::move(bd));
        }
        p->flatten();
        *out = p.release();
    });
}

const neng_planned_model* nref_planned_view(const nref_planned* p) { return &p->view; }

void nref_planned_stats(const nref_planned* p, double* contiguous_read_fraction,
                        int64_t* gather_row_count, int32_t* groups_per_step) {
    *contiguous_read_fraction = p->pm.stats.contiguous_read_fraction;
    *gather_row_count = p->pm.stats.gather_row_count;
    *groups_per_step = p->pm.stats.groups_per_step;
}

/// Read blocks (passes.hpp:87-99): per block (group, position, buffer,
/// n_refs) in meta[4*i..], refs flattened (signal, start, stop).
int32_t nref_planned_num_read_blocks(const nref_planned* p) {
    return static_cast<int32_t>(p->pm.read_blocks.size());
}
int64_t nref_planned_read_block_refs(const nref_planned* p) {
    int64_t n = 0;
    for (const auto& b : p->pm.read_blocks) n += static_cast<int64_t>(b.refs.size());
    return n;
}
void nref_planned_read_blocks(const nref_planned* p, int32_t* meta, int32_t* refs) {
    int64_t at = 0;
    for (size_t i = 0; i < p->pm.read_blocks.size(); ++i) {
        const neng::ReadBlock& b = p->pm.read_blocks[i];
        meta[4 * i] = b.group;
        meta[4 * i + 1] = b.position;
        meta[4 * i + 2] = b.buffer;
        meta[4 * i + 3] = static_cast<int32_t>(b.refs.size());
        for (const auto& r : b.refs) {
            refs[3 * at] = r.signal;
            refs[3 * at + 1] = r.start;
            refs[3 * at + 2] = r.stop;
            ++at;
        }
    }
}

void nref_planned_destroy(nref_planned* p) { delete p; }

/// EngineCore<float> (fp64 == 0) or EngineCore<double> (fp64 != 0) over a
/// copy of the planned model (the reference ctor takes it by value).
neng_status nref_engine_create(const nref_planned* p, int32_t batch, int32_t unroll, int32_t fp64,
                               nref_engine** out) {
    return guarded([&] {
        auto e = std::make_unique<nref_engine>();
        if (fp64)
            e->f64 = std::make_unique<neng::EngineCore<double>>(p->pm, batch, unroll);
        else
            e->f32 = std::make_unique<neng::EngineCore<float>>(p->pm, batch, unroll);
        *out = e.release();
    });
}

neng_status nref_engine_run(nref_engine* e, int32_t n_steps, int32_t n_feeds,
                            const neng_feed* feeds, double* probes_out) {
    return guarded([&] {
        neng::FeedData fd = to_feeds(n_feeds, feeds);
        if (e->f32) {
            neng::ProbeOutput out = e->f32->run(n_steps, fd);
            if (probes_out) write_probes(e->f32->planned().model, out, probes_out);
            e->last = std::move(out);
        } else {
            neng::ProbeOutput out = e->f64->run(n_steps, fd);
            if (probes_out) write_probes(e->f64->planned().model, out, probes_out);
            e->last = std::move(out);
        }
    });
}

/* the reference's own write_probe_binary / write_probe_csv (export.cpp) of the last run */
neng_status nref_engine_write_probe_binary(const nref_engine* e, const char* path) {
    return guarded([&] { neng::write_probe_binary(std::string(path), e->last); });
}

neng_status nref_engine_write_probe_csv(const nref_engine* e, const char* path, double dt) {
    return guarded([&] { neng::write_probe_csv(std::string(path), e->last, dt); });
}

neng_status nref_engine_reset(nref_engine* e) {
    return guarded([&] { e->f32 ? e->f32->reset() : e->f64->reset(); });
}

neng_status nref_engine_read_signal(const nref_engine* e, int32_t sig, int32_t b, double* out,
                                    int64_t capacity, int64_t* n_out) {
    return guarded([&] {
        std::vector<double> v = e->f32 ? e->f32->read_signal(sig, b) : e->f64->read_signal(sig, b);
        *n_out = static_cast<int64_t>(v.size());
        if (out) {
            if (capacity < static_cast<int64_t>(v.size()))
                throw std::invalid_argument("read_signal: capacity too small");
            std::copy(v.begin(), v.end(), out);
        }
    });
}

int32_t nref_engine_steps_completed(const nref_engine* e) {
    return e->f32 ? e->f32->steps_completed() : e->f64->steps_completed();
}

int32_t nref_engine_buffer_storage(const nref_engine* e, int32_t buffer) {
    neng::StorageMode m = e->f32 ? e->f32->buffer_storage(buffer) : e->f64->buffer_storage(buffer);
    return m == neng::StorageMode::PerBatch ? NENG_STORAGE_PER_BATCH : NENG_STORAGE_SHARED;
}

void nref_engine_destroy(nref_engine* e) { delete e; }

/// run_reference (reference.cpp:194-226): the f64 interpreter.
neng_status nref_run_reference(const neng_built_model* m, int32_t n_steps, int32_t n_feeds,
                               const neng_feed* feeds, int32_t minibatch, double* probes_out) {
    return guarded([&] {
        neng::BuiltModel model = to_model(m);
        neng::ProbeOutput out = neng::run_reference(model, n_steps, to_feeds(n_feeds, feeds), minibatch);
        if (probes_out) write_probes(model, out, probes_out);
    });
}

/// CPU baseline timing harness (bench.py --impl reference / cpu_baseline):
/// `threads` independent EngineCore<float> instances, each advancing
/// `rows_per_engine` batch rows, following the reference protocol
/// (warm-up run, reset, timed run — bench.cpp:218-225). Batch rows are
/// independent (test_exec.cpp:246-267), so splitting them across engines is
/// exact. Returns the wall seconds of the timed run (max over threads).
}  // extern "C"

namespace {

template <class T>
double time_engines_t(const nref_planned* p, int threads, int rows, int warm_steps, int timed_steps,
                      uint64_t feed_seed) {
    // white-noise feeds N(0, 1) for every feed slot, per engine (seeded, generated before timing)
    const neng::BuiltModel& m = p->pm.model;
    const int steps = std::max(std::max(warm_steps, timed_steps), 1);
    std::vector<neng::FeedData> feeds(threads);
    if (feed_seed)
        for (int t = 0; t < threads; ++t) {
            std::mt19937_64 rng(feed_seed + 1000003ull * t);
            std::normal_distribution<double> nd(0.0, 1.0);
            for (const neng::FeedSlot& fs : m.feed_slots) {
                neng::Tensor3 x(rows, steps, fs.dim);
                for (double& v : x.data) v = nd(rng);
                feeds[t].emplace(fs.node_id, std::move(x));
            }
        }
    std::vector<std::unique_ptr<neng::EngineCore<T>>> engines(threads);
    std::vector<std::thread> pool;
    std::vector<double> secs(threads, 0.0);
    std::vector<std::string> errs(threads);
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            try {
                engines[t] = std::make_unique<neng::EngineCore<T>>(p->pm, rows, 1);
                if (warm_steps > 0) engines[t]->run(warm_steps, feeds[t]);  // warm-up, excluded (bench.cpp:221)
                engines[t]->reset();
            } catch (const std::exception& ex) {
                errs[t] = ex.what();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& s : errs)
        if (!s.empty()) throw neng::RunError(s);
    pool.clear();
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            try {
                auto t0 = std::chrono::steady_clock::now();
                engines[t]->run(timed_steps, feeds[t]);
                secs[t] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            } catch (const std::exception& ex) {
                errs[t] = ex.what();
            }
        });
    for (auto& th : pool) th.join();
    for (auto& s : errs)
        if (!s.empty()) throw neng::RunError(s);
    double mx = 0.0;
    for (double s : secs) mx = std::max(mx, s);
    return mx;
}

}  // namespace

extern "C" {

neng_status nref_time_engines(const nref_planned* p, int32_t threads, int32_t rows_per_engine,
                              int32_t warm_steps, int32_t timed_steps, double* seconds_out) {
    return guarded([&] { *seconds_out = time_engines_t<float>(p, threads, rows_per_engine, warm_steps, timed_steps, 0); });
}

/// nref_time_engines with the engine precision (fp64: EngineCore<double>, what the
/// reference's run_bench times, bench.cpp:218) and seeded white-noise feeds on every
/// feed slot (feed_seed 0: no feeds).
neng_status nref_time_engines2(const nref_planned* p, int32_t threads, int32_t rows_per_engine, int32_t warm_steps,
                               int32_t timed_steps, int32_t fp64, uint64_t feed_seed, double* seconds_out) {
    return guarded([&] {
        *seconds_out = fp64 ? time_engines_t<double>(p, threads, rows_per_engine, warm_steps, timed_steps, feed_seed)
                            : time_engines_t<float>(p, threads, rows_per_engine, warm_steps, timed_steps, feed_seed);
    });
}

}  // extern "C"
