// host_capi.cpp — extern "C" host tooling (include/neng_host.h): validation,
// dependency graph, the planner, and parity diagnostics.
#include <cstring>
#include <new>
#include <string>

#include "engine.hpp"
#include "neng_host.h"
#include "passes.hpp"

namespace nengb {
cudaError_t launch_libm_eval(int func, uint32_t lo, int64_t n, uint32_t* out, const LibmTables& t,
                             cudaStream_t stream);
}

namespace {

thread_local std::string g_err;

template <class F>
neng_status guarded(F&& f) {
    auto fail = [&](neng_status s, const char* m) {
        g_err = m;
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
    } catch (const std::bad_alloc&) {
        return fail(NENG_OUT_OF_MEMORY, "out of memory");
    } catch (const std::exception& x) {
        return fail(NENG_INVALID_ARGUMENT, x.what());
    }
}

}  // namespace

struct neng_plan {
    nengb::PlannedModel pm;
    nengb::PlannedView view;
};

extern "C" {

const char* neng_host_last_error(void) { return g_err.c_str(); }

neng_status neng_model_validate(const neng_built_model* model) {
    return guarded([&] {
        nengb::BuiltModel m = nengb::model_from_view(*model);
        nengb::build_dependency_graph(m.signals, m.operators);
    });
}

neng_status neng_model_toposort(const neng_built_model* model, int32_t* order_out) {
    return guarded([&] {
        nengb::BuiltModel m = nengb::model_from_view(*model);
        auto g = nengb::build_dependency_graph(m.signals, m.operators);
        auto order = nengb::toposort_schedule(g);
        std::memcpy(order_out, order.data(), order.size() * sizeof(int32_t));
    });
}

neng_status neng_model_dependency_edges(const neng_built_model* model, int64_t* n_edges, int32_t* pairs) {
    return guarded([&] {
        nengb::BuiltModel m = nengb::model_from_view(*model);
        auto g = nengb::build_dependency_graph(m.signals, m.operators);
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

neng_status neng_solve_decoders(const double* a, int32_t m, int32_t n, const double* y, int32_t d, double reg,
                                double* decoders_out) {
    return guarded([&] {
        if (!a || !y || !decoders_out) throw nengb::InvalidArgument("neng_solve_decoders: null argument");
        const std::vector<double> dec = nengb::solve_decoders(a, m, n, y, d, reg);
        std::memcpy(decoders_out, dec.data(), dec.size() * sizeof(double));
    });
}

neng_status neng_run_passes(const neng_built_model* model, int32_t merge, int32_t simplify, int32_t planner,
                            int32_t tree_depth, int32_t sort, neng_plan** out) {
    return guarded([&] {
        nengb::PipelineConfig cfg;
        cfg.merge = merge != 0;
        cfg.simplify = simplify != 0;
        cfg.planner = static_cast<nengb::Planner>(planner);
        cfg.tree_depth = tree_depth;
        cfg.sort = sort != 0;
        auto* p = new neng_plan();
        try {
            p->pm = nengb::run_passes(nengb::model_from_view(*model), cfg);
            p->view.build(p->pm);
        } catch (...) {
            delete p;
            throw;
        }
        *out = p;
    });
}

const neng_planned_model* neng_plan_view(const neng_plan* p) { return &p->view.view; }

void neng_plan_stats(const neng_plan* p, double* frac, int64_t* rows, int32_t* groups) {
    *frac = p->pm.stats.contiguous_read_fraction;
    *rows = p->pm.stats.gather_row_count;
    *groups = p->pm.stats.groups_per_step;
}

void neng_plan_destroy(neng_plan* p) { delete p; }

neng_status neng_debug_libm_eval(int32_t device, int32_t func, uint32_t lo, int64_t n, uint32_t* out_host) {
    return guarded([&] {
        nengb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
        const nengb::LibmTables& t = nengb::libm_tables(device);
        nengb::DevMem buf;
        const int64_t chunk = int64_t{1} << 26;
        buf.ensure(static_cast<size_t>(std::min(n, chunk)) * 4 + 16);
        for (int64_t at = 0; at < n; at += chunk) {
            int64_t m = std::min(chunk, n - at);
            nengb::cuda_check(nengb::launch_libm_eval(func, lo + static_cast<uint32_t>(at), m, buf.as<uint32_t>(), t,
                                                      nullptr),
                              "libm eval");
            nengb::cuda_check(cudaMemcpy(out_host + at, buf.p, m * 4, cudaMemcpyDeviceToHost), "libm eval D2H");
        }
    });
}

}  // extern "C"
