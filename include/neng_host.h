/*
 * neng_host.h — host-side tooling exported by libneng_gpu.so next to the
 * engine ABI (neng_gpu.h): structural validation and the dependency graph
 * (reference: proj/src/ir.cpp:310-488), the merge planner / layout passes
 * (proj/src/passes.cpp:663-694, PlannedModel passes.hpp:131-139), and
 * diagnostics used by the parity tests.
 */
#ifndef NENG_HOST_H
#define NENG_HOST_H

#include <stdint.h>

#include "neng_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* validate_operators + build_dependency_graph (ir.cpp:310-317, 396-463). */
neng_status neng_model_validate(const neng_built_model* model);

/* toposort_schedule (ir.cpp:465-488): order_out receives n_operators ids. */
neng_status neng_model_toposort(const neng_built_model* model, int32_t* order_out);

/* Dependency edges as (from_id, to_id) pairs; pairs == NULL queries the count. */
neng_status neng_model_dependency_edges(const neng_built_model* model, int64_t* n_edges, int32_t* pairs);

/* run_passes (passes.cpp:663-694) with PipelineConfig fields (passes.hpp:122-128);
 * planner: 0 greedy, 1 tree, 2 transitive closure (BuildError, as in the reference). */
typedef struct neng_plan neng_plan;
neng_status neng_run_passes(const neng_built_model* model, int32_t merge, int32_t simplify, int32_t planner,
                            int32_t tree_depth, int32_t sort, neng_plan** out);
/* The planned model (operators after simplification); valid until neng_plan_destroy. */
const neng_planned_model* neng_plan_view(const neng_plan* p);
void neng_plan_stats(const neng_plan* p, double* contiguous_read_fraction, int64_t* gather_row_count,
                     int32_t* groups_per_step);
void neng_plan_destroy(neng_plan* p);

/* solve_decoders (frontend.cpp:56-76) without Eigen: D solves
 * (A^T A + m sigma^2 I) D = A^T Y with sigma = reg * max|A|; A [m][n], Y [m][d],
 * decoders_out [n][d], all row-major doubles.  BuildError for an empty system,
 * negative reg, or singular normal equations (reg too small). */
neng_status neng_solve_decoders(const double* a, int32_t m, int32_t n, const double* y, int32_t d, double reg,
                                double* decoders_out);

/* Diagnostics: evaluate the device's glibc-parity expm1f (func 0) or log1pf
 * (func 1) on every float whose bit pattern is in [lo, lo + n); out_host gets
 * the result bit patterns. */
neng_status neng_debug_libm_eval(int32_t device, int32_t func, uint32_t lo, int64_t n, uint32_t* out_host);

#ifdef __cplusplus
}
#endif
#endif /* NENG_HOST_H */
