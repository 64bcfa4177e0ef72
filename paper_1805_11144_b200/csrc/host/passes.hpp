// passes.hpp — the build-time passes that produce a PlannedModel
// (semantics of proj/src/passes.cpp): simplify and merge planning in
// passes.cpp, the signal layout in layout.cpp.
#pragma once

#include "host_ir.hpp"

namespace nengb {

std::vector<Operator> simplify_operators(const std::vector<Signal>& signals, std::vector<Operator> ops);
Plan plan_tree_search(const std::vector<Signal>& signals, const std::vector<Operator>& ops, int depth);
Plan plan_greedy(const std::vector<Signal>& signals, const std::vector<Operator>& ops);
void validate_plan(const std::vector<Signal>& signals, const std::vector<Operator>& ops, const Plan& plan);
BufferAssignment create_base_buffers(const std::vector<Signal>& signals, const std::vector<Operator>& ops,
                                     const Plan& plan);
std::vector<ReadBlock> collect_read_blocks(const std::vector<Operator>& ops, const Plan& plan,
                                           const BufferAssignment& buffers);
void sort_buffers(const std::vector<Signal>& signals, Plan& plan, BufferAssignment& buffers,
                  std::vector<ReadBlock>& blocks);
ContiguityStats contiguity_stats(const std::vector<ReadBlock>& blocks, const BufferAssignment& buffers,
                                 const Plan& plan);
PlannedModel run_passes(BuiltModel model, const PipelineConfig& config = {});

// decoders.cpp: the frontend's regularised least-squares decoder solve (frontend.cpp:56-76)
std::vector<double> solve_decoders(const double* A, int m, int n, const double* Y, int d, double reg);

}  // namespace nengb
