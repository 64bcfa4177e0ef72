// host_ir.hpp — the product's own C++ model types (namespace nengb).
//
// Field-for-field mirrors of the reference's model containers so the planner
// and the engine compiler read like the reference: Signal/SignalRef/Operator
// (proj/include/nengine/ir.hpp:37-137), BuiltModel/FeedSlot/ProbeRegistration
// (model.hpp:35-60), BufferDesc/BufferAssignment/ReadBlock/ContiguityStats/
// PipelineConfig/PlannedModel (passes.hpp:35-139).  Written from scratch; the
// only way in and out is the POD view in include/neng_gpu.h.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "neng_gpu.h"

namespace nengb {

struct StructuralError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct BuildError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct RunError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::runtime_error {
    using std::runtime_error::runtime_error;
};

enum class OpKind : int32_t {
    Reset = NENG_OP_RESET,
    Copy = NENG_OP_COPY,
    ElementwiseInc = NENG_OP_ELEMENTWISE_INC,
    DotInc = NENG_OP_DOT_INC,
    SimNeurons = NENG_OP_SIM_NEURONS,
    SimProcess = NENG_OP_SIM_PROCESS,
    SimPES = NENG_OP_SIM_PES,
    TimeUpdate = NENG_OP_TIME_UPDATE,
};
const char* op_kind_name(OpKind k);

enum class NeuronKind : int32_t {
    LIF = NENG_NEURON_LIF,
    LIFRate = NENG_NEURON_LIF_RATE,
    RectifiedLinear = NENG_NEURON_RECTIFIED_LINEAR
};

enum class AccessMode { Read, Set, Inc, Update };

using SignalId = int;
using OpId = int;

struct Signal {
    SignalId id = -1;
    std::string label;
    std::vector<int> shape;
    int32_t elem = NENG_ELEM_F64;
    std::vector<double> initial;
    bool constant = false, minibatched = false, trainable = false;

    int rows() const { return shape.empty() ? 0 : shape[0]; }
    long long elems_per_row() const {
        long long n = 1;
        for (size_t i = 1; i < shape.size(); ++i) n *= shape[i];
        return n;
    }
    long long size() const { return rows() * elems_per_row(); }
    std::vector<int> trailing_shape() const {
        return shape.empty() ? std::vector<int>{} : std::vector<int>(shape.begin() + 1, shape.end());
    }
};

struct SignalRef {
    SignalId signal = -1;
    int start = 0, stop = 0;
    int rows() const { return stop - start; }
    bool operator==(const SignalRef& o) const = default;
};

inline bool refs_overlap(const SignalRef& a, const SignalRef& b) {
    return a.signal == b.signal && a.start < b.stop && b.start < a.stop;
}

struct NeuronModel {
    NeuronKind kind = NeuronKind::LIF;
    double tau_rc = 0.02, tau_ref = 0.002, amplitude = 1.0;
    bool has_state() const { return kind == NeuronKind::LIF; }
    bool operator==(const NeuronModel& o) const = default;
};

struct Operator {
    OpId id = -1;
    OpKind kind = OpKind::Reset;
    std::vector<SignalRef> operands;
    std::vector<double> value;
    bool inc = false;
    NeuronModel neuron;
    double tau = 0.0, learning_rate = 0.0, dt = 0.0;
};

struct ProbeRegistration {
    int key = -1;
    SignalId signal = -1;
    std::string label;
};

struct FeedSlot {
    int node_id = -1;
    SignalId signal = -1;
    int dim = 0;
    bool has_default = true;
    std::string label;
};

struct BuiltModel {
    std::vector<Signal> signals;
    std::vector<Operator> operators;
    std::vector<ProbeRegistration> probes;
    std::vector<FeedSlot> feed_slots;
    double dt = 0.001;
};

struct OpGroup {
    std::vector<OpId> members;
};
using Plan = std::vector<OpGroup>;

struct BufferDesc {
    std::vector<int> trailing;
    int32_t elem = NENG_ELEM_F64;
    bool minibatched = false, trainable = false;
    int rows = 0;
    std::vector<SignalId> order;
};

struct BufferAssignment {
    std::vector<int> buffer_of, row_offset;
    std::vector<BufferDesc> buffers;
};

struct ReadBlock {
    int id = 0, group = 0, position = 0, buffer = 0;
    std::vector<SignalRef> refs;
    int total_rows() const {
        int n = 0;
        for (const auto& r : refs) n += r.rows();
        return n;
    }
};

struct ContiguityStats {
    double contiguous_read_fraction = 1.0;
    long long gather_row_count = 0;
    int groups_per_step = 0;
};

enum class Planner { Greedy = 0, Tree = 1, TransitiveClosure = 2 };

struct PipelineConfig {
    bool merge = true, simplify = true;
    Planner planner = Planner::Tree;
    int tree_depth = 3;
    bool sort = true;
};

struct PlannedModel {
    BuiltModel model;
    Plan plan;
    BufferAssignment buffers;
    std::vector<ReadBlock> read_blocks;
    ContiguityStats stats;
};

// ---- conversions at the ABI -------------------------------------------------
BuiltModel model_from_view(const neng_built_model& v);
PlannedModel planned_from_view(const neng_planned_model& v);

/// Owns a flattened POD view of a PlannedModel (pointers into `pm`).
struct PlannedView {
    const PlannedModel* pm = nullptr;
    std::vector<neng_signal> sig;
    std::vector<neng_operator> ops;
    std::vector<std::vector<neng_ref>> refs;
    std::vector<neng_probe> probes;
    std::vector<neng_feed_slot> slots;
    std::vector<int32_t> goff, gmem;
    std::vector<neng_buffer_desc> bufs;
    neng_planned_model view{};
    void build(const PlannedModel& p);
};

// ---- IR helpers (semantics of ir.cpp) --------------------------------------
/// (operand index, mode) per operand (operand_modes ir.cpp:130-167).
std::vector<std::pair<int, AccessMode>> operand_modes(const Operator& op);
/// validate_operators (ir.cpp:310-317): StructuralError on the first failure.
void validate_operators(const std::vector<Signal>& signals, const std::vector<Operator>& ops);

struct DependencyGraph {
    std::vector<OpId> op_ids;
    std::vector<std::vector<int>> succ, pred;
    std::vector<int> index_of_id;  // dense: op id -> node index (-1 if absent)
    int index(OpId id) const {
        return id >= 0 && id < static_cast<int>(index_of_id.size()) ? index_of_id[id] : -1;
    }
    size_t node_count() const { return op_ids.size(); }
};
/// build_dependency_graph (ir.cpp:396-463): BuildError on write conflicts/cycles.
DependencyGraph build_dependency_graph(const std::vector<Signal>& signals,
                                       const std::vector<Operator>& ops);
/// toposort_schedule (ir.cpp:465-488): Kahn, ties to the lowest operator id.
std::vector<OpId> toposort_schedule(const DependencyGraph& g);

}  // namespace nengb
