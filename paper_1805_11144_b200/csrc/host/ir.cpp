// ir.cpp — model conversion at the ABI plus the IR semantics the planner and
// engine need: operand access modes, structural validation, the within-step
// dependency graph and its deterministic topological order.  Semantics follow
// proj/src/ir.cpp (cited per function); the implementation is our own.
#include <algorithm>
#include <queue>
#include <sstream>
#include <unordered_map>

#include "host_ir.hpp"

namespace nengb {

const char* op_kind_name(OpKind k) {
    switch (k) {
        case OpKind::Reset: return "Reset";
        case OpKind::Copy: return "Copy";
        case OpKind::ElementwiseInc: return "ElementwiseInc";
        case OpKind::DotInc: return "DotInc";
        case OpKind::SimNeurons: return "SimNeurons";
        case OpKind::SimProcess: return "SimProcess";
        case OpKind::SimPES: return "SimPES";
        case OpKind::TimeUpdate: return "TimeUpdate";
    }
    return "?";
}

BuiltModel model_from_view(const neng_built_model& v) {
    if (v.n_signals < 0 || v.n_operators < 0 || v.n_probes < 0 || v.n_feed_slots < 0)
        throw InvalidArgument("negative element count in model view");
    BuiltModel m;
    m.dt = v.dt;
    m.signals.resize(v.n_signals);
    for (int i = 0; i < v.n_signals; ++i) {
        const neng_signal& s = v.signals[i];
        Signal& d = m.signals[i];
        d.id = s.id;
        d.label = s.label ? s.label : "";
        if (s.ndim > 0) d.shape.assign(s.shape, s.shape + s.ndim);
        d.elem = s.elem;
        if (s.n_initial > 0) d.initial.assign(s.initial, s.initial + s.n_initial);
        d.constant = s.constant != 0;
        d.minibatched = s.minibatched != 0;
        d.trainable = s.trainable != 0;
    }
    m.operators.resize(v.n_operators);
    for (int i = 0; i < v.n_operators; ++i) {
        const neng_operator& o = v.operators[i];
        Operator& d = m.operators[i];
        d.id = o.id;
        d.kind = static_cast<OpKind>(o.kind);
        for (int k = 0; k < o.n_operands; ++k)
            d.operands.push_back({o.operands[k].signal, o.operands[k].start, o.operands[k].stop});
        if (o.n_value > 0) d.value.assign(o.value, o.value + o.n_value);
        d.inc = o.inc != 0;
        d.neuron = {static_cast<NeuronKind>(o.neuron_kind), o.tau_rc, o.tau_ref, o.amplitude};
        d.tau = o.tau;
        d.learning_rate = o.learning_rate;
        d.dt = o.dt;
    }
    for (int i = 0; i < v.n_probes; ++i)
        m.probes.push_back({v.probes[i].key, v.probes[i].signal, v.probes[i].label ? v.probes[i].label : ""});
    for (int i = 0; i < v.n_feed_slots; ++i) {
        const neng_feed_slot& f = v.feed_slots[i];
        m.feed_slots.push_back({f.node_id, f.signal, f.dim, f.has_default != 0, f.label ? f.label : ""});
    }
    return m;
}

PlannedModel planned_from_view(const neng_planned_model& v) {
    PlannedModel p;
    p.model = model_from_view(v.model);
    if (v.n_groups < 0 || v.n_buffers < 0) throw InvalidArgument("negative count in planned view");
    for (int g = 0; g < v.n_groups; ++g) {
        OpGroup og;
        og.members.assign(v.group_members + v.group_offsets[g], v.group_members + v.group_offsets[g + 1]);
        p.plan.push_back(std::move(og));
    }
    int ns = v.model.n_signals;
    if (ns > 0) {
        p.buffers.buffer_of.assign(v.buffer_of, v.buffer_of + ns);
        p.buffers.row_offset.assign(v.row_offset, v.row_offset + ns);
    }
    for (int b = 0; b < v.n_buffers; ++b) {
        const neng_buffer_desc& d = v.buffers[b];
        BufferDesc bd;
        if (d.n_trailing > 0) bd.trailing.assign(d.trailing, d.trailing + d.n_trailing);
        bd.elem = d.elem;
        bd.minibatched = d.minibatched != 0;
        bd.trainable = d.trainable != 0;
        bd.rows = d.rows;
        if (d.n_order > 0) bd.order.assign(d.order, d.order + d.n_order);
        p.buffers.buffers.push_back(std::move(bd));
    }
    p.stats.groups_per_step = static_cast<int>(p.plan.size());
    return p;
}

void PlannedView::build(const PlannedModel& p) {
    pm = &p;
    const BuiltModel& m = p.model;
    sig.resize(m.signals.size());
    for (size_t i = 0; i < m.signals.size(); ++i) {
        const Signal& s = m.signals[i];
        sig[i] = {s.id, static_cast<int32_t>(s.shape.size()), s.shape.data(), s.elem,
                  static_cast<int64_t>(s.initial.size()), s.initial.data(), s.constant, s.minibatched,
                  s.trainable, s.label.c_str()};
    }
    ops.resize(m.operators.size());
    refs.resize(m.operators.size());
    for (size_t i = 0; i < m.operators.size(); ++i) {
        const Operator& o = m.operators[i];
        refs[i].clear();
        for (const SignalRef& r : o.operands) refs[i].push_back({r.signal, r.start, r.stop});
        neng_operator& d = ops[i];
        d = neng_operator{};
        d.id = o.id;
        d.kind = static_cast<int32_t>(o.kind);
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
    for (const auto& pr : m.probes) probes.push_back({pr.key, pr.signal, pr.label.c_str()});
    slots.clear();
    for (const auto& f : m.feed_slots) slots.push_back({f.node_id, f.signal, f.dim, f.has_default, f.label.c_str()});
    goff.assign(1, 0);
    gmem.clear();
    for (const OpGroup& g : p.plan) {
        gmem.insert(gmem.end(), g.members.begin(), g.members.end());
        goff.push_back(static_cast<int32_t>(gmem.size()));
    }
    bufs.resize(p.buffers.buffers.size());
    for (size_t i = 0; i < bufs.size(); ++i) {
        const BufferDesc& b = p.buffers.buffers[i];
        bufs[i] = {static_cast<int32_t>(b.trailing.size()), b.trailing.data(), b.elem, b.minibatched,
                   b.trainable, b.rows, static_cast<int32_t>(b.order.size()), b.order.data()};
    }
    view.model = {static_cast<int32_t>(sig.size()), sig.data(), static_cast<int32_t>(ops.size()), ops.data(),
                  static_cast<int32_t>(probes.size()), probes.data(), static_cast<int32_t>(slots.size()),
                  slots.data(), m.dt};
    view.n_groups = static_cast<int32_t>(p.plan.size());
    view.group_offsets = goff.data();
    view.group_members = gmem.data();
    view.buffer_of = p.buffers.buffer_of.data();
    view.row_offset = p.buffers.row_offset.data();
    view.n_buffers = static_cast<int32_t>(bufs.size());
    view.buffers = bufs.data();
}

// ---------------------------------------------------------------------------

namespace {

[[noreturn]] void structural_fail(const Operator& op, const std::string& what) {
    std::ostringstream os;
    os << "operator " << op.id << " (" << op_kind_name(op.kind) << "): " << what;
    throw StructuralError(os.str());
}

/// The operand signature of an operator kind: how many operands it takes and
/// how it accesses each (the reference's table, ir.cpp:130-167).  Positions
/// past the table read as Update (SimNeurons' state operands).
struct Signature {
    size_t arity;
    std::vector<AccessMode> modes;
};

Signature signature_of(const Operator& op) {
    using M = AccessMode;
    switch (op.kind) {
        case OpKind::Reset: return {1, {M::Set}};
        case OpKind::Copy: return {2, {M::Read, op.inc ? M::Inc : M::Set}};
        case OpKind::ElementwiseInc:
        case OpKind::DotInc: return {3, {M::Read, M::Read, M::Inc}};
        case OpKind::SimNeurons: return {op.neuron.has_state() ? size_t{4} : size_t{2}, {M::Read, M::Set}};
        case OpKind::SimProcess:
            return op.tau > 0.0 ? Signature{3, {M::Read, M::Update, M::Update}} : Signature{2, {M::Read, M::Set}};
        case OpKind::SimPES: return {3, {M::Read, M::Read, M::Update}};
        case OpKind::TimeUpdate: return {2, {M::Update, M::Update}};
    }
    structural_fail(op, "unknown kind");
}

}  // namespace

std::vector<std::pair<int, AccessMode>> operand_modes(const Operator& op) {
    const Signature sg = signature_of(op);
    if (op.operands.size() != sg.arity)
        structural_fail(op, "expected " + std::to_string(sg.arity) + " operands, got " +
                                std::to_string(op.operands.size()));
    std::vector<std::pair<int, AccessMode>> out;
    out.reserve(sg.arity);
    for (size_t i = 0; i < sg.arity; ++i)
        out.emplace_back(static_cast<int>(i), i < sg.modes.size() ? sg.modes[i] : AccessMode::Update);
    return out;
}

namespace {

/// Structural checks of one operator against the signal table; every failure
/// is a StructuralError naming the operator (messages as the reference's,
/// ir.cpp:228-306, which the tests compare).
class OperandCheck {
public:
    OperandCheck(const std::vector<Signal>& signals, const Operator& op) : sig_(signals), op_(op) {}

    void run() {
        const auto modes = operand_modes(op_);
        for (const SignalRef& r : op_.operands) in_bounds(r);
        const int32_t width = sig_[op_.operands[0].signal].elem;
        require(std::all_of(op_.operands.begin(), op_.operands.end(),
                            [&](const SignalRef& r) { return sig_[r.signal].elem == width; }),
                "operands mix element widths");
        for (auto [pos, mode] : modes) {
            const Signal& s = sig_[op_.operands[pos].signal];
            if (mode != AccessMode::Read && s.constant) fail("writes constant signal '" + s.label + "'");
        }
        kind_rules();
    }

private:
    [[noreturn]] void fail(const std::string& what) const { structural_fail(op_, what); }
    void require(bool ok, const std::string& what) const {
        if (!ok) fail(what);
    }
    const SignalRef& arg(size_t i) const { return op_.operands[i]; }
    std::vector<int> trailing(const SignalRef& r) const { return sig_[r.signal].trailing_shape(); }
    long long elems(const SignalRef& r) const {
        return static_cast<long long>(r.rows()) * sig_[r.signal].elems_per_row();
    }

    void in_bounds(const SignalRef& r) const {
        require(r.signal >= 0 && static_cast<size_t>(r.signal) < sig_.size(),
                "ref to unknown signal " + std::to_string(r.signal));
        const Signal& s = sig_[r.signal];
        require(r.start >= 0 && r.stop <= s.rows() && r.start < r.stop,
                "slice [" + std::to_string(r.start) + ", " + std::to_string(r.stop) + ") out of bounds for signal '" +
                    s.label + "' with " + std::to_string(s.rows()) + " rows");
    }
    void same_shape(const SignalRef& a, const SignalRef& b, const char* pair) const {
        require(a.rows() == b.rows() && trailing(a) == trailing(b), std::string(pair) + " shapes do not agree");
    }
    void is_vector(const SignalRef& r, const char* what) const {
        require(trailing(r).empty(), std::string(what) + " must be a vector signal");
    }

    void kind_rules() const {
        switch (op_.kind) {
            case OpKind::Reset:
                require(static_cast<long long>(op_.value.size()) == elems(arg(0)),
                        "value length does not match destination");
                return;
            case OpKind::Copy: same_shape(arg(0), arg(1), "src/dst"); return;
            case OpKind::ElementwiseInc:
                same_shape(arg(1), arg(2), "x/y");
                if (!(arg(0).rows() == 1 && sig_[arg(0).signal].elems_per_row() == 1))  // a scalar scale broadcasts
                    same_shape(arg(0), arg(1), "a/x");
                return;
            case OpKind::DotInc: {
                const std::vector<int> at = trailing(arg(0));
                require(at.size() == 1, "a must be a matrix signal");
                is_vector(arg(1), "x");
                is_vector(arg(2), "y");
                require(at[0] == arg(1).rows(), "a columns do not match x rows");
                require(arg(0).rows() == arg(2).rows(), "a rows do not match y rows");
                require(!refs_overlap(arg(2), arg(1)) && !refs_overlap(arg(2), arg(0)), "y aliases an input operand");
                return;
            }
            case OpKind::SimNeurons:
                for (const SignalRef& r : op_.operands) is_vector(r, "operand");
                for (const SignalRef& r : op_.operands) require(r.rows() == arg(0).rows(), "operand row counts differ");
                return;
            case OpKind::SimProcess:
                same_shape(arg(0), arg(1), "in/out");
                if (op_.operands.size() == 3) same_shape(arg(1), arg(2), "out/state");
                return;
            case OpKind::SimPES: {
                is_vector(arg(0), "pre");
                is_vector(arg(1), "error");
                const std::vector<int> wt = trailing(arg(2));
                require(wt.size() == 1, "weights must be a matrix signal");
                require(arg(2).rows() == arg(1).rows() && wt[0] == arg(0).rows(),
                        "weights shape does not match error x pre");
                return;
            }
            case OpKind::TimeUpdate:
                for (const SignalRef& r : op_.operands) require(elems(r) == 1, "step/time must be scalar signals");
                return;
        }
    }

    const std::vector<Signal>& sig_;
    const Operator& op_;
};

void validate_one(const std::vector<Signal>& signals, const Operator& op) { OperandCheck(signals, op).run(); }

// phase_edge (ir.cpp:351-360): Set < Inc < Read < Update, no Update -> Read.
bool phase_edge(AccessMode from, AccessMode to) {
    using M = AccessMode;
    switch (from) {
        case M::Set: return to == M::Inc || to == M::Read || to == M::Update;
        case M::Inc: return to == M::Read || to == M::Update;
        case M::Read: return to == M::Update;
        case M::Update: return false;
    }
    return false;
}

}  // namespace

void validate_operators(const std::vector<Signal>& signals, const std::vector<Operator>& ops) {
    std::vector<char> seen;
    for (const Operator& op : ops) {
        if (op.id < 0) throw StructuralError("negative operator id " + std::to_string(op.id));
        if (static_cast<size_t>(op.id) >= seen.size()) seen.resize(static_cast<size_t>(op.id) + 1, 0);
        if (seen[op.id]) throw StructuralError("duplicate operator id " + std::to_string(op.id));
        seen[op.id] = 1;
        validate_one(signals, op);
    }
}

DependencyGraph build_dependency_graph(const std::vector<Signal>& signals, const std::vector<Operator>& ops) {
    validate_operators(signals, ops);
    DependencyGraph g;
    size_t n = ops.size();
    g.op_ids.reserve(n);
    int max_id = -1;
    for (const Operator& op : ops) max_id = std::max(max_id, op.id);
    g.index_of_id.assign(static_cast<size_t>(max_id + 1), -1);
    for (size_t i = 0; i < n; ++i) {
        g.op_ids.push_back(ops[i].id);
        g.index_of_id[ops[i].id] = static_cast<int>(i);
    }
    struct Access {
        int node;
        SignalRef ref;
        AccessMode mode;
    };
    std::vector<std::vector<Access>> by_signal(signals.size());
    for (size_t i = 0; i < n; ++i)
        for (auto [pos, mode] : operand_modes(ops[i]))
            by_signal[ops[i].operands[pos].signal].push_back({static_cast<int>(i), ops[i].operands[pos], mode});

    std::vector<std::pair<int, int>> edges;
    for (size_t sid = 0; sid < by_signal.size(); ++sid) {
        const auto& acc = by_signal[sid];
        for (size_t i = 0; i < acc.size(); ++i)
            for (size_t j = i + 1; j < acc.size(); ++j) {
                const Access &a = acc[i], &b = acc[j];
                if (a.node == b.node || !refs_overlap(a.ref, b.ref)) continue;
                if ((a.mode == AccessMode::Set && b.mode == AccessMode::Set) ||
                    (a.mode == AccessMode::Update && b.mode == AccessMode::Update)) {
                    std::ostringstream os;
                    os << "write conflict on signal '" << signals[sid].label << "': operators " << ops[a.node].id
                       << " (" << op_kind_name(ops[a.node].kind) << ") and " << ops[b.node].id << " ("
                       << op_kind_name(ops[b.node].kind) << ") both "
                       << (a.mode == AccessMode::Set ? "set" : "update") << " overlapping rows";
                    throw BuildError(os.str());
                }
                if (phase_edge(a.mode, b.mode)) edges.emplace_back(a.node, b.node);
                if (phase_edge(b.mode, a.mode)) edges.emplace_back(b.node, a.node);
            }
    }
    std::sort(edges.begin(), edges.end());
    edges.erase(std::unique(edges.begin(), edges.end()), edges.end());
    g.succ.assign(n, {});
    g.pred.assign(n, {});
    for (auto [f, t] : edges) {
        g.succ[f].push_back(t);
        g.pred[t].push_back(f);
    }
    for (auto& v : g.pred) std::sort(v.begin(), v.end());

    // cycle check (Kahn)
    std::vector<int> indeg(n);
    std::vector<int> ready;
    for (size_t i = 0; i < n; ++i) {
        indeg[i] = static_cast<int>(g.pred[i].size());
        if (!indeg[i]) ready.push_back(static_cast<int>(i));
    }
    size_t done = 0;
    while (!ready.empty()) {
        int v = ready.back();
        ready.pop_back();
        ++done;
        for (int w : g.succ[v])
            if (--indeg[w] == 0) ready.push_back(w);
    }
    if (done != n) {
        // report one cycle (DFS), like find_cycle (ir.cpp:362-392)
        std::vector<int> color(n, 0), parent(n, -1), cycle;
        for (size_t root = 0; root < n && cycle.empty(); ++root) {
            if (color[root]) continue;
            std::vector<std::pair<int, size_t>> stack{{static_cast<int>(root), 0}};
            color[root] = 1;
            while (!stack.empty() && cycle.empty()) {
                int v = stack.back().first;
                size_t& ei = stack.back().second;
                if (ei < g.succ[v].size()) {
                    int w = g.succ[v][ei++];
                    if (color[w] == 0) {
                        color[w] = 1;
                        parent[w] = v;
                        stack.emplace_back(w, 0);
                    } else if (color[w] == 1) {
                        cycle.push_back(w);
                        for (int u = v; u != w; u = parent[u]) cycle.push_back(u);
                        cycle.push_back(w);
                        std::reverse(cycle.begin(), cycle.end());
                    }
                } else {
                    color[v] = 2;
                    stack.pop_back();
                }
            }
        }
        std::ostringstream os;
        os << "dependency cycle:";
        for (int v : cycle) os << " " << ops[v].id;
        throw BuildError(os.str());
    }
    return g;
}

std::vector<OpId> toposort_schedule(const DependencyGraph& g) {
    size_t n = g.node_count();
    std::vector<int> indeg(n);
    std::priority_queue<std::pair<OpId, int>, std::vector<std::pair<OpId, int>>, std::greater<>> ready;
    for (size_t i = 0; i < n; ++i) {
        indeg[i] = static_cast<int>(g.pred[i].size());
        if (!indeg[i]) ready.push({g.op_ids[i], static_cast<int>(i)});
    }
    std::vector<OpId> order;
    order.reserve(n);
    while (!ready.empty()) {
        auto [id, v] = ready.top();
        ready.pop();
        order.push_back(id);
        for (int w : g.succ[v])
            if (--indeg[w] == 0) ready.push({g.op_ids[w], w});
    }
    if (order.size() != n) throw BuildError("toposort on cyclic graph");
    return order;
}

}  // namespace nengb
