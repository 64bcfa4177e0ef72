// layout.cpp — signal layout after merge planning: which base buffer every
// signal lives in, its row offset there, and the read blocks whose contiguity
// the layout optimises.  The results are the reference's (passes.cpp:330-661:
// create_base_buffers, collect_read_blocks, sort_buffers, contiguity_stats),
// checked plan-for-plan by tests/test_planner.py (up to the 78,849-operator
// config-4 graph); the organisation here is our own:
//   * buffers are the connected components of the graph "two signals sit at the
//     same operand position of one merged group", labelled by a depth-first
//     walk from the smallest signal id;
//   * the layout sort (the paper's Alg. 1 + Alg. 2) is a LayoutSorter object:
//     "spans" (signals of a buffer read by exactly the same read blocks) are
//     chained greedily by block similarity, then groups' member order and
//     spans' signal order are aligned alternately until nothing moves.
#include <algorithm>
#include <numeric>
#include <unordered_map>

#include "passes.hpp"

namespace nengb {

namespace {

std::unordered_map<OpId, const Operator*> index_ops(const std::vector<Operator>& ops) {
    std::unordered_map<OpId, const Operator*> idx;
    idx.reserve(ops.size());
    for (const Operator& op : ops) idx.emplace(op.id, &op);
    return idx;
}

/// Row layout of a signal (what every signal of one buffer must share).
struct RowKind {
    std::vector<int> trailing;
    int32_t elem;
    bool minibatched, trainable;
    explicit RowKind(const Signal& s)
        : trailing(s.trailing_shape()), elem(s.elem), minibatched(s.minibatched), trainable(s.trainable) {}
    bool operator==(const RowKind&) const = default;
};

/// First row (in buffer rows) a ref reads.
int first_row_of(const BufferAssignment& ba, const SignalRef& r) { return ba.row_offset[r.signal] + r.start; }

}  // namespace

BufferAssignment create_base_buffers(const std::vector<Signal>& signals, const std::vector<Operator>& ops,
                                     const Plan& plan) {
    const int nsig = static_cast<int>(signals.size());
    // edges: operand p of every member of a merged group shares member 0's buffer
    std::vector<std::vector<int>> adj(nsig);
    const auto idx = index_ops(ops);
    for (const OpGroup& g : plan) {
        const Operator& lead = *idx.at(g.members.front());
        for (size_t m = 1; m < g.members.size(); ++m) {
            const Operator& op = *idx.at(g.members[m]);
            for (size_t p = 0; p < lead.operands.size(); ++p) {
                const int a = lead.operands[p].signal, b = op.operands[p].signal;
                if (a == b) continue;
                adj[a].push_back(b);
                adj[b].push_back(a);
            }
        }
    }
    // components in order of their smallest signal id (the walk starts from ascending ids)
    std::vector<int> comp(nsig, -1);
    std::vector<int> stack;
    int ncomp = 0;
    for (int s = 0; s < nsig; ++s) {
        if (comp[s] != -1) continue;
        comp[s] = ncomp;
        stack.assign(1, s);
        while (!stack.empty()) {
            const int u = stack.back();
            stack.pop_back();
            for (int v : adj[u])
                if (comp[v] == -1) {
                    comp[v] = ncomp;
                    stack.push_back(v);
                }
        }
        ++ncomp;
    }
    BufferAssignment out;
    out.buffer_of = comp;
    out.row_offset.assign(nsig, 0);
    out.buffers.resize(ncomp);
    std::vector<int> lead(ncomp, -1);  // the component's smallest signal: its row kind is the buffer's
    for (int s = 0; s < nsig; ++s) {
        BufferDesc& d = out.buffers[comp[s]];
        if (lead[comp[s]] == -1) {
            lead[comp[s]] = s;
            const RowKind k(signals[s]);
            d.trailing = k.trailing;
            d.elem = k.elem;
            d.minibatched = k.minibatched;
            d.trainable = k.trainable;
        } else if (!(RowKind(signals[s]) == RowKind(signals[lead[comp[s]]]))) {
            throw BuildError("signals " + signals[lead[comp[s]]].label + " and " + signals[s].label +
                             " share a buffer but not a row layout");
        }
        out.row_offset[s] = d.rows;  // signals stacked in id order
        d.rows += signals[s].rows();
        d.order.push_back(s);
    }
    return out;
}

std::vector<ReadBlock> collect_read_blocks(const std::vector<Operator>& ops, const Plan& plan,
                                           const BufferAssignment& buffers) {
    const auto idx = index_ops(ops);
    std::vector<ReadBlock> out;
    for (int gi = 0; gi < static_cast<int>(plan.size()); ++gi) {
        const std::vector<OpId>& members = plan[gi].members;
        const Operator& lead = *idx.at(members.front());
        for (auto [pos, mode] : operand_modes(lead)) {
            if (mode != AccessMode::Read) continue;
            ReadBlock rb;
            rb.id = static_cast<int>(out.size());
            rb.group = gi;
            rb.position = pos;
            rb.buffer = buffers.buffer_of[lead.operands[pos].signal];
            rb.refs.reserve(members.size());
            for (OpId id : members) rb.refs.push_back(idx.at(id)->operands[pos]);
            out.push_back(std::move(rb));
        }
    }
    return out;
}

namespace {

/// The layout sort of one planned model (paper Alg. 1 and 2).
class LayoutSorter {
public:
    LayoutSorter(const std::vector<Signal>& sig, Plan& plan, BufferAssignment& ba, std::vector<ReadBlock>& blocks)
        : sig_(sig), plan_(plan), ba_(ba), blocks_(blocks), nbuf_(ba.buffers.size()) {
        size_.resize(blocks.size());
        for (const ReadBlock& b : blocks) size_[b.id] = b.total_rows();
        of_buffer_.resize(nbuf_);
        of_group_.resize(plan.size());
        for (const ReadBlock& b : blocks) {
            of_buffer_[b.buffer].push_back(b.id);
            of_group_[b.group].push_back(b.id);
        }
        make_spans();
    }

    void run() {
        for (size_t bi = 0; bi < nbuf_; ++bi) {
            Buf& B = bufs_[bi];
            B.chain.resize(B.spans.size());
            std::iota(B.chain.begin(), B.chain.end(), 0);
            if (!of_buffer_[bi].empty() && B.spans.size() >= 2) B.chain = chain_spans(bi);
            if (!B.chain.empty()) lay_out(bi);
        }
        align();
    }

private:
    struct Span {
        std::vector<int> sigs;    // layout order inside the span
        std::vector<int> blocks;  // read blocks touching every signal of the span (ascending)
        bool reads(int block) const { return std::binary_search(blocks.begin(), blocks.end(), block); }
    };
    struct Buf {
        std::vector<Span> spans;
        std::vector<int> chain;  // span order in the buffer
    };

    struct VecHash {
        size_t operator()(const std::vector<int>& v) const {
            size_t h = v.size() * 0x9E3779B97F4A7C15ULL;
            for (int x : v) h = (h ^ static_cast<size_t>(x)) * 0x100000001B3ULL;
            return h;
        }
    };

    // spans: signals of a buffer with the same set of reading blocks, in order of
    // their smallest signal id (and signals ascending inside)
    void make_spans() {
        std::vector<std::vector<int>> readers(ba_.buffer_of.size());
        for (const ReadBlock& b : blocks_)
            for (const SignalRef& r : b.refs)
                if (readers[r.signal].empty() || readers[r.signal].back() != b.id) readers[r.signal].push_back(b.id);
        bufs_.resize(nbuf_);
        for (size_t bi = 0; bi < nbuf_; ++bi) {
            std::vector<int> sigs = ba_.buffers[bi].order;
            std::sort(sigs.begin(), sigs.end());
            std::unordered_map<std::vector<int>, int, VecHash> where;
            for (int s : sigs) {
                auto [it, fresh] = where.emplace(readers[s], static_cast<int>(bufs_[bi].spans.size()));
                if (fresh) bufs_[bi].spans.push_back(Span{{}, readers[s]});
                bufs_[bi].spans[it->second].sigs.push_back(s);
            }
        }
    }

    /// The largest read block of `ids` (first on ties).
    int biggest(const std::vector<int>& ids) const {
        return *std::max_element(ids.begin(), ids.end(), [&](int l, int r) { return size_[l] < size_[r]; });
    }

    static size_t differ(const std::vector<int>& a, const std::vector<int>& b) {
        std::vector<int> common;
        std::set_intersection(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(common));
        return a.size() + b.size() - 2 * common.size();
    }

    /// Alg. 1: start from the span holding the buffer's largest read block, then
    /// repeatedly append the most similar remaining span — narrowing candidates
    /// to those sharing the anchor block, then to supersets of the current
    /// span's blocks, then to the fewest differing blocks, then by the current
    /// span's blocks from largest down.
    std::vector<int> chain_spans(size_t bi) const {
        const std::vector<Span>& spans = bufs_[bi].spans;
        int anchor = biggest(of_buffer_[bi]);
        int cur = 0;
        for (int i = 0; i < static_cast<int>(spans.size()); ++i)
            if (spans[i].reads(anchor)) {
                cur = i;
                break;
            }
        std::vector<int> chain{cur};
        std::vector<int> left;
        for (int i = 0; i < static_cast<int>(spans.size()); ++i)
            if (i != cur) left.push_back(i);
        auto keep = [](std::vector<int>& cand, auto&& pred) {
            std::vector<int> kept;
            std::copy_if(cand.begin(), cand.end(), std::back_inserter(kept), pred);
            if (!kept.empty()) cand.swap(kept);
            return !kept.empty() || cand.empty();
        };
        while (!left.empty()) {
            const Span& c = spans[cur];
            std::vector<int> cand;
            std::copy_if(left.begin(), left.end(), std::back_inserter(cand), [&](int i) { return spans[i].reads(anchor); });
            if (cand.empty()) {
                cand = left;
                if (!c.blocks.empty()) anchor = biggest(c.blocks);
            }
            keep(cand, [&](int i) {
                return std::includes(spans[i].blocks.begin(), spans[i].blocks.end(), c.blocks.begin(), c.blocks.end());
            });
            size_t fewest = SIZE_MAX;
            for (int i : cand) fewest = std::min(fewest, differ(spans[i].blocks, c.blocks));
            std::vector<int> best;
            for (int i : cand)
                if (differ(spans[i].blocks, c.blocks) == fewest) best.push_back(i);
            if (best.size() > 1) {
                std::vector<int> by_rows = c.blocks;
                std::sort(by_rows.begin(), by_rows.end(),
                          [&](int l, int r) { return size_[l] != size_[r] ? size_[l] > size_[r] : l < r; });
                for (int blk : by_rows) {
                    std::vector<int> narrowed;
                    for (int i : best)
                        if (spans[i].reads(blk)) narrowed.push_back(i);
                    if (!narrowed.empty()) best.swap(narrowed);
                    if (best.size() == 1) break;
                }
            }
            cur = best.front();
            chain.push_back(cur);
            left.erase(std::find(left.begin(), left.end(), cur));
        }
        return chain;
    }

    /// Row offsets and order of buffer bi from its span chain.
    void lay_out(size_t bi) {
        BufferDesc& d = ba_.buffers[bi];
        d.order.clear();
        int row = 0;
        for (int si : bufs_[bi].chain)
            for (int s : bufs_[bi].spans[si].sigs) {
                d.order.push_back(s);
                ba_.row_offset[s] = row;
                row += sig_[s].rows();
            }
    }

    /// Alg. 2: visiting read blocks from smallest to largest, put each group's
    /// members in the order their reads sit in memory, then order each span's
    /// signals by the first member reading them; up to 10 rounds, until stable.
    void align() {
        std::vector<int> visit(blocks_.size());
        std::iota(visit.begin(), visit.end(), 0);
        std::sort(visit.begin(), visit.end(),
                  [&](int l, int r) { return size_[l] != size_[r] ? size_[l] < size_[r] : l < r; });
        std::vector<int> first_reader(ba_.buffer_of.size(), -1);
        for (int round = 0; round < 10; ++round) {
            bool moved = false;
            for (int bid : visit) {
                moved |= sort_members(bid);
                for (int cid : of_group_[blocks_[bid].group]) moved |= sort_span_signals(cid, first_reader);
            }
            if (!moved) break;
        }
    }

    /// Members of block bid's group in ascending order of the rows bid reads
    /// (stable); every block of the group follows the permutation.
    bool sort_members(int bid) {
        const ReadBlock& b = blocks_[bid];
        const size_t k = b.refs.size();
        std::vector<int> perm(k);
        std::iota(perm.begin(), perm.end(), 0);
        std::stable_sort(perm.begin(), perm.end(), [&](int l, int r) {
            return first_row_of(ba_, b.refs[l]) < first_row_of(ba_, b.refs[r]);
        });
        if (std::is_sorted(perm.begin(), perm.end())) return false;
        OpGroup& g = plan_[b.group];
        auto apply = [&](auto& v) {
            std::remove_reference_t<decltype(v)> out;
            out.reserve(k);
            for (int i : perm) out.push_back(v[i]);
            v = std::move(out);
        };
        apply(g.members);
        for (int cid : of_group_[b.group]) apply(blocks_[cid].refs);
        return true;
    }

    /// Signals of the spans block cid reads, ordered by the first member of its
    /// group that reads them (signals it does not read keep their place in front).
    bool sort_span_signals(int cid, std::vector<int>& first_reader) {
        const ReadBlock& c = blocks_[cid];
        for (int m = 0; m < static_cast<int>(c.refs.size()); ++m)
            if (first_reader[c.refs[m].signal] == -1) first_reader[c.refs[m].signal] = m;
        bool moved = false;
        for (Span& sp : bufs_[c.buffer].spans) {
            if (!sp.reads(cid)) continue;
            std::vector<int> next = sp.sigs;
            std::stable_sort(next.begin(), next.end(),
                             [&](int l, int r) { return first_reader[l] < first_reader[r]; });
            if (next != sp.sigs) {
                sp.sigs.swap(next);
                moved = true;
            }
        }
        for (const SignalRef& r : c.refs) first_reader[r.signal] = -1;
        if (moved) lay_out(c.buffer);
        return moved;
    }

    const std::vector<Signal>& sig_;
    Plan& plan_;
    BufferAssignment& ba_;
    std::vector<ReadBlock>& blocks_;
    size_t nbuf_;
    std::vector<int> size_;                    // rows of each read block
    std::vector<std::vector<int>> of_buffer_;  // read blocks per buffer
    std::vector<std::vector<int>> of_group_;   // read blocks per plan group
    std::vector<Buf> bufs_;
};

}  // namespace

void sort_buffers(const std::vector<Signal>& signals, Plan& plan, BufferAssignment& buffers,
                  std::vector<ReadBlock>& blocks) {
    LayoutSorter(signals, plan, buffers, blocks).run();
}

ContiguityStats contiguity_stats(const std::vector<ReadBlock>& blocks, const BufferAssignment& buffers,
                                 const Plan& plan) {
    ContiguityStats st;
    st.groups_per_step = static_cast<int>(plan.size());
    if (blocks.empty()) return st;
    auto contiguous = [&](const ReadBlock& b) {
        for (size_t m = 1; m < b.refs.size(); ++m) {
            const SignalRef& prev = b.refs[m - 1];
            if (first_row_of(buffers, b.refs[m]) != first_row_of(buffers, prev) + prev.rows()) return false;
        }
        return true;
    };
    int ok = 0;
    for (const ReadBlock& b : blocks) {
        if (contiguous(b))
            ++ok;
        else
            st.gather_row_count += b.total_rows();
    }
    st.contiguous_read_fraction = static_cast<double>(ok) / static_cast<double>(blocks.size());
    return st;
}

}  // namespace nengb
