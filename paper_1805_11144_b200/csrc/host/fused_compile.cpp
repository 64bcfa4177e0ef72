// fused_compile.cpp — recognise an ensemble network in a PlannedModel and
// compile it to the fused two-phase pipeline (kernels/fused.cu).
//
// Recognised structure (the reference frontend's lowering, frontend.cpp:305-517,
// in the unfolded form of SURVEY §8(d)):
//   ensemble   Reset(in), Reset(J, bias), DotInc(E, in, J), SimNeurons(LIF, J, out, [v, r]),
//              Reset(xhat), DotInc(D, out, xhat)
//   connection Reset(acc), DotInc(T, src, acc), SimProcess(tau > 0, acc, filt, state),
//              optionally Copy(filt -> in_dst, inc)          src = an ensemble's xhat or a fed node
//   clock      TimeUpdate(step, time)
// with no other accessor of any of these signals, every operand a full-signal
// ref, every state per-batch and every weight a shared constant.  Anything
// else returns nullptr and the engine keeps the generic interpreter.
//
// Why the two-phase schedule is the reference's arithmetic: every ordering
// the plan imposes is a dependency edge (Set<Inc<Read<Update, ir.cpp:351-360)
// except the order of increments into one target, and the only target with
// several increments is `in`, whose Copy incs are summed in plan-group order
// here.  The Copy reads `filt` before the SimProcess updates it (Read->Update
// edge), so in(k) sums filt(k-1) == state(k-1); the connection DotInc reads
// xhat(k) after its decoder increment and the fed value of step k.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <random>
#include <sstream>
#include <unordered_map>

#include "../kernels/fused.hpp"
#include "engine.hpp"
#include "fused.hpp"

namespace nengb {

int fused_dmax_for(int d);
size_t fused_smem_bytes(const FusedProgram& p, int dmax);
cudaError_t launch_fused(const FusedProgram& p, int dmax, int grid, int k0, int k1, cudaStream_t stream);
cudaError_t launch_fused_small(const FusedProgram& p, int dmax, int k0, int k1, cudaStream_t stream);
cudaError_t launch_feed_projection(const FProj* proj, int nproj, const float* weights, const float* feed_data,
                                   const int64_t* feed_off, const int32_t* present, const float* arena, float* out,
                                   int n_steps, int k0, int k1, int B, cudaStream_t stream);
int fused_max_grid(const FusedProgram& p, int dmax, int device);

namespace {

struct Access {
    int op;  // index into model.operators
    int pos;
    AccessMode mode;
};

struct Fail {
    std::string why;
};

class FusedImpl : public FusedPlan {
  public:
    FusedProgram prog;
    int dmax = 8, grid = 1, steps_per_launch = 0;
    bool small = false;  // fused_small_kernel: the whole step on one CTA (programs too small to fill the GPU)
    DevMem d_ens, d_conns, d_incoming, d_orphans, d_my_conns, d_values, d_probes, d_feeds, d_call, d_prof, d_work, d_xbuf, d_df, d_proj, d_projw, d_projout;
    int n_proj = 0, proj_rows = 0;  // fed-node projections (FProj)
    std::vector<FProj> h_proj;
    std::string desc;

    FusedProgram call;  // the open call's program (begin .. step)

    void begin(int n_steps, const float* d_feed_data, const int64_t* feed_off, const int* present, float* d_ring,
               const int64_t* ring_off, cudaStream_t stream) override {
        // per-call tables: feed offsets, presence, ring offsets
        cuda_check(cudaStreamSynchronize(stream), "fused call tables");  // the previous call's tables are free
        // feed slots, then one slot per fed-node projection (computed per launch)
        const int nf0 = prog.n_feeds, nf = nf0 + n_proj, np = n_probe_total;
        const float* base = d_feed_data;
        if (n_proj) {
            d_projout.ensure(static_cast<size_t>(std::max(n_steps, 1)) * proj_rows * prog.batch * sizeof(float));
            if (!base) base = d_projout.as<float>();
        }
        std::vector<int64_t> offs(feed_off, feed_off + nf0);
        std::vector<int32_t> pres(present, present + nf0);
        for (int q = 0; q < n_proj; ++q) {
            offs.push_back((d_projout.as<float>() - base) + static_cast<int64_t>(h_proj[q].dd_prefix) * n_steps * prog.batch);
            pres.push_back(1);
        }
        std::vector<char> blob(static_cast<size_t>(nf) * 8 + static_cast<size_t>(np) * 8 + static_cast<size_t>(nf) * 4 + 64);
        std::memcpy(blob.data(), offs.data(), nf * 8);
        std::memcpy(blob.data() + nf * 8, ring_off, np * 8);
        std::memcpy(blob.data() + nf * 8 + np * 8, pres.data(), nf * 4);
        cuda_check(cudaStreamSynchronize(stream), "fused call tables");  // the previous call's tables are free
        d_call.ensure(blob.size());
        cuda_check(cudaMemcpyAsync(d_call.p, blob.data(), blob.size(), cudaMemcpyHostToDevice, stream), "fused call H2D");
        FusedProgram p = prog;
        p.feed_data = base;
        p.feed_off = d_call.as<int64_t>();
        p.ring_off = reinterpret_cast<const int64_t*>(d_call.as<char>() + nf * 8);
        p.feed_present = reinterpret_cast<const int32_t*>(d_call.as<char>() + nf * 8 + np * 8);
        p.ring = d_ring;
        p.call_steps = n_steps;
        p.prof = nullptr;
        if (std::getenv("NENG_FUSED_PROFILE") != nullptr) {
            d_prof.ensure((FS_COUNT + 4) * 8);
            cuda_check(cudaMemsetAsync(d_prof.p, 0, (FS_COUNT + 4) * 8, stream), "profile reset");
            p.prof = d_prof.as<unsigned long long>();
        }
        p.trace = nullptr;
        if (std::getenv("NENG_FUSED_TRACE") != nullptr) {  // fault localisation (-DNENG_FUSED_TRACE builds)
            const size_t words = static_cast<size_t>(grid) * 8 * 2;
            if (!trace_host) {
                cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&trace_host), words * 4, cudaHostAllocMapped),
                           "trace alloc");
                cuda_check(cudaHostGetDevicePointer(reinterpret_cast<void**>(&trace_dev), trace_host, 0), "trace map");
            }
            std::memset(trace_host, 0, words * 4);
            p.trace = trace_dev;
        }
        d_work.ensure(16 + static_cast<size_t>(units) * 4);
        sched = 0;
        p.work = d_work.as<int32_t>();
        p.done = p.work + 4;
        call = p;
    }

    void step(int k, int flags, cudaStream_t stream) override {
        launch(k, k < call.call_steps ? k + 1 : k, flags, stream);  // k == n_steps: the epilogue of step n - 1
    }

    void launch(int k0, int k1, int flags, cudaStream_t stream) override {
        FusedProgram p = call;
        p.dataflow = 0;  // stepped calls: one barrier per step (the host exchanges xhat between them)
        p.first_update = (flags & NENG_STEP_FIRST_UPDATE) ? 1 : 0;
        p.epilogue = (flags & NENG_STEP_EPILOGUE) ? 1 : 0;
        cuda_check(cudaMemsetAsync(d_work.p, 0, 8, stream), "fused work reset");
        sched |= small ? NENG_SCHED_FUSED_SMALL : NENG_SCHED_FUSED_STEPPED;
        project(p, k0, k1, stream);
        cuda_check(small ? launch_fused_small(p, dmax, k0, k1, stream) : launch_fused(p, dmax, grid, k0, k1, stream),
                   "fused kernel launch");
        trace_check(stream);
    }

    /// Steps [k0, k1) of the open call as one self-contained launch (the
    /// previous launch's epilogue did step k0-1's connection updates): the
    /// barrier-free schedule when the engine owns its xhat buffer, else one
    /// grid barrier per step.  run() and the chunked host-buffer path of
    /// Engine::run both advance through this.
    void launch_chunk(int k0, int k1, cudaStream_t stream) override {
        FusedProgram p = call;
        p.first_update = 0;
        p.epilogue = 1;
        p.dataflow = dataflow ? 1 : 0;
        cuda_check(cudaMemsetAsync(d_work.p, 0, dataflow ? 16 + static_cast<size_t>(units) * 4 : 8, stream),
                   "fused work reset");
        sched |= small ? NENG_SCHED_FUSED_SMALL : dataflow ? NENG_SCHED_FUSED_BARRIER_FREE : NENG_SCHED_FUSED_STEPPED;
        project(p, k0, k1, stream);
        cuda_check(small ? launch_fused_small(p, dmax, k0, k1, stream) : launch_fused(p, dmax, grid, k0, k1, stream),
                   "fused kernel launch");
        trace_check(stream);
    }

    int32_t* trace_host = nullptr;
    int32_t* trace_dev = nullptr;
    /// NENG_FUSED_TRACE: wait for the launch; on a fault print every warp's last checkpoint
    void trace_check(cudaStream_t stream) {
        if (!call.trace) return;
        if (cudaStreamSynchronize(stream) == cudaSuccess) return;
        for (int c = 0; c < grid; ++c) {
            std::fprintf(stderr, "[fused trace] cta %d:", c);
            for (int w = 0; w < 8; ++w)
                std::fprintf(stderr, " %d/%d", trace_host[2 * (c * 8 + w)], trace_host[2 * (c * 8 + w) + 1]);
            std::fprintf(stderr, "\n");
        }
    }

    /// the fed-node projections of steps [k0, k1) (before the launch that reads them)
    void project(const FusedProgram& p, int k0, int k1, cudaStream_t stream) {
        if (!n_proj) return;
        cuda_check(launch_feed_projection(d_proj.as<FProj>(), n_proj, d_projw.as<float>(), p.feed_data, p.feed_off,
                                          p.feed_present, p.arena, d_projout.as<float>(), p.call_steps, k0, k1,
                                          p.batch, stream),
                   "feed projection");
    }

    void xhat_layout(int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf) const override {
        if (xbuf_floats) *xbuf_floats = static_cast<int64_t>(2) * prog.xrows * prog.batch;
        if (rank_floats) *rank_floats = static_cast<int64_t>(xstride) * prog.batch;
        if (xbuf) *xbuf = prog.xbuf;
    }

    void set_xhat_buffer(float* d_buf) override {
        dataflow = false;  // a caller's buffer holds two parity slots
        prog.xbuf = d_buf;
        call.xbuf = d_buf;
    }

    int xstride = 0;  // parity-buffer rows per shard
    bool dataflow = false;  // barrier-free stepping in run() (unsharded, own xhat buffer)
    int units = 0;

    int64_t run(int n_steps, const float* d_feed_data, const int64_t* feed_off, const int* present, float* d_ring,
                const int64_t* ring_off, cudaStream_t stream) override {
        begin(n_steps, d_feed_data, feed_off, present, d_ring, ring_off, stream);
        int K = steps_per_launch > 0 ? steps_per_launch : n_steps;
        if (dataflow) K = std::max(1, std::min<int>(K, static_cast<int>((int64_t{1} << 30) / std::max(units, 1))));
        int64_t launches = 0;
        for (int k = 0; k < n_steps; k += K) {
            launch_chunk(k, std::min(n_steps, k + K), stream);
            ++launches;
        }
        cuda_check(cudaStreamSynchronize(stream), "fused run");  // call tables are reused next call
        if (call.prof) {
            unsigned long long h[FS_COUNT + 4];
            cuda_check(cudaMemcpy(h, d_prof.p, sizeof h, cudaMemcpyDeviceToHost), "profile D2H");
            static const char* names[FS_COUNT] = {"deferred", "in+conn", "sweep", "unit-barrier", "fixup",
                                                  "decode",   "barrier", "epilogue"};
            double tot = 0;
            for (int s = 0; s < FS_COUNT; ++s) tot += static_cast<double>(h[s]);
            std::fprintf(stderr, "[fused profile] %d steps, grid %d: per-step per-CTA us:", n_steps, grid);
            for (int s = 0; s < FS_COUNT; ++s)
                std::fprintf(stderr, " %s=%.1f", names[s], h[s] / 1e3 / grid / n_steps);
            std::fprintf(stderr, " (total %.1f)\n", tot / 1e3 / grid / n_steps);
            std::fprintf(stderr, "[fused profile] per step: queued transcendental lane evaluations %.0f, exact path %.0f\n",
                         double(h[FS_COUNT]) / n_steps, double(h[FS_COUNT + 1]) / n_steps);
        }
        return launches;
    }
    void materialize(cudaStream_t) override {}
    void load_from_arena(cudaStream_t) override {}
    std::string describe() const override { return desc; }
    int n_probe_total = 0;
};

/// Claim order for barrier-free stepping: a permutation of the ensembles such
/// that a source's position in step t is not within `window` (the units in
/// flight at once, with margin) of the end when its destination's position in
/// step t+1 comes up — the wait a unit would otherwise spend.  Random pair swaps
/// that do not increase the number of such edges (deterministic seed).
std::vector<int> dataflow_order(int n, const std::vector<std::vector<int>>& srcs,
                                const std::vector<std::vector<int>>& dsts, int window) {
    std::vector<int> order(n), pos(n);
    for (int i = 0; i < n; ++i) order[i] = pos[i] = i;
    const int thr = n - (window * 8 + 4) / 5;  // an edge s -> e is late when pos[s] - pos[e] > thr
    if (n < 4 || thr <= 0) return order;
    auto cost = [&](int x) {
        int c = 0;
        for (int s : srcs[x]) c += pos[s] - pos[x] > thr;
        for (int d : dsts[x]) c += pos[x] - pos[d] > thr;
        return c;
    };
    std::mt19937 rng(12345u);
    std::uniform_int_distribution<int> pick(0, n - 1);
    const int64_t iters = std::min<int64_t>(int64_t{40} * n, 400000);
    for (int64_t it = 0; it < iters; ++it) {
        const int a = pick(rng), b = pick(rng);
        if (a == b) continue;
        const int ea = order[a], eb = order[b];
        const int c0 = cost(ea) + cost(eb);
        pos[ea] = b;
        pos[eb] = a;
        if (cost(ea) + cost(eb) <= c0) {
            order[a] = eb;
            order[b] = ea;
        } else {
            pos[ea] = a;
            pos[eb] = b;
        }
    }
    return order;
}

bool is_full(const BuiltModel& m, const SignalRef& r) { return r.start == 0 && r.stop == m.signals[r.signal].rows(); }

}  // namespace

std::unique_ptr<FusedPlan> try_compile_fused(Engine& eng, std::string* why) {
    const PlannedModel& pm = eng.planned();
    const BuiltModel& m = pm.model;
    const auto& L = eng.layout();
    const int B = eng.batch();
    try {
        auto fail = [](const std::string& w) -> void { throw Fail{w}; };
        const int nops = static_cast<int>(m.operators.size());
        std::vector<std::vector<Access>> acc(m.signals.size());
        for (int i = 0; i < nops; ++i) {
            const Operator& op = m.operators[i];
            for (auto [pos, mode] : operand_modes(op)) {
                if (!is_full(m, op.operands[pos])) fail("operator " + std::to_string(op.id) + " uses a slice");
                acc[op.operands[pos].signal].push_back({i, pos, mode});
            }
        }
        std::unordered_map<int, int> group_of;  // op id -> plan group
        for (size_t g = 0; g < pm.plan.size(); ++g)
            for (int id : pm.plan[g].members) group_of[id] = static_cast<int>(g);
        std::vector<char> claimed(nops, 0);
        auto claim = [&](int i) {
            if (claimed[i]) fail("operator " + std::to_string(m.operators[i].id) + " has two roles");
            claimed[i] = 1;
        };
        auto per_batch = [&](int sig) { return L[pm.buffers.buffer_of[sig]].per_batch != 0; };
        auto need_pb = [&](int sig, const char* what) {
            if (!per_batch(sig)) fail(std::string(what) + " is not in per-batch storage");
        };
        auto need_shared_const = [&](int sig, const char* what) {
            if (per_batch(sig) || !m.signals[sig].constant) fail(std::string(what) + " is not a shared constant");
        };
        auto op_at = [&](const Access& a) -> const Operator& { return m.operators[a.op]; };
        // find the single Reset(Set) of a signal among its accessors
        auto find_reset = [&](int sig) -> int {
            int r = -1;
            for (const Access& a : acc[sig])
                if (op_at(a).kind == OpKind::Reset) {
                    if (r >= 0) fail("signal '" + m.signals[sig].label + "' has two resets");
                    r = a.op;
                }
            if (r < 0) fail("signal '" + m.signals[sig].label + "' has no reset");
            return r;
        };

        std::vector<float> values;
        auto push_values = [&](const std::vector<double>& v) {
            int off = static_cast<int>(values.size());
            for (double x : v) values.push_back(static_cast<float>(x));
            return off;
        };

        struct EnsInfo {
            int sn, enc, dec, rin, rj, rx;
            int in, j, out, v, r, xhat, E, D;
            std::vector<std::pair<int, int>> incs;  // (group, copy op index)
        };
        std::vector<EnsInfo> ens;
        std::unordered_map<int, int> ens_of_in, ens_of_xhat;
        std::unordered_map<int, std::pair<int, int>> ens_state_of;  // neuron signal -> (ensemble, FStateCap)
        for (int i = 0; i < nops; ++i) {
            const Operator& op = m.operators[i];
            if (op.kind != OpKind::SimNeurons) continue;
            if (op.neuron.kind != NeuronKind::LIF) fail("non-LIF neurons");
            EnsInfo e{};
            e.sn = i;
            e.j = op.operands[0].signal;
            e.out = op.operands[1].signal;
            e.v = op.operands[2].signal;
            e.r = op.operands[3].signal;
            for (int s : {e.j, e.out, e.v, e.r}) need_pb(s, "ensemble state");
            for (int s : {e.v, e.r})
                if (acc[s].size() != 1) fail("voltage/refractory has other accessors");
            // J: Reset + DotInc(E, in, J) + this SimNeurons
            if (acc[e.j].size() != 3) fail("J has extra accessors");
            e.rj = find_reset(e.j);
            e.enc = -1;
            for (const Access& a : acc[e.j])
                if (op_at(a).kind == OpKind::DotInc && a.pos == 2) e.enc = a.op;
            if (e.enc < 0) fail("J has no encoder");
            const Operator& enc = m.operators[e.enc];
            e.E = enc.operands[0].signal;
            e.in = enc.operands[1].signal;
            need_shared_const(e.E, "encoders");
            need_pb(e.in, "ensemble input");
            // in: Reset + Copy incs + the encoder read
            e.rin = find_reset(e.in);
            for (const Access& a : acc[e.in]) {
                const Operator& o = op_at(a);
                if (a.op == e.rin || a.op == e.enc) continue;
                if (o.kind == OpKind::Copy && o.inc && a.pos == 1)
                    e.incs.push_back({group_of.at(o.id), a.op});
                else
                    fail("ensemble input has an unsupported accessor");
            }
            // out: this SimNeurons + one decoder DotInc
            if (acc[e.out].size() != 2) fail("neuron output has extra readers");
            e.dec = -1;
            for (const Access& a : acc[e.out])
                if (op_at(a).kind == OpKind::DotInc && a.pos == 1) e.dec = a.op;
            if (e.dec < 0) fail("neuron output has no decoder");
            const Operator& dec = m.operators[e.dec];
            e.D = dec.operands[0].signal;
            e.xhat = dec.operands[2].signal;
            need_shared_const(e.D, "decoders");
            need_pb(e.xhat, "decoded value");
            e.rx = find_reset(e.xhat);
            for (const Access& a : acc[e.xhat]) {
                const Operator& o = op_at(a);
                if (a.op == e.rx || a.op == e.dec) continue;
                if (!(o.kind == OpKind::DotInc && a.pos == 1)) fail("decoded value has an unsupported accessor");
            }
            const Signal& Es = m.signals[e.E];
            const Signal& Ds = m.signals[e.D];
            int n = m.signals[e.j].rows(), d = m.signals[e.in].rows();
            if (Es.shape.size() != 2 || Es.shape[0] != n || Es.shape[1] != d) fail("encoder shape");
            if (Ds.shape.size() != 2 || Ds.shape[1] != n) fail("decoder shape");
            if (!fused_dmax_for(std::max(d, Ds.shape[0]))) fail("dimension above 32");
            for (double x : Ds.initial)
                if (!std::isfinite(static_cast<float>(x))) fail("non-finite decoder weight");
            for (int o : {e.sn, e.enc, e.dec, e.rin, e.rj, e.rx}) claim(o);
            ens_state_of[e.out] = {static_cast<int>(ens.size()), SC_OUT};
            ens_state_of[e.v] = {static_cast<int>(ens.size()), SC_VOLTAGE};
            ens_state_of[e.r] = {static_cast<int>(ens.size()), SC_REFRACTORY};
            ens_state_of[e.j] = {static_cast<int>(ens.size()), SC_J};
            ens_of_in[e.in] = static_cast<int>(ens.size());
            ens_of_xhat[e.xhat] = static_cast<int>(ens.size());
            ens.push_back(std::move(e));
        }
        if (ens.empty()) fail("no LIF ensembles");

        std::unordered_map<int, int> slot_of_sig;
        for (size_t f = 0; f < m.feed_slots.size(); ++f) slot_of_sig[m.feed_slots[f].signal] = static_cast<int>(f);

        struct ConnInfo {
            int dot, rst, sp, copy;
            int src, T, accs, filt, state;
            int dst_ens;
            bool proj;  // fed node wider than the fused rows: projected ahead of the kernel (FProj)
        };
        std::vector<ConnInfo> conns;
        std::unordered_map<int, int> conn_of_copy, conn_of_filt, conn_of_state;
        for (int i = 0; i < nops; ++i) {
            const Operator& op = m.operators[i];
            if (op.kind != OpKind::DotInc || claimed[i]) continue;
            ConnInfo c{};
            c.dot = i;
            c.T = op.operands[0].signal;
            c.src = op.operands[1].signal;
            c.accs = op.operands[2].signal;
            need_shared_const(c.T, "transform");
            need_pb(c.accs, "connection accumulator");
            if (!ens_of_xhat.count(c.src)) {
                if (!slot_of_sig.count(c.src)) fail("connection source is neither a decoded value nor a fed node");
                need_pb(c.src, "fed node");
                for (const Access& a : acc[c.src])
                    if (!(op_at(a).kind == OpKind::DotInc && a.pos == 1)) fail("fed node has a writer or other reader");
            }
            if (acc[c.accs].size() != 3) fail("connection accumulator has extra accessors");
            c.rst = find_reset(c.accs);
            c.sp = -1;
            for (const Access& a : acc[c.accs])
                if (op_at(a).kind == OpKind::SimProcess && a.pos == 0) c.sp = a.op;
            if (c.sp < 0) fail("connection without a lowpass synapse");
            const Operator& sp = m.operators[c.sp];
            if (!(sp.tau > 0.0) || sp.operands.size() != 3) fail("passthrough synapse (tau = 0)");
            c.filt = sp.operands[1].signal;
            c.state = sp.operands[2].signal;
            need_pb(c.filt, "filtered value");
            need_pb(c.state, "filter state");
            if (acc[c.state].size() != 1) fail("filter state has other accessors");
            {
                const Signal& fs = m.signals[c.filt];
                const Signal& ss = m.signals[c.state];
                std::vector<double> fi = fs.initial, si = ss.initial;
                if (fi.empty()) fi.assign(fs.size(), 0.0);
                if (si.empty()) si.assign(ss.size(), 0.0);
                if (fi != si) fail("filtered value and filter state start differently");
            }
            c.copy = -1;
            c.dst_ens = -1;
            for (const Access& a : acc[c.filt]) {
                if (a.op == c.sp) continue;
                const Operator& o = op_at(a);
                if (o.kind == OpKind::Copy && a.pos == 0 && o.inc && ens_of_in.count(o.operands[1].signal) &&
                    c.copy < 0) {
                    c.copy = a.op;
                    c.dst_ens = ens_of_in[o.operands[1].signal];
                } else {
                    fail("filtered value has an unsupported reader");
                }
            }
            const Signal& Ts = m.signals[c.T];
            int dd = m.signals[c.accs].rows(), ds = m.signals[c.src].rows();
            if (Ts.shape.size() != 2 || Ts.shape[0] != dd || Ts.shape[1] != ds) fail("transform shape");
            c.proj = false;
            if (!fused_dmax_for(std::max(dd, ds))) {
                if (slot_of_sig.count(c.src) && fused_dmax_for(dd))
                    c.proj = true;
                else
                    fail("dimension above 32");
            }
            for (int o : {c.dot, c.rst, c.sp}) claim(o);
            if (c.copy >= 0) {
                claim(c.copy);
                conn_of_copy[c.copy] = static_cast<int>(conns.size());
            }
            conn_of_filt[c.filt] = static_cast<int>(conns.size());
            conn_of_state[c.state] = static_cast<int>(conns.size());
            conns.push_back(c);
        }
        int time_op = -1;
        for (int i = 0; i < nops; ++i) {
            const Operator& op = m.operators[i];
            if (op.kind == OpKind::TimeUpdate && !claimed[i]) {
                if (time_op >= 0) fail("two clocks");
                for (const SignalRef& r : op.operands) {
                    if (acc[r.signal].size() != (op.operands[0].signal == op.operands[1].signal ? 2u : 1u))
                        fail("clock signals have other accessors");
                    if (per_batch(r.signal)) fail("per-batch clock");
                }
                time_op = i;
                claim(i);
            }
        }
        for (int i = 0; i < nops; ++i)
            if (!claimed[i])
                fail("operator " + std::to_string(m.operators[i].id) + " (" + op_kind_name(m.operators[i].kind) +
                     ") is outside the ensemble pattern");
        for (const EnsInfo& e : ens)
            for (auto [g, ci] : e.incs)
                if (!conn_of_copy.count(ci)) fail("ensemble input increment is not a connection");

        // ---- descriptors -----------------------------------------------------
        auto impl = std::make_unique<FusedImpl>();
        FusedProgram& p = impl->prog;
        const float dt = static_cast<float>(m.dt);
        std::vector<FEns> fe;
        std::vector<int32_t> incoming, orphans, my_conns;
        int nmax = 0, dmax_need = 1, pmax_floats = 0, xrows = 0;
        for (const EnsInfo& e : ens)
            dmax_need = std::max({dmax_need, m.signals[e.in].rows(), m.signals[e.xhat].rows()});
        for (const ConnInfo& c : conns)
            dmax_need = std::max({dmax_need, m.signals[c.accs].rows(), c.proj ? 0 : m.signals[c.src].rows()});
        const int DMAX = fused_dmax_for(dmax_need);
        auto align4 = [&] {
            while (values.size() % 4) values.push_back(0.0f);
            return static_cast<int64_t>(values.size());
        };
        // ensemble sharding: shard s owns ensembles [lo_s, hi_s) and writes its
        // xhat rows at s * xstride of the parity buffers (in-place all-gather)
        const int W = eng.shard_count(), R = eng.shard_rank();
        const int n_all = static_cast<int>(ens.size());
        auto shard_lo = [&](int sidx) { return static_cast<int>(static_cast<int64_t>(sidx) * n_all / W); };
        int xstride = 0;
        for (int sidx = 0; sidx < W; ++sidx) {
            int rows = 0;
            for (int i = shard_lo(sidx); i < shard_lo(sidx + 1); ++i) rows += m.signals[ens[i].xhat].rows();
            xstride = std::max(xstride, rows);
        }
        const int ens_lo = shard_lo(R), ens_hi = shard_lo(R + 1);
        std::vector<int> shard_row(W, 0);
        int ens_index = 0;
        for (EnsInfo& e : ens) {
            const int my_shard = [&] {
                int sidx = 0;
                while (shard_lo(sidx + 1) <= ens_index) ++sidx;
                return sidx;
            }();
            ++ens_index;
            std::stable_sort(e.incs.begin(), e.incs.end());  // plan-group order of the Copy incs
            for (size_t q = 1; q < e.incs.size(); ++q)
                if (e.incs[q].first == e.incs[q - 1].first) fail("two increments of one input in one group");
            FEns x{};
            x.in_base = eng.resolve_full(e.in).base;
            x.j_base = eng.resolve_full(e.j).base;
            x.out_base = eng.resolve_full(e.out).base;
            x.v_base = eng.resolve_full(e.v).base;
            x.r_base = eng.resolve_full(e.r).base;
            x.xhat_base = eng.resolve_full(e.xhat).base;
            x.n = m.signals[e.j].rows();
            x.d = m.signals[e.in].rows();
            x.dx = m.signals[e.xhat].rows();
            x.inc_begin = static_cast<int32_t>(incoming.size());
            for (auto [g, ci] : e.incs) incoming.push_back(conn_of_copy.at(ci));
            x.inc_count = static_cast<int32_t>(e.incs.size());
            x.n_pad = (x.n + 3) / 4 * 4;
            x.bias_off = align4();
            push_values(m.operators[e.rj].value);
            while (static_cast<int64_t>(values.size()) < x.bias_off + x.n_pad) values.push_back(0.0f);
            {
                // encoder rows zero padded to DMAX (exact: see fused.cu), n rounded
                // up to even with a zero row (phase A takes neurons in pairs)
                const Signal& Es = m.signals[e.E];
                x.epad_off = align4();
                // neuron pairs interleaved, [i / 2][j][i % 2]: the sweep sums two neurons side by side
                const int n2 = (x.n + 1) & ~1;
                for (int i2 = 0; i2 < n2; i2 += 2)
                    for (int jj = 0; jj < DMAX; ++jj)
                        for (int ii = i2; ii < i2 + 2; ++ii)
                            values.push_back(ii < x.n && jj < x.d && !Es.initial.empty()
                                                 ? static_cast<float>(Es.initial[static_cast<size_t>(ii) * x.d + jj])
                                                 : 0.0f);
            }
            x.in_init_off = push_values(m.operators[e.rin].value);
            x.xhat_init_off = push_values(m.operators[e.rx].value);
            x.xb_row = my_shard * xstride + shard_row[my_shard];
            shard_row[my_shard] += x.dx;
            const NeuronModel& nm = m.operators[e.sn].neuron;
            x.dt = dt;
            x.tau_rc = static_cast<float>(nm.tau_rc);
            x.tau_ref = static_cast<float>(nm.tau_ref);
            x.amplitude = static_cast<float>(nm.amplitude);
            volatile float num = x.amplitude, den = x.dt;  // float division, as amplitude / dt in T
            x.amp_dt = num / den;
            volatile float mdt = -x.dt, trc = x.tau_rc;
            float arg = mdt / trc;
            x.em_dt = expm1f(arg);  // the host libm result the reference uses
            x.inv_tau_rc = 1.0 / static_cast<double>(x.tau_rc);
            {
                // spike products fp32(D[r,i]) * amp_dt: the DotInc term for out[i] = amp/dt
                const Signal& Ds = m.signals[e.D];
                x.dec_scaled_off = align4();
                x.dec_bytes = (x.n * x.dx * 4 + 15) / 16 * 16;
                pmax_floats = std::max(pmax_floats, x.dec_bytes / 4);
                for (int ii = 0; ii < x.n; ++ii)  // transposed: [n][dx]
                    for (int rr = 0; rr < x.dx; ++rr) {
                        double dv = Ds.initial.empty() ? 0.0 : Ds.initial[static_cast<size_t>(rr) * x.n + ii];
                        volatile float w = static_cast<float>(dv);
                        values.push_back(w * x.amp_dt);
                    }
            }
            nmax = std::max(nmax, x.n);
            dmax_need = std::max({dmax_need, x.d, x.dx});
            fe.push_back(x);
        }
        xrows = W * xstride;
        {
            // a unit applies its incoming connections one after another (a chain of
            // dependent loads); past this fan-in the generic executor is faster
            // (config 1's 132-way inverse DFT: 2.6 vs 0.6 ms/step), so AUTO keeps it
            int fan_in = 0;
            for (const FEns& x : fe) fan_in = std::max(fan_in, x.inc_count);
            if (fan_in > 64 && eng.requested_mode() == NENG_MODE_AUTO && W == 1)
                fail("fan-in " + std::to_string(fan_in) + " above 64 (the generic executor is faster)");
            // programs too small to fill the GPU (fewer than 4 units per step, or batch
            // columns that leave most lanes of a tile idle) run the whole step on one
            // CTA with lanes over neurons (fused_small_kernel; config 0, one ensemble at
            // B=1: the multi-CTA pipeline took 113 us/step, the interpreter 29.5)
            const int64_t step_units = static_cast<int64_t>(fe.size()) * ((B + 255) / 256);
            int64_t neuron_cols = 0, words = 0;
            for (const FEns& x : fe) {
                neuron_cols += static_cast<int64_t>(x.n) * B;
                words += static_cast<int64_t>((x.n + 31) / 32) * B;
            }
            int64_t pfloats = 0;
            for (const FEns& x : fe) pfloats += static_cast<int64_t>(x.n) * x.dx;
            const char* se = std::getenv("NENG_FUSED_SMALL");  // 0: never, 1: whenever it fits
            int64_t nmax_cols = 0;  // the decode's index lists: (nmax rounded to 32 + 1) x B ints
            for (const FEns& x : fe) nmax_cols = std::max<int64_t>(nmax_cols, (static_cast<int64_t>(x.n) + 31) / 32 * 32);
            const int64_t fixed = words + (nmax_cols + 1) * B;
            const bool fits = W == 1 && fixed * 4 <= 200 * 1024;
            p.small_pfloats = (fixed + pfloats) * 4 <= 200 * 1024 ? static_cast<int32_t>(pfloats) : 0;
            impl->small = fits && (se ? std::atoi(se) != 0
                                      : (step_units < 4 || B < 32) && neuron_cols <= 65536);
            p.small_words = static_cast<int32_t>(words);
            if (step_units < 4 && !impl->small && eng.requested_mode() == NENG_MODE_AUTO && W == 1)
                fail("only " + std::to_string(step_units) + " unit(s) per step (the generic executor is faster)");
        }
        std::vector<FConn> fc;
        std::vector<FProj> projs;
        std::vector<float> proj_w;
        int proj_rows = 0;
        for (const ConnInfo& c : conns) {
            FConn x{};
            x.src_base = eng.resolve_full(c.src).base;
            x.acc_base = eng.resolve_full(c.accs).base;
            x.filt_base = eng.resolve_full(c.filt).base;
            x.state_base = eng.resolve_full(c.state).base;
            x.dd = m.signals[c.accs].rows();
            x.ds = m.signals[c.src].rows();
            x.src_feed = -1;
            x.src_xb = ens_of_xhat.count(c.src) ? fe[ens_of_xhat.at(c.src)].xb_row : -1;
            x.src_ens = ens_of_xhat.count(c.src) ? ens_of_xhat.at(c.src) : -1;
            if (c.dst_ens < 0) orphans.push_back(static_cast<int32_t>(fc.size()));
            if ((c.dst_ens < 0 && R == 0) || (c.dst_ens >= ens_lo && c.dst_ens < ens_hi))
                my_conns.push_back(static_cast<int32_t>(fc.size()));
            if (slot_of_sig.count(c.src)) {
                x.src_feed = slot_of_sig[c.src];
                if (m.feed_slots[x.src_feed].dim != x.ds) fail("feed slot dim differs from its signal");
            }
            x.acc_init_off = push_values(m.operators[c.rst].value);
            if (c.proj) {
                // T . u computed ahead of the kernel into projection slot n_feeds + q; the
                // connection reads it through an identity transform (see FProj)
                const Signal& Ts = m.signals[c.T];
                FProj pj{};
                pj.t_off = static_cast<int64_t>(proj_w.size());
                for (size_t i = 0; i < static_cast<size_t>(x.dd) * x.ds; ++i)
                    proj_w.push_back(Ts.initial.empty() ? 0.0f : static_cast<float>(Ts.initial[i]));
                pj.node_base = x.src_base;
                pj.slot = x.src_feed;
                pj.dd = x.dd;
                pj.ds = x.ds;
                pj.copies = per_batch(c.src) ? B : 1;
                pj.dd_prefix = proj_rows;
                proj_rows += x.dd;
                x.src_feed = static_cast<int32_t>(m.feed_slots.size() + projs.size());
                projs.push_back(pj);
                x.ds = x.dd;
                x.tpad_off = align4();
                for (int rr = 0; rr < x.dd; ++rr)
                    for (int jj = 0; jj < DMAX; ++jj) values.push_back(jj == rr ? 1.0f : 0.0f);
            } else {
                const Signal& Ts = m.signals[c.T];
                x.tpad_off = align4();
                for (int rr = 0; rr < x.dd; ++rr)
                    for (int jj = 0; jj < DMAX; ++jj)
                        values.push_back(jj < x.ds && !Ts.initial.empty()
                                             ? static_cast<float>(Ts.initial[static_cast<size_t>(rr) * x.ds + jj])
                                             : 0.0f);
            }
            const Operator& sp = m.operators[c.sp];
            double a = std::exp(-m.dt / sp.tau);  // lowpass_coefficients (neuron_math.hpp:33-37)
            x.a = static_cast<float>(a);
            x.b = static_cast<float>(1.0 - a);
            x.probe_filt = x.probe_state = -1;
            dmax_need = std::max({dmax_need, x.dd, x.ds});
            fc.push_back(x);
        }
        // probes
        std::vector<FProbe> fp;
        std::vector<int> fp_ens;  // producing ensemble of each capture (-1: a fed node)
        std::vector<std::vector<std::pair<int32_t, int32_t>>> scaps_of(fe.size());  // per ensemble (kind, probe)
        p.time_probe_step = p.time_probe_time = -1;
        for (size_t q = 0; q < m.probes.size(); ++q) {
            int s = m.probes[q].signal;
            if (ens_of_xhat.count(s) || slot_of_sig.count(s)) {
                FProbe pr{};
                pr.base = eng.resolve_full(s).base;
                pr.dim = static_cast<int32_t>(m.signals[s].size());
                pr.per_batch = per_batch(s);
                pr.index = static_cast<int32_t>(q);
                pr.feed_slot = slot_of_sig.count(s) ? slot_of_sig[s] : -1;
                pr.xb_row = ens_of_xhat.count(s) ? fe[ens_of_xhat.at(s)].xb_row : -1;
                if (pr.feed_slot >= 0 && m.feed_slots[pr.feed_slot].dim != pr.dim)
                    fail("feed slot dim differs from its signal");
                // captured by the shard that produces the value (fed nodes: shard 0)
                const bool mine = ens_of_xhat.count(s) ? (ens_of_xhat.at(s) >= ens_lo && ens_of_xhat.at(s) < ens_hi)
                                                       : R == 0;
                if (mine) {
                    fp.push_back(pr);
                    fp_ens.push_back(ens_of_xhat.count(s) ? ens_of_xhat.at(s) : -1);
                }
            } else if (ens_state_of.count(s)) {
                const auto [ei, kind] = ens_state_of.at(s);
                scaps_of[ei].push_back({kind, static_cast<int32_t>(q)});  // captured by the unit stepping it
            } else if (conn_of_filt.count(s)) {
                FConn& x = fc[conn_of_filt[s]];
                if (x.probe_filt >= 0) fail("two probes on one filtered value");
                x.probe_filt = static_cast<int32_t>(q);
            } else if (conn_of_state.count(s)) {
                FConn& x = fc[conn_of_state[s]];
                if (x.probe_state >= 0) fail("two probes on one filter state");
                x.probe_state = static_cast<int32_t>(q);
            } else if (time_op >= 0 && s == m.operators[time_op].operands[0].signal && p.time_probe_step < 0) {
                p.time_probe_step = static_cast<int32_t>(q);
            } else if (time_op >= 0 && s == m.operators[time_op].operands[1].signal && p.time_probe_time < 0) {
                p.time_probe_time = static_cast<int32_t>(q);
            } else {
                fail("probe on '" + m.signals[s].label + "' (an on-chip intermediate)");
            }
        }
        std::vector<FFeed> ff;
        for (size_t f = 0; f < m.feed_slots.size(); ++f) {
            FFeed x{};
            x.base = eng.resolve_full(m.feed_slots[f].signal).base;
            x.dim = m.feed_slots[f].dim;
            x.copies = per_batch(m.feed_slots[f].signal) ? B : 1;
            x.slot = static_cast<int32_t>(f);
            ff.push_back(x);
        }

        // barrier-free stepping tables: per-ensemble waits, destination-less
        // connections by source, xhat captures; the epilogue's connections
        std::vector<int32_t> df_deps, df_orph, df_free, df_xp, df_dest, sc_flat;
        std::vector<std::vector<int>> ens_srcs(fe.size()), ens_dsts(fe.size());
        {
            std::vector<std::vector<int>> orph(fe.size()), xps(fe.size());
            for (size_t ci = 0; ci < conns.size(); ++ci) {
                const ConnInfo& c = conns[ci];
                const int s = ens_of_xhat.count(c.src) ? ens_of_xhat.at(c.src) : -1;
                if (c.dst_ens >= 0) {
                    df_dest.push_back(static_cast<int32_t>(ci));
                    if (s >= 0) {
                        ens_srcs[c.dst_ens].push_back(s);
                        ens_dsts[s].push_back(c.dst_ens);
                    }
                } else if (s >= 0) {
                    orph[s].push_back(static_cast<int>(ci));
                } else {
                    df_free.push_back(static_cast<int32_t>(ci));
                }
            }
            for (size_t q = 0; q < fp.size(); ++q)
                if (fp_ens[q] >= 0) xps[fp_ens[q]].push_back(static_cast<int>(q));
            for (size_t e = 0; e < fe.size(); ++e) {
                std::vector<int> pre = ens_srcs[e];
                pre.push_back(static_cast<int>(e));
                std::sort(pre.begin(), pre.end());
                pre.erase(std::unique(pre.begin(), pre.end()), pre.end());
                std::vector<int> post = ens_dsts[e];
                std::sort(post.begin(), post.end());
                post.erase(std::unique(post.begin(), post.end()), post.end());
                fe[e].dep_begin = static_cast<int32_t>(df_deps.size());
                for (int x : pre) df_deps.push_back(x << 1);
                for (int x : post)
                    if (!std::binary_search(pre.begin(), pre.end(), x)) df_deps.push_back((x << 1) | 1);
                fe[e].dep_count = static_cast<int32_t>(df_deps.size()) - fe[e].dep_begin;
                fe[e].orph_begin = static_cast<int32_t>(df_orph.size());
                for (int c : orph[e]) df_orph.push_back(c);
                fe[e].orph_count = static_cast<int32_t>(orph[e].size());
                fe[e].xp_begin = static_cast<int32_t>(df_xp.size());
                for (int q : xps[e]) df_xp.push_back(q);
                fe[e].xp_count = static_cast<int32_t>(xps[e].size());
                fe[e].sc_begin = static_cast<int32_t>(sc_flat.size() / 2);
                for (auto [kind, q] : scaps_of[e]) {
                    sc_flat.push_back(kind);
                    sc_flat.push_back(q);
                }
                fe[e].sc_count = static_cast<int32_t>(scaps_of[e].size());
            }
        }

        auto upload = [](DevMem& d, const void* src, size_t bytes) {
            d.ensure(std::max<size_t>(bytes, 16));
            if (bytes) cuda_check(cudaMemcpy(d.p, src, bytes, cudaMemcpyHostToDevice), "fused H2D");
        };
        upload(impl->d_ens, fe.data(), fe.size() * sizeof(FEns));
        upload(impl->d_conns, fc.data(), fc.size() * sizeof(FConn));
        upload(impl->d_incoming, incoming.data(), incoming.size() * sizeof(int32_t));
        upload(impl->d_orphans, orphans.data(), orphans.size() * sizeof(int32_t));
        // three slots: parity with a barrier per step, k % 3 barrier-free
        impl->d_xbuf.ensure(static_cast<size_t>(3) * std::max(xrows, 1) * B * sizeof(float));
        cuda_check(cudaMemset(impl->d_xbuf.p, 0, static_cast<size_t>(3) * std::max(xrows, 1) * B * sizeof(float)),
                   "xbuf clear");
        upload(impl->d_values, values.data(), values.size() * sizeof(float));
        upload(impl->d_probes, fp.data(), fp.size() * sizeof(FProbe));
        upload(impl->d_feeds, ff.data(), ff.size() * sizeof(FFeed));
        upload(impl->d_proj, projs.data(), projs.size() * sizeof(FProj));
        upload(impl->d_projw, proj_w.data(), proj_w.size() * sizeof(float));
        impl->n_proj = static_cast<int>(projs.size());
        impl->h_proj = projs;
        impl->proj_rows = proj_rows;
        p.arena = eng.arena();
        p.values = impl->d_values.as<float>();
        p.ens = impl->d_ens.as<FEns>();
        p.conns = impl->d_conns.as<FConn>();
        p.incoming = impl->d_incoming.as<int32_t>();
        p.orphans = impl->d_orphans.as<int32_t>();
        p.xbuf = impl->d_xbuf.as<float>();
        p.xrows = xrows;
        p.n_orphans = R == 0 ? static_cast<int32_t>(orphans.size()) : 0;
        upload(impl->d_my_conns, my_conns.data(), my_conns.size() * sizeof(int32_t));
        p.my_conns = impl->d_my_conns.as<int32_t>();
        p.n_my_conns = static_cast<int32_t>(my_conns.size());
        p.ens_lo = ens_lo;
        p.ens_hi = ens_hi;
        impl->xstride = xstride;
        if (R != 0) p.time_probe_step = p.time_probe_time = -1;  // the clock's captures live on shard 0
        p.probes = impl->d_probes.as<FProbe>();
        p.feeds = impl->d_feeds.as<FFeed>();
        p.n_ens = static_cast<int32_t>(fe.size());
        p.n_conn = static_cast<int32_t>(fc.size());
        p.n_probes = static_cast<int32_t>(fp.size());
        p.n_feeds = static_cast<int32_t>(ff.size());
        p.batch = B;
        p.btiles = (B + 31) / 32;
        p.nmax = (nmax + 31) / 32 * 32;
        p.pmax_floats = pmax_floats;
        p.libm = libm_tables(eng.device());
        // tiles per unit (one warp each) and warps per tile (neuron slices)
        {
            int tu = 1, tu_max = 8;
            if (const char* env = std::getenv("NENG_FUSED_TILES_PER_UNIT")) tu_max = std::max(1, std::min(8, std::atoi(env)));
            while (tu < tu_max && tu < p.btiles) tu *= 2;
            p.tu = tu;
            p.slices = 8 / tu;
            p.groups = (p.btiles + tu - 1) / tu;
        }
        // stage the decoder products with the encoders (else they replace the encoders
        // after the sweep) when that keeps as many CTAs per SM (at most 3: the register
        // budget); config 2's 1024-neuron ensembles: 2 CTAs/SM late vs 1 staged, +17%
        {
            auto per_sm = [](size_t b) { return std::min<size_t>(3, (228 * 1024) / (b + 1024)); };
            p.stage_dec = 1;
            const size_t with = fused_smem_bytes(p, DMAX);
            p.stage_dec = 0;
            const size_t without = fused_smem_bytes(p, DMAX);
            p.stage_dec = (with <= 227 * 1024 && per_sm(with) >= per_sm(without)) ? 1 : 0;
            if (const char* env = std::getenv("NENG_FUSED_STAGE_DEC")) p.stage_dec = std::atoi(env) ? 1 : 0;  // experiments
        }
        p.dt = dt;
        if (time_op >= 0) {
            p.has_time = 1;
            p.step_base = eng.resolve_full(m.operators[time_op].operands[0].signal).base;
            p.time_base = eng.resolve_full(m.operators[time_op].operands[1].signal).base;
        }
        impl->steps_per_launch = eng.steps_per_launch();
        impl->n_probe_total = static_cast<int>(m.probes.size());
        impl->dmax = fused_dmax_for(dmax_need);
        int cap = fused_max_grid(p, impl->dmax, eng.device());
        if (cap <= 0) fail("fused kernel does not fit on the device");
        int64_t work = std::max<int64_t>(static_cast<int64_t>(ens_hi - ens_lo) * p.groups,
                                         (static_cast<int64_t>(p.n_conn) * B + 255) / 256);
        impl->grid = static_cast<int>(std::min<int64_t>(cap, std::max<int64_t>(1, work)));
        if (const char* env = std::getenv("NENG_FUSED_GRID"))  // experiments: co-resident CTAs (<= cap)
            impl->grid = std::max(1, std::min(cap, std::atoi(env)));

        // barrier-free stepping (unsharded): claim order of the units
        impl->units = (ens_hi - ens_lo) * p.groups;
        const char* dfe = std::getenv("NENG_FUSED_DATAFLOW");
        impl->dataflow = W == 1 && !(dfe && std::atoi(dfe) == 0) && !impl->small;
        if (impl->small) impl->grid = 1;
        {
            const int NE = static_cast<int>(fe.size());
            const int window = (impl->grid + p.groups - 1) / p.groups;  // ensembles in flight at once
            std::vector<int> perm = dataflow_order(NE, ens_srcs, ens_dsts, window);
            std::vector<int32_t> order;
            if (W == 1)
                for (int e : perm)
                    for (int g = 0; g < p.groups; ++g) order.push_back(e * p.groups + g);
            const size_t n_order = order.size(), n_deps = df_deps.size(), n_orph = df_orph.size(),
                         n_xp = df_xp.size(), n_free = df_free.size();
            std::vector<int32_t> blob;
            // the (kind, probe) pairs first: int2 loads need 8-B alignment
            for (auto* v : {&sc_flat, &order, &df_deps, &df_orph, &df_xp, &df_free, &df_dest})
                blob.insert(blob.end(), v->begin(), v->end());
            upload(impl->d_df, blob.data(), blob.size() * sizeof(int32_t));
            const int32_t* base = impl->d_df.as<int32_t>();
            p.scaps = base;
            base += sc_flat.size();
            p.order = base;
            p.deps = base + n_order;
            p.ens_orph = p.deps + n_deps;
            p.xprobes = p.ens_orph + n_orph;
            p.free_orph = p.xprobes + n_xp;
            p.n_free_orph = static_cast<int32_t>(n_free);
            p.dest_conns = p.free_orph + n_free;
            p.n_dest_conns = static_cast<int32_t>(df_dest.size());
            upload(impl->d_ens, fe.data(), fe.size() * sizeof(FEns));  // with the dep / orphan / capture ranges
        }

        std::ostringstream os;
        os << "fused: " << p.n_ens << " ensembles, " << p.n_conn << " connections, dmax " << impl->dmax << ", grid "
           << impl->grid << ", tiles/unit " << p.tu << ", slices " << p.slices << ", stage_dec " << p.stage_dec
           << ", smem " << fused_smem_bytes(p, impl->dmax) << (impl->dataflow ? ", barrier-free" : "")
           << (impl->small ? ", small (one CTA, lanes over neurons)" : "");
        impl->desc = os.str();
        return impl;
    } catch (const Fail& f) {
        if (why) *why = f.why;
        return nullptr;
    }
}

}  // namespace nengb
