// test_drop_in.cpp — the reference's EngineCore<float> and neng::gpu::GpuEngine
// (include/neng_gpu_engine.hpp) driven side by side through the reference's
// own C++ API, in one process.  Built by oracle/Makefile (target `dropin`)
// against the reference's unchanged sources; run by tests/test_drop_in.py on
// the GPU box.  Exit 0 = every check bit-exact.
//
// Model: the §8(d) ensemble lowering (frontend.cpp:305-341, 419-517) built
// directly with the reference IR — per ensemble Reset(in), Reset(J, bias),
// DotInc(E, in, J), SimNeurons(LIF, J, out, [v, r]), Reset(xhat), DotInc(D,
// out, xhat); per connection Reset(acc), DotInc(T, src, acc),
// SimProcess(tau, acc, filt, state), Copy(filt -> in_dst, inc); fed input
// nodes; a TimeUpdate; probes on xhat, a filtered value and the clock.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "neng_gpu_engine.hpp"
#include "nengine/exec.hpp"
#include "nengine/passes.hpp"

using namespace neng;

namespace {

int g_checks = 0, g_failed = 0;

void expect(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        ++g_failed;
        std::fprintf(stderr, "FAIL: %s\n", what.c_str());
    }
}

void expect_same(const std::string& ref, const std::string& gpu, const std::string& what) {
    expect(ref == gpu, what + " (reference \"" + ref + "\", gpu \"" + gpu + "\")");
}

struct Builder {
    BuiltModel m;
    int next_op = 0;

    SignalId signal(const std::string& label, std::vector<int> shape, std::vector<double> init, bool minibatched,
                    bool constant = false) {
        Signal s;
        s.id = static_cast<SignalId>(m.signals.size());
        s.label = label;
        s.shape = std::move(shape);
        s.elem = Elem::f32;
        s.initial = std::move(init);
        s.minibatched = minibatched;
        s.constant = constant;
        m.signals.push_back(s);
        return s.id;
    }
    SignalRef full(SignalId s) const { return SignalRef::full(m.signals[s]); }
    void op(Operator o) { m.operators.push_back(std::move(o)); }
    int id() { return next_op++; }
};

struct Net {
    PlannedModel planned;
    std::vector<int> fed_nodes;
    std::vector<int> fed_dims;
    std::vector<SignalId> voltages;
};

Net build_network(unsigned seed, int n_ens, int n, int d, int k_out, int n_inputs) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    std::uniform_real_distribution<double> uni(0.0, 1.0);
    Builder b;
    Net net;
    std::vector<SignalId> in(n_ens), xhat(n_ens);
    for (int e = 0; e < n_ens; ++e) {
        const std::string p = "ens" + std::to_string(e);
        std::vector<double> enc(static_cast<size_t>(n) * d), dec(static_cast<size_t>(d) * n), bias(n);
        for (auto& x : enc) x = 3.0 * gauss(rng);
        for (auto& x : dec) x = gauss(rng) / std::sqrt(static_cast<double>(n));
        for (auto& x : bias) x = 0.5 + 2.0 * uni(rng);
        in[e] = b.signal(p + ".in", {d}, {}, true);
        SignalId J = b.signal(p + ".J", {n}, {}, true);
        SignalId out = b.signal(p + ".out", {n}, {}, true);
        SignalId v = b.signal(p + ".voltage", {n}, {}, true);
        SignalId r = b.signal(p + ".refractory", {n}, {}, true);
        SignalId E = b.signal(p + ".encoders", {n, d}, enc, false, true);
        SignalId D = b.signal(p + ".decoders", {d, n}, dec, false, true);
        xhat[e] = b.signal(p + ".xhat", {d}, {}, true);
        net.voltages.push_back(v);
        b.op(Operator::reset(b.id(), b.full(in[e]), std::vector<double>(d, 0.0)));
        b.op(Operator::reset(b.id(), b.full(J), bias));
        b.op(Operator::dot_inc(b.id(), b.full(E), b.full(in[e]), b.full(J)));
        NeuronModel lif;
        b.op(Operator::sim_neurons(b.id(), lif, b.full(J), b.full(out), {b.full(v), b.full(r)}));
        b.op(Operator::reset(b.id(), b.full(xhat[e]), std::vector<double>(d, 0.0)));
        b.op(Operator::dot_inc(b.id(), b.full(D), b.full(out), b.full(xhat[e])));
    }
    auto connect = [&](const std::string& p, SignalId src, int ds, int dst) {
        std::vector<double> t(static_cast<size_t>(d) * ds);
        for (auto& x : t) x = 0.5 * gauss(rng) / std::sqrt(static_cast<double>(ds));
        SignalId T = b.signal(p + ".transform", {d, ds}, t, false, true);
        SignalId acc = b.signal(p + ".accum", {d}, {}, true);
        SignalId filt = b.signal(p + ".filtered", {d}, {}, true);
        SignalId state = b.signal(p + ".state", {d}, {}, true);
        b.op(Operator::reset(b.id(), b.full(acc), std::vector<double>(d, 0.0)));
        b.op(Operator::dot_inc(b.id(), b.full(T), b.full(src), b.full(acc)));
        b.op(Operator::sim_process(b.id(), 0.01, b.full(acc), b.full(filt), b.full(state)));
        b.op(Operator::copy(b.id(), b.full(filt), b.full(in[dst]), true));
        return filt;
    };
    SignalId probe_filt = -1;
    for (int e = 0; e < n_ens; ++e)
        for (int k = 0; k < k_out; ++k) {
            int dst = static_cast<int>(rng() % static_cast<unsigned>(n_ens - 1));
            if (dst >= e) ++dst;
            SignalId f = connect("c" + std::to_string(e) + "_" + std::to_string(k), xhat[e], d, dst);
            if (probe_filt < 0) probe_filt = f;
        }
    for (int i = 0; i < n_inputs; ++i) {
        const int node = 1000 + i;
        SignalId sig = b.signal("node" + std::to_string(node) + ".out", {d}, {}, true);
        b.m.feed_slots.push_back({node, sig, d, true, "input" + std::to_string(i)});
        connect("in" + std::to_string(i), sig, d, static_cast<int>(rng() % static_cast<unsigned>(n_ens)));
        net.fed_nodes.push_back(node);
        net.fed_dims.push_back(d);
    }
    SignalId step = b.signal("step", {1}, {}, false), time = b.signal("time", {1}, {}, false);
    b.op(Operator::time_update(b.id(), b.m.dt, b.full(step), b.full(time)));
    b.m.probes.push_back({0, xhat[0], "xhat0"});
    b.m.probes.push_back({1, probe_filt, "filt0"});
    b.m.probes.push_back({2, time, "time"});
    net.planned = run_passes(std::move(b.m));
    return net;
}

FeedData make_feeds(const Net& net, int batch, int steps, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    FeedData f;
    for (size_t i = 0; i < net.fed_nodes.size(); ++i) {
        Tensor3 t(batch, steps, net.fed_dims[i]);
        for (auto& x : t.data) x = gauss(rng);
        f.emplace(net.fed_nodes[i], std::move(t));
    }
    return f;
}

FeedData step_slice(const FeedData& f, int s0, int s1) {
    FeedData out;
    for (const auto& [node, t] : f) {
        Tensor3 u(t.batch, s1 - s0, t.dim);
        for (int b = 0; b < t.batch; ++b)
            for (int s = s0; s < s1; ++s)
                for (int d = 0; d < t.dim; ++d) u.at(b, s - s0, d) = t.at(b, s, d);
        out.emplace(node, std::move(u));
    }
    return out;
}

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

void compare_outputs(const ProbeOutput& ref, const ProbeOutput& gpu, const std::string& what) {
    expect(ref.size() == gpu.size(), what + ": probe count");
    for (const auto& [key, t] : ref) {
        auto it = gpu.find(key);
        if (it == gpu.end()) {
            expect(false, what + ": missing probe " + std::to_string(key));
            continue;
        }
        const Tensor3& g = it->second;
        expect(t.batch == g.batch && t.steps == g.steps && t.dim == g.dim, what + ": probe shape");
        size_t bad = 0;
        for (size_t i = 0; i < t.data.size() && i < g.data.size(); ++i)
            if (std::memcmp(&t.data[i], &g.data[i], sizeof(double)) != 0) ++bad;
        expect(bad == 0, what + ": probe " + std::to_string(key) + " differs in " + std::to_string(bad) + " of " +
                             std::to_string(t.data.size()) + " values");
    }
}

template <class Fn>
std::string error_of(Fn&& fn, const char* type) {
    try {
        fn();
    } catch (const RunError& e) {
        return std::string("RunError:") + e.what();
    } catch (const BuildError& e) {
        return std::string("BuildError:") + e.what();
    } catch (const StructuralError& e) {
        return std::string("StructuralError:") + e.what();
    } catch (const std::exception& e) {
        return std::string("other:") + e.what();
    }
    return std::string("none:") + type;
}

void run_case(const char* name, unsigned seed, int batch, int mode) {
    Net net = build_network(seed, 6, 96, 4, 2, 2);
    const int steps = 40, split = 17;
    FeedData feeds = make_feeds(net, batch, steps, seed + 7);
    EngineCore<float> ref(net.planned, batch, 3);
    neng_device_cfg cfg{};
    cfg.mode = mode;
    gpu::GpuEngine gpu(net.planned, batch, 3, &cfg);
    const std::string tag = std::string(name) + (gpu.mode() == NENG_MODE_FUSED ? " [fused]" : " [generic]");
    expect(mode == NENG_MODE_AUTO || gpu.mode() == mode, tag + ": executor mode");
    expect(ref.batch() == gpu.batch() && ref.unroll() == gpu.unroll(), tag + ": batch/unroll");

    // one call vs two calls (state and clock persist), then reset and rerun
    compare_outputs(ref.run(split, step_slice(feeds, 0, split)), gpu.run(split, step_slice(feeds, 0, split)),
                    tag + " first call");
    compare_outputs(ref.run(steps - split, step_slice(feeds, split, steps)),
                    gpu.run(steps - split, step_slice(feeds, split, steps)), tag + " second call");
    expect(ref.steps_completed() == gpu.steps_completed(), tag + ": steps_completed");
    for (SignalId v : net.voltages)
        for (int bi = 0; bi < batch; bi += std::max(1, batch / 3))
            expect(same_bits(ref.read_signal(v, bi), gpu.read_signal(v, bi)), tag + ": read_signal voltage");
    for (size_t i = 0; i < net.planned.buffers.buffers.size(); ++i)
        expect(ref.buffer_storage(static_cast<int>(i)) == gpu.buffer_storage(static_cast<int>(i)),
               tag + ": buffer_storage " + std::to_string(i));
    ref.reset();
    gpu.reset();
    expect(gpu.steps_completed() == 0, tag + ": reset rewinds the clock");
    compare_outputs(ref.run(steps, feeds), gpu.run(steps, feeds), tag + " after reset");

    // error behaviour: same exception type and message
    FeedData bad = feeds;
    bad.begin()->second = Tensor3(batch + 1, steps, net.fed_dims[0]);
    expect_same(error_of([&] { ref.run(steps, bad); }, "run"), error_of([&] { gpu.run(steps, bad); }, "run"), tag + ": bad feed shape error");
    FeedData unknown = feeds;
    unknown.emplace(424242, Tensor3(batch, steps, 1));
    expect_same(error_of([&] { ref.run(steps, unknown); }, "run"), error_of([&] { gpu.run(steps, unknown); }, "run"), tag + ": unknown node error");
    expect_same(error_of([&] { ref.run(0); }, "run"), error_of([&] { gpu.run(0); }, "run"), tag + ": n_steps error");
    expect_same(error_of([&] { ref.read_signal(-1); }, "read"), error_of([&] { gpu.read_signal(-1); }, "read"), tag + ": read_signal id error");
    expect_same(error_of([&] { ref.read_signal(0, batch); }, "read"), error_of([&] { gpu.read_signal(0, batch); }, "read"), tag + ": read_signal batch error");
}

}  // namespace

int main() {
    {
        Net net = build_network(1, 3, 32, 2, 1, 1);
        expect_same(error_of([&] { EngineCore<float>(net.planned, 0); }, "ctor"), error_of([&] { gpu::GpuEngine(net.planned, 0); }, "ctor"), "batch < 1 error");
        expect_same(error_of([&] { EngineCore<float>(net.planned, 1, 0); }, "ctor"), error_of([&] { gpu::GpuEngine(net.planned, 1, 0); }, "ctor"), "unroll < 1 error");
    }
    try {
        run_case("seed 3, batch 32", 3, 32, NENG_MODE_AUTO);
        run_case("seed 4, batch 5", 4, 5, NENG_MODE_AUTO);
        run_case("seed 5, batch 8", 5, 8, NENG_MODE_GENERIC);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "ERROR: %s\n", e.what());
        return 2;
    }
    std::printf("%s: %d checks, %d failed\n", g_failed ? "FAIL" : "PASS", g_checks, g_failed);
    return g_failed ? 1 : 0;
}
