// engine.cpp — compile a PlannedModel into device storage + a device program,
// and step it (the B200 counterpart of EngineCore<T>::compile/run/reset/
// read_signal, proj/src/exec.cpp:41-377).
#include "engine.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <unordered_map>

#include "fused.hpp"

namespace nengb {

// kernels (generic.cu)
cudaError_t launch_generic(const GenericProgram& p, int grid, int k_begin, int k_end, int call_k0,
                           cudaStream_t stream, int64_t small_arena_floats = 0);
size_t generic_small_arena_limit();
size_t generic_small_smem_bytes(const GenericProgram& p, int64_t arena_floats);
int generic_max_coresident_blocks(int device);
cudaError_t launch_reset(float* arena, const float* pristine, const int64_t* base, const int64_t* pbase,
                         const int64_t* span, const int32_t* per_batch, int nbuf, int B, cudaStream_t stream);
cudaError_t launch_probe_transpose(const float* ring, float* out, const int64_t* off, const int32_t* dims,
                                   int nprobes, int steps, int B, cudaStream_t stream);
cudaError_t launch_feed_transpose(const float* in, float* out, const int64_t* offs, const int32_t* cols, int nslots,
                                  int max_cols, int B, cudaStream_t stream);
cudaError_t launch_libm_hash_build(unsigned long long* slots, uint32_t mask, int shift, const uint32_t* keys,
                                   const uint32_t* results, int64_t n, cudaStream_t stream);

void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void DevMem::ensure(size_t n) {
    if (n <= bytes && p) return;
    release();
    if (n == 0) n = 16;
    cuda_check(cudaMalloc(&p, n), "cudaMalloc");
    bytes = n;
}

void PinnedMem::ensure(size_t n) {
    if (n <= bytes && p) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    if (n == 0) n = 16;
    cuda_check(cudaMallocHost(&p, n), "cudaMallocHost");
    bytes = n;
}

// ---------------------------------------------------------------------------
// libm parity tables

namespace {

std::string library_dir() {
    Dl_info info{};
    if (dladdr(reinterpret_cast<void*>(&library_dir), &info) && info.dli_fname) {
        std::string p = info.dli_fname;
        auto s = p.find_last_of('/');
        return s == std::string::npos ? std::string(".") : p.substr(0, s);
    }
    return ".";
}

struct HostTable {
    std::vector<uint32_t> keys, results;
    double tmin = 0.0, tmin_hot = 0.0;
    uint32_t region_shift = 0;
    std::vector<float> regions;  // per-region minimum exception distance on [-1/16, 0)
};

std::vector<HostTable> load_libm_file() {
    const char* env = std::getenv("NENG_LIBM_TABLES");
    std::string path = env ? env : library_dir() + "/data/libm_tables.bin";
    std::ifstream f(path, std::ios::binary);
    if (!f) throw BuildError("libm parity tables not found at " + path + " (run the package build)");
    std::vector<char> buf((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
    size_t at = 0;
    auto take = [&](void* dst, size_t n) {
        if (at + n > buf.size()) throw BuildError("libm parity table file truncated: " + path);
        std::memcpy(dst, buf.data() + at, n);
        at += n;
    };
    char magic[8];
    take(magic, 8);
    if (std::memcmp(magic, "NENGLIBM", 8)) throw BuildError("bad libm parity table file: " + path);
    uint32_t ver[2];
    take(ver, 8);
    if (ver[0] != 4) throw BuildError("libm parity table file has version " + std::to_string(ver[0]) + ", want 4");
    std::vector<HostTable> out(3);
    for (uint32_t t = 0; t < ver[1]; ++t) {
        uint32_t hdr[2], rh[2];
        uint64_t nkb;
        double tmin, tmin_hot;
        take(hdr, 8);
        take(&tmin, 8);
        take(&tmin_hot, 8);
        take(rh, 8);
        std::vector<float> regions(rh[0]);
        take(regions.data(), 4 * static_cast<size_t>(rh[0]));
        take(&nkb, 8);
        if (hdr[0] > 2) throw BuildError("bad libm table index");
        HostTable& ht = out[hdr[0]];
        ht.tmin = tmin;
        ht.tmin_hot = tmin_hot;
        ht.region_shift = rh[1];
        ht.regions = std::move(regions);
        size_t n = hdr[1];
        ht.keys.resize(n);
        ht.results.resize(n);
        const unsigned char* kb = reinterpret_cast<const unsigned char*>(buf.data() + at);
        size_t kp = 0;
        uint32_t prev = 0;
        for (size_t i = 0; i < n; ++i) {
            uint32_t d = 0;
            int shift = 0;
            unsigned char c;
            do {
                c = kb[kp++];
                d |= static_cast<uint32_t>(c & 0x7f) << shift;
                shift += 7;
            } while (c & 0x80);
            prev += d;
            ht.keys[i] = prev;
        }
        at += nkb;
        const unsigned char* cb = reinterpret_cast<const unsigned char*>(buf.data() + at);
        at += (n + 3) / 4;
        // results = host double-then-round +- 1 ulp (code 2: equal)
        int func = hdr[0] == 0 ? 0 : 1;
        unsigned nth = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < nth; ++w)
            pool.emplace_back([&, w] {
                for (size_t i = w; i < n; i += nth) {
                    float x;
                    std::memcpy(&x, &ht.keys[i], 4);
                    float r = func == 0 ? static_cast<float>(std::expm1(static_cast<double>(x)))
                                        : static_cast<float>(std::log1p(static_cast<double>(x)));
                    uint32_t rb;
                    std::memcpy(&rb, &r, 4);
                    int code = (cb[i / 4] >> (2 * (i % 4))) & 3;
                    ht.results[i] = code == 0 ? rb - 1 : code == 1 ? rb + 1 : rb;
                }
            });
        for (auto& th : pool) th.join();
    }
    return out;
}

struct DeviceLibm {
    LibmTables tables;
    std::vector<void*> allocs;
};

std::mutex g_libm_mu;
std::map<int, DeviceLibm*> g_libm;  // intentionally leaked for the process lifetime

}  // namespace

const LibmTables& libm_tables(int device) {
    std::lock_guard<std::mutex> lock(g_libm_mu);
    auto it = g_libm.find(device);
    if (it != g_libm.end()) return it->second->tables;
    std::vector<HostTable> host = load_libm_file();
    auto* dl = new DeviceLibm();
    // open-addressing table at load factor <= 1/2 over (keys, results)
    auto build = [&](const uint32_t* keys, const uint32_t* results, size_t n, const unsigned long long** slots_out,
                     uint32_t* mask_out, int32_t* shift_out) {
        int log2cap = 4;
        while ((size_t{1} << log2cap) < 2 * n + 16) ++log2cap;
        size_t cap = size_t{1} << log2cap;
        void* slots = nullptr;
        cuda_check(cudaMalloc(&slots, cap * sizeof(unsigned long long)), "cudaMalloc libm");
        cuda_check(cudaMemset(slots, 0, cap * sizeof(unsigned long long)), "cudaMemset libm");
        void *dk = nullptr, *dr = nullptr;
        cuda_check(cudaMalloc(&dk, std::max<size_t>(n, 1) * 4), "cudaMalloc libm keys");
        cuda_check(cudaMalloc(&dr, std::max<size_t>(n, 1) * 4), "cudaMalloc libm results");
        cuda_check(cudaMemcpy(dk, keys, n * 4, cudaMemcpyHostToDevice), "libm H2D");
        cuda_check(cudaMemcpy(dr, results, n * 4, cudaMemcpyHostToDevice), "libm H2D");
        cuda_check(launch_libm_hash_build(static_cast<unsigned long long*>(slots), static_cast<uint32_t>(cap - 1),
                                          32 - log2cap, static_cast<uint32_t*>(dk), static_cast<uint32_t*>(dr),
                                          static_cast<int64_t>(n), nullptr),
                   "libm hash build");
        cuda_check(cudaDeviceSynchronize(), "libm hash build");
        cudaFree(dk);
        cudaFree(dr);
        *slots_out = static_cast<const unsigned long long*>(slots);
        *mask_out = static_cast<uint32_t>(cap - 1);
        *shift_out = 32 - log2cap;
        dl->allocs.push_back(slots);
    };
    for (int t = 0; t < 3; ++t) {
        const HostTable& ht = host[t];
        build(ht.keys.data(), ht.results.data(), ht.keys.size(), &dl->tables.t[t].slots, &dl->tables.t[t].mask,
              &dl->tables.t[t].shift);
        // the LIF range x in [-1/16, 0) (bit patterns 0x80000001..0xBD800000) as a small, L2-resident table
        auto lo = std::lower_bound(ht.keys.begin(), ht.keys.end(), 0x80000001u);
        auto hi = std::upper_bound(ht.keys.begin(), ht.keys.end(), 0xBD800000u);
        size_t a = static_cast<size_t>(lo - ht.keys.begin()), b = static_cast<size_t>(hi - ht.keys.begin());
        build(ht.keys.data() + a, ht.results.data() + a, b > a ? b - a : 0, &dl->tables.t[t].hot_slots,
              &dl->tables.t[t].hot_mask, &dl->tables.t[t].hot_shift);
        {
            // bucketed key set of the same LIF-range keys (load <= 1/4 per slot on average)
            const size_t nk = b > a ? b - a : 0;
            int lb = 4;
            while ((size_t{4} << lb) < 4 * nk + 64) ++lb;  // 4 * 2^lb slots >= 4 * nk: load <= 0.25
            const size_t nb = size_t{1} << lb;
            std::vector<uint32_t> bk(nb * 4, 0u), br(nb * 4, 0u);
            for (size_t q = a; q < b; ++q) {
                const uint32_t key = ht.keys[q];
                const uint32_t res = ht.results[q];
                size_t bi = static_cast<uint32_t>(key * 0x9E3779B1u) >> (32 - lb);
                for (;;) {
                    uint32_t* slot = bk.data() + bi * 4;
                    int j = 0;
                    while (j < 4 && slot[j] != 0u) ++j;
                    if (j < 4) {
                        slot[j] = key;
                        br[bi * 4 + j] = res;
                        break;
                    }
                    bi = (bi + 1) & (nb - 1);
                }
            }
            void* db = nullptr;
            cuda_check(cudaMalloc(&db, bk.size() * 4), "cudaMalloc libm buckets");
            cuda_check(cudaMemcpy(db, bk.data(), bk.size() * 4, cudaMemcpyHostToDevice), "libm buckets H2D");
            dl->allocs.push_back(db);
            dl->tables.t[t].hot_buckets = static_cast<const uint4*>(db);
            void* dr2 = nullptr;
            cuda_check(cudaMalloc(&dr2, br.size() * 4), "cudaMalloc libm bucket results");
            cuda_check(cudaMemcpy(dr2, br.data(), br.size() * 4, cudaMemcpyHostToDevice), "libm bucket results H2D");
            dl->allocs.push_back(dr2);
            dl->tables.t[t].bucket_results = static_cast<const uint32_t*>(dr2);
            dl->tables.t[t].bucket_mask = static_cast<uint32_t>(nb - 1);
            dl->tables.t[t].bucket_shift = 32 - lb;
        }
        {
            // block filter over k = key - 0x80000001 in [0, 0x3D800000): bit (k >> 6)
            std::vector<uint32_t> filt((0x3D800000u >> 11) + 1, 0u);
            for (size_t q = a; q < b; ++q) {
                const uint32_t k = ht.keys[q] - 0x80000001u;
                filt[k >> 11] |= 1u << ((k >> 6) & 31u);
            }
            void* df = nullptr;
            cuda_check(cudaMalloc(&df, filt.size() * 4), "cudaMalloc libm filter");
            cuda_check(cudaMemcpy(df, filt.data(), filt.size() * 4, cudaMemcpyHostToDevice), "libm filter H2D");
            dl->allocs.push_back(df);
            dl->tables.t[t].hot_filter = static_cast<const uint32_t*>(df);
        }
        // skip lookups whose double result is farther than this from a float
        // rounding midpoint (all exceptions are closer); margin covers the
        // device/host double results differing by a few double ulps
        dl->tables.t[t].lookup_from = static_cast<float>(host[t].tmin - 0.01);
        dl->tables.t[t].lookup_from_hot = static_cast<float>(host[t].tmin_hot - 0.01);
        std::vector<float> reg(ht.regions.size());
        for (size_t i = 0; i < reg.size(); ++i) reg[i] = ht.regions[i] - 0.01f;  // same margin
        void* dreg = nullptr;
        cuda_check(cudaMalloc(&dreg, std::max<size_t>(reg.size(), 1) * 4), "cudaMalloc libm regions");
        cuda_check(cudaMemcpy(dreg, reg.data(), reg.size() * 4, cudaMemcpyHostToDevice), "libm regions H2D");
        dl->allocs.push_back(dreg);
        dl->tables.t[t].region_from = static_cast<const float*>(dreg);
        // screening window of the fast polynomials: the exact window, and never
        // less than 0.004 ulp (the fast polynomials are within 0.002 ulp)
        std::vector<uint32_t> win(reg.size());
        for (size_t i = 0; i < win.size(); ++i) {
            double w = std::max(0.5 - static_cast<double>(reg[i]), 0.004) * 536870912.0;  // x 2^29
            win[i] = static_cast<uint32_t>(std::ceil(w));
        }
        void* dwin = nullptr;
        cuda_check(cudaMalloc(&dwin, std::max<size_t>(win.size(), 1) * 4), "cudaMalloc libm windows");
        cuda_check(cudaMemcpy(dwin, win.data(), win.size() * 4, cudaMemcpyHostToDevice), "libm windows H2D");
        dl->allocs.push_back(dwin);
        dl->tables.t[t].region_win = static_cast<const uint32_t*>(dwin);
        // byte screen for shared memory: doubtful when (d >> 21) <= w8 (d <= win implies it)
        std::vector<uint8_t> w8(win.size());
        for (size_t i = 0; i < win.size(); ++i) w8[i] = static_cast<uint8_t>(std::min<uint32_t>(win[i] >> 21, 255u));
        void* dw8 = nullptr;
        cuda_check(cudaMalloc(&dw8, std::max<size_t>(w8.size(), 16)), "cudaMalloc libm byte windows");
        cuda_check(cudaMemcpy(dw8, w8.data(), w8.size(), cudaMemcpyHostToDevice), "libm byte windows H2D");
        dl->allocs.push_back(dw8);
        dl->tables.t[t].region_w8 = static_cast<const uint8_t*>(dw8);
        dl->tables.t[t].region_shift = ht.region_shift;
        dl->tables.t[t].n_regions = static_cast<uint32_t>(reg.size());
    }
    g_libm[device] = dl;
    return dl->tables;
}

// ---------------------------------------------------------------------------

namespace {

std::vector<int> written_positions(const Operator& op) {
    std::vector<int> w;
    for (auto [pos, mode] : operand_modes(op))
        if (mode != AccessMode::Read) w.push_back(pos);
    return w;
}

}  // namespace

Engine::Engine(PlannedModel planned, int batch, int unroll, const neng_device_cfg* cfg)
    : pm_(std::move(planned)), batch_(batch), unroll_(unroll) {
    // exec.cpp:10-16
    if (batch_ < 1) throw BuildError("engine batch size must be at least 1");
    if (unroll_ < 1) throw BuildError("engine unroll factor must be at least 1");
    if (cfg) {
        device_ = cfg->device;
        requested_mode_ = cfg->mode;
        steps_per_launch_ = cfg->steps_per_launch;
        shard_rank_ = cfg->shard_rank;
        shard_count_ = cfg->shard_count > 0 ? cfg->shard_count : 1;
        precision_ = cfg->precision;
    }
    if (precision_ != NENG_PRECISION_STRICT_FP32 && precision_ != NENG_PRECISION_TF32 &&
        precision_ != NENG_PRECISION_BF16X3)
        throw BuildError("unknown precision mode " + std::to_string(precision_));
    if (shard_count_ < 1 || shard_rank_ < 0 || shard_rank_ >= shard_count_)
        throw BuildError("shard rank " + std::to_string(shard_rank_) + " is outside [0, " +
                         std::to_string(shard_count_) + ")");
    if (shard_count_ > 1 && requested_mode_ == NENG_MODE_GENERIC)
        throw BuildError("ensemble sharding needs the fused pipeline");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    compile();
}

Engine::~Engine() {
    fused_.reset();
    for (cudaEvent_t& ev : feed_events_)
        if (ev) cudaEventDestroy(ev);
    for (cudaEvent_t& ev : xpose_events_)
        if (ev) cudaEventDestroy(ev);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (stream_) cudaStreamDestroy(stream_);
}

DArg Engine::resolve(const SignalRef& r) const {
    // resolve (exec.cpp:18-25) in the transposed device layout
    int bi = pm_.buffers.buffer_of[r.signal];
    const BufLayout& L = bufs_[bi];
    int64_t off = (static_cast<int64_t>(pm_.buffers.row_offset[r.signal]) + r.start) * L.epr;
    DArg a;
    a.elems = static_cast<int64_t>(r.rows()) * L.epr;
    a.es = L.per_batch ? batch_ : 1;
    a.bs = L.per_batch ? 1 : 0;
    a.base = L.base + off * a.es;
    return a;
}

DArg Engine::resolve_full(int sig) const { return resolve({sig, 0, pm_.model.signals[sig].rows()}); }

void Engine::compile() {
    const BuiltModel& m = pm_.model;
    const BufferAssignment& ba = pm_.buffers;
    if (ba.buffer_of.size() != m.signals.size() || ba.row_offset.size() != m.signals.size())
        throw BuildError("planned model buffer assignment does not cover every signal");
    for (size_t i = 0; i < m.signals.size(); ++i)
        if (m.signals[i].id != static_cast<int>(i)) throw StructuralError("signals must be id-indexed");
    size_t nbuf = ba.buffers.size();
    bufs_.assign(nbuf, {});
    // elements per row (exec.cpp:46-51); promoted PES buffers (:54-59)
    std::vector<char> promoted(nbuf, 0);
    for (const Operator& op : m.operators)
        if (op.kind == OpKind::SimPES && op.operands.size() == 3) promoted[ba.buffer_of[op.operands[2].signal]] = 1;
    int64_t total = 0;
    std::vector<int64_t> pbase(nbuf);
    int64_t ptotal = 0;
    for (size_t bi = 0; bi < nbuf; ++bi) {
        BufLayout& L = bufs_[bi];
        L.epr = 1;
        for (int d : ba.buffers[bi].trailing) L.epr *= d;
        L.span = static_cast<int64_t>(ba.buffers[bi].rows) * L.epr;
        L.per_batch = ba.buffers[bi].minibatched || promoted[bi];
        L.base = total;
        int64_t n = L.span * (L.per_batch ? batch_ : 1);
        total += (n + 31) / 32 * 32;  // 128-B aligned bases
        pbase[bi] = ptotal;
        ptotal += L.span;
    }
    arena_floats_ = total;
    arena_.ensure(static_cast<size_t>(std::max<int64_t>(total, 1)) * sizeof(float));

    // pristine image (exec.cpp:61-79), fp32
    std::vector<float> pristine(static_cast<size_t>(std::max<int64_t>(ptotal, 1)), 0.0f);
    for (const Signal& s : m.signals) {
        if (s.initial.empty()) continue;
        int bi = ba.buffer_of[s.id];
        int64_t at = pbase[bi] + static_cast<int64_t>(ba.row_offset[s.id]) * bufs_[bi].epr;
        for (size_t k = 0; k < s.initial.size(); ++k) pristine[at + k] = static_cast<float>(s.initial[k]);
    }
    pristine_.ensure(pristine.size() * sizeof(float));
    cuda_check(cudaMemcpy(pristine_.p, pristine.data(), pristine.size() * sizeof(float), cudaMemcpyHostToDevice),
               "pristine H2D");
    // reset metadata: base, pbase, span (int64 x3) + per_batch (int32)
    {
        std::vector<int64_t> meta(3 * nbuf + 1);
        std::vector<int32_t> pb(nbuf + 1);
        for (size_t bi = 0; bi < nbuf; ++bi) {
            meta[bi] = bufs_[bi].base;
            meta[nbuf + bi] = pbase[bi];
            meta[2 * nbuf + bi] = bufs_[bi].span;
            pb[bi] = bufs_[bi].per_batch;
        }
        reset_meta_.ensure(meta.size() * 8 + pb.size() * 4);
        cuda_check(cudaMemcpy(reset_meta_.p, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice), "meta H2D");
        cuda_check(cudaMemcpy(static_cast<char*>(reset_meta_.p) + meta.size() * 8, pb.data(), pb.size() * 4,
                              cudaMemcpyHostToDevice),
                   "meta H2D");
    }

    for (const Operator& op : m.operators)
        if (op.kind == OpKind::SimNeurons &&
            (op.neuron.kind == NeuronKind::LIF || op.neuron.kind == NeuronKind::LIFRate))
            needs_libm_ = true;

    compile_generic();

    mode_ = NENG_MODE_GENERIC;
    if (requested_mode_ != NENG_MODE_GENERIC) {
        std::string why;
        fused_ = try_compile_fused(*this, &why);
        if (fused_)
            mode_ = NENG_MODE_FUSED;
        else if (requested_mode_ == NENG_MODE_FUSED || shard_count_ > 1)
            throw BuildError("fused pipeline unavailable for this model: " + why);
    }
    reset();
}

void Engine::compile_generic() {
    const BuiltModel& m = pm_.model;
    std::unordered_map<int, const Operator*> by_id;
    for (const Operator& op : m.operators) by_id.emplace(op.id, &op);

    std::vector<DGroup> groups;
    std::vector<DMember> members;
    std::vector<DTile> tiles;
    std::vector<float> values;
    int max_tiles = 1;
    std::vector<char> written_sig;  // lazily: signals some operator writes
    for (const OpGroup& og : pm_.plan) {
        if (og.members.empty()) throw BuildError("plan has an empty group");
        auto fit = by_id.find(og.members[0]);
        if (fit == by_id.end())
            throw BuildError("plan names operator " + std::to_string(og.members[0]) + " which does not exist");
        const Operator& first = *fit->second;
        DGroup g;
        g.kind = static_cast<int32_t>(first.kind);
        if (first.kind == OpKind::Copy && first.inc) g.flags |= GF_INC;
        g.dt = static_cast<float>(m.dt);  // Instr::dt = (T)model.dt (exec.cpp:88)
        if (first.kind == OpKind::SimNeurons) {
            g.neuron = static_cast<int32_t>(first.neuron.kind);
            g.tau_rc = static_cast<float>(first.neuron.tau_rc);
            g.tau_ref = static_cast<float>(first.neuron.tau_ref);
            g.amplitude = static_cast<float>(first.neuron.amplitude);
            volatile float mdt = -g.dt, trc = g.tau_rc;  // -delta / tau_rc in float, delta = dt
            const float arg = mdt / trc;
            g.em_dt = expm1f(arg);  // the host libm result the reference uses
        } else if (first.kind == OpKind::SimProcess) {
            double a = 0.0, b = 1.0;  // lowpass_coefficients (neuron_math.hpp:33-37)
            if (first.tau > 0.0) {
                a = std::exp(-m.dt / first.tau);
                b = 1.0 - a;
            }
            g.tau_a = static_cast<float>(a);
            g.tau_b = static_cast<float>(b);
            if (first.operands.size() >= 3) g.flags |= GF_HAS_STATE;
        }
        auto modes = operand_modes(first);
        auto wpos = written_positions(first);
        // per_batch (exec.cpp:122-125) from member 0's buffers
        int wpb = 0, wshared = 0;
        for (int p : wpos) {
            int bi = pm_.buffers.buffer_of[first.operands[p].signal];
            if (bufs_[bi].per_batch)
                wpb = 1;
            else
                wshared = 1;
        }
        if (wpb) g.flags |= GF_PER_BATCH;
        g.copies = wpb ? batch_ : 1;
        if (wpb && wshared && batch_ > 1) g.flags |= GF_SERIAL_B;
        g.member_begin = static_cast<int32_t>(members.size());
        g.tile_begin = static_cast<int32_t>(tiles.size());
        for (OpId id : og.members) {
            auto it = by_id.find(id);
            if (it == by_id.end())
                throw BuildError("plan names operator " + std::to_string(id) + " which does not exist");
            const Operator& op = *it->second;
            if (op.kind != first.kind) throw BuildError("plan group mixes operator kinds");
            DMember dm;
            for (size_t p = 0; p < op.operands.size() && p < 4; ++p) dm.a[p] = resolve(op.operands[p]);
            if (op.kind == OpKind::Reset) {
                dm.value_at = static_cast<int64_t>(values.size());
                for (double v : op.value) values.push_back(static_cast<float>(v));
            }
            switch (op.kind) {
                case OpKind::Reset: dm.items = dm.a[0].elems; break;
                case OpKind::Copy: dm.items = dm.a[0].elems; break;
                case OpKind::ElementwiseInc:
                    dm.items = dm.a[1].elems;
                    if (dm.a[0].elems == 1) dm.flags |= MF_SCALAR_A;
                    break;
                case OpKind::DotInc: {
                    dm.items = dm.a[2].elems;
                    const Signal& As = m.signals[op.operands[0].signal];
                    if (As.constant && std::all_of(As.initial.begin(), As.initial.end(),
                                                   [](double v) { return std::isfinite(static_cast<float>(v)); }))
                        dm.flags |= MF_SKIP_ZERO_X;
                    break;
                }
                case OpKind::SimNeurons: dm.items = dm.a[0].elems; break;
                case OpKind::SimProcess: dm.items = dm.a[0].elems; break;
                case OpKind::SimPES:
                    dm.items = dm.a[0].elems * dm.a[1].elems;
                    dm.pes_scale = static_cast<float>(first.learning_rate * m.dt /
                                                      static_cast<double>(dm.a[0].elems));
                    break;
                case OpKind::TimeUpdate: dm.items = 1; break;
            }
            // self-aliasing with an offset -> reference loop order (GF_SERIAL_ALL)
            auto wp = written_positions(op);
            for (int p : wp)
                for (size_t q = 0; q < op.operands.size(); ++q) {
                    if (static_cast<int>(q) == p) continue;
                    int bp = pm_.buffers.buffer_of[op.operands[p].signal];
                    int bq = pm_.buffers.buffer_of[op.operands[q].signal];
                    if (bp != bq) continue;
                    const DArg &A = dm.a[p], &Q = dm.a[q];
                    bool overlap = A.base < Q.base + Q.elems * A.es && Q.base < A.base + A.elems * A.es;
                    if (!overlap) continue;
                    bool elementwise_same = A.base == Q.base && A.elems == Q.elems &&
                                            !(op.kind == OpKind::ElementwiseInc && (dm.flags & MF_SCALAR_A));
                    if (!elementwise_same) g.flags |= GF_SERIAL_ALL;
                }
            int64_t total_items = dm.items * g.copies;
            int mi = static_cast<int>(members.size());
            // light items (Reset, Copy, ElementwiseInc, SimProcess) of large members: 4 per
            // thread per tile (amortises the descriptor loads); heavy ones (a DotInc k loop,
            // a neuron step) and small members: 1 per thread, for load balance and latency
            const bool heavy = op.kind == OpKind::DotInc || op.kind == OpKind::SimNeurons || op.kind == OpKind::SimPES;
            const int64_t per_tile = heavy || total_items < (int64_t{1} << 18) ? kTile : kTileItems;
            for (int64_t s = 0; s < total_items; s += per_tile)
                tiles.push_back(
                    {mi, static_cast<int32_t>(s), static_cast<int32_t>(std::min<int64_t>(per_tile, total_items - s))});
            if (total_items > (int64_t{1} << 30)) throw BuildError("group member too large for the generic path");
            members.push_back(dm);
        }
        g.n_members = static_cast<int32_t>(members.size()) - g.member_begin;
        g.n_tiles = static_cast<int32_t>(tiles.size()) - g.tile_begin;
        g.flags |= GF_BARRIER;
        if (first.kind == OpKind::DotInc && batch_ >= 64 && (g.flags & GF_PER_BATCH) &&
            !(g.flags & (GF_SERIAL_ALL | GF_SERIAL_B)) && std::getenv("NENG_GENERIC_DENSE_OFF") == nullptr) {
            // dense members (shared row-major A, per-batch x and y, K >= 32): CTA
            // tiles of 32 rows x 64 batch columns (dense_dot_tile) instead of one thread per output
            bool dense = true;
            for (int mi = g.member_begin; mi < static_cast<int>(members.size()) && dense; ++mi) {
                const DArg &A = members[mi].a[0], &X = members[mi].a[1], &Y = members[mi].a[2];
                dense = A.bs == 0 && A.es == 1 && A.elems == Y.elems * X.elems && X.es == batch_ && X.bs == 1 &&
                        Y.es == batch_ && Y.bs == 1 && X.elems >= 32;  // any rows: a long k loop per thread is latency-bound
            }
            if (dense) {
                tiles.resize(g.tile_begin);
                for (int mi = g.member_begin; mi < static_cast<int>(members.size()); ++mi)
                    for (int64_t r0 = 0; r0 < members[mi].a[2].elems; r0 += 32)
                        for (int c0 = 0; c0 < batch_; c0 += 64)
                            tiles.push_back({mi, static_cast<int32_t>(r0), c0});
                g.n_tiles = static_cast<int32_t>(tiles.size()) - g.tile_begin;
                g.flags |= GF_DENSE;
            }
        }
        if (precision_ != NENG_PRECISION_STRICT_FP32 && first.kind == OpKind::DotInc && batch_ >= 32 &&
            (g.flags & GF_PER_BATCH) && !(g.flags & (GF_SERIAL_ALL | GF_SERIAL_B))) {
            // Y[M][B] += A[M][K] X[K][B]: shared row-major weights, per-batch input and output,
            // every member on the tensor cores or the whole group stays in the interpreter
            TcGroup tg;
            tg.group = static_cast<int>(groups.size());
            const int mode = precision_ == NENG_PRECISION_TF32 ? TC_TF32 : TC_BF16X3;
            float* Ab = arena_.as<float>();
            if (written_sig.empty()) {  // signals some operator writes (BF16X3 splits A once per call)
                written_sig.assign(m.signals.size(), 0);
                for (const Operator& o : m.operators)
                    for (int wp : written_positions(o)) written_sig[o.operands[wp].signal] = 1;
            }
            bool ok = true;
            for (int mi = g.member_begin; mi < static_cast<int>(members.size()) && ok; ++mi) {
                const Operator& mop = *by_id.at(og.members[mi - g.member_begin]);
                if (mode == TC_BF16X3 && written_sig[mop.operands[0].signal]) {
                    ok = false;
                    break;
                }
                const DMember& dm = members[mi];
                const DArg &A = dm.a[0], &X = dm.a[1], &Y = dm.a[2];
                const int64_t M = Y.elems, K = X.elems;
                ok = A.bs == 0 && A.es == 1 && A.elems == M * K && X.es == batch_ && X.bs == 1 && Y.es == batch_ &&
                     Y.bs == 1 && M >= 1 && K >= 32 && M < (1 << 30) && K < (1 << 30);
                // the output rows must not overlap the operands (they are read by TMA while it is written)
                ok = ok && (Y.base + M * batch_ <= X.base || X.base + K * batch_ <= Y.base) &&
                     (Y.base + M * batch_ <= A.base || A.base + M * K <= Y.base);
                if (!ok) break;
                void* scr = nullptr;
                if (mode == TC_BF16X3) {
                    tg.scratch.push_back(std::make_unique<DevMem>());
                    tg.scratch.back()->ensure(tc_dot_scratch_bytes(static_cast<int>(M), static_cast<int>(K), batch_));
                    scr = tg.scratch.back()->p;
                }
                TcDotDesc d;
                const char* why = tc_dot_prepare(&d, Ab + A.base, Ab + X.base, Ab + Y.base, static_cast<int>(M),
                                                 static_cast<int>(K), batch_, batch_, batch_, mode, scr);
                ok = *why == 0;
                if (ok) tg.dots.push_back(d);
            }
            if (ok) tc_groups_.push_back(std::move(tg));
        }
        if (!(g.flags & (GF_SERIAL_ALL | GF_SERIAL_B))) max_tiles = std::max(max_tiles, g.n_tiles);
        groups.push_back(g);
    }

    // feeds / probes (exec.cpp:150-159)
    feeds_.clear();
    for (const FeedSlot& fs : m.feed_slots) {
        DFeed f;
        f.dst = resolve_full(fs.signal);
        f.dim = fs.dim;
        f.copies = bufs_[pm_.buffers.buffer_of[fs.signal]].per_batch ? batch_ : 1;
        feeds_.push_back(f);
    }
    probes_.clear();
    int64_t roff = 0;
    for (const ProbeRegistration& p : m.probes) {
        DProbe q;
        q.src = resolve_full(p.signal);
        q.dim = static_cast<int32_t>(m.signals[p.signal].size());
        q.per_batch = bufs_[pm_.buffers.buffer_of[p.signal]].per_batch;
        q.ring_off = roff;
        roff += q.dim;  // scaled by n_steps*B per call
        probes_.push_back(q);
    }

    auto upload = [](DevMem& dst, const void* src, size_t bytes) {
        dst.ensure(std::max<size_t>(bytes, 16));
        if (bytes) cuda_check(cudaMemcpy(dst.p, src, bytes, cudaMemcpyHostToDevice), "program H2D");
    };
    prof_kinds_.clear();
    for (const DGroup& g : groups) prof_kinds_.push_back(g.kind | (g.flags << 8));
    upload(d_groups_, groups.data(), groups.size() * sizeof(DGroup));
    upload(d_members_, members.data(), members.size() * sizeof(DMember));
    upload(d_tiles_, tiles.data(), tiles.size() * sizeof(DTile));
    upload(d_values_, values.data(), values.size() * sizeof(float));

    prog_ = GenericProgram{};
    prog_.arena = arena_.as<float>();
    prog_.groups = d_groups_.as<DGroup>();
    prog_.members = d_members_.as<DMember>();
    prog_.tiles = d_tiles_.as<DTile>();
    prog_.values = d_values_.as<float>();
    prog_.n_groups = static_cast<int32_t>(groups.size());
    prog_.n_feeds = static_cast<int32_t>(feeds_.size());
    prog_.n_probes = static_cast<int32_t>(probes_.size());
    prog_.batch = batch_;
    if (needs_libm_) prog_.libm = libm_tables(device_);

    int maxco = generic_max_coresident_blocks(device_);
    {
        // at most 2 CTAs per SM: every group ends in a grid barrier, whose cost grows with
        // the CTA count (config 3 strict: 0.30 ms/step at 2 per SM, 0.35 at 3)
        int sms = 0;
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "SM count");
        maxco = std::min(maxco, 2 * std::max(sms, 1));
    }
    if (const char* env = std::getenv("NENG_GENERIC_GRID")) maxco = std::max(1, std::min(maxco, std::atoi(env)));
    grid_ = std::max(1, std::min(maxco, max_tiles));
    // tiny programs: one CTA, block-level barriers only (config 0: 42 vs 60 us/step on 4 CTAs)
    if (max_tiles <= 16 && !std::getenv("NENG_GENERIC_GRID")) grid_ = 1;
    // ... and when the whole arena fits in shared memory, the arena lives there during a launch
    small_arena_floats_ = 0;
    // (dense DotInc tiles are written for exactly kTile threads: those programs keep the plain kernel)
    const bool any_dense =
        std::any_of(groups.begin(), groups.end(), [](const DGroup& g) { return (g.flags & GF_DENSE) != 0; });
    prog_.n_members = static_cast<int32_t>(members.size());
    prog_.n_tiles = static_cast<int32_t>(tiles.size());
    if (grid_ == 1 && tc_groups_.empty() && !any_dense && !std::getenv("NENG_GENERIC_NO_SMEM") &&
        generic_small_smem_bytes(prog_, arena_floats_) <= generic_small_arena_limit())
        small_arena_floats_ = arena_floats_;
    if (std::getenv("NENG_GENERIC_VERBOSE"))
        std::fprintf(stderr, "[generic] %zu groups, max tiles %d, grid %d\n", groups.size(), max_tiles, grid_);
}

void Engine::reset() {
    // exec.cpp:164-174
    if (call_steps_) throw RunError("reset: a stepped call is open");
    size_t nbuf = bufs_.size();
    const int64_t* meta = reset_meta_.as<int64_t>();
    const int32_t* pb = reinterpret_cast<const int32_t*>(reset_meta_.as<char>() + (3 * nbuf + 1) * 8);
    cuda_check(launch_reset(arena_.as<float>(), pristine_.as<float>(), meta, meta + nbuf, meta + 2 * nbuf, pb,
                            static_cast<int>(nbuf), batch_, stream_),
               "reset");
    if (fused_) fused_->load_from_arena(stream_);
    cuda_check(cudaStreamSynchronize(stream_), "reset");
    steps_done_ = 0;
}

void Engine::validate_feeds(int n_feeds, const neng_feed* feeds, int n_steps) const {
    // validate_feeds (model.hpp:62-83); FeedData iterates in node-id order
    const BuiltModel& m = pm_.model;
    std::vector<const neng_feed*> order;
    for (int i = 0; i < n_feeds; ++i) order.push_back(&feeds[i]);
    std::stable_sort(order.begin(), order.end(),
                     [](const neng_feed* a, const neng_feed* b) { return a->node_id < b->node_id; });
    for (const neng_feed* t : order) {
        const FeedSlot* slot = nullptr;
        for (const FeedSlot& s : m.feed_slots)
            if (s.node_id == t->node_id) slot = &s;
        if (!slot) throw RunError("feed for unknown node " + std::to_string(t->node_id));
        if (t->batch != batch_ || t->steps < n_steps || t->dim != slot->dim) {
            std::ostringstream os;
            os << "feed for node " << t->node_id << " ('" << slot->label << "') has shape (" << t->batch << ", "
               << t->steps << ", " << t->dim << "), expected (" << batch_ << ", >=" << n_steps << ", " << slot->dim
               << ")";
            throw RunError(os.str());
        }
        if (!t->data && static_cast<int64_t>(t->batch) * t->steps * t->dim > 0)
            throw InvalidArgument("feed data pointer is null");
    }
    for (const FeedSlot& s : m.feed_slots) {
        bool found = false;
        for (int i = 0; i < n_feeds; ++i) found |= feeds[i].node_id == s.node_id;
        if (!s.has_default && !found)
            throw RunError("node " + std::to_string(s.node_id) + " ('" + s.label +
                           "') has no default output and no feed was supplied");
    }
}

void Engine::launch_steps(int n_steps, const float* d_feed_data, const std::vector<int>& present, float* d_ring,
                          cudaStream_t stream) {
    last_launches_ = 0;
    std::vector<int64_t> feed_off, ring_off;
    call_offsets(n_steps, present, &feed_off, &ring_off);
    if (fused_) {
        last_launches_ = fused_->run(n_steps, d_feed_data, feed_off.data(), present.data(), d_ring, ring_off.data(),
                                     stream);
        return;
    }
    // refresh per-call feed/probe descriptors
    bool any = false;
    for (size_t f = 0; f < feeds_.size(); ++f) {
        feeds_[f].present = present[f];
        feeds_[f].data_off = feed_off[f];
        any |= present[f] != 0;
    }
    for (size_t q = 0; q < probes_.size(); ++q) probes_[q].ring_off = ring_off[q];
    size_t fb = feeds_.size() * sizeof(DFeed), pbytes = probes_.size() * sizeof(DProbe);
    d_feeds_.ensure(std::max<size_t>(fb, 16));
    d_probes_.ensure(std::max<size_t>(pbytes, 16));
    if (fb) cuda_check(cudaMemcpyAsync(d_feeds_.p, feeds_.data(), fb, cudaMemcpyHostToDevice, stream), "feeds H2D");
    if (pbytes)
        cuda_check(cudaMemcpyAsync(d_probes_.p, probes_.data(), pbytes, cudaMemcpyHostToDevice, stream), "probes H2D");
    GenericProgram p = prog_;
    p.feeds = d_feeds_.as<DFeed>();
    p.probes = d_probes_.as<DProbe>();
    p.any_feed = any ? 1 : 0;
    p.feed_data = d_feed_data;
    p.ring = d_ring;
    p.call_steps = n_steps;
    if (!tc_groups_.empty()) {
        // BF16X3: the weights' bf16 halves, once per call (a DotInc's weights are shared and
        // constant inside a call: no operator of a dense group writes its own A)
        for (const TcGroup& tg : tc_groups_)
            for (const TcDotDesc& d : tg.dots) {
                cuda_check(tc_dot_split_a(d, stream), "tensor-core weight split");
                if (d.mode == TC_BF16X3) ++last_launches_;
            }
        // per step: interpreter segments between the tensor-core groups (feeds with the
        // first segment, probe captures with the last), the GEMMs in stream order between
        for (int k = 0; k < n_steps; ++k) {
            int seg = 0;
            for (const TcGroup& tg : tc_groups_) {
                if (tg.group > seg || seg == 0) {
                    GenericProgram q = p;
                    q.g_begin = seg;
                    q.g_end = tg.group;
                    cuda_check(launch_generic(q, grid_, k, k + 1, 0, stream), "generic kernel launch");
                    ++last_launches_;
                }
                run_tc_dots(tg, stream);
                last_launches_ += static_cast<int64_t>(tg.dots.size()) * (precision_ == NENG_PRECISION_BF16X3 ? 2 : 1);
                seg = tg.group + 1;
            }
            GenericProgram q = p;
            q.g_begin = seg;
            q.g_end = -1;
            cuda_check(launch_generic(q, grid_, k, k + 1, 0, stream), "generic kernel launch");
            ++last_launches_;
        }
    } else {
        int K = steps_per_launch_ > 0 ? steps_per_launch_ : n_steps;
        for (int k = 0; k < n_steps; k += K) {
            const bool prof = std::getenv("NENG_GENERIC_PROFILE") != nullptr;
            DevMem dprof;
            if (prof) {
                dprof.ensure((prog_.n_groups + 1) * 8);
                cuda_check(cudaMemsetAsync(dprof.p, 0, (prog_.n_groups + 1) * 8, stream), "profile reset");
                p.prof = dprof.as<unsigned long long>();
            }
            cuda_check(launch_generic(p, grid_, k, std::min(n_steps, k + K), 0, stream, small_arena_floats_),
                       "generic kernel launch");
            if (prof) {
                std::vector<unsigned long long> h(prog_.n_groups);
                cuda_check(cudaMemcpyAsync(h.data(), dprof.p, h.size() * 8, cudaMemcpyDeviceToHost, stream), "prof");
                cuda_check(cudaStreamSynchronize(stream), "prof");
                const int nk = std::min(n_steps, k + K) - k;
                std::fprintf(stderr, "[generic profile] cycles per step per group (CTA 0):");
                for (int gi = 0; gi < prog_.n_groups; ++gi)
                    std::fprintf(stderr, " g%d:%s/f%d=%.0f", gi, op_kind_name(static_cast<OpKind>(prof_kinds_[gi] & 255)),
                                 prof_kinds_[gi] >> 8, static_cast<double>(h[gi]) / nk);
                std::fprintf(stderr, "\n");
                p.prof = nullptr;
            }
            ++last_launches_;
        }
    }
    // the descriptor upload must finish before the host vectors change again
    cuda_check(cudaStreamSynchronize(stream), "generic run");
}

void Engine::run_tc_dots(const TcGroup& tg, cudaStream_t stream) {
    for (const TcDotDesc& d : tg.dots) cuda_check(tc_dot_launch(d, stream), "tensor-core DotInc launch");
}

void Engine::run(int n_steps, int n_feeds, const neng_feed* feeds, double* probes_out) {
    // exec.cpp:340-366
    if (n_steps <= 0) throw RunError("n_steps must be positive");
    if (call_steps_) throw RunError("run: a stepped call is open");
    if (shard_count_ > 1) throw RunError("run: a sharded engine advances through neng_gpu_call_*");
    if (n_feeds < 0 || (n_feeds > 0 && !feeds)) throw InvalidArgument("bad feed array");
    validate_feeds(n_feeds, feeds, n_steps);
    const BuiltModel& m = pm_.model;
    const int B = batch_;
    // stage feeds as f32 [slot][step][dim][B] (the write_feeds cast, exec.cpp:323)
    std::vector<int> present(feeds_.size(), 0);
    std::vector<const neng_feed*> src(feeds_.size(), nullptr);
    int64_t feed_floats = 0;
    for (size_t f = 0; f < m.feed_slots.size(); ++f) {
        for (int i = 0; i < n_feeds; ++i)
            if (feeds[i].node_id == m.feed_slots[f].node_id) src[f] = &feeds[i];
        if (src[f]) {
            present[f] = 1;
            feed_floats += static_cast<int64_t>(n_steps) * feeds_[f].dim * B;
        }
    }
    int64_t ring_floats = 0;
    for (const DProbe& q : probes_) ring_floats += static_cast<int64_t>(n_steps) * q.dim * B;
    ring_.ensure(static_cast<size_t>(std::max<int64_t>(ring_floats, 1)) * sizeof(float));

    // Feeds: narrowed f64 -> f32 on the host cores in the host's own order ([b][step][dim],
    // contiguous per batch row), copied, and transposed to [step][dim][B] on the device, in
    // chunks of steps; with the fused pipeline chunk c+1 is staged while chunk c runs.
    std::vector<int64_t> full_off, ring_off;
    call_offsets(n_steps, present, &full_off, &ring_off);
    int64_t per_step = 0;  // floats per step over the present slots
    std::vector<size_t> slots;
    for (size_t f = 0; f < feeds_.size(); ++f)
        if (present[f]) {
            slots.push_back(f);
            per_step += static_cast<int64_t>(feeds_[f].dim) * B;
        }
    // chunk sizes grow geometrically from a small first chunk (the only staging
    // not overlapped with the kernel) to the largest staging buffer
    int cs = n_steps, cs0 = n_steps;
    if (fused_ && per_step > 0) {
        cs = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(n_steps, (int64_t{1} << 24) / per_step)));
        cs0 = std::max(1, std::min(cs, 4));
    }
    const int nbuf = cs0 < n_steps ? 2 : 1;
    feed_buf_.ensure(static_cast<size_t>(std::max<int64_t>(feed_floats, 1)) * sizeof(float));
    const size_t chunk_floats = static_cast<size_t>(std::max<int64_t>(per_step * cs, 1));
    feed_stage_.ensure(chunk_floats * nbuf * sizeof(float));
    feed_raw_.ensure(chunk_floats * nbuf * sizeof(float));
    const size_t meta_stride = (slots.size() * 20 + 16 + 15) / 16 * 16;  // 8-B aligned offsets in each half
    feed_meta_.ensure(meta_stride * nbuf);
    feed_meta_host_.ensure(meta_stride * nbuf);
    if (!feed_events_[0]) {
        cuda_check(cudaEventCreateWithFlags(&feed_events_[0], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&feed_events_[1], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&xpose_events_[0], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventCreateWithFlags(&xpose_events_[1], cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    double t_conv = 0.0;
    auto stage_chunk = [&](int c0, int c1, int buf) {
        if (slots.empty()) return;
        const int n = c1 - c0;
        float* stage = feed_stage_.as<float>() + chunk_floats * buf;
        float* raw = feed_raw_.as<float>() + chunk_floats * buf;
        cuda_check(cudaEventSynchronize(feed_events_[buf]), "feed staging buffer");  // its last copy is done
        std::vector<int64_t> offs(2 * slots.size());
        std::vector<int32_t> cols(slots.size());
        int64_t at = 0;
        for (size_t j = 0; j < slots.size(); ++j) {
            const size_t f = slots[j];
            offs[j] = at;
            offs[slots.size() + j] = full_off[f] + static_cast<int64_t>(c0) * feeds_[f].dim * B;
            cols[j] = n * feeds_[f].dim;
            at += static_cast<int64_t>(n) * feeds_[f].dim * B;
        }
        const int64_t rows = static_cast<int64_t>(slots.size()) * B;  // (slot, batch row) pieces
        auto work = [&](int64_t q0, int64_t q1) {
            for (int64_t q = q0; q < q1; ++q) {
                const size_t j = static_cast<size_t>(q / B);
                const int b = static_cast<int>(q % B);
                const neng_feed* t = src[slots[j]];
                const int64_t len = static_cast<int64_t>(n) * t->dim;
                const double* in = t->data + (static_cast<int64_t>(b) * t->steps + c0) * t->dim;
                float* out = stage + offs[j] + static_cast<int64_t>(b) * len;
                for (int64_t i = 0; i < len; ++i) out[i] = static_cast<float>(in[i]);
            }
        };
        const auto tc = std::chrono::steady_clock::now();
        const int64_t nt = std::min<int64_t>(rows, std::max(1u, std::thread::hardware_concurrency()));
        if (nt <= 1 || at < (int64_t{1} << 20)) {
            work(0, rows);
        } else {
            std::vector<std::thread> pool;
            for (int64_t t = 0; t < nt; ++t) pool.emplace_back(work, rows * t / nt, rows * (t + 1) / nt);
            for (auto& th : pool) th.join();
        }
        t_conv += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
        char* meta = feed_meta_.as<char>() + meta_stride * buf;
        // the copies run on their own stream so they overlap the previous chunk's kernel:
        // they wait for the last transpose that read raw/meta[buf], and the transpose
        // of this chunk waits for them
        cuda_check(cudaStreamWaitEvent(copy_stream_, xpose_events_[buf], 0), "feed copy wait");
        cuda_check(cudaMemcpyAsync(raw, stage, at * sizeof(float), cudaMemcpyHostToDevice, copy_stream_), "feed H2D");
        // the metadata goes through pinned memory too, so no copy on copy_stream_ waits for the host
        char* hmeta = feed_meta_host_.as<char>() + meta_stride * buf;
        std::memcpy(hmeta, offs.data(), offs.size() * 8);
        std::memcpy(hmeta + offs.size() * 8, cols.data(), cols.size() * 4);
        cuda_check(cudaMemcpyAsync(meta, hmeta, offs.size() * 8 + cols.size() * 4, cudaMemcpyHostToDevice, copy_stream_),
                   "feed meta");
        cuda_check(cudaEventRecord(feed_events_[buf], copy_stream_), "feed event");
        cuda_check(cudaStreamWaitEvent(stream_, feed_events_[buf], 0), "feed wait");
        const int max_cols = *std::max_element(cols.begin(), cols.end());
        cuda_check(launch_feed_transpose(raw, feed_buf_.as<float>(), reinterpret_cast<const int64_t*>(meta),
                                         reinterpret_cast<const int32_t*>(meta + offs.size() * 8),
                                         static_cast<int>(slots.size()), max_cols, B, stream_),
                   "feed transpose");
        cuda_check(cudaEventRecord(xpose_events_[buf], stream_), "transpose event");
    };
    const bool tprof = std::getenv("NENG_RUN_PROFILE") != nullptr;  // host-side phase times (stderr)
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_start = now();
    double t_stage = 0.0;
    if (fused_ && cs0 < n_steps) {
        fused_->begin(n_steps, feed_buf_.as<float>(), full_off.data(), present.data(), ring_.as<float>(),
                      ring_off.data(), stream_);
        last_launches_ = 0;
        for (int c0 = 0, i = 0, n = cs0; c0 < n_steps; c0 += n, n = std::min(cs, 2 * n), ++i) {
            const int c1 = std::min(n_steps, c0 + n);
            const auto t0 = now();
            stage_chunk(c0, c1, i & 1);
            t_stage += std::chrono::duration<double>(now() - t0).count();
            fused_->launch_chunk(c0, c1, stream_);
            ++last_launches_;
        }
    } else {
        stage_chunk(0, n_steps, 0);
        launch_steps(n_steps, feed_buf_.as<float>(), present, ring_.as<float>(), stream_);
    }

    const auto t_issued = now();
    if (tprof) {
        cuda_check(cudaStreamSynchronize(stream_), "run");
        std::fprintf(stderr,
                     "[run profile] %d steps in %lld launches (chunks %d..%d): staging %.1f ms (conversion %.1f), issue "
                     "%.1f ms, device done %.1f ms\n",
                     n_steps, static_cast<long long>(last_launches_), cs0, cs, t_stage * 1e3, t_conv * 1e3,
                     std::chrono::duration<double>(t_issued - t_start).count() * 1e3,
                     std::chrono::duration<double>(now() - t_start).count() * 1e3);
    }
    if (ring_floats) {
        // ring [probe][step][dim][B] -> [probe][B][step][dim], D2H, widen to f64
        std::vector<int64_t> off(probes_.size());
        std::vector<int32_t> dims(probes_.size());
        int64_t o = 0;
        for (size_t q = 0; q < probes_.size(); ++q) {
            off[q] = o;
            dims[q] = probes_[q].dim;
            o += static_cast<int64_t>(n_steps) * probes_[q].dim * B;
        }
        probe_meta_.ensure(probes_.size() * 12 + 16);
        cuda_check(cudaMemcpyAsync(probe_meta_.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice, stream_),
                   "probe meta");
        cuda_check(cudaMemcpyAsync(probe_meta_.as<char>() + off.size() * 8, dims.data(), dims.size() * 4,
                                   cudaMemcpyHostToDevice, stream_),
                   "probe meta");
        probe_out_.ensure(ring_floats * sizeof(float));
        cuda_check(launch_probe_transpose(ring_.as<float>(), probe_out_.as<float>(), probe_meta_.as<int64_t>(),
                                          reinterpret_cast<int32_t*>(probe_meta_.as<char>() + off.size() * 8),
                                          static_cast<int>(probes_.size()), n_steps, B, stream_),
                   "probe transpose");
        probe_stage_.ensure(ring_floats * sizeof(float));
        cuda_check(cudaMemcpyAsync(probe_stage_.p, probe_out_.p, ring_floats * sizeof(float), cudaMemcpyDeviceToHost,
                                   stream_),
                   "probe D2H");
        cuda_check(cudaStreamSynchronize(stream_), "run");
        if (probes_out) {
            const float* ps = probe_stage_.as<float>();
            for (int64_t i = 0; i < ring_floats; ++i) probes_out[i] = static_cast<double>(ps[i]);
        }
    } else {
        cuda_check(cudaStreamSynchronize(stream_), "run");
    }
    if (tprof)
        std::fprintf(stderr, "[run profile] total %.1f ms\n", std::chrono::duration<double>(now() - t_start).count() * 1e3);
    steps_done_ += n_steps;
    last_run_steps_ = n_steps;
}

// ---- probe export (export.cpp:53-101) from the last run's transposed probe block ----

namespace {
/// The traces ProbeOutput holds: one per key in key order (std::map); with a
/// key registered twice capture_probes leaves the last binding's values.
std::vector<int> export_order(const PlannedModel& pm) {
    std::map<int, int> last;
    for (size_t i = 0; i < pm.model.probes.size(); ++i) last[pm.model.probes[i].key] = static_cast<int>(i);
    std::vector<int> order;
    for (auto [k, i] : last) order.push_back(i);
    return order;
}
}  // namespace

int64_t Engine::probe_dump_bytes() const {
    if (last_run_steps_ <= 0) throw RunError("no probe traces: run() has not been called");
    int64_t n = 5 + 1 + 4;
    for (int i : export_order(pm_)) n += 16 + int64_t{8} * batch_ * last_run_steps_ * probe_dim(i);
    return n;
}

void Engine::probe_dump(char* out, int64_t capacity) const {
    const int64_t need = probe_dump_bytes();
    if (capacity < need) throw InvalidArgument("probe dump: output capacity too small");
    std::vector<int64_t> at(pm_.model.probes.size());  // float offset of probe i in the block
    int64_t o = 0;
    for (size_t i = 0; i < at.size(); ++i) {
        at[i] = o;
        o += int64_t{1} * batch_ * last_run_steps_ * probe_dim(static_cast<int>(i));
    }
    const float* blk = probe_stage_.as<float>();
    char* p = out;
    auto put = [&](const void* v, size_t n) {
        std::memcpy(p, v, n);
        p += n;
    };
    put("NENG1", 5);
    const uint8_t width = 8;
    put(&width, 1);
    const std::vector<int> order = export_order(pm_);
    const uint32_t count = static_cast<uint32_t>(order.size());
    put(&count, 4);
    for (int i : order) {
        const int32_t hdr[4] = {pm_.model.probes[i].key, batch_, last_run_steps_, probe_dim(i)};
        put(hdr, sizeof hdr);
        const int64_t n = int64_t{1} * batch_ * last_run_steps_ * probe_dim(i);  // (batch, step, dim) order
        for (int64_t j = 0; j < n; ++j) {
            const double v = static_cast<double>(blk[at[i] + j]);
            put(&v, 8);
        }
    }
}

std::string Engine::probe_csv(double dt) const {
    if (last_run_steps_ <= 0) throw RunError("no probe traces: run() has not been called");
    std::string s = "step,time,batch,probe_key,dim_index,value\n";
    const std::vector<int> order = export_order(pm_);
    if (order.empty()) return s;
    std::vector<int64_t> at(pm_.model.probes.size());
    int64_t o = 0;
    for (size_t i = 0; i < at.size(); ++i) {
        at[i] = o;
        o += int64_t{1} * batch_ * last_run_steps_ * probe_dim(static_cast<int>(i));
    }
    const float* blk = probe_stage_.as<float>();
    const int S = last_run_steps_;
    // rows by step, batch, key, dim; steps formatted in parallel blocks
    const int nt = static_cast<int>(std::max(1u, std::min(16u, std::thread::hardware_concurrency())));
    std::vector<std::string> part(nt);
    auto work = [&](int t) {
        std::string& r = part[t];
        char buf[64];
        for (int st = S * t / nt; st < S * (t + 1) / nt; ++st) {
            std::snprintf(buf, sizeof buf, "%.9g", (st + 1) * dt);
            const std::string stamp = std::to_string(st) + ',' + buf + ',';
            for (int b = 0; b < batch_; ++b)
                for (int i : order) {
                    const int D = probe_dim(i);
                    for (int d = 0; d < D; ++d) {
                        std::snprintf(buf, sizeof buf, "%.17g",
                                      static_cast<double>(blk[at[i] + (int64_t{1} * b * S + st) * D + d]));
                        r += stamp;
                        r += std::to_string(b);
                        r += ',';
                        r += std::to_string(pm_.model.probes[i].key);
                        r += ',';
                        r += std::to_string(d);
                        r += ',';
                        r += buf;
                        r += '\n';
                    }
                }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    for (auto& r : part) s += r;
    return s;
}

void Engine::device_call_args(int n_steps, const float* const* d_feeds, float* const* d_probes, const float** base_out,
                              std::vector<int>* present_out, float** ring_out) const {
    const BuiltModel& m = pm_.model;
    // feeds: per slot pointer -> gather offsets relative to the first present block
    std::vector<int>& present = *present_out;
    present.assign(feeds_.size(), 0);
    for (size_t f = 0; f < m.feed_slots.size(); ++f) {
        present[f] = d_feeds && d_feeds[f] ? 1 : 0;
        if (!present[f] && !m.feed_slots[f].has_default)
            throw RunError("node " + std::to_string(m.feed_slots[f].node_id) + " ('" + m.feed_slots[f].label +
                           "') has no default output and no feed was supplied");
    }
    // the device program addresses feed and probe blocks by offset from one
    // base; require the caller's blocks to be packed in model order
    const float* base = nullptr;
    int64_t expect = 0;
    for (size_t f = 0; f < feeds_.size(); ++f) {
        if (!present[f]) continue;
        if (!base) base = d_feeds[f];
        if (d_feeds[f] != base + expect) throw InvalidArgument("run_device: feed blocks must be packed in slot order");
        expect += static_cast<int64_t>(n_steps) * feeds_[f].dim * batch_;
    }
    float* ring = nullptr;
    int64_t rexp = 0;
    for (size_t q = 0; q < probes_.size(); ++q) {
        if (!d_probes || !d_probes[q]) throw InvalidArgument("run_device: every probe needs an output block");
        if (!ring) ring = d_probes[q];
        if (d_probes[q] != ring + rexp) throw InvalidArgument("run_device: probe blocks must be packed in order");
        rexp += static_cast<int64_t>(n_steps) * probes_[q].dim * batch_;
    }
    *base_out = base;
    *ring_out = ring;
}

void Engine::call_offsets(int n_steps, const std::vector<int>& present, std::vector<int64_t>* feed_off,
                          std::vector<int64_t>* ring_off) const {
    feed_off->assign(feeds_.size(), 0);
    ring_off->assign(probes_.size(), 0);
    int64_t at = 0;
    for (size_t f = 0; f < feeds_.size(); ++f) {
        (*feed_off)[f] = at;
        if (present[f]) at += static_cast<int64_t>(n_steps) * feeds_[f].dim * batch_;
    }
    at = 0;
    for (size_t q = 0; q < probes_.size(); ++q) {
        (*ring_off)[q] = at;
        at += static_cast<int64_t>(n_steps) * probes_[q].dim * batch_;
    }
}

void Engine::run_device(int n_steps, const float* const* d_feeds, float* const* d_probes, cudaStream_t stream) {
    if (n_steps <= 0) throw RunError("n_steps must be positive");
    if (call_steps_) throw RunError("run_device: a stepped call is open");
    if (shard_count_ > 1) throw RunError("run_device: a sharded engine advances through neng_gpu_call_*");
    if (!stream) stream = stream_;
    const float* base = nullptr;
    float* ring = nullptr;
    std::vector<int> present;
    device_call_args(n_steps, d_feeds, d_probes, &base, &present, &ring);
    launch_steps(n_steps, base, present, ring, stream);
    steps_done_ += n_steps;
    last_run_steps_ = 0;  // the probe block no longer holds the engine's latest traces
}

void Engine::call_begin(int n_steps, const float* const* d_feeds, float* const* d_probes, cudaStream_t stream) {
    if (n_steps <= 0) throw RunError("n_steps must be positive");
    if (!fused_) throw RunError("stepped calls need the fused pipeline");
    if (call_steps_) throw RunError("call_begin: a stepped call is already open");
    if (!stream) stream = stream_;
    const float* base = nullptr;
    float* ring = nullptr;
    std::vector<int> present;
    device_call_args(n_steps, d_feeds, d_probes, &base, &present, &ring);
    std::vector<int64_t> feed_off, ring_off;
    call_offsets(n_steps, present, &feed_off, &ring_off);
    fused_->begin(n_steps, base, feed_off.data(), present.data(), ring, ring_off.data(), stream);
    call_steps_ = n_steps;
    call_stream_ = stream;
    last_run_steps_ = 0;  // the probe block no longer holds the engine's latest traces
    last_launches_ = 0;
}

void Engine::call_step(int k, int flags) {
    if (!call_steps_) throw RunError("call_step: no stepped call is open");
    if (k < 0 || k > call_steps_ || (k == call_steps_ && !(flags & NENG_STEP_EPILOGUE)))
        throw RunError("call_step: step " + std::to_string(k) + " is outside the call");
    fused_->step(k, flags, call_stream_);
    ++last_launches_;
}

void Engine::call_end() {
    if (!call_steps_) throw RunError("call_end: no stepped call is open");
    cuda_check(cudaStreamSynchronize(call_stream_), "stepped call");
    steps_done_ += call_steps_;
    call_steps_ = 0;
}

void Engine::shard_layout(int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf) const {
    if (!fused_) throw RunError("shard_layout: the engine runs the generic interpreter");
    fused_->xhat_layout(xbuf_floats, rank_floats, xbuf);
}

void Engine::set_xhat_buffer(float* d_buf) {
    if (!fused_) throw RunError("set_xhat_buffer: the engine runs the generic interpreter");
    if (!d_buf) throw InvalidArgument("set_xhat_buffer: null buffer");
    if (call_steps_) throw RunError("set_xhat_buffer: a stepped call is open");
    fused_->set_xhat_buffer(d_buf);
}

int Engine::last_schedule() const { return fused_ ? fused_->sched : (last_launches_ ? NENG_SCHED_GENERIC : 0); }

void Engine::synchronize() { cuda_check(cudaStreamSynchronize(stream_), "synchronize"); }

std::vector<double> Engine::read_signal(int sig, int batch_index) const {
    // exec.cpp:368-377
    if (sig < 0 || sig >= static_cast<int>(pm_.model.signals.size())) throw RunError("read_signal: no such signal");
    if (batch_index < 0 || batch_index >= batch_) throw RunError("read_signal: batch index out of range");
    if (fused_) fused_->materialize(stream_);
    DArg a = resolve_full(sig);
    std::vector<float> tmp(static_cast<size_t>(std::max<int64_t>(a.elems, 1)));
    int b = a.bs ? batch_index : 0;
    if (a.elems) {
        const float* src = arena_.as<float>() + a.base + static_cast<int64_t>(b) * a.bs;
        cuda_check(cudaMemcpy2DAsync(tmp.data(), sizeof(float), src, static_cast<size_t>(a.es) * sizeof(float),
                                     sizeof(float), static_cast<size_t>(a.elems), cudaMemcpyDeviceToHost, stream_),
                   "read_signal D2H");
        cuda_check(cudaStreamSynchronize(stream_), "read_signal");
    }
    return std::vector<double>(tmp.begin(), tmp.begin() + a.elems);
}

int Engine::buffer_storage(int buffer) const {
    if (buffer < 0 || buffer >= static_cast<int>(bufs_.size())) throw RunError("buffer_storage: no such buffer");
    return bufs_[buffer].per_batch ? NENG_STORAGE_PER_BATCH : NENG_STORAGE_SHARED;
}

}  // namespace nengb
