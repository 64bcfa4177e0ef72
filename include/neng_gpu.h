/*
 * neng_gpu.h — C ABI of the B200 executor that drops in for the reference's
 * `neng::EngineCore<float>` (reference: proj/include/nengine/exec.hpp:18-120,
 * proj/src/exec.cpp:10-380).
 *
 * Everything crossing this boundary is plain C: POD views of the reference's
 * model types, caller-owned host buffers, status codes. No STL, no exceptions,
 * no torch types.  The engine owns its device memory.
 *
 *   reference C++                                  this ABI
 *   ---------------------------------------------  ----------------------------------
 *   neng::Signal            ir.hpp:37-58           neng_signal
 *   neng::SignalRef         ir.hpp:61-73           neng_ref
 *   neng::Operator          ir.hpp:114-137         neng_operator
 *   neng::ProbeRegistration model.hpp:35-39        neng_probe
 *   neng::FeedSlot          model.hpp:41-47        neng_feed_slot
 *   neng::BuiltModel        model.hpp:54-60        neng_built_model
 *   neng::BufferDesc        passes.hpp:63-70       neng_buffer_desc
 *   neng::PlannedModel      passes.hpp:131-137     neng_planned_model (plan + buffers)
 *   neng::Tensor3 (feed)    model.hpp:15-31        neng_feed
 *   EngineCore(planned, batch, unroll) exec.cpp:10-16   neng_gpu_create
 *   EngineCore::run         exec.cpp:340-366       neng_gpu_run / neng_gpu_run_device
 *   EngineCore::reset       exec.cpp:164-174       neng_gpu_reset
 *   EngineCore::read_signal exec.cpp:368-377       neng_gpu_read_signal
 *   EngineCore::buffer_storage exec.hpp:41-43      neng_gpu_buffer_storage
 *   EngineCore::{batch,unroll,steps_completed} exec.hpp:36-38  neng_gpu_{batch,unroll,steps_completed}
 *   StructuralError/BuildError/RunError ir.hpp:15-25  neng_status codes
 *
 * Host-side model tooling (validation, the merge planner) is exported by the
 * same library under neng_model_* / neng_plan_* — see neng_host.h.
 */
#ifndef NENG_GPU_H
#define NENG_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: map 1:1 onto the reference's exception types ---------- */
typedef enum neng_status {
    NENG_OK = 0,
    NENG_STRUCTURAL_ERROR = 1, /* neng::StructuralError  ir.hpp:15-17 */
    NENG_BUILD_ERROR = 2,      /* neng::BuildError       ir.hpp:19-21 */
    NENG_RUN_ERROR = 3,        /* neng::RunError         ir.hpp:23-25 */
    NENG_CUDA_ERROR = 4,       /* device failure (no reference equivalent) */
    NENG_OUT_OF_MEMORY = 5,
    NENG_INVALID_ARGUMENT = 6  /* null pointers, bad sizes at the ABI level */
} neng_status;

/* ---- IR enums: same order as the reference enums ------------------------- */
enum { /* neng::OpKind ir.hpp:78-87 */
    NENG_OP_RESET = 0,
    NENG_OP_COPY = 1,
    NENG_OP_ELEMENTWISE_INC = 2,
    NENG_OP_DOT_INC = 3,
    NENG_OP_SIM_NEURONS = 4,
    NENG_OP_SIM_PROCESS = 5,
    NENG_OP_SIM_PES = 6,
    NENG_OP_TIME_UPDATE = 7
};
enum { /* neng::NeuronKind ir.hpp:91 */
    NENG_NEURON_LIF = 0,
    NENG_NEURON_LIF_RATE = 1,
    NENG_NEURON_RECTIFIED_LINEAR = 2
};
enum { NENG_ELEM_F32 = 0, NENG_ELEM_F64 = 1 }; /* neng::Elem ir.hpp:27 */
enum { NENG_STORAGE_SHARED = 0, NENG_STORAGE_PER_BATCH = 1 }; /* exec.hpp:16 */

/* ---- model views (all pointers borrowed for the duration of the call) ---- */
typedef struct neng_signal {
    int32_t id;              /* must equal its index (BuiltModel is id-indexed) */
    int32_t ndim;
    const int32_t* shape;    /* shape[ndim], every dim >= 1 */
    int32_t elem;            /* NENG_ELEM_* */
    int64_t n_initial;       /* 0 = all zeros, else == prod(shape) */
    const double* initial;   /* flattened row-major */
    int32_t constant, minibatched, trainable;
    const char* label;       /* may be NULL */
} neng_signal;

typedef struct neng_ref { /* contiguous first-axis slice [start, stop) */
    int32_t signal, start, stop;
} neng_ref;

typedef struct neng_operator {
    int32_t id;
    int32_t kind;            /* NENG_OP_* */
    int32_t n_operands;
    const neng_ref* operands;
    int64_t n_value;         /* Reset payload */
    const double* value;
    int32_t inc;             /* Copy */
    int32_t neuron_kind;     /* SimNeurons: NENG_NEURON_* */
    double tau_rc, tau_ref, amplitude;
    double tau;              /* SimProcess (0 = passthrough) */
    double learning_rate;    /* SimPES */
    double dt;               /* TimeUpdate */
} neng_operator;

typedef struct neng_probe {
    int32_t key, signal;
    const char* label;
} neng_probe;

typedef struct neng_feed_slot {
    int32_t node_id, signal, dim, has_default;
    const char* label;
} neng_feed_slot;

typedef struct neng_built_model {
    int32_t n_signals;
    const neng_signal* signals;
    int32_t n_operators;
    const neng_operator* operators;
    int32_t n_probes;
    const neng_probe* probes;
    int32_t n_feed_slots;
    const neng_feed_slot* feed_slots;
    double dt;
} neng_built_model;

typedef struct neng_buffer_desc {
    int32_t n_trailing;
    const int32_t* trailing;
    int32_t elem, minibatched, trainable, rows;
    int32_t n_order;
    const int32_t* order;    /* signal ids in layout order */
} neng_buffer_desc;

typedef struct neng_planned_model {
    neng_built_model model;  /* operators AFTER simplification */
    int32_t n_groups;
    const int32_t* group_offsets; /* n_groups + 1 */
    const int32_t* group_members; /* operator ids, plan order then member order */
    const int32_t* buffer_of;     /* per signal */
    const int32_t* row_offset;    /* per signal */
    int32_t n_buffers;
    const neng_buffer_desc* buffers;
} neng_planned_model;

/* A Tensor3 feed view: data is [batch][steps][dim] row-major, f64. */
typedef struct neng_feed {
    int32_t node_id;
    int32_t batch, steps, dim;
    const double* data;
} neng_feed;

/* ---- device configuration ------------------------------------------------ */
enum {
    NENG_MODE_AUTO = 0,    /* fused ensemble pipeline when the model allows it */
    NENG_MODE_GENERIC = 1, /* one pass per plan group (any model) */
    NENG_MODE_FUSED = 2    /* require the fused pipeline; BuildError if impossible */
};

typedef struct neng_device_cfg {
    int32_t device;            /* CUDA ordinal */
    int32_t mode;              /* NENG_MODE_* */
    int32_t steps_per_launch;  /* K steps per persistent launch; 0 = engine default */
    /* Ensemble sharding (fused pipeline only; shard_count 0 or 1 = unsharded):
     * this engine owns shard shard_rank of shard_count contiguous ensemble
     * ranges and the connections into them; the caller all-gathers the xhat
     * parity buffer between per-step calls (neng_gpu_call_*). */
    int32_t shard_rank, shard_count;
    /* NENG_PRECISION_*: STRICT_FP32 (default) reproduces EngineCore<float> bit for
     * bit; TF32 and BF16X3 run dense DotInc groups (shared 2-D weights with K >= 32,
     * per-batch input and output, batch >= 32, 16-byte aligned rows) on the
     * tcgen05 tensor cores with fp32 accumulation in TMEM: TF32 products (10-bit
     * mantissa), or BF16X3 (each operand split into bf16 hi + lo, three MMAs:
     * ~16-bit products) — a stated tolerance instead of bit-exact results. */
    int32_t precision;
    int32_t reserved[2];
} neng_device_cfg;

enum { NENG_PRECISION_STRICT_FP32 = 0, NENG_PRECISION_TF32 = 1, NENG_PRECISION_BF16X3 = 2 };

typedef struct neng_engine neng_engine;

/* EngineCore<float>(PlannedModel planned, int batch = 1, int unroll = 1).
 * BuildError when batch < 1 or unroll < 1 (exec.cpp:11-12). cfg may be NULL. */
neng_status neng_gpu_create(const neng_planned_model* planned, int32_t batch, int32_t unroll,
                            const neng_device_cfg* cfg, neng_engine** out);
void neng_gpu_destroy(neng_engine* e);

/* EngineCore::run. feeds: one view per fed node; validated exactly like
 * validate_feeds (model.hpp:62-83) with the same messages. probes_out: caller
 * allocated, the concatenation over the model's probes in registration order
 * of [batch][n_steps][dim] f64 blocks (neng_gpu_probe_info gives the sizes). */
neng_status neng_gpu_run(neng_engine* e, int32_t n_steps, int32_t n_feeds,
                         const neng_feed* feeds, double* probes_out);

/* Device-resident variant (inputs already in HBM, outputs left in HBM).
 * d_feeds: per feed slot (model order) a [n_steps][dim][batch] f32 block, or
 * NULL for slots left at their current value; d_probes: per probe a
 * [n_steps][dim][batch] f32 block (may be NULL when the model has no probes).
 * stream: a cudaStream_t or NULL for the engine's stream. Returns after
 * enqueueing; call neng_gpu_synchronize to wait. */
neng_status neng_gpu_run_device(neng_engine* e, int32_t n_steps, const float* const* d_feeds,
                                float* const* d_probes, void* stream);
neng_status neng_gpu_synchronize(neng_engine* e);

/* Stepped device-resident call (the building block of sharded runs; same
 * buffers and packing as neng_gpu_run_device):
 *   neng_gpu_call_begin(e, n, feeds, probes, stream)
 *   for k in [0, n): neng_gpu_call_step(e, k, k ? NENG_STEP_FIRST_UPDATE : 0)
 *                    ... all-gather xhat parity buffer k & 1 across shards ...
 *   neng_gpu_call_step(e, n, NENG_STEP_EPILOGUE)   (completes step n - 1)
 *   neng_gpu_call_end(e)
 * Bits and state are those of one neng_gpu_run_device call. */
enum { NENG_STEP_FIRST_UPDATE = 1, NENG_STEP_EPILOGUE = 2 };
neng_status neng_gpu_call_begin(neng_engine* e, int32_t n_steps, const float* const* d_feeds, float* const* d_probes,
                                void* stream);
neng_status neng_gpu_call_step(neng_engine* e, int32_t k, int32_t flags);
neng_status neng_gpu_call_end(neng_engine* e);

/* The fused pipeline's xhat parity buffers: 2 x xbuf_floats/2 floats (parity p
 * at xbuf + p * xbuf_floats / 2); shard r's rows are the rank_floats floats at
 * r * rank_floats within a parity buffer (an in-place all-gather layout). */
neng_status neng_gpu_shard_layout(const neng_engine* e, int64_t* xbuf_floats, int64_t* rank_floats, float** xbuf);
/* Use a caller-owned device buffer (>= xbuf_floats floats) for the parity
 * buffers, e.g. one a collective library writes into. */
neng_status neng_gpu_set_xhat_buffer(neng_engine* e, float* d_buf);

neng_status neng_gpu_reset(neng_engine* e);

/* read_signal(sig, batch_index): RunError on a bad id or batch index. n_out
 * receives the element count; out may be NULL to query the size. */
neng_status neng_gpu_read_signal(const neng_engine* e, int32_t signal, int32_t batch_index,
                                 double* out, int64_t capacity, int64_t* n_out);

/* Probe export of the last neng_gpu_run call, replacing the reference's
 * write_probe_binary / write_probe_csv on the ProbeOutput that run returned
 * (export.hpp:17-25, export.cpp:53-101): the traces come from the engine's
 * device-transposed probe block, in key order, byte-identical to the
 * reference's output.  RunError before the first run. */
neng_status neng_gpu_probe_dump_size(const neng_engine* e, int64_t* bytes);           /* NENG1 size */
neng_status neng_gpu_probe_dump(const neng_engine* e, void* out, int64_t capacity);   /* NENG1 bytes */
neng_status neng_gpu_write_probe_binary(const neng_engine* e, const char* path);
neng_status neng_gpu_write_probe_csv(const neng_engine* e, const char* path, double dt);

neng_status neng_gpu_buffer_storage(const neng_engine* e, int32_t buffer, int32_t* mode_out);
int32_t neng_gpu_batch(const neng_engine* e);
int32_t neng_gpu_unroll(const neng_engine* e);
int32_t neng_gpu_steps_completed(const neng_engine* e);

/* probe i (registration order): key and dim */
neng_status neng_gpu_probe_info(const neng_engine* e, int32_t i, int32_t* key, int32_t* dim);
int32_t neng_gpu_num_probes(const neng_engine* e);

/* Which executor the engine compiled to: NENG_MODE_GENERIC or NENG_MODE_FUSED. */
int32_t neng_gpu_mode(const neng_engine* e);

/* Kernel launches issued by the most recent run call (for the bench). */
int64_t neng_gpu_last_launch_count(const neng_engine* e);

/* Schedules the most recent run / run_device / stepped call used (bit set):
 * the generic interpreter, the fused pipeline with one grid barrier per step,
 * the fused pipeline's barrier-free stepping, the fused step on one CTA
 * (programs too small to fill the GPU). */
#define NENG_SCHED_GENERIC 1
#define NENG_SCHED_FUSED_STEPPED 2
#define NENG_SCHED_FUSED_BARRIER_FREE 4
#define NENG_SCHED_FUSED_SMALL 8
int32_t neng_gpu_last_schedule(const neng_engine* e);

/* The tensor-core DotInc of the TF32 / BF16X3 precision modes on its own
 * (tc_dot.cu), for tests and measurement:  Y[m][n] += A[m][k] X[k][n] with
 * row-major host arrays (n, k multiples of 4; BF16X3: n, k multiples of 8).
 * mode: NENG_PRECISION_TF32 or NENG_PRECISION_BF16X3.  y receives the result
 * of one launch; *ms_out (may be NULL) = the mean device time of a launch over
 * `reps` further back-to-back launches (CUDA events), the split of X included
 * for BF16X3. */
neng_status neng_gpu_tc_dot(int32_t mode, int32_t m, int32_t k, int32_t n, const float* a, const float* x,
                            float* y, int32_t reps, double* ms_out);

/* Error text of the engine's last failing call ("" if none). */
const char* neng_gpu_last_error(const neng_engine* e);
/* Error text of the calling thread's last failing call (covers create). */
const char* neng_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NENG_GPU_H */
