/* oracle/engine_port.c — TEST INFRASTRUCTURE ONLY (the "port" oracle).
 *
 * A plain-C restatement of the reference executor neng::EngineCore<T>
 * (proj/src/exec.cpp, proj/include/nengine/exec.hpp) for T = float and
 * T = double, consuming the same neng_planned_model view as the product ABI.
 * It exists so the CPU algorithm is written down independently of both the
 * reference's C++ and the CUDA product: tests pin it bit-for-bit against the
 * reference build (oracle/_ref) and against the reference's golden vectors
 * (tests/golden/), then use it as a second checker.  Compiled with
 * -ffp-contract=off and no -march, like the reference's Release build, so the
 * float arithmetic rounds exactly as EngineCore<float> does (glibc
 * expm1f/log1pf included).  Never linked into the product.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "neng_gpu.h"

static _Thread_local char g_err[512];

static int fail(int status, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return status;
}

typedef struct {
    int buffer;
    long long offset;
    long long elems;
} PArg;

static long long signal_size(const neng_signal* s) {
    long long n = 1;
    for (int k = 0; k < s->ndim; ++k) n *= s->shape[k];
    return n;
}

/* Written operand positions of an operator (operand_modes ir.cpp:130-167,
 * every mode except Read). Returns the count. */
static int operand_write_positions(const neng_operator* op, int* pos) {
    int n = 0;
    switch (op->kind) {
    case NENG_OP_RESET: pos[n++] = 0; break;
    case NENG_OP_COPY: pos[n++] = 1; break;
    case NENG_OP_ELEMENTWISE_INC:
    case NENG_OP_DOT_INC: pos[n++] = 2; break;
    case NENG_OP_SIM_NEURONS:
        for (int i = 1; i < op->n_operands; ++i) pos[n++] = i;
        break;
    case NENG_OP_SIM_PROCESS:
        pos[n++] = 1;
        if (op->tau > 0.0) pos[n++] = 2;
        break;
    case NENG_OP_SIM_PES: pos[n++] = 2; break;
    case NENG_OP_TIME_UPDATE:
        pos[n++] = 0;
        pos[n++] = 1;
        break;
    }
    return n;
}

/* validate_feeds (model.hpp:62-83), same messages */
static int validate_feeds(const neng_built_model* m, int n_feeds, const neng_feed* feeds, int n_steps,
                          int batch) {
    /* FeedData is a std::map: iterate in ascending node id */
    int* order = (int*)malloc(sizeof(int) * (size_t)(n_feeds + 1));
    for (int i = 0; i < n_feeds; ++i) order[i] = i;
    for (int i = 1; i < n_feeds; ++i)
        for (int k = i; k > 0 && feeds[order[k - 1]].node_id > feeds[order[k]].node_id; --k) {
            int t = order[k];
            order[k] = order[k - 1];
            order[k - 1] = t;
        }
    for (int q = 0; q < n_feeds; ++q) {
        const neng_feed* t = &feeds[order[q]];
        const neng_feed_slot* slot = NULL;
        for (int s = 0; s < m->n_feed_slots; ++s)
            if (m->feed_slots[s].node_id == t->node_id) slot = &m->feed_slots[s];
        if (!slot) {
            char buf[128];
            snprintf(buf, sizeof buf, "feed for unknown node %d", t->node_id);
            free(order);
            return fail(NENG_RUN_ERROR, buf);
        }
        if (t->batch != batch || t->steps < n_steps || t->dim != slot->dim) {
            char buf[400];
            snprintf(buf, sizeof buf, "feed for node %d ('%s') has shape (%d, %d, %d), expected (%d, >=%d, %d)",
                     t->node_id, slot->label ? slot->label : "", t->batch, t->steps, t->dim, batch, n_steps,
                     slot->dim);
            free(order);
            return fail(NENG_RUN_ERROR, buf);
        }
    }
    free(order);
    for (int s = 0; s < m->n_feed_slots; ++s) {
        const neng_feed_slot* fs = &m->feed_slots[s];
        if (fs->has_default) continue;
        int found = 0;
        for (int q = 0; q < n_feeds; ++q) found |= feeds[q].node_id == fs->node_id;
        if (!found) {
            char buf[300];
            snprintf(buf, sizeof buf, "node %d ('%s') has no default output and no feed was supplied",
                     fs->node_id, fs->label ? fs->label : "");
            return fail(NENG_RUN_ERROR, buf);
        }
    }
    return NENG_OK;
}

#define T float
#define SFX(name) name##_f32
#define EXPM1 expm1f
#define LOG1P log1pf
#include "engine_port_core.inc"
#undef T
#undef SFX
#undef EXPM1
#undef LOG1P

#define T double
#define SFX(name) name##_f64
#define EXPM1 expm1
#define LOG1P log1p
#include "engine_port_core.inc"
#undef T
#undef SFX
#undef EXPM1
#undef LOG1P

typedef struct {
    int fp64;
    neng_built_model model; /* shallow copy for feed validation (pointers borrowed from creator) */
    /* deep-copied pieces used at run time */
    int n_slots;
    neng_feed_slot* slots;
    char** slot_labels;
    Engine_f32* f32;
    Engine_f64* f64;
} PortEngine;

const char* nport_last_error(void) { return g_err; }

int nport_create(const neng_planned_model* pm, int batch, int unroll, int fp64, PortEngine** out) {
    PortEngine* pe = (PortEngine*)calloc(1, sizeof(PortEngine));
    pe->fp64 = fp64;
    int st = fp64 ? create_f64(pm, batch, unroll, &pe->f64) : create_f32(pm, batch, unroll, &pe->f32);
    if (st) {
        free(pe);
        return st;
    }
    pe->n_slots = pm->model.n_feed_slots;
    pe->slots = (neng_feed_slot*)calloc((size_t)pe->n_slots + 1, sizeof(neng_feed_slot));
    pe->slot_labels = (char**)calloc((size_t)pe->n_slots + 1, sizeof(char*));
    for (int i = 0; i < pe->n_slots; ++i) {
        pe->slots[i] = pm->model.feed_slots[i];
        const char* l = pm->model.feed_slots[i].label ? pm->model.feed_slots[i].label : "";
        pe->slot_labels[i] = strdup(l);
        pe->slots[i].label = pe->slot_labels[i];
    }
    memset(&pe->model, 0, sizeof pe->model);
    pe->model.n_feed_slots = pe->n_slots;
    pe->model.feed_slots = pe->slots;
    *out = pe;
    return NENG_OK;
}

int nport_run(PortEngine* pe, int n_steps, int n_feeds, const neng_feed* feeds, double* probes_out) {
    if (n_steps <= 0) return fail(NENG_RUN_ERROR, "n_steps must be positive");
    int batch = pe->fp64 ? pe->f64->batch : pe->f32->batch;
    int st = validate_feeds(&pe->model, n_feeds, feeds, n_steps, batch);
    if (st) return st;
    return pe->fp64 ? run_f64(pe->f64, NULL, n_steps, n_feeds, feeds, probes_out)
                    : run_f32(pe->f32, NULL, n_steps, n_feeds, feeds, probes_out);
}

int nport_reset(PortEngine* pe) {
    if (pe->fp64)
        reset_f64(pe->f64);
    else
        reset_f32(pe->f32);
    return NENG_OK;
}

/* read_signal (exec.cpp:368-377) */
int nport_read_signal(const PortEngine* pe, int sig, int b, double* out, long long capacity, long long* n_out) {
    int nsig = pe->fp64 ? pe->f64->nsig : pe->f32->nsig;
    int batch = pe->fp64 ? pe->f64->batch : pe->f32->batch;
    if (sig < 0 || sig >= nsig) return fail(NENG_RUN_ERROR, "read_signal: no such signal");
    if (b < 0 || b >= batch) return fail(NENG_RUN_ERROR, "read_signal: batch index out of range");
    if (pe->fp64) {
        Engine_f64* e = pe->f64;
        PArg a = e->sig_arg[sig];
        *n_out = a.elems;
        if (out) {
            if (capacity < a.elems) return fail(NENG_INVALID_ARGUMENT, "capacity too small");
            double* src = ptr_f64(e, a, e->store[a.buffer].stride > 0 ? b : 0);
            for (long long i = 0; i < a.elems; ++i) out[i] = src[i];
        }
    } else {
        Engine_f32* e = pe->f32;
        PArg a = e->sig_arg[sig];
        *n_out = a.elems;
        if (out) {
            if (capacity < a.elems) return fail(NENG_INVALID_ARGUMENT, "capacity too small");
            float* src = ptr_f32(e, a, e->store[a.buffer].stride > 0 ? b : 0);
            for (long long i = 0; i < a.elems; ++i) out[i] = (double)src[i];
        }
    }
    return NENG_OK;
}

int nport_steps_completed(const PortEngine* pe) { return pe->fp64 ? pe->f64->steps_done : pe->f32->steps_done; }

int nport_buffer_storage(const PortEngine* pe, int buffer) {
    long long stride = pe->fp64 ? pe->f64->store[buffer].stride : pe->f32->store[buffer].stride;
    return stride > 0 ? NENG_STORAGE_PER_BATCH : NENG_STORAGE_SHARED;
}

void nport_destroy(PortEngine* pe) {
    if (!pe) return;
    if (pe->fp64)
        destroy_f64(pe->f64);
    else
        destroy_f32(pe->f32);
    for (int i = 0; i < pe->n_slots; ++i) free(pe->slot_labels[i]);
    free(pe->slot_labels);
    free(pe->slots);
    free(pe);
}
