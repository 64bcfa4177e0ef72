/* gen_libm_tables.c — build-time calibration of the host libm.
 *
 * The reference's EngineCore<float> calls glibc's expm1f/log1pf inside the
 * LIF step (proj/include/nengine/neuron_math.hpp:62,67) and log1pf inside the
 * LIFRate curve (:15).  Those glibc routines are not correctly rounded: on
 * glibc 2.39 about 0.2-23% of inputs (by binade) round one ulp away from
 * (float)f((double)x).  The device computes (float)f((double)x) and patches
 * the exceptions from this table, which is produced by sweeping every float in
 * the ranges the engine can feed these functions and recording, black-box,
 * where the host's float result differs from the host's double-then-round.
 *
 * Tables (keys = IEEE-754 bit patterns, ascending):
 *   0  expm1f  x in [-104, 0)   (LIF: x = -delta/tau_rc; below -104 both give -1)
 *   1  log1pf  x in [-1, 0)     (LIF spike time: x = -(v-1)/(j-1))
 *   2  log1pf  x in (0, +inf)   (LIFRate: x = 1/(j-1))
 * plus, on the LIF range x in [-1/16, 0), every input where the device's
 * speculative polynomial (libm_fast.h) rounds differently from glibc although
 * glibc is not an exception there (code 2), and, per table, any keys listed in
 * device_overrides.txt (inputs where the device's double-then-round was found
 * to differ from the host's).
 *
 * File format (little endian):
 *   "NENGLIBM" u32 version=4 u32 n_tables
 *   per table: u32 index, u32 count, f64 tmin, f64 tmin on [-1/16,0),
 *              u32 n_regions, u32 region_shift, f32 region tmin[n_regions],
 *              u64 n_key_bytes, varint key deltas,
 *              2-bit codes (0: host_dtr-1ulp, 1: host_dtr+1ulp, 2: host_dtr), 4 per byte
 * Usage: gen_libm_tables OUT [THREADS] [OVERRIDES]
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../kernels/libm_fast.h"

static float f_of(uint32_t u) {
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static uint32_t u_of(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
}

/* host results: glibc float function and double-then-round */
static uint32_t host_f(int func, uint32_t key) {
    float x = f_of(key);
    return func == 0 ? u_of(expm1f(x)) : u_of(log1pf(x));
}
static uint32_t host_dtr(int func, uint32_t key) {
    float x = f_of(key);
    return func == 0 ? u_of((float)expm1((double)x)) : u_of((float)log1p((double)x));
}

typedef struct {
    int func;
    uint32_t lo, hi; /* inclusive key range */
    uint32_t* keys;
    uint8_t* codes;
    size_t n, cap;
} Job;

static void push(Job* j, uint32_t key, uint8_t code) {
    if (j->n == j->cap) {
        j->cap = j->cap ? j->cap * 2 : 4096;
        j->keys = realloc(j->keys, j->cap * sizeof(uint32_t));
        j->codes = realloc(j->codes, j->cap);
    }
    j->keys[j->n] = key;
    j->codes[j->n] = code;
    j->n++;
}

/* the device's speculative value on the LIF range (libm_fast.h) */
static uint32_t host_fast(int func, uint32_t key) {
    double x = (double)f_of(key);
    return u_of((float)(func == 0 ? neng_expm1_fast(x) : neng_log1p_fast(x)));
}

static void* sweep(void* arg) {
    Job* j = (Job*)arg;
    for (uint64_t u = j->lo; u <= j->hi; ++u) {
        uint32_t a = host_f(j->func, (uint32_t)u), b = host_dtr(j->func, (uint32_t)u);
        if (a == b) {
            /* not an exception, but the speculative polynomial rounds the other
             * way: listed (code 2) so the device's fix-up resolves it exactly */
            if (u >= 0x80000001u && u <= 0xBD800000u && host_fast(j->func, (uint32_t)u) != a) push(j, (uint32_t)u, 2);
            continue;
        }
        int64_t d = (int64_t)a - (int64_t)b;
        if (d != 1 && d != -1) {
            fprintf(stderr, "func %d key %08x: glibc differs from double-then-round by %lld ulp\n", j->func,
                    (unsigned)u, (long long)d);
            exit(2);
        }
        push(j, (uint32_t)u, d < 0 ? 0 : 1);
    }
    return NULL;
}

typedef struct {
    uint32_t* keys;
    uint8_t* codes;
    size_t n;
} Table;

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

static Table run_table(int func, uint32_t lo, uint32_t hi, int threads) {
    Job* jobs = calloc((size_t)threads, sizeof(Job));
    pthread_t* tid = calloc((size_t)threads, sizeof(pthread_t));
    /* negative-float patterns ascend with |x|; split evenly by key */
    uint64_t span = (uint64_t)hi - lo + 1;
    for (int t = 0; t < threads; ++t) {
        jobs[t].func = func;
        jobs[t].lo = (uint32_t)(lo + span * t / threads);
        jobs[t].hi = (uint32_t)(lo + span * (t + 1) / threads - 1);
        pthread_create(&tid[t], NULL, sweep, &jobs[t]);
    }
    Table tb = {0};
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    for (int t = 0; t < threads; ++t) tb.n += jobs[t].n;
    tb.keys = malloc((tb.n + 1) * sizeof(uint32_t));
    tb.codes = malloc(tb.n + 1);
    size_t at = 0;
    for (int t = 0; t < threads; ++t) {
        memcpy(tb.keys + at, jobs[t].keys, jobs[t].n * sizeof(uint32_t));
        memcpy(tb.codes + at, jobs[t].codes, jobs[t].n);
        at += jobs[t].n;
        free(jobs[t].keys);
        free(jobs[t].codes);
    }
    free(jobs);
    free(tid);
    return tb;
}

/* merge override keys (func, key) into a table: code 2 = host dtr, or the
 * real glibc correction if the key is an exception anyway */
static void add_overrides(Table* tb, int func, const char* path) {
    if (!path) return;
    FILE* f = fopen(path, "r");
    if (!f) return;
    char line[256];
    size_t extra = 0;
    uint32_t* add = NULL;
    while (fgets(line, sizeof line, f)) {
        unsigned fn, key;
        if (line[0] == '#') continue;
        if (sscanf(line, "%u %x", &fn, &key) != 2 || (int)fn != func) continue;
        add = realloc(add, (extra + 1) * sizeof(uint32_t));
        add[extra++] = key;
    }
    fclose(f);
    if (!extra) return;
    qsort(add, extra, sizeof(uint32_t), cmp_u32);
    uint32_t* keys = malloc((tb->n + extra) * sizeof(uint32_t));
    uint8_t* codes = malloc(tb->n + extra);
    size_t i = 0, k = 0, o = 0;
    while (i < tb->n || k < extra) {
        if (k >= extra || (i < tb->n && tb->keys[i] <= add[k])) {
            if (k < extra && tb->keys[i] == add[k]) ++k; /* already present */
            keys[o] = tb->keys[i];
            codes[o++] = tb->codes[i++];
        } else {
            if (o == 0 || keys[o - 1] != add[k]) {
                keys[o] = add[k];
                codes[o++] = 2;
            }
            ++k;
        }
    }
    free(tb->keys);
    free(tb->codes);
    free(add);
    tb->keys = keys;
    tb->codes = codes;
    tb->n = o;
}

/* Distance (in float ulps) of the double result from the float it rounds
 * to, for the smallest such distance among a table's exceptions.  glibc's
 * float routines are ~0.53 ulp accurate, so every exception lies near a
 * rounding midpoint (t close to 0.5); the device skips the table lookup when
 * its own t is below this minimum (minus a margin). */
static double exception_tmin(int func, const Table* tb, int hot_only) {
    double tmin = 0.5;
    for (size_t i = 0; i < tb->n; ++i) {
        float x = f_of(tb->keys[i]);
        if (hot_only && !(x >= -0.0625f && x < 0.0f)) continue;
        double y = func == 0 ? expm1((double)x) : log1p((double)x);
        float r = (float)y;
        float up = nextafterf(r, INFINITY), dn = nextafterf(r, -INFINITY);
        double ulp = (double)up - (double)r;
        if (y < (double)r) ulp = (double)r - (double)dn;
        if (!(ulp > 0)) continue;
        double t = fabs(y - (double)r) / ulp;
        if (t < tmin) tmin = t;
    }
    return tmin;
}

/* Per-region minimum exception distance over the LIF range x in [-1/16, 0)
 * (bit patterns 0x80000001..0xBD800000, region = (key - 0x80000000) >> 18):
 * 1.0 for regions without exceptions.  Lets the device skip ~2/3 of the
 * probes the single hot-range bound would take. */
#define REGION_SHIFT 18
#define REGIONS (((0xBD800000u - 0x80000000u) >> REGION_SHIFT) + 1)
static void region_tmin(int func, const Table* tb, float* out) {
    for (unsigned i = 0; i < REGIONS; ++i) out[i] = 1.0f;
    for (size_t i = 0; i < tb->n; ++i) {
        uint32_t k = tb->keys[i];
        if (k < 0x80000001u || k > 0xBD800000u) continue;
        float x = f_of(k);
        double y = func == 0 ? expm1((double)x) : log1p((double)x);
        float r = (float)y;
        float up = nextafterf(r, INFINITY), dn = nextafterf(r, -INFINITY);
        double ulp = y < (double)r ? (double)r - (double)dn : (double)up - (double)r;
        if (!(ulp > 0)) continue;
        double t = fabs(y - (double)r) / ulp;
        unsigned reg = (k - 0x80000000u) >> REGION_SHIFT;
        if (t < out[reg]) out[reg] = (float)t;
    }
}

static void write_table(FILE* out, int func, const Table* tb, double tmin, double tmin_hot) {
    uint8_t* kb = malloc(tb->n * 5 + 16);
    size_t nk = 0;
    uint32_t prev = 0;
    for (size_t i = 0; i < tb->n; ++i) {
        uint32_t d = tb->keys[i] - prev;
        prev = tb->keys[i];
        do {
            uint8_t b = d & 0x7f;
            d >>= 7;
            kb[nk++] = (uint8_t)(b | (d ? 0x80 : 0));
        } while (d);
    }
    uint32_t hdr[2] = {(uint32_t)func, (uint32_t)tb->n};
    uint64_t nkb = nk;
    fwrite(hdr, 4, 2, out);
    fwrite(&tmin, 8, 1, out);
    fwrite(&tmin_hot, 8, 1, out);
    {
        static float reg[REGIONS];
        uint32_t rh[2] = {REGIONS, REGION_SHIFT};
        region_tmin(func == 0 ? 0 : 1, tb, reg);
        fwrite(rh, 4, 2, out);
        fwrite(reg, 4, REGIONS, out);
    }
    fwrite(&nkb, 8, 1, out);
    fwrite(kb, 1, nk, out);
    size_t ncb = (tb->n + 3) / 4;
    uint8_t* cb = calloc(ncb + 1, 1);
    for (size_t i = 0; i < tb->n; ++i) cb[i / 4] |= (uint8_t)(tb->codes[i] << (2 * (i % 4)));
    fwrite(cb, 1, ncb, out);
    free(kb);
    free(cb);
}

int main(int argc, char** argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s OUT [THREADS] [OVERRIDES]\n", argv[0]);
        return 1;
    }
    int threads = argc > 2 ? atoi(argv[2]) : 8;
    if (threads < 1) threads = 1;
    const char* overrides = argc > 3 ? argv[3] : NULL;
    struct {
        int func;
        uint32_t lo, hi;
    } spec[3] = {
        {0, 0x80000001u, 0xC2D00000u}, /* expm1f over [-104, 0) */
        {1, 0x80000001u, 0xBF800000u}, /* log1pf over [-1, 0)   */
        {1, 0x00000001u, 0x7F7FFFFFu}, /* log1pf over (0, FLT_MAX] */
    };
    char tmp[4096];
    snprintf(tmp, sizeof tmp, "%s.tmp", argv[1]);
    FILE* out = fopen(tmp, "wb");
    if (!out) {
        perror("open");
        return 1;
    }
    fwrite("NENGLIBM", 1, 8, out);
    uint32_t ver[2] = {4, 3};
    fwrite(ver, 4, 2, out);
    for (int t = 0; t < 3; ++t) {
        Table tb = run_table(spec[t].func, spec[t].lo, spec[t].hi, threads);
        /* overrides are keyed by table index */
        add_overrides(&tb, t, overrides);
        double tmin = exception_tmin(spec[t].func, &tb, 0);
        double tmin_hot = exception_tmin(spec[t].func, &tb, 1);
        write_table(out, t, &tb, tmin, tmin_hot);
        fprintf(stderr, "table %d: %zu entries, min exception distance %.4f ulp (%.4f on [-1/16, 0))\n", t, tb.n,
                tmin, tmin_hot);
        free(tb.keys);
        free(tb.codes);
    }
    fclose(out);
    if (rename(tmp, argv[1])) {
        perror("rename");
        return 1;
    }
    return 0;
}
