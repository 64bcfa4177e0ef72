/* oracle/libm_host.c — TEST INFRASTRUCTURE ONLY.
 * The host glibc expm1f / log1pf that the reference's EngineCore<float> calls
 * (neuron_math.hpp:62,67,15), evaluated over a contiguous range of IEEE-754
 * bit patterns with all host threads.  tests/test_libm_parity.py compares the
 * device's parity functions against this, exhaustively. */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

typedef struct { int func; uint32_t lo; int64_t begin, end; uint32_t* out; } Job;

static void* work(void* p) {
    Job* j = (Job*)p;
    for (int64_t i = j->begin; i < j->end; ++i) {
        uint32_t k = j->lo + (uint32_t)i;
        float x, r;
        memcpy(&x, &k, 4);
        r = j->func == 0 ? expm1f(x) : log1pf(x);
        memcpy(&j->out[i], &r, 4);
    }
    return NULL;
}

/* func 0 = expm1f, 1 = log1pf; out[i] = bits(f(bits_to_float(lo + i))) */
void nlibm_eval(int func, uint32_t lo, int64_t n, uint32_t* out, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    Job jobs[256];
    for (int t = 0; t < threads; ++t) {
        jobs[t].func = func;
        jobs[t].lo = lo;
        jobs[t].begin = n * t / threads;
        jobs[t].end = n * (t + 1) / threads;
        jobs[t].out = out;
        pthread_create(&tid[t], NULL, work, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}
