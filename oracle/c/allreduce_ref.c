/* Plain threaded C oracle of the AllReduce result — TEST INFRASTRUCTURE ONLY.
 *
 * The same definition as oracle/allreduce.py (SURVEY.md §8(c) "Definition of
 * the result"): every rank ends with
 *     y[i] = op(... op(op(x_0[i], x_1[i]), x_2[i]) ..., x_{n-1}[i])
 * folded left to right in rank order, one element at a time.  Written as plain
 * loops (no intrinsics, no blocking, no reordering) and split over threads by
 * contiguous element ranges only, so it computes exactly what the numpy oracle
 * computes; SURVEY.md §8(d) "a plain threaded C++ variant (no intrinsics) on
 * all cores, cross-checked bit-exactly against numpy" — the CPU baseline timed
 * beside the GPU.  Compiled with -ffp-contract=off (no FMA) and without
 * -ffast-math: every float add is one IEEE binary32 RNE add.
 *   i32 / i64 : two's-complement wrap (computed unsigned), signed max / min
 *   f32       : binary32 adds in rank order; fmaxf / fminf
 *   bf16      : widen bits << 16, accumulate in binary32, round once (RNE)
 * Shares no code with the CUDA path.
 * Pinned by tests/test_oracle_cref.py (bit-exact against oracle/allreduce.py,
 * which is itself pinned by brute force and closed forms).
 */
#include <math.h>
#include <pthread.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

enum { DT_I32 = 2, DT_I64 = 4, DT_F32 = 7, DT_BF16 = 9 };   /* nccl.h numbering */
enum { OP_SUM = 0, OP_MAX = 2, OP_MIN = 3 };

typedef struct {
    const void* const* xs;
    void* y;
    size_t lo, hi;
    int n, dtype, op;
} job_t;

static float bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static uint16_t f32_to_bf16_rne(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

static void fold(const job_t* j) {
    const int n = j->n;
    for (size_t i = j->lo; i < j->hi; ++i) {
        switch (j->dtype) {
            case DT_I32: {
                uint32_t acc = ((const uint32_t*)j->xs[0])[i];
                for (int r = 1; r < n; ++r) {
                    uint32_t v = ((const uint32_t*)j->xs[r])[i];
                    if (j->op == OP_SUM) acc = acc + v;
                    else if (j->op == OP_MAX) acc = ((int32_t)v > (int32_t)acc) ? v : acc;
                    else acc = ((int32_t)v < (int32_t)acc) ? v : acc;
                }
                ((uint32_t*)j->y)[i] = acc;
                break;
            }
            case DT_I64: {
                uint64_t acc = ((const uint64_t*)j->xs[0])[i];
                for (int r = 1; r < n; ++r) {
                    uint64_t v = ((const uint64_t*)j->xs[r])[i];
                    if (j->op == OP_SUM) acc = acc + v;
                    else if (j->op == OP_MAX) acc = ((int64_t)v > (int64_t)acc) ? v : acc;
                    else acc = ((int64_t)v < (int64_t)acc) ? v : acc;
                }
                ((uint64_t*)j->y)[i] = acc;
                break;
            }
            case DT_F32: {
                float acc = ((const float*)j->xs[0])[i];
                for (int r = 1; r < n; ++r) {
                    float v = ((const float*)j->xs[r])[i];
                    if (j->op == OP_SUM) acc = acc + v;
                    else if (j->op == OP_MAX) acc = fmaxf(acc, v);
                    else acc = fminf(acc, v);
                }
                ((float*)j->y)[i] = acc;
                break;
            }
            case DT_BF16: {
                float acc = bf16_to_f32(((const uint16_t*)j->xs[0])[i]);
                for (int r = 1; r < n; ++r) {
                    float v = bf16_to_f32(((const uint16_t*)j->xs[r])[i]);
                    if (j->op == OP_SUM) acc = acc + v;
                    else if (j->op == OP_MAX) acc = fmaxf(acc, v);
                    else acc = fminf(acc, v);
                }
                ((uint16_t*)j->y)[i] = f32_to_bf16_rne(acc);
                break;
            }
        }
    }
}

static void* run(void* arg) {
    fold((const job_t*)arg);
    return NULL;
}

/* y = rank-ordered AllReduce of xs[0..n-1] (count elements each), computed by
 * `nthreads` threads over contiguous element ranges.  Returns 0, or -1 on bad
 * arguments. */
int oracle_allreduce(const void* const* xs, void* y, size_t count, int n, int dtype, int op, int nthreads) {
    if (n < 1 || n > 64 || nthreads < 1 || nthreads > 1024) return -1;
    if (dtype != DT_I32 && dtype != DT_I64 && dtype != DT_F32 && dtype != DT_BF16) return -1;
    if (op != OP_SUM && op != OP_MAX && op != OP_MIN) return -1;
    if (count == 0) return 0;
    job_t jobs[1024];
    pthread_t th[1024];
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].xs = xs;
        jobs[t].y = y;
        jobs[t].n = n;
        jobs[t].dtype = dtype;
        jobs[t].op = op;
        jobs[t].lo = count * (size_t)t / (size_t)nthreads;
        jobs[t].hi = count * (size_t)(t + 1) / (size_t)nthreads;
    }
    for (int t = 1; t < nthreads; ++t) {
        if (pthread_create(&th[t], NULL, run, &jobs[t]) != 0) break;
        started = t;
    }
    fold(&jobs[0]);
    for (int t = started + 1; t < nthreads; ++t) fold(&jobs[t]);   /* threads that failed to start */
    for (int t = 1; t <= started; ++t) pthread_join(th[t], NULL);
    return 0;
}
