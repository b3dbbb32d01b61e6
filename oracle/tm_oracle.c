/*
 * tm_oracle.c -- CPU restatement of the reference Tsetlin-machine hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: it is linked
 * only by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  The product path (paper_2405_04212_b200) never
 * loads it and fails loudly when its CUDA library is missing.
 *
 * It restates, in plain C, the algorithm of the reference package
 * `tsetlinkit` (pure Python + numba, /root/reference/pkg/src/tsetlinkit).
 * The arithmetic lives in the reference's own files (numba 0.65 / numpy 2.3
 * only compile / vectorise it; no library numerics are involved), and each
 * function below cites the file:line it follows.  The restatement is pinned
 * against golden vectors produced by importing the reference itself
 * (tests/golden/make_golden.py writes the .npz fixtures, checked by
 * tests/test_oracle_golden.py) and against the reference's own known-answer
 * values (test_core.py:104-106, :132-137).
 *
 * Where the two reference backends differ on inputs outside the documented
 * state range (numpy clips the whole row, numba only guards the moved
 * position: kernels/_numpy.py:63 vs kernels/_numba.py:78-86) the oracle
 * follows numba, the reference's default backend (kernels/__init__.py:31-44).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

#define OR_GOLDEN 0x9E3779B97F4A7C15ULL
#define OR_C1 0xBF58476D1CE4E5B9ULL
#define OR_C2 0x94D049BB133111EBULL
#define OR_INV53 (1.0 / 9007199254740992.0) /* 2^-53 */

/* Minimal pthread parallel-for over [0, n): harness parallelism for the CPU
 * baseline (the reference shards its nogil numba kernels the same way). */
typedef void (*or_range_fn)(void *ctx, int64_t lo, int64_t hi);
typedef struct { or_range_fn fn; void *ctx; int64_t lo, hi; } or_job;
static void *or_job_main(void *p) {
    or_job *j = (or_job *)p;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}
static void or_parallel_for(int64_t n, int nthreads, or_range_fn fn, void *ctx) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads == 1 || n < 2 * nthreads) { fn(ctx, 0, n); return; }
    pthread_t th[256];
    or_job jobs[256];
    for (int t = 0; t < nthreads; ++t) {
        jobs[t].fn = fn; jobs[t].ctx = ctx;
        jobs[t].lo = n * t / nthreads; jobs[t].hi = n * (t + 1) / nthreads;
        pthread_create(&th[t], NULL, or_job_main, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

/* ---------------------------------------------------------------- RNG -- */

/* core.py:66-71 */
uint64_t or_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * OR_C1;
    z = (z ^ (z >> 27)) * OR_C2;
    return z ^ (z >> 31);
}

/* core.py:74-85 */
uint64_t or_derive_stream(uint64_t seed, uint64_t index) {
    uint64_t v = index + 1;
    uint64_t rot = (v << 32) | (v >> 32);
    return or_mix64(seed ^ rot);
}

/* core.py:88-90 */
uint64_t or_stream_u64(uint64_t seed, uint64_t k) {
    return or_mix64(seed + OR_GOLDEN * (k + 1));
}

/* core.py:93-95 */
double or_stream_u01(uint64_t seed, uint64_t k) {
    return (double)(or_stream_u64(seed, k) >> 11) * OR_INV53;
}

/* core.py:98-109 */
void or_stream_u64_block(uint64_t seed, uint64_t start, int64_t count, uint64_t *out) {
    for (int64_t i = 0; i < count; ++i) out[i] = or_stream_u64(seed, start + (uint64_t)i);
}

void or_stream_u01_block(uint64_t seed, uint64_t start, int64_t count, double *out) {
    for (int64_t i = 0; i < count; ++i) out[i] = or_stream_u01(seed, start + (uint64_t)i);
}

/* ----------------------------------------------------------- clause eval -- */

/* kernels/_numba.py:36-50 (and dense.evaluate_clause, dense.py:29-48) */
static uint8_t one_output(const int8_t *row, int64_t P, const uint8_t *lits,
                          int training, int64_t budget) {
    int64_t n_inc = 0;
    for (int64_t k = 0; k < P; ++k) {
        if (row[k] >= 0) {
            if (lits[k] == 0) return 0;
            ++n_inc;
        }
    }
    if (training) return n_inc > budget ? 0 : 1;
    return n_inc == 0 ? 0 : 1;
}

/* kernels/_numba.py:53-58 */
void or_clause_outputs(const int8_t *states, int64_t C, int64_t P,
                       const uint8_t *lits, int training, int64_t budget,
                       uint8_t *out) {
    for (int64_t j = 0; j < C; ++j)
        out[j] = one_output(states + j * P, P, lits, training, budget);
}

/* kernels/_numba.py:61-68; parallel over examples (harness parallelism) */
typedef struct {
    const int8_t *states; int64_t C, P; const uint8_t *x_lit; int training;
    int64_t budget; uint8_t *out;
} or_cob_ctx;
static void or_cob_range(void *p, int64_t lo, int64_t hi) {
    or_cob_ctx *c = (or_cob_ctx *)p;
    for (int64_t e = lo; e < hi; ++e)
        for (int64_t j = 0; j < c->C; ++j)
            c->out[e * c->C + j] = one_output(c->states + j * c->P, c->P,
                                              c->x_lit + e * c->P, c->training, c->budget);
}
void or_clause_outputs_batch(const int8_t *states, int64_t C, int64_t P,
                             const uint8_t *x_lit, int64_t N, int training,
                             int64_t budget, uint8_t *out, int nthreads) {
    or_cob_ctx c = {states, C, P, x_lit, training, budget, out};
    or_parallel_for(N, nthreads, or_cob_range, &c);
}

static void or_argmax_store(const int64_t *v, int64_t K, int64_t e, int64_t *votes, int64_t *pred) {
    if (votes) memcpy(votes + e * K, v, sizeof(int64_t) * (size_t)K);
    if (pred) {
        int64_t best = 0;
        for (int64_t k = 1; k < K; ++k) if (v[k] > v[best]) best = k;
        pred[e] = best;
    }
}

/* dense.py:171-174 (batch_votes) followed by executor.py:382 (argmax, ties
 * to the lowest class as np.argmax does).  votes / pred may be NULL. */
typedef struct {
    const int8_t *states; const int32_t *weights; int64_t C, P, K;
    const uint8_t *x_lit; int64_t *votes, *pred;
} or_bv_ctx;
static void or_bv_range(void *p, int64_t lo, int64_t hi) {
    or_bv_ctx *c = (or_bv_ctx *)p;
    int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)c->K);
    for (int64_t e = lo; e < hi; ++e) {
        for (int64_t k = 0; k < c->K; ++k) v[k] = 0;
        for (int64_t j = 0; j < c->C; ++j)
            if (one_output(c->states + j * c->P, c->P, c->x_lit + e * c->P, 0, c->P))
                for (int64_t k = 0; k < c->K; ++k) v[k] += c->weights[j * c->K + k];
        or_argmax_store(v, c->K, e, c->votes, c->pred);
    }
    free(v);
}
void or_batch_votes(const int8_t *states, const int32_t *weights, int64_t C,
                    int64_t P, int64_t K, const uint8_t *x_lit, int64_t N,
                    int64_t *votes, int64_t *pred, int nthreads) {
    or_bv_ctx c = {states, weights, C, P, K, x_lit, votes, pred};
    or_parallel_for(N, nthreads, or_bv_range, &c);
}

/* Include-list (RuleSet) inference: predictor.py:79-91.  Rules are given in
 * CSR form: rule r includes positions inc_idx[inc_ptr[r] .. inc_ptr[r+1]).
 * x is the RAW feature matrix [N, F]; augment_literals (core.py:232-242) is
 * applied implicitly: position p < F is x[p], p >= F is 1 - x[p - F]. */
typedef struct {
    const int64_t *inc_ptr, *inc_idx; int64_t R; const int32_t *weights; int64_t K;
    const uint8_t *x; int64_t F; int negations; int64_t *votes, *pred;
} or_rs_ctx;
static void or_rs_range(void *p, int64_t lo, int64_t hi) {
    or_rs_ctx *c = (or_rs_ctx *)p;
    int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)c->K);
    for (int64_t e = lo; e < hi; ++e) {
        const uint8_t *xe = c->x + e * c->F;
        for (int64_t k = 0; k < c->K; ++k) v[k] = 0;
        for (int64_t r = 0; r < c->R; ++r) {
            int fire = 1;
            for (int64_t q = c->inc_ptr[r]; q < c->inc_ptr[r + 1]; ++q) {
                int64_t pos = c->inc_idx[q];
                uint8_t lit = (c->negations && pos >= c->F) ? (uint8_t)(1 - xe[pos - c->F]) : xe[pos];
                if (lit == 0) { fire = 0; break; }
            }
            if (fire) for (int64_t k = 0; k < c->K; ++k) v[k] += c->weights[r * c->K + k];
        }
        or_argmax_store(v, c->K, e, c->votes, c->pred);
    }
    free(v);
}
void or_ruleset_votes(const int64_t *inc_ptr, const int64_t *inc_idx, int64_t R,
                      const int32_t *weights, int64_t K, const uint8_t *x,
                      int64_t N, int64_t F, int negations, int64_t *votes,
                      int64_t *pred, int nthreads) {
    or_rs_ctx c = {inc_ptr, inc_idx, R, weights, K, x, F, negations, votes, pred};
    or_parallel_for(N, nthreads, or_rs_range, &c);
}

/* ------------------------------------------------------------- feedback -- */

typedef struct {
    double s;
    int boost;
    int state_min, state_max;
} or_fb_params;

/* kernels/_numba.py:71-90.  u01 draw for position k is supplied either by
 * the stream (draws == NULL: stream_u01(seed, base + k)) or by an explicit
 * row (draws != NULL: draws[k]) -- the explicit-draws test hook.  The stream
 * loop is written branch-free so the compiler vectorises the 64-bit
 * SplitMix64 arithmetic the way numba/LLVM does for the reference (AVX-512DQ
 * vpmullq); target_clones keeps the .so portable across host CPUs. */
/* Draw phase of Type I for positions [k0, k0+n): bit i of inc_bits / dec_bits
 * = (u_{k0+i} < p_inc) / (u_{k0+i} < p_dec), computed as the exact integer
 * compare (z >> 11) < ceil(p * 2^53) (u = (z >> 11) * 2^-53 is a multiple of
 * 2^-53, tests/test_oracle_golden.py::test_integer_threshold_identity).  An
 * AVX-512DQ path (8 SplitMix64 lanes per vpmullq) is chosen at run time when
 * the host supports it -- the reference's numba kernels are likewise compiled
 * for the host CPU. */
#include <immintrin.h>
#define OR_CHUNK 512

static uint64_t or_threshold(double p) {
    double x = p * 9007199254740992.0;
    if (x <= 0.0) return 0;
    if (x >= 9007199254740992.0) return 1ULL << 53;
    return (uint64_t)ceil(x);
}

__attribute__((target("avx512f,avx512dq")))
static void or_draw_bits_avx512(uint64_t zb, int64_t k0, int64_t n, uint64_t t_inc,
                                uint64_t t_dec, uint8_t *inc_bits, uint8_t *dec_bits) {
    const __m512i G = _mm512_set1_epi64((long long)OR_GOLDEN);
    const __m512i C1 = _mm512_set1_epi64((long long)OR_C1);
    const __m512i C2 = _mm512_set1_epi64((long long)OR_C2);
    const __m512i TI = _mm512_set1_epi64((long long)t_inc);
    const __m512i TD = _mm512_set1_epi64((long long)t_dec);
    const __m512i lane = _mm512_set_epi64(7, 6, 5, 4, 3, 2, 1, 0);
    const __m512i ZB = _mm512_set1_epi64((long long)zb);
    for (int64_t i = 0; i < n; i += 8) {
        __m512i k = _mm512_add_epi64(_mm512_set1_epi64(k0 + i), lane);
        __m512i z = _mm512_add_epi64(ZB, _mm512_mullo_epi64(G, k));
        z = _mm512_mullo_epi64(_mm512_xor_si512(z, _mm512_srli_epi64(z, 30)), C1);
        z = _mm512_mullo_epi64(_mm512_xor_si512(z, _mm512_srli_epi64(z, 27)), C2);
        z = _mm512_xor_si512(z, _mm512_srli_epi64(z, 31));
        __m512i m = _mm512_srli_epi64(z, 11);
        inc_bits[i >> 3] = (uint8_t)_mm512_cmplt_epu64_mask(m, TI);
        dec_bits[i >> 3] = (uint8_t)_mm512_cmplt_epu64_mask(m, TD);
    }
}

static void or_draw_bits_scalar(uint64_t zb, int64_t k0, int64_t n, uint64_t t_inc,
                                uint64_t t_dec, uint8_t *inc_bits, uint8_t *dec_bits) {
    for (int64_t i = 0; i < n; i += 8) {
        uint8_t a = 0, b = 0;
        for (int q = 0; q < 8; ++q) {
            uint64_t m = or_mix64(zb + OR_GOLDEN * (uint64_t)(k0 + i + q)) >> 11;
            a |= (uint8_t)((m < t_inc) << q);
            b |= (uint8_t)((m < t_dec) << q);
        }
        inc_bits[i >> 3] = a;
        dec_bits[i >> 3] = b;
    }
}

static int or_have_avx512 = -1;

/* Byte phase, 64 positions per step (AVX-512BW masked adds). */
__attribute__((target("avx512f,avx512bw")))
static void or_apply_avx512(int8_t *row, const uint8_t *lits, int64_t n, int output, int boost,
                            int smin, int smax, const uint8_t *ib, const uint8_t *db) {
    const __m512i one = _mm512_set1_epi8(1);
    const __m512i vmax = _mm512_set1_epi8((char)smax), vmin = _mm512_set1_epi8((char)smin);
    int64_t i = 0;
    for (; i + 64 <= n; i += 64) {
        __m512i st = _mm512_loadu_si512((const void *)(row + i));
        __m512i li = _mm512_loadu_si512((const void *)(lits + i));
        __mmask64 on = output ? _mm512_cmpeq_epi8_mask(li, one) : 0;
        uint64_t ibits, dbits;
        memcpy(&ibits, ib + (i >> 3), 8);
        memcpy(&dbits, db + (i >> 3), 8);
        __mmask64 inc = on & (boost ? ~0ULL : ibits) & _mm512_cmplt_epi8_mask(st, vmax);
        __mmask64 dec = ~on & dbits & _mm512_cmpgt_epi8_mask(st, vmin);
        st = _mm512_mask_add_epi8(st, inc, st, one);
        st = _mm512_mask_sub_epi8(st, dec, st, one);
        _mm512_storeu_si512((void *)(row + i), st);
    }
    for (; i < n; ++i) {
        int st = row[i];
        int on = output & (lits[i] == 1);
        int inc = on & (boost | ((ib[i >> 3] >> (i & 7)) & 1)) & (st < smax);
        int dec = (!on) & ((db[i >> 3] >> (i & 7)) & 1) & (st > smin);
        row[i] = (int8_t)(st + inc - dec);
    }
}

static void type_i_stream_row(int8_t *row, int64_t P, const uint8_t *lits, int output,
                              double p_inc, double p_dec, int boost, int smin, int smax,
                              uint64_t seed, uint64_t base) {
    if (or_have_avx512 < 0) {
        __builtin_cpu_init();
        or_have_avx512 = __builtin_cpu_supports("avx512f") &&
                         __builtin_cpu_supports("avx512dq") && __builtin_cpu_supports("avx512bw");
    }
    const uint64_t zb = seed + OR_GOLDEN * (base + 1);
    const uint64_t t_inc = or_threshold(p_inc), t_dec = or_threshold(p_dec);
    uint8_t ib[OR_CHUNK / 8 + 8], db[OR_CHUNK / 8 + 8];
    for (int64_t k0 = 0; k0 < P; k0 += OR_CHUNK) {
        int64_t n = P - k0 < OR_CHUNK ? P - k0 : OR_CHUNK;
        int64_t n8 = (n + 7) & ~7LL;
        if (or_have_avx512) {
            or_draw_bits_avx512(zb, k0, n8, t_inc, t_dec, ib, db);
            or_apply_avx512(row + k0, lits + k0, n, output, boost, smin, smax, ib, db);
            continue;
        }
        or_draw_bits_scalar(zb, k0, n8, t_inc, t_dec, ib, db);
        for (int64_t i = 0; i < n; ++i) {
            int st = row[k0 + i];
            int on = output & (lits[k0 + i] == 1);
            int inc = on & (boost | ((ib[i >> 3] >> (i & 7)) & 1)) & (st < smax);
            int dec = (!on) & ((db[i >> 3] >> (i & 7)) & 1) & (st > smin);
            row[k0 + i] = (int8_t)(st + inc - dec);
        }
    }
}

static void type_i(int8_t *row, int64_t P, const uint8_t *lits, int output,
                   const or_fb_params *fp, uint64_t seed, uint64_t base,
                   const double *draws) {
    double p_inc = (fp->s - 1.0) / fp->s;
    double p_dec = 1.0 / fp->s;
    if (!draws) {
        type_i_stream_row(row, P, lits, output == 1, p_inc, p_dec, fp->boost != 0,
                          fp->state_min, fp->state_max, seed, base);
        return;
    }
    for (int64_t k = 0; k < P; ++k) {
        double u = draws[k];
        int st = row[k];
        if (output == 1 && lits[k] == 1) {
            if ((fp->boost || u < p_inc) && st < fp->state_max) row[k] = (int8_t)(st + 1);
        } else {
            if (u < p_dec && st > fp->state_min) row[k] = (int8_t)(st - 1);
        }
    }
}

/* kernels/_numba.py:93-98 */
static void type_ii(int8_t *row, int64_t P, const uint8_t *lits, int output) {
    if (output != 1) return;
    for (int64_t k = 0; k < P; ++k)
        if (lits[k] == 0 && row[k] < 0) row[k] = (int8_t)(row[k] + 1);
}

/* kernels/_numba.py:101-125.  Returns the new event counter.  When draws is
 * non-NULL it is an [n_draw_rows, P] row-major float64 array; applied event
 * number i (0-based, in clause-then-direction order) reads row i, whether or
 * not it is a Type I event (a Type II event still consumes its window:
 * dense.py:111, kernels/_numba.py:115,124). */
static uint64_t bank_feedback_impl(int8_t *states, int32_t *weights, int64_t C,
                                   int64_t P, int64_t K, const uint8_t *lits,
                                   const uint8_t *outputs, int64_t label,
                                   int64_t negative, const uint8_t *ut,
                                   const uint8_t *un, const or_fb_params *fp,
                                   uint64_t seed, uint64_t counter,
                                   const double *draws, int64_t n_draw_rows) {
    int64_t ev = 0;
    for (int64_t j = 0; j < C; ++j) {
        int8_t *row = states + j * P;
        int output = outputs[j];
        if (ut[j]) {
            const double *d = (draws && ev < n_draw_rows) ? draws + ev * P : NULL;
            if (weights[j * K + label] >= 0)
                type_i(row, P, lits, output, fp, seed, counter << 32, draws ? d : NULL);
            else
                type_ii(row, P, lits, output);
            if (output == 1) weights[j * K + label] += 1;
            counter += 1;
            ev += 1;
        }
        if (un[j]) {
            const double *d = (draws && ev < n_draw_rows) ? draws + ev * P : NULL;
            if (weights[j * K + negative] >= 0)
                type_ii(row, P, lits, output);
            else
                type_i(row, P, lits, output, fp, seed, counter << 32, draws ? d : NULL);
            if (output == 1) weights[j * K + negative] -= 1;
            counter += 1;
            ev += 1;
        }
    }
    return counter;
}

uint64_t or_bank_feedback(int8_t *states, int32_t *weights, int64_t C, int64_t P,
                          int64_t K, const uint8_t *lits, const uint8_t *outputs,
                          int64_t label, int64_t negative, const uint8_t *ut,
                          const uint8_t *un, double s, int boost, int state_min,
                          int state_max, uint64_t seed, uint64_t counter) {
    or_fb_params fp = {s, boost, state_min, state_max};
    return bank_feedback_impl(states, weights, C, P, K, lits, outputs, label,
                              negative, ut, un, &fp, seed, counter, NULL, 0);
}

uint64_t or_bank_feedback_draws(int8_t *states, int32_t *weights, int64_t C,
                                int64_t P, int64_t K, const uint8_t *lits,
                                const uint8_t *outputs, int64_t label,
                                int64_t negative, const uint8_t *ut,
                                const uint8_t *un, double s, int boost,
                                int state_min, int state_max, uint64_t counter,
                                const double *draws, int64_t n_draw_rows) {
    or_fb_params fp = {s, boost, state_min, state_max};
    return bank_feedback_impl(states, weights, C, P, K, lits, outputs, label,
                              negative, ut, un, &fp, 0, counter, draws, n_draw_rows);
}

/* ------------------------------------------------------ feedback block -- */

/* feedback.py:20-22 */
static int64_t clip_votes(int64_t v, int64_t T) {
    return v < -T ? -T : (v > T ? T : v);
}

/* feedback.py:33-44.  Consumes one draw at fb_counter.  u is either the
 * stream draw or an explicit value (u_explicit >= 0). */
void or_update_probabilities(const int64_t *votes, int64_t K, int64_t label,
                             int64_t T, double u, int64_t *negative,
                             double *p_target, double *p_negative) {
    int64_t offset = 1 + (int64_t)(u * (double)(K - 1));
    *negative = (label + offset) % K;
    *p_target = (double)(T - clip_votes(votes[label], T)) / (2.0 * (double)T);
    *p_negative = (double)(T + clip_votes(votes[*negative], T)) / (2.0 * (double)T);
}

/* feedback.py:47-53 */
void or_sample_updates(double p_target, double p_negative, int64_t C,
                       uint64_t fb_seed, uint64_t fb_counter, uint8_t *ut,
                       uint8_t *un) {
    for (int64_t j = 0; j < C; ++j)
        ut[j] = or_stream_u01(fb_seed, fb_counter + (uint64_t)j) < p_target;
    for (int64_t j = 0; j < C; ++j)
        un[j] = or_stream_u01(fb_seed, fb_counter + (uint64_t)C + (uint64_t)j) < p_negative;
}

/* ------------------------------------------------------------ executor -- */

/* executor.py:50-58.  Returns the advanced stream counter. */
uint64_t or_shuffle_permutation(int64_t n, uint64_t seed, uint64_t counter, int64_t *perm) {
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    if (n > 1) {
        int64_t t = 0;
        for (int64_t i = n - 1; i > 0; --i, ++t) {
            double u = or_stream_u01(seed, counter + (uint64_t)t);
            int64_t j = (int64_t)(u * (double)(i + 1));
            int64_t tmp = perm[i];
            perm[i] = perm[j];
            perm[j] = tmp;
        }
        counter += (uint64_t)(n - 1);
    }
    return counter;
}

/* executor.py:36-47 */
static void partition(int64_t C, int64_t nb, int64_t b, int64_t *start, int64_t *stop) {
    int64_t base = C / nb, extra = C % nb;
    int64_t s = b * base + (b < extra ? b : extra);
    *start = s;
    *stop = s + base + (b < extra ? 1 : 0);
}

typedef struct {
    int64_t n_literals;   /* F */
    int64_t n_positions;  /* P (2F with negations) */
    int64_t n_clauses;
    int64_t n_classes;
    int64_t n_blocks;
    int64_t threshold;
    int64_t budget;       /* effective budget (core.py:220-226) */
    double s;
    int boost;
    int state_min, state_max;
    uint64_t seed;
} or_train_cfg;

/* executor.py:275-340 for dense data, serial driver.  Runs `n_steps`
 * examples in the given order starting from the supplied RNG counters
 * (block_counters[n_blocks], *fb_counter) and updates them.  x_lit is the
 * augmented literal matrix [N, P] (executor.py:105-106). */
void or_train_steps(const or_train_cfg *cfg, int8_t *states, int32_t *weights,
                    const uint8_t *x_lit, const int64_t *labels,
                    const int64_t *order, int64_t n_steps,
                    uint64_t *block_counters, uint64_t *fb_counter) {
    int64_t C = cfg->n_clauses, P = cfg->n_positions, K = cfg->n_classes;
    uint8_t *outputs = (uint8_t *)malloc((size_t)C);
    uint8_t *ut = (uint8_t *)malloc((size_t)C);
    uint8_t *un = (uint8_t *)malloc((size_t)C);
    int64_t *votes = (int64_t *)malloc(sizeof(int64_t) * (size_t)K);
    uint64_t fb_seed = or_derive_stream(cfg->seed, 0xFEED);
    or_fb_params fp = {cfg->s, cfg->boost, cfg->state_min, cfg->state_max};
    for (int64_t st = 0; st < n_steps; ++st) {
        int64_t idx = order[st];
        const uint8_t *lits = x_lit + idx * P;
        int64_t label = labels[idx];
        /* eval_block for every block: executor.py:296-300 */
        or_clause_outputs(states, C, P, lits, 1, cfg->budget, outputs);
        for (int64_t k = 0; k < K; ++k) votes[k] = 0;
        for (int64_t j = 0; j < C; ++j)
            if (outputs[j]) for (int64_t k = 0; k < K; ++k) votes[k] += weights[j * K + k];
        /* decide: executor.py:302-309 */
        double u = or_stream_u01(fb_seed, *fb_counter);
        int64_t negative;
        double pt, pn;
        or_update_probabilities(votes, K, label, cfg->threshold, u, &negative, &pt, &pn);
        or_sample_updates(pt, pn, C, fb_seed, *fb_counter + 1, ut, un);
        *fb_counter += 1 + 2 * (uint64_t)C;
        /* update_block for every block: executor.py:311-317 */
        for (int64_t b = 0; b < cfg->n_blocks; ++b) {
            int64_t c0, c1;
            partition(C, cfg->n_blocks, b, &c0, &c1);
            uint64_t bseed = or_derive_stream(cfg->seed, (uint64_t)b);
            block_counters[b] = bank_feedback_impl(
                states + c0 * P, weights + c0 * K, c1 - c0, P, K, lits, outputs + c0,
                label, negative, ut + c0, un + c0, &fp, bseed, block_counters[b], NULL, 0);
        }
    }
    free(outputs); free(ut); free(un); free(votes);
}

/* ---------------------------------------------------------------- sparse -- */
/*
 * SparseClauseBank feedback for ONE clause and ONE event (sparse.py:162-239).
 * The clause's sorted pair list is (lits_in[0..n_in), sts_in[0..n_in)); the
 * new list is written to (lits_out, sts_out) and its length returned.  The
 * output buffers must hold n_in + n_domain_extra pairs.  `kind` is 1 for
 * Type I, 2 for Type II.  active: sorted example indices; candidates: sorted
 * candidate set (sparse.py:65-69, executor.py:287-289).  capacity < 0 means
 * None.
 */
static int64_t sparse_keep(int was_stored, int64_t lit, int st, int floor_,
                           int64_t capacity, int64_t *lo, int8_t *so, int64_t n) {
    /* sparse.py:212-220 */
    if (st <= floor_) return n;
    if (!was_stored && capacity >= 0 && n >= capacity) return n;
    lo[n] = lit;
    so[n] = (int8_t)st;
    return n + 1;
}

int64_t or_sparse_event(const int64_t *lits_in, const int8_t *sts_in, int64_t n_in,
                        const int64_t *active, int64_t n_active,
                        const int64_t *candidates, int64_t n_cand, int kind,
                        int output, double s, int boost, int floor_, int state_max,
                        int64_t capacity, uint64_t seed, uint64_t base,
                        int64_t *lits_out, int8_t *sts_out) {
    double p_inc = (s - 1.0) / s, p_dec = 1.0 / s;
    int64_t n = 0;
    if (kind == 2 && output != 1) {
        /* sparse.py:193-194: no-op */
        memcpy(lits_out, lits_in, sizeof(int64_t) * (size_t)n_in);
        memcpy(sts_out, sts_in, (size_t)n_in);
        return n_in;
    }
    /* merge walk over union(stored, other) in ascending order, other =
     * active (Type I, sparse.py:171) or candidates (Type II, :198) */
    const int64_t *oth = kind == 1 ? active : candidates;
    int64_t n_oth = kind == 1 ? n_active : n_cand;
    int64_t i = 0, q = 0, a = 0;
    while (i < n_in || q < n_oth) {
        int64_t lit;
        int was_stored;
        int st;
        if (q >= n_oth || (i < n_in && lits_in[i] < oth[q])) {
            lit = lits_in[i]; st = sts_in[i]; was_stored = 1; ++i;
        } else if (i >= n_in || oth[q] < lits_in[i]) {
            lit = oth[q]; st = floor_; was_stored = 0; ++q;
        } else {
            lit = lits_in[i]; st = sts_in[i]; was_stored = 1; ++i; ++q;
        }
        while (a < n_active && active[a] < lit) ++a;
        int is_active = (a < n_active && active[a] == lit);
        if (kind == 1) {
            double u = or_stream_u01(seed, base + (uint64_t)lit);
            if (output == 1) {
                if (is_active) {
                    if ((boost || u < p_inc) && st < state_max) st += 1;
                } else if (u < p_dec && st > floor_) {
                    st -= 1;
                }
            } else if (u < p_dec && st > floor_) {
                st -= 1;
            }
        } else {
            if (!is_active && st < 0) st += 1;
        }
        n = sparse_keep(was_stored, lit, st, floor_, capacity, lits_out, sts_out, n);
    }
    return n;
}
