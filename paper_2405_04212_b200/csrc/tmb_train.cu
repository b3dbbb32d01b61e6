// tmb_train.cu -- the fused, persistent Coalesced-TM training kernels.
//
// One launch runs a whole epoch (or any run of consecutive examples) of
// executor.train's per-example loop (executor.py:275-340):
//
//   eval_block   (dense.py:147-154, kernels/_numba.py:36-58)  -> per-CTA clause
//                outputs + partial class sums
//   vote all-reduce (votes summed over ALL blocks, executor.py:303)
//   decide       (feedback.py:33-53) -- recomputed redundantly by every CTA
//                from random-access feedback-stream draws
//   update_block (kernels/_numba.py:101-125) -- event windows from a scan of
//                the update flags, Type I / II per literal position, weights
//
// Each CTA owns a contiguous clause range [c0, c1) for the whole launch: its
// include bitmasks and weights (and its int8 TA states when they fit) stay in
// shared memory; otherwise states stream through L2/HBM.  Two
// synchronisation domains:
//
//   CLUSTER mode (n_cta <= 16): one thread-block cluster.  Partial votes and
//     per-CTA event prefixes are exchanged through distributed shared memory
//     and two hardware cluster barriers per example -- no global memory
//     round trips on the critical path.
//   GRID mode (n_cta > 16, cooperative launch, up to one CTA per SM): two
//     relaxed 64-bit atomics per CTA + a spin per example; the CTA's block
//     range of update-flag draws is computed while the spin is pending.
//
//   FAST grid mode (k_train_fast: one block, C <= 65536, the common case):
//     a pre-pass (k_step_records) builds one record per step -- example,
//     label, negative class, literal row and the step's update-flag draws as
//     16-bit keys bucketed by their top byte -- which the trainer streams two
//     steps ahead into shared memory with cp.async.  Next-example clause
//     outputs are computed while the all-reduce is pending (only clauses the
//     feedback changed are re-evaluated afterwards), and the events of a step
//     are read straight off the key buckets below the decision thresholds.
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"

namespace cg = cooperative_groups;

namespace tmb {

struct TrainK {
    int C, P, K, W, Ppad, n_blocks, n_cta, cmax, fmax_words, bmax;
    int vec4;  // states rows 4-byte addressable in global memory
    int fast, Wp, Cp, R;  // fast path: padded literal words / clauses, record words
    int MW;         // include-mask row stride in shared memory (W, or Wp for k_train_spec)
    int dbg;        // timing ablations only (tmb_set_option "train.debug_skip")
    int64_t budget, T;
    FbParams fp;
    uint64_t fb_seed, fb_counter0;
    int64_t n_steps;
    const uint32_t *lit_words;
    const int32_t *labels, *order;
    const uint32_t *recs;  // fast: [n_steps][R] step records (k_step_records)
    int8_t *states;
    int32_t *weights;
    uint64_t *block_counters;
    const uint64_t *block_seeds;
    unsigned long long *rec;   // grid mode: [n_steps][2] {arrivals:24 | biased vote sum:40}
    // grid-balanced feedback (generic grid kernel, HBM-resident states):
    // every CTA publishes its work list, the union is split evenly over the
    // CTAs by quads, and the owners pull the rebuilt include masks back
    int gbal;
    unsigned *gsync;           // [n_steps][2] arrivals: work lists published / feedback done
    int *gcount;               // [2][n_cta] work items per CTA this step, their summed cost weights
    int gbw[3];                // gbal cost weights of an event: Type II (firing), Type I silent, Type I firing
    unsigned *gdirty;          // [C] gbal: an include bit of the clause flipped since its owner's last pull
    int *gw_clause, *gw_info;  // [n_cta][cmax] work items (global clause id, info bits)
    uint64_t *gw_sk;           // [n_cta][cmax][2] event stream keys (target, negative)
    uint32_t *gmask;           // [C][W] every clause's include mask (gbal: rewritten where include bits flip)
    unsigned long long *phase;  // optional [n_cta][8] clock64 per phase (profiling)
    tmb_train_stats *stats;
    long long *trace;  // optional [n_steps][4]: negative, votes[label], votes[neg], events
    // fast path: update thresholds for every numerator a in [0, 2T]
    // (threshold_of(a, T), feedback.py:33-44) -- copied to shared memory when
    // it fits, so the decision is one lookup instead of an f64 division
    const uint64_t *thr_tab;
    int thr_smem;
    // speculative windows (k_train_spec): examples per window, 0 = k_train_fast
    int spec;
    int spec_ent;              // spec: flag entries per stream staged with each step head
    const uint32_t *thr32;     // spec: threshold_of(a, T) >> 21 for a in [0, 2T] (k.thr_smem)
};

// CTA owning clause c (inverse of cta_begin).
__device__ __forceinline__ int cta_of(int c, int C, int n_cta) {
    int r = (int)(((int64_t)c * n_cta + n_cta - 1) / C);
    while (r > 0 && cta_begin(r, C, n_cta) > c) --r;
    while (r + 1 < n_cta && cta_begin(r + 1, C, n_cta) <= c) ++r;
    return r;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned *p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Strong (morally strong, gpu scope) accesses for the vote records.  Weak
// loads (ld.global.cg) may be served from the other L2 partition's stale
// copy of the line and never observe the update.
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
enum : int { I_TEV = 1, I_NEV = 2, I_T1 = 4, I_N1 = 8, I_OUT = 16 };
enum : int { MODE_CLUSTER = 0, MODE_GRID = 1 };

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Flag-draw precompute capacity (entries per stream) in shared memory.
constexpr int kMaxPrecompute = 4096;

struct Smem {
    uint32_t *lit0, *lit1, *masks, *ut_bits, *un_bits;
    int32_t *word_cum, *weights, *work, *info, *cnt;
    uint64_t *sk_t, *sk_n, *blk_ctr, *blk_seed, *draw_t, *draw_n;
    int8_t *states;
    long long *vin;    // cluster: [2][16][2] (label, negative) vote inbox
    long long *vsum;   // grid: [2] summed votes
    int *misc;         // [0]=n_work [3..5]=example ring [8..10]=label ring
    uint64_t *thr;     // grid: [0]=t_t [1]=t_n [2]=negative
    uint32_t *rec3;    // fast: [4][R] step records in flight (ring i & 3)
    int *nout, *oflag; // fast: [2][cmax] next-example outputs; [cmax] own event flags
    long long *clo;    // fast: [2 parity][2 class][cmax] shadow-time vote contributions
    unsigned long long *vsh;  // fast: [2 parity][2] shadow-time partial sums
    uint64_t *thr_tab;        // fast: [2T + 1] update thresholds (k.thr_smem)
    unsigned *wcnt;    // per-warp event counts [32]
    unsigned long long *vacc;  // grid: [2] CTA partial votes (label, negative)
    uint32_t *hring;           // spec: [3 * spec][spec_hsz] staged step heads (ring i % HR)
    uint32_t *obs;             // spec: [3 * spec][cmax / 32] clause-output bitset per kept step
    long long *vst;            // spec: [3 * spec][2] partial class sums per kept step
    long long *part;           // spec: [warp][lane] per-warp class-sum partials of a window
    int *gpref;                // gbal: [n_cta + 1] prefix of the published work counts
    int *gwpref;               // gbal: [n_cta + 1] prefix of the published cost weights
    long long *gcut;           // gbal: [2] this CTA's share [q_begin, q_end) of the union's quads
    int *rc_clause, *rc_info;  // gbal: [cmax + 4] work items of this CTA's quad range
    uint64_t *rc_sk;           // gbal: [cmax + 4][2]
};

// Shared-memory carve-up; identical on host (size) and device (pointers).
__host__ __device__ inline size_t smem_layout(const TrainK &k, bool smem_states, int mode,
                                              char *base, Smem *s) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> char * {
        off = align_up(off, 16);
        char *p = base ? base + off : nullptr;
        off += bytes;
        return p;
    };
    Smem t;
    t.sk_t = (uint64_t *)take(8 * k.cmax);
    t.sk_n = (uint64_t *)take(8 * k.cmax);
    t.blk_ctr = (uint64_t *)take(8 * (k.bmax + 1));
    t.blk_seed = (uint64_t *)take(8 * (k.bmax + 1));
    t.thr = (uint64_t *)take(8 * 4);
    t.vin = mode == MODE_CLUSTER ? (long long *)take(8 * 2 * 16 * 2) : nullptr;
    t.vsum = (long long *)take(8 * 2);
    t.lit0 = (uint32_t *)take(4 * k.W);
    t.lit1 = (uint32_t *)take(4 * k.W);
    t.masks = (uint32_t *)take(4 * (size_t)k.cmax * k.MW);
    t.weights = (int32_t *)take(4 * (size_t)k.cmax * k.K);
    t.work = (int32_t *)take(4 * k.cmax);
    t.info = (int32_t *)take(4 * k.cmax);
    t.cnt = (int32_t *)take(4 * k.cmax);
    t.misc = (int *)take(4 * 16);
    t.ut_bits = (uint32_t *)take(4 * k.fmax_words);
    t.un_bits = (uint32_t *)take(4 * k.fmax_words);
    t.word_cum = (int32_t *)take(4 * (k.fmax_words + 1));
    const bool pre = 32 * k.fmax_words <= kMaxPrecompute;
    t.draw_t = pre && !k.fast ? (uint64_t *)take(8 * 32 * k.fmax_words) : nullptr;
    t.draw_n = pre && !k.fast ? (uint64_t *)take(8 * 32 * k.fmax_words) : nullptr;
    const bool fs = k.fast && !k.spec;  // k_train_fast's record ring and shadow sums
    t.rec3 = fs ? (uint32_t *)take(4 * 4 * (size_t)k.R) : nullptr;
    t.nout = fs ? (int *)take(4 * 2 * (size_t)k.cmax) : nullptr;
    t.oflag = k.fast ? (int *)take(4 * (size_t)k.cmax) : nullptr;
    t.wcnt = (unsigned *)take(4 * 64);  // [0, 32): per-warp prefix counts, [32, 64): totals
    t.vacc = (unsigned long long *)take(8 * 2);
    t.clo = fs ? (long long *)take(8 * 4 * (size_t)k.cmax) : nullptr;
    t.vsh = fs ? (unsigned long long *)take(8 * 4) : nullptr;
    const bool sp = k.fast && k.spec;
    t.hring = sp ? (uint32_t *)take(4 * (size_t)(3 * k.spec) * (size_t)(4 + k.Wp + 260 + 2 * k.spec_ent))
                 : nullptr;
    t.obs = sp ? (uint32_t *)take(4 * (size_t)(3 * k.spec) * (size_t)((k.cmax + 31) / 32)) : nullptr;
    t.vst = sp ? (long long *)take(8 * 2 * (size_t)(3 * k.spec)) : nullptr;
    t.part = sp ? (long long *)take(8 * 32 * 32) : nullptr;
    // k_train_spec keeps the table in 32 bits (bucket + all but the low 21
    // bits of each threshold; the exact value is recomputed on a key tie)
    t.thr_tab = k.fast && k.thr_smem ? (uint64_t *)take((k.spec ? 4 : 8) * (size_t)(2 * k.T + 1))
                                     : nullptr;
    t.states = smem_states ? (int8_t *)take((size_t)k.cmax * k.Ppad) : nullptr;
    const bool gb = k.gbal && !k.fast && !smem_states && mode == MODE_GRID;
    t.gcut = gb ? (long long *)take(16) : nullptr;
    t.gpref = gb ? (int *)take(4 * (size_t)(k.n_cta + 1)) : nullptr;
    t.gwpref = gb ? (int *)take(4 * (size_t)(k.n_cta + 1)) : nullptr;
    t.rc_clause = gb ? (int *)take(4 * (size_t)(k.cmax + 4)) : nullptr;
    t.rc_info = gb ? (int *)take(4 * (size_t)(k.cmax + 4)) : nullptr;
    t.rc_sk = gb ? (uint64_t *)take(16 * (size_t)(k.cmax + 4)) : nullptr;
    if (s) *s = t;
    return align_up(off, 16);
}

struct Counters {
    uint64_t draws = 0, upd = 0, events = 0, t1 = 0, t2 = 0;
};

// Per-position feedback over the CTA's work list, four positions per thread
// (one 32-bit state word), include masks + include counts rebuilt from the
// new states.  kernels/_numba.py:71-98 per position, target event then
// negative event.  Up to four state words per thread are loaded
// before any is processed so the L2 round trips of HBM-resident states
// overlap.
template <bool SMEM_STATES>
__device__ __forceinline__ void feedback_quads(const TrainK &k, const Smem &s, int c0,
                                               const uint32_t *lit, int n_work, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;  // quads per (padded) row; multiple of 32
    const int total = n_work * QP;
    constexpr int B = 4;
    // quad index it = (work item wc, quad rem), advanced by nthr per unit
    // without a division (nthr < 2 * QP is not assumed: a short loop)
    int wc_next = tid / QP, rem_next = tid - (tid / QP) * QP;
    const uint64_t t_inc = k.fp.t_inc, t_dec = k.fp.t_dec;
    const int smin = k.fp.smin, smax = k.fp.smax, boost = k.fp.boost ? 1 : 0;
    unsigned nd = 0, nupd = 0;  // draws consumed / states changed (statistics)
    for (int it0 = tid; it0 < total; it0 += B * nthr) {
        uint32_t word[B];
        int jj[B], pp[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int it = it0 + u * nthr;
            const int wc = wc_next, rem = rem_next;
            rem_next += nthr;
            while (rem_next >= QP) {
                rem_next -= QP;
                ++wc_next;
            }
            jj[u] = -1;
            word[u] = 0xFFFFFFFFu;
            if (it < total) {
                const int p0 = rem << 2;
                const int j = s.work[wc];
                jj[u] = j;
                pp[u] = p0;
                if (SMEM_STATES) {
                    word[u] = *reinterpret_cast<const uint32_t *>(s.states + (size_t)j * k.Ppad + p0);
                } else {
                    const int8_t *grow = k.states + (int64_t)(c0 + j) * k.P;
                    if (k.vec4 && p0 + 4 <= k.P) {
                        word[u] = __ldcg(reinterpret_cast<const unsigned int *>(grow + p0));
                    } else {
                        for (int b = 0; b < 4; ++b)
                            if (p0 + b < k.P)
                                word[u] = (word[u] & ~(0xFFu << (8 * b))) |
                                          ((uint32_t)(uint8_t)grow[p0 + b] << (8 * b));
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (it0 + u * nthr >= total) break;  // warp-uniform (total % 32 == 0)
            const int j = jj[u], p0 = pp[u];
            const int info = s.info[j];
            const int out = (info & I_OUT) ? 1 : 0;
            const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
            const int lim = k.P - p0;  // positions b < lim are real (the rest is row padding)
            int st[4], s0[4];
#pragma unroll
            for (int b = 0; b < 4; ++b) s0[b] = st[b] = (int)(int8_t)(word[u] >> (8 * b));
            // Type I (kernels/_numba.py:71-90) on the quad with draw
            // mix64(z0 + b*G) for position p0 + b, branch-free: the draw is
            // computed for every position and counted / used only where the
            // reference consumes it.  Type II (:93-98) likewise.
            auto type_i = [&](uint64_t z0) {
                if (!out) {  // warp-uniform: every position moves down w.p. 1/s
#pragma unroll
                    for (int b = 0; b < 4; ++b) {
                        const int above = (b < lim ? 1 : 0) & (st[b] > smin ? 1 : 0);
                        const int hit = (mix64(z0 + kGolden * (uint64_t)b) >> 11) < t_dec ? 1 : 0;
                        nd += above;
                        st[b] -= above & hit;
                    }
                    return;
                }
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int vb = b < lim ? 1 : 0;
                    const int inc = out & (int)((litn >> b) & 1u);
                    const uint64_t thr = inc ? t_inc : t_dec;
                    const int hit = (mix64(z0 + kGolden * (uint64_t)b) >> 11) < thr ? 1 : 0;
                    const int room = st[b] < smax ? 1 : 0;
                    const int above = st[b] > smin ? 1 : 0;
                    nd += vb & (inc ? (room & (boost ^ 1)) : above);
                    const int delta = (inc & room & (boost | hit)) - ((inc ^ 1) & above & hit);
                    st[b] += vb ? delta : 0;
                }
            };
            auto type_ii = [&]() {
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    st[b] += (b < lim ? 1 : 0) & out & (int)(((litn >> b) & 1u) ^ 1u) & (st[b] < 0 ? 1 : 0);
            };
            if (info & I_TEV) {
                if (info & I_T1) type_i(s.sk_t[j] + kGolden * (uint64_t)p0);
                else type_ii();
            }
            if (info & I_NEV) {
                if (info & I_N1) type_i(s.sk_n[j] + kGolden * (uint64_t)p0);
                else type_ii();
            }
            uint32_t nib = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                nupd += st[b] != s0[b] ? 1 : 0;
                nib |= (uint32_t)(b < lim && st[b] >= 0) << b;
            }
            const uint32_t nw = __byte_perm(__byte_perm((uint32_t)st[0], (uint32_t)st[1], 0x0040),
                                            __byte_perm((uint32_t)st[2], (uint32_t)st[3], 0x0040),
                                            0x5410);
            if (nw != word[u]) {
                if (SMEM_STATES) {
                    *reinterpret_cast<uint32_t *>(s.states + (size_t)j * k.Ppad + p0) = nw;
                } else {
                    int8_t *grow = k.states + (int64_t)(c0 + j) * k.P;
                    if (k.vec4 && p0 + 4 <= k.P) {
                        __stcg(reinterpret_cast<unsigned int *>(grow + p0), nw);
                    } else {
                        for (int b = 0; b < 4; ++b)
                            if (p0 + b < k.P) grow[p0 + b] = (int8_t)(nw >> (8 * b));
                    }
                }
            }
            // mask word for positions 32w..32w+31: lanes 8g..8g+7 hold its nibbles
            uint32_t m = nib << ((lane & 7) * 4);
            m |= __shfl_xor_sync(0xffffffffu, m, 1);
            m |= __shfl_xor_sync(0xffffffffu, m, 2);
            m |= __shfl_xor_sync(0xffffffffu, m, 4);
            if ((lane & 7) == 0) {
                const int w = p0 >> 5;
                if (w < k.W) {
                    const uint32_t old = s.masks[j * k.MW + w];
                    if (old != m) {
                        s.masks[j * k.MW + w] = m;
                        atomicAdd(&s.cnt[j], __popc(m) - __popc(old));
                    }
                }
            }
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// Compact per-position feedback for k_train_spec: the arithmetic of
// feedback_quads (kernels/_numba.py:71-98, target event then negative event,
// SPEC.md:369) with one quad per thread and iteration and both events
// through one code path -- a fraction of the instructions.  The non-empty-
// step path runs every few microseconds with its code fetched cold, so code
// size is latency here.  Type I with the clause not firing is the general
// rule with inc = 0 (every position decrements w.p. 1/s).
// ABL (microbenchmark ablations only): 1 no mask rebuild, 2 a cheap hash
// instead of SplitMix64, 4 no state load / store
template <bool SMEM_STATES, int ABL = 0>
__device__ __forceinline__ void feedback_compact(const TrainK &k, const Smem &s, int c0,
                                                 const uint32_t *lit, int n_work, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;  // quads per (padded) row; multiple of 32
    const int total = n_work * QP;
    int wc = tid / QP, rem = tid - (tid / QP) * QP;
    const uint64_t t_inc = k.fp.t_inc, t_dec = k.fp.t_dec;
    const int smin = k.fp.smin, smax = k.fp.smax, boost = k.fp.boost ? 1 : 0;
    unsigned nd = 0, nupd = 0;
    for (int it = tid; it < total; it += nthr) {  // warp-uniform: a warp's quads share a row
        const int j = s.work[wc], p0 = rem << 2;
        uint32_t word = 0xFFFFFFFFu;
        int8_t *grow = SMEM_STATES ? nullptr : k.states + (int64_t)(c0 + j) * k.P;
        if (ABL & 4) {
            word = (uint32_t)(it * 0x9E3779B9u);
        } else if (SMEM_STATES) {
            word = *reinterpret_cast<const uint32_t *>(s.states + (size_t)j * k.Ppad + p0);
        } else if (k.vec4 && p0 + 4 <= k.P) {
            word = __ldcg(reinterpret_cast<const unsigned int *>(grow + p0));
        } else {
            for (int b = 0; b < 4; ++b)
                if (p0 + b < k.P)
                    word = (word & ~(0xFFu << (8 * b))) | ((uint32_t)(uint8_t)grow[p0 + b] << (8 * b));
        }
        const int info = s.info[j];
        const int out = (info & I_OUT) ? 1 : 0;
        const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
        const int lim = k.P - p0;
        int st[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) st[b] = (int)(int8_t)(word >> (8 * b));
#pragma unroll 1
        for (int ev = 0; ev < 2; ++ev) {
            if (!(info & (ev ? I_NEV : I_TEV))) continue;
            if (info & (ev ? I_N1 : I_T1)) {  // Type I
                const uint64_t z0 = (ev ? s.sk_n[j] : s.sk_t[j]) + kGolden * (uint64_t)p0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const int vb = b < lim ? 1 : 0;
                    const int inc = out & (int)((litn >> b) & 1u);
                    const uint64_t zz = (ABL & 2) ? (z0 + kGolden * (uint64_t)b) * kMixC1
                                                  : mix64(z0 + kGolden * (uint64_t)b);
                    const int hit = (zz >> 11) < (inc ? t_inc : t_dec) ? 1 : 0;
                    const int room = st[b] < smax ? 1 : 0;
                    const int above = st[b] > smin ? 1 : 0;
                    nd += vb & (inc ? (room & (boost ^ 1)) : above);
                    const int delta = (inc & room & (boost | hit)) - ((inc ^ 1) & above & hit);
                    st[b] += vb ? delta : 0;
                }
            } else {  // Type II
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    st[b] += (b < lim ? 1 : 0) & out & (int)(((litn >> b) & 1u) ^ 1u) & (st[b] < 0 ? 1 : 0);
            }
        }
        uint32_t nib = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            nupd += st[b] != (int)(int8_t)(word >> (8 * b)) ? 1 : 0;
            nib |= (uint32_t)(b < lim && st[b] >= 0) << b;
        }
        const uint32_t nw = __byte_perm(__byte_perm((uint32_t)st[0], (uint32_t)st[1], 0x0040),
                                        __byte_perm((uint32_t)st[2], (uint32_t)st[3], 0x0040), 0x5410);
        if (nw != word && !(ABL & 4)) {
            if (SMEM_STATES) {
                *reinterpret_cast<uint32_t *>(s.states + (size_t)j * k.Ppad + p0) = nw;
            } else if (k.vec4 && p0 + 4 <= k.P) {
                __stcg(reinterpret_cast<unsigned int *>(grow + p0), nw);
            } else {
                for (int b = 0; b < 4; ++b)
                    if (p0 + b < k.P) grow[p0 + b] = (int8_t)(nw >> (8 * b));
            }
        }
        // mask word for positions 32w..32w+31: lanes 8g..8g+7 hold its nibbles
        if (!(ABL & 1)) {
            uint32_t m = nib << ((lane & 7) * 4);
            m |= __shfl_xor_sync(0xffffffffu, m, 1);
            m |= __shfl_xor_sync(0xffffffffu, m, 2);
            m |= __shfl_xor_sync(0xffffffffu, m, 4);
            if ((lane & 7) == 0) {
                const int w = p0 >> 5;
                if (w < k.W) {
                    const uint32_t old = s.masks[j * k.MW + w];
                    if (old != m) {
                        s.masks[j * k.MW + w] = m;
                        atomicAdd(&s.cnt[j], __popc(m) - __popc(old));
                    }
                }
            }
        } else {
            cn.t2 += nib;
        }
        rem += nthr;
        while (rem >= QP) {
            rem -= QP;
            ++wc;
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// Byte-SIMD per-quad feedback for k_train_spec: feedback_compact's
// arithmetic (kernels/_numba.py:71-98, target then negative event) on the
// four int8 states of a 32-bit word at once -- per-byte compares, the
// +1 / -1 applied by carry-free SWAR add / subtract (states stay in
// [state_min, state_max] within int8, so no byte over/underflows).  Only the
// SplitMix64 draws remain per position; u < p is tested as z < t << 11 on
// the full 64-bit draw (t < 2^53, exact).
__device__ __forceinline__ uint32_t spread4(uint32_t nib) {  // bit b -> byte b = 0xFF
    return ((nib * 0x204081u) & 0x01010101u) * 0xFFu;
}
__device__ __forceinline__ uint32_t swar_inc(uint32_t w, uint32_t one) {  // bytes + {0,1}
    return ((w & 0x7F7F7F7Fu) + one) ^ (w & 0x80808080u);
}
__device__ __forceinline__ uint32_t swar_dec(uint32_t w, uint32_t one) {  // bytes - {0,1}
    return ((w | 0x80808080u) - one) ^ ((w ^ ~one) & 0x80808080u);
}

// The four draws z0 + kGolden * b (b = 0..3) against 64-bit thresholds, as a
// 0x01-per-byte mask of the positions with draw < threshold.  SELECT: byte b
// uses T_inc where bit 8b of incb is set, else T_dec.  (Measured and rejected,
// tmb_microbench_feedback on the silent path, cycles per clause: deciding on
// the high word alone with a full compare on ties +5%, the same with the
// high-word shifts as IMAD.HI on the FMA pipe +12%.)
template <bool SELECT>
__device__ __forceinline__ uint32_t quad_hits(uint64_t z0, uint64_t T_dec, uint64_t T_inc,
                                              uint32_t incb) {
    uint32_t h = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const uint64_t t = SELECT && ((incb >> (8 * b)) & 1u) ? T_inc : T_dec;
        h |= mix64(z0 + kGolden * (uint64_t)b) < t ? (1u << (8 * b)) : 0u;
    }
    return h;
}

// One quad of feedback_simd: the four states of word w after the clause's
// events (info bits), literal nibble litn, valid positions lim; zt / zn =
// event key + kGolden * p0 of the target / negative event.  Adds the
// reference's draw count to nd.
__device__ __forceinline__ uint32_t quad_update_simd(const TrainK &k, uint32_t w, int info,
                                                     uint32_t litn, int lim, uint64_t zt,
                                                     uint64_t zn, unsigned &nd) {
    const uint64_t T_inc = k.fp.t_inc << 11, T_dec = k.fp.t_dec << 11;
    const uint32_t smin4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smin;
    const uint32_t smax4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smax;
    const uint32_t boostm = k.fp.boost ? 0xFFFFFFFFu : 0u;
    const uint32_t outm = (info & I_OUT) ? 0xFFFFFFFFu : 0u;
    const uint32_t vb = lim >= 4 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - lim))));
    const uint32_t litb = spread4(litn);
    const uint32_t incb = litb & outm & vb;  // Type I: positions that may increment
#pragma unroll 1
    for (int ev = 0; ev < 2; ++ev) {
        if (!(info & (ev ? I_NEV : I_TEV))) continue;
        if (info & (ev ? I_N1 : I_T1)) {  // Type I
            const uint32_t hit = quad_hits<true>(ev ? zn : zt, T_dec, T_inc, incb);  // 0x01 bytes
            const uint32_t room = __vcmplts4(w, smax4), above = __vcmpgts4(w, smin4);
            nd += __popc(((incb & room & ~boostm) | (~incb & above & vb)) & 0x01010101u);
            const uint32_t up = incb & room & (boostm | hit);
            const uint32_t dn = ~incb & vb & above & hit;
            w = swar_dec(swar_inc(w, up & 0x01010101u), dn & 0x01010101u);
        } else {  // Type II
            const uint32_t neg = __vcmplts4(w, 0u);
            w = swar_inc(w, outm & ~litb & vb & neg & 0x01010101u);
        }
    }
    return w;
}

// Include bits (state >= 0) of the valid positions of a quad, as a nibble.
__device__ __forceinline__ uint32_t quad_include_nibble(uint32_t w, int lim) {
    const uint32_t vb = lim >= 4 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - lim))));
    return (((~w & 0x80808080u) >> 7) & vb & 0x01010101u) * 0x01020408u >> 24;
}

template <bool SMEM_STATES>
__device__ __forceinline__ void feedback_simd_v1(const TrainK &k, const Smem &s, int c0,
                                              const uint32_t *lit, int n_work, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;  // quads per (padded) row; multiple of 32
    const int total = n_work * QP;
    int wc = tid / QP, rem = tid - (tid / QP) * QP;
    unsigned nd = 0, nupd = 0;
    for (int it = tid; it < total; it += nthr) {  // warp-uniform: a warp's quads share a row
        const int j = s.work[wc], p0 = rem << 2;
        uint32_t word = 0xFFFFFFFFu;
        int8_t *grow = SMEM_STATES ? nullptr : k.states + (int64_t)(c0 + j) * k.P;
        if (SMEM_STATES) {
            word = *reinterpret_cast<const uint32_t *>(s.states + (size_t)j * k.Ppad + p0);
        } else if (k.vec4 && p0 + 4 <= k.P) {
            word = __ldcg(reinterpret_cast<const unsigned int *>(grow + p0));
        } else {
            for (int b = 0; b < 4; ++b)
                if (p0 + b < k.P)
                    word = (word & ~(0xFFu << (8 * b))) | ((uint32_t)(uint8_t)grow[p0 + b] << (8 * b));
        }
        const int info = s.info[j];
        const int lim = k.P - p0;
        const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
        const uint64_t zp = kGolden * (uint64_t)p0;
        const uint32_t w = quad_update_simd(k, word, info, litn, lim,
                                            (info & I_TEV) ? s.sk_t[j] + zp : 0,
                                            (info & I_NEV) ? s.sk_n[j] + zp : 0, nd);
        nupd += __popc(__vcmpne4(w, word) & 0x01010101u);
        const uint32_t nib = quad_include_nibble(w, lim);
        if (w != word) {
            if (SMEM_STATES) {
                *reinterpret_cast<uint32_t *>(s.states + (size_t)j * k.Ppad + p0) = w;
            } else if (k.vec4 && p0 + 4 <= k.P) {
                __stcg(reinterpret_cast<unsigned int *>(grow + p0), w);
            } else {
                for (int b = 0; b < 4; ++b)
                    if (p0 + b < k.P) grow[p0 + b] = (int8_t)(w >> (8 * b));
            }
        }
        // mask word for positions 32w..32w+31: lanes 8g..8g+7 hold its nibbles
        uint32_t m = nib << ((lane & 7) * 4);
        m |= __shfl_xor_sync(0xffffffffu, m, 1);
        m |= __shfl_xor_sync(0xffffffffu, m, 2);
        m |= __shfl_xor_sync(0xffffffffu, m, 4);
        if ((lane & 7) == 0) {
            const int wd = p0 >> 5;
            if (wd < k.W) {
                const uint32_t old = s.masks[j * k.MW + wd];
                if (old != m) {
                    s.masks[j * k.MW + wd] = m;
                    atomicAdd(&s.cnt[j], __popc(m) - __popc(old));
                }
            }
        }
        rem += nthr;
        while (rem >= QP) {
            rem -= QP;
            ++wc;
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// feedback_simd, second cut.  A warp's 32 quads share a work row, so the row's
// event class is warp-uniform and the common one gets its own straight-line
// path: ONE Type I event on a silent clause (kernels/_numba.py:84-90 with
// clause_out == 0: every valid position above state_min decrements w.p. 1/s)
// needs no literal bits, no threshold selection and no increment arithmetic.
// The pre-shifted thresholds are loop invariants, and the include-mask word is
// rebuilt only when some state of the warp's 128 positions crossed the include
// boundary (the sign byte changed) -- the masks always equal the states' signs,
// so an unchanged sign pattern means an unchanged word.  Same results as
// feedback_simd_v1 (the microbenchmark compares cycles, the trainers' parity
// tests the states).
__device__ __forceinline__ uint32_t quad_silent_type1(uint32_t w, uint32_t vb, uint32_t smin4,
                                                      uint64_t T_dec, uint64_t z0, unsigned &nd,
                                                      unsigned &nupd) {
    const uint32_t above = __vcmpgts4(w, smin4) & vb & 0x01010101u;
    const uint32_t dn = above & quad_hits<false>(z0, T_dec, T_dec, 0u);
    nd += __popc(above);
    nupd += __popc(dn);
    return swar_dec(w, dn);
}

// ONE Type I event on a firing clause (kernels/_numba.py:71-83): positions
// whose literal is 1 increment w.p. (s-1)/s (always with boost), the others
// decrement w.p. 1/s -- quad_update_simd's Type I branch without the event loop.
__device__ __forceinline__ uint32_t quad_firing_type1(const TrainK &k, uint32_t w, uint32_t litn,
                                                      uint32_t vb, uint64_t z0, unsigned &nd,
                                                      unsigned &nupd) {
    const uint32_t smin4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smin;
    const uint32_t smax4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smax;
    const uint32_t boostm = k.fp.boost ? 0xFFFFFFFFu : 0u;
    const uint32_t incb = spread4(litn) & vb;
    const uint32_t hit = quad_hits<true>(z0, k.fp.t_dec << 11, k.fp.t_inc << 11, incb);
    const uint32_t room = __vcmplts4(w, smax4), above = __vcmpgts4(w, smin4);
    nd += __popc(((incb & room & ~boostm) | (~incb & above & vb)) & 0x01010101u);
    const uint32_t up = incb & room & (boostm | hit) & 0x01010101u;
    const uint32_t dn = ~incb & vb & above & hit & 0x01010101u;
    nupd += __popc(up | dn);
    return swar_dec(swar_inc(w, up), dn);
}
// ONE Type II event on a firing clause (kernels/_numba.py:93-98): excluded
// positions whose literal is 0 move one step towards inclusion; no draws.
__device__ __forceinline__ uint32_t quad_type2(uint32_t w, uint32_t litn, uint32_t vb,
                                               unsigned &nupd) {
    const uint32_t up = ~spread4(litn) & vb & __vcmplts4(w, 0u) & 0x01010101u;
    nupd += __popc(up);
    return swar_inc(w, up);
}
// Warp-uniform class of a work row's events: 1 one Type I event on a silent
// clause, 2 one Type I event on a firing clause, 3 one Type II event (firing),
// 0 anything else (both events) -- the general quad_update_simd.
__device__ __forceinline__ int fb_class(int info) {
    const int e = info & (I_TEV | I_NEV);
    if (e == (I_TEV | I_NEV) || e == 0) return 0;
    const bool t1 = e == I_TEV ? (info & I_T1) : (info & I_N1);
    if (!(info & I_OUT)) return t1 ? 1 : 0;
    return t1 ? 2 : 3;
}

// PRECLS: s.info[j] carries the row's event class in bits 8.. (spec_events).
template <bool SMEM_STATES, bool PRECLS = false>
__device__ __forceinline__ void feedback_simd(const TrainK &k, const Smem &s, int c0,
                                              const uint32_t *lit, int n_work, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;  // quads per (padded) row; multiple of 32
    const int total = n_work * QP;
    int wc = tid / QP, rem = tid - (tid / QP) * QP;
    const uint64_t T_dec = k.fp.t_dec << 11;
    const uint32_t smin4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smin;
    unsigned nd = 0, nupd = 0;
    for (int it = tid; it < total; it += nthr) {  // warp-uniform: a warp's quads share a row
        const int j = s.work[wc], p0 = rem << 2;
        uint32_t word = 0xFFFFFFFFu;
        int8_t *grow = SMEM_STATES ? nullptr : k.states + (int64_t)(c0 + j) * k.P;
        if (SMEM_STATES) {
            word = *reinterpret_cast<const uint32_t *>(s.states + (size_t)j * k.Ppad + p0);
        } else if (k.vec4 && p0 + 4 <= k.P) {
            word = __ldcg(reinterpret_cast<const unsigned int *>(grow + p0));
        } else {
            for (int b = 0; b < 4; ++b)
                if (p0 + b < k.P)
                    word = (word & ~(0xFFu << (8 * b))) | ((uint32_t)(uint8_t)grow[p0 + b] << (8 * b));
        }
        const int info = s.info[j];
        const int lim = k.P - p0;
        const uint64_t zp = kGolden * (uint64_t)p0;
        uint32_t w;
        const int cls = PRECLS ? (info >> 8) : fb_class(info);
        // valid-position byte mask: all ones except in a row's last warp
        uint32_t vb = 0xFFFFFFFFu;
        if (__any_sync(0xffffffffu, lim < 4))
            vb = lim >= 4 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - lim))));
        if (cls == 1) {
            w = quad_silent_type1(word, vb, smin4, T_dec, ((info & I_TEV) ? s.sk_t[j] : s.sk_n[j]) + zp,
                                  nd, nupd);
        } else {
            const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
            if (cls == 2) {
                w = quad_firing_type1(k, word, litn, vb, ((info & I_TEV) ? s.sk_t[j] : s.sk_n[j]) + zp,
                                      nd, nupd);
            } else if (cls == 3) {
                w = quad_type2(word, litn, vb, nupd);
            } else {
                w = quad_update_simd(k, word, info, litn, lim, (info & I_TEV) ? s.sk_t[j] + zp : 0,
                                     (info & I_NEV) ? s.sk_n[j] + zp : 0, nd);
                nupd += __popc(__vcmpne4(w, word) & 0x01010101u);
            }
        }
        if (w != word) {
            if (SMEM_STATES) {
                *reinterpret_cast<uint32_t *>(s.states + (size_t)j * k.Ppad + p0) = w;
            } else if (k.vec4 && p0 + 4 <= k.P) {
                __stcg(reinterpret_cast<unsigned int *>(grow + p0), w);
            } else {
                for (int b = 0; b < 4; ++b)
                    if (p0 + b < k.P) grow[p0 + b] = (int8_t)(w >> (8 * b));
            }
        }
        // mask word for positions 32w..32w+31 (lanes 8g..8g+7 hold its
        // nibbles), only when an include bit of the warp's positions flipped
        if (__any_sync(0xffffffffu, ((w ^ word) & 0x80808080u) != 0)) {
            uint32_t m = quad_include_nibble(w, lim) << ((lane & 7) * 4);
            m |= __shfl_xor_sync(0xffffffffu, m, 1);
            m |= __shfl_xor_sync(0xffffffffu, m, 2);
            m |= __shfl_xor_sync(0xffffffffu, m, 4);
            if ((lane & 7) == 0) {
                const int wd = p0 >> 5;
                if (wd < k.W) {
                    const uint32_t old = s.masks[j * k.MW + wd];
                    if (old != m) {
                        s.masks[j * k.MW + wd] = m;
                        atomicAdd(&s.cnt[j], __popc(m) - __popc(old));
                    }
                }
            }
        }
        rem += nthr;
        while (rem >= QP) {
            rem -= QP;
            ++wc;
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// Wide feedback for shared-memory states: a thread owns NQ consecutive quads
// (4 * NQ positions) of one work row, a row takes RW whole warps.  The row's
// index, info bits, event keys, the literal bits and kGolden * p0 are fetched
// or computed once per 4 * NQ positions instead of once per quad, the states
// move as one 8- or 16-byte shared access, and the include-mask word needs
// log2(8 / NQ) shuffles instead of three -- about 40% fewer instructions per
// position than feedback_simd (same arithmetic: quad_update_simd).
template <int NQ, int UNR>
__device__ __forceinline__ void feedback_wide(const TrainK &k, const Smem &s,
                                              const uint32_t *lit, int n_work, Counters &cn) {
    static_assert(NQ == 2 || NQ == 4, "NQ: 2 or 4 quads per thread");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    constexpr int LPW = 8 / NQ;             // lanes per include-mask word
    const int UP = k.Ppad / (4 * NQ);       // units per padded row (Ppad % 128 == 0)
    const int RW = (UP + 31) >> 5;          // warps per row
    const int total = n_work * RW;
    unsigned nd = 0, nupd = 0;
    for (int v = warp; v < total; v += nwarp) {
        const int wc = v / RW, u = (v - wc * RW) * 32 + lane;
        const int j = s.work[wc];
        const int p0 = u * (4 * NQ);
        const bool valid = u < UP;
        uint32_t nibs = 0;
        if (valid) {
            const int info = s.info[j];
            const uint32_t litu = p0 < k.P ? lit[p0 >> 5] >> (p0 & 31) : 0u;
            const uint64_t zp = kGolden * (uint64_t)p0;
            uint64_t zt = (info & I_TEV) ? s.sk_t[j] + zp : 0;
            uint64_t zn = (info & I_NEV) ? s.sk_n[j] + zp : 0;
            int8_t *row = s.states + (size_t)j * k.Ppad + p0;
            uint32_t in[NQ], out[NQ];
            if (NQ == 4) {
                const uint4 t = *reinterpret_cast<const uint4 *>(row);
                in[0] = t.x; in[1] = t.y; in[NQ - 2] = t.z; in[NQ - 1] = t.w;
            } else {
                const uint2 t = *reinterpret_cast<const uint2 *>(row);
                in[0] = t.x; in[1] = t.y;
            }
            bool changed = false;
            if (UNR >= NQ) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const int lim = k.P - p0 - 4 * q;
                    out[q] = quad_update_simd(k, in[q], info, (litu >> (4 * q)) & 0xFu, lim,
                                              zt + kGolden * (uint64_t)(4 * q),
                                              zn + kGolden * (uint64_t)(4 * q), nd);
                    nupd += __popc(__vcmpne4(out[q], in[q]) & 0x01010101u);
                    nibs |= quad_include_nibble(out[q], lim) << (4 * q);
                    changed |= out[q] != in[q];
                }
            } else {
                // rolled: the words rotate through in[0] / out[NQ - 1]
                int lim = k.P - p0;
                uint32_t lq = litu;
#pragma unroll 1
                for (int q = 0; q < NQ; ++q) {
                    const uint32_t wi = in[0];
                    const uint32_t wo = quad_update_simd(k, wi, info, lq & 0xFu, lim, zt, zn, nd);
                    nupd += __popc(__vcmpne4(wo, wi) & 0x01010101u);
                    nibs = (nibs >> 4) | (quad_include_nibble(wo, lim) << (4 * (NQ - 1)));
                    changed |= wo != wi;
#pragma unroll
                    for (int r = 0; r + 1 < NQ; ++r) {
                        in[r] = in[r + 1];
                        out[r] = out[r + 1];
                    }
                    out[NQ - 1] = wo;
                    zt += 4 * kGolden;
                    zn += 4 * kGolden;
                    lq >>= 4;
                    lim -= 4;
                }
            }
            if (changed) {
                if (NQ == 4)
                    *reinterpret_cast<uint4 *>(row) = make_uint4(out[0], out[1], out[NQ - 2], out[NQ - 1]);
                else
                    *reinterpret_cast<uint2 *>(row) = make_uint2(out[0], out[1]);
            }
        }
        // mask word for positions 32w..32w+31: LPW adjacent lanes hold its parts
        uint32_t m = nibs << ((lane & (LPW - 1)) * 4 * NQ);
#pragma unroll
        for (int o = 1; o < LPW; o <<= 1) m |= __shfl_xor_sync(0xffffffffu, m, o);
        if (valid && (lane & (LPW - 1)) == 0) {
            const int wd = p0 >> 5;
            if (wd < k.W) {
                const uint32_t old = s.masks[j * k.MW + wd];
                if (old != m) {
                    s.masks[j * k.MW + wd] = m;
                    atomicAdd(&s.cnt[j], __popc(m) - __popc(old));
                }
            }
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// Cost weight of a work item for the balanced split (relative SM time of its
// quads: a Type II event has no draws, Type I on a silent clause runs the
// straight-line decrement path, Type I on a firing clause the general one).
__device__ __forceinline__ int gbal_weight(const TrainK &k, int info) {
    const int out = (info & I_OUT) ? 1 : 0;
    int w = 0;
    if (info & I_TEV) w += (info & I_T1) ? k.gbw[1 + out] : out * k.gbw[0];
    if (info & I_NEV) w += (info & I_N1) ? k.gbw[1 + out] : out * k.gbw[0];
    return w > 0 ? w : 1;
}

// Grid-balanced feedback (HBM-resident states): this CTA's share
// [q_begin, q_end) of the quads of all CTAs' work items (the union of the
// published work lists in CTA order; q_begin, q_end multiples of 32, so a
// warp's 32 quads lie in one row).  rc_*[g - g_lo] hold the work items.
// Same per-position arithmetic as feedback_quads; the rebuilt include-mask
// words go to k.gmask for the owners to pull.
#ifndef TMB_GB_B
#define TMB_GB_B 1  // state words in flight per thread of the 1024-thread build (2: +5% time, 3: +4%)
#endif
template <int B>  // state words in flight per thread
__device__ __forceinline__ void feedback_quads_global(const TrainK &k, const Smem &s,
                                                      const uint32_t *lit, int64_t q_begin,
                                                      int64_t q_end, int64_t g_lo, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;
    unsigned nd = 0, nupd = 0;
    const uint64_t T_dec = k.fp.t_dec << 11;
    const uint32_t smin4 = 0x01010101u * (uint32_t)(uint8_t)k.fp.smin;
    // quad it = (work item g_lo + gnext, quad rem) advanced by nthr per unit
    // without a division (nthr < QP is not assumed: a short loop)
    int gnext = (int)((q_begin + tid) / QP - g_lo);
    int rnext = (int)((q_begin + tid) % QP);
    for (int64_t it0 = q_begin + tid; it0 < q_end; it0 += (int64_t)B * nthr) {
        uint32_t word[B];
        int gi[B], pp[B];
        int8_t *gp[B];  // the quad's states in HBM
#pragma unroll
        for (int u = 0; u < B; ++u) {
            const int64_t it = it0 + (int64_t)u * nthr;
            const int g = gnext, rem = rnext;
            rnext += nthr;
            while (rnext >= QP) {
                rnext -= QP;
                ++gnext;
            }
            gi[u] = -1;
            word[u] = 0xFFFFFFFFu;
            if (it < q_end) {
                const int p0 = rem << 2;
                gi[u] = g;
                pp[u] = p0;
                gp[u] = k.states + (int64_t)s.rc_clause[gi[u]] * k.P + p0;
                if (k.vec4 && p0 + 4 <= k.P) {
                    word[u] = __ldcg(reinterpret_cast<const unsigned int *>(gp[u]));
                } else {
                    for (int b = 0; b < 4; ++b)
                        if (p0 + b < k.P)
                            word[u] = (word[u] & ~(0xFFu << (8 * b))) |
                                      ((uint32_t)(uint8_t)__ldcg(gp[u] + b) << (8 * b));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < B; ++u) {
            if (it0 + (int64_t)u * nthr >= q_end) break;  // warp-uniform
            const int g = gi[u], p0 = pp[u];
            const int c = s.rc_clause[g];
            const int info = s.rc_info[g] & 0xFF, cls = s.rc_info[g] >> 8;
            const int lim = k.P - p0;
            const uint64_t zp = kGolden * (uint64_t)p0;
            // valid-position byte mask: all ones except in a row's last warp
            uint32_t vb = 0xFFFFFFFFu;
            if (__any_sync(0xffffffffu, lim < 4))
                vb = lim >= 4 ? 0xFFFFFFFFu : (lim <= 0 ? 0u : (0xFFFFFFFFu >> (8 * (4 - lim))));
            uint32_t nw;
            // warp-uniform: a warp's quads share a work item (see feedback_simd)
            if (cls == 1) {
                nw = quad_silent_type1(word[u], vb, smin4, T_dec, s.rc_sk[2 * g] + zp, nd, nupd);
            } else {
                const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
                if (cls == 2) {
                    nw = quad_firing_type1(k, word[u], litn, vb, s.rc_sk[2 * g] + zp, nd, nupd);
                } else if (cls == 3) {
                    nw = quad_type2(word[u], litn, vb, nupd);
                } else {
                    nw = quad_update_simd(k, word[u], info, litn, lim,
                                          (info & I_TEV) ? s.rc_sk[2 * g] + zp : 0,
                                          (info & I_NEV) ? s.rc_sk[2 * g + 1] + zp : 0, nd);
                    nupd += __popc(__vcmpne4(nw, word[u]) & 0x01010101u);
                }
            }
            if (nw != word[u]) {
                if (k.vec4 && p0 + 4 <= k.P) {
                    __stcg(reinterpret_cast<unsigned int *>(gp[u]), nw);
                } else {
                    for (int b = 0; b < 4; ++b)
                        if (p0 + b < k.P) __stcg(gp[u] + b, (int8_t)(nw >> (8 * b)));
                }
            }
            // mask word for positions 32w..32w+31 (lanes 8g..8g+7 hold its
            // nibbles), only when an include bit of the warp's positions
            // flipped: k.gmask holds every clause's current mask (k_train
            // writes the own rows at launch), so an unchanged word is current
            if (__any_sync(0xffffffffu, ((nw ^ word[u]) & 0x80808080u) != 0)) {
                uint32_t m = quad_include_nibble(nw, lim) << ((lane & 7) * 4);
                m |= __shfl_xor_sync(0xffffffffu, m, 1);
                m |= __shfl_xor_sync(0xffffffffu, m, 2);
                m |= __shfl_xor_sync(0xffffffffu, m, 4);
                if ((lane & 7) == 0) {
                    const int w = p0 >> 5;
                    if (w < k.W) __stcg(&k.gmask[(int64_t)c * k.W + w], m);
                }
                if (lane == 0) __stcg(&k.gdirty[c], 1u);
            }
        }
    }
    cn.draws += nd;
    cn.upd += nupd;
}

// Grid-wide arrival + wait on a per-step counter (release / acquire; thread 0
// spins, the CTA waits at a barrier).  Callers: __syncthreads() before.
__device__ __forceinline__ void grid_arrive_step(unsigned *ctr) {
    if (threadIdx.x == 0) {
        __threadfence();
        red_release_add(ctr, 1u);
    }
}
__device__ __forceinline__ void grid_wait_step(const unsigned *ctr, unsigned want) {
    if (threadIdx.x == 0) {
        while (ld_acquire_u32(ctr) < want) {
        }
    }
    __syncthreads();
}

// Load the model slice into shared memory, build include masks and counts.
template <bool SMEM_STATES>
__device__ __forceinline__ void load_slice(const TrainK &k, const Smem &s, int c0, int cown) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int warp = tid >> 5, nwarps = nthr >> 5;
    for (int i = tid; i < cown * k.K; i += nthr) s.weights[i] = k.weights[(int64_t)c0 * k.K + i];
    for (int i = tid; i < cown; i += nthr) s.cnt[i] = 0;
    if (k.MW > k.W)  // row padding of the masks stays 0 (never an include)
        for (int i = tid; i < cown * (k.MW - k.W); i += nthr)
            s.masks[(i / (k.MW - k.W)) * k.MW + k.W + i % (k.MW - k.W)] = 0u;
    if (SMEM_STATES) {
        for (int i = tid; i < cown * k.Ppad; i += nthr) {
            int j = i / k.Ppad, p = i - j * k.Ppad;
            s.states[i] = p < k.P ? k.states[(int64_t)(c0 + j) * k.P + p] : (int8_t)-1;
        }
    }
    __syncthreads();
    for (int it = warp; it < cown * k.W; it += nwarps) {
        int j = it / k.W, w = it - j * k.W;
        int p = w * 32 + lane;
        int st;
        if (SMEM_STATES) st = s.states[j * k.Ppad + p];
        else st = p < k.P ? k.states[(int64_t)(c0 + j) * k.P + p] : -1;
        unsigned m = __ballot_sync(0xffffffffu, st >= 0);
        if (lane == 0) {
            s.masks[j * k.MW + w] = m;
            if (m) atomicAdd(&s.cnt[j], __popc(m));
        }
    }
}

template <bool SMEM_STATES>
__device__ __forceinline__ void store_slice(const TrainK &k, const Smem &s, int c0, int cown) {
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int i = tid; i < cown * k.K; i += nthr) k.weights[(int64_t)c0 * k.K + i] = s.weights[i];
    if (SMEM_STATES) {
        for (int i = tid; i < cown * k.Ppad; i += nthr) {
            int j = i / k.Ppad, p = i - j * k.Ppad;
            if (p < k.P) k.states[(int64_t)(c0 + j) * k.P + p] = s.states[i];
        }
    }
}

__device__ __forceinline__ void flush_stats(const TrainK &k, Counters &cn, bool add_examples) {
    if (!k.stats) return;
    const int lane = threadIdx.x & 31;
    for (int o = 16; o; o >>= 1) {
        cn.draws += __shfl_xor_sync(0xffffffffu, cn.draws, o);
        cn.upd += __shfl_xor_sync(0xffffffffu, cn.upd, o);
        cn.events += __shfl_xor_sync(0xffffffffu, cn.events, o);
        cn.t1 += __shfl_xor_sync(0xffffffffu, cn.t1, o);
        cn.t2 += __shfl_xor_sync(0xffffffffu, cn.t2, o);
    }
    if (lane == 0) {
        atomicAdd((unsigned long long *)&k.stats->draws, (unsigned long long)cn.draws);
        atomicAdd((unsigned long long *)&k.stats->state_updates, (unsigned long long)cn.upd);
        atomicAdd((unsigned long long *)&k.stats->events, (unsigned long long)cn.events);
        atomicAdd((unsigned long long *)&k.stats->type_i, (unsigned long long)cn.t1);
        atomicAdd((unsigned long long *)&k.stats->type_ii, (unsigned long long)cn.t2);
    }
    if (add_examples && threadIdx.x == 0)
        atomicAdd((unsigned long long *)&k.stats->examples, (unsigned long long)k.n_steps);
}

// Example ring in shared memory: misc[3 + (i % 3)] = order[i]; the literal
// row of example i lives in lit{i&1}.  Issued one / two examples ahead so
// the dependent global loads overlap the current example.
// Next-example prefetch, split so the global loads are issued at the top of
// example i (into registers) and committed to shared memory at its end --
// their latency hides behind the whole example instead of stalling it.
constexpr int kRowRegs = 4;  // literal words per thread (W <= 4 * blockDim)
struct Prefetch {
    uint32_t row[kRowRegs];
    int label, ex2;
};

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ void prefetch_issue(const TrainK &k, const Smem &s, int64_t i,
                                               Prefetch &pf) {
    if (i + 1 >= k.n_steps) return;
    const int ex = s.misc[3 + (int)((i + 1) % 3)];
#pragma unroll
    for (int q = 0; q < kRowRegs; ++q) {
        const int w = threadIdx.x + q * blockDim.x;
        if (w < k.W) pf.row[q] = __ldg(&k.lit_words[(int64_t)ex * k.W + w]);
    }
    if (threadIdx.x == blockDim.x - 1) {
        pf.label = __ldg(&k.labels[ex]);
        if (i + 2 < k.n_steps) pf.ex2 = __ldg(&k.order[i + 2]);
    }
}

__device__ __forceinline__ void prefetch_commit(const TrainK &k, const Smem &s, int64_t i,
                                                const Prefetch &pf) {
    if (i + 1 >= k.n_steps) return;
    uint32_t *dst = ((i + 1) & 1) ? s.lit1 : s.lit0;
#pragma unroll
    for (int q = 0; q < kRowRegs; ++q) {
        const int w = threadIdx.x + q * blockDim.x;
        if (w < k.W) dst[w] = pf.row[q];
    }
    if (threadIdx.x == blockDim.x - 1) {
        s.misc[8 + (int)((i + 1) % 3)] = pf.label;
        if (i + 2 < k.n_steps) s.misc[3 + (int)((i + 2) % 3)] = pf.ex2;
    }
}

__device__ __forceinline__ void prologue_ring(const TrainK &k, const Smem &s) {
    if (threadIdx.x == 0) {
        s.misc[3] = __ldg(&k.order[0]);
        s.misc[8] = __ldg(&k.labels[s.misc[3]]);
        if (k.n_steps > 1) s.misc[4] = __ldg(&k.order[1]);
        s.vacc[0] = 0;
        s.vacc[1] = 0;
    }
    __syncthreads();
    const int ex = s.misc[3];
    for (int w = threadIdx.x; w < k.W; w += blockDim.x)
        s.lit0[w] = __ldg(&k.lit_words[(int64_t)ex * k.W + w]);
}

__device__ __forceinline__ void decide(const TrainK &k, long long vl, long long vn,
                                       uint64_t &t_t, uint64_t &t_n) {
    const long long T = k.T;
    const long long cl = vl < -T ? -T : (vl > T ? T : vl);
    const long long cn = vn < -T ? -T : (vn > T ? T : vn);
    t_t = threshold_of(T - cl, T);
    t_n = threshold_of(T + cn, T);
}

__device__ __forceinline__ int negative_class(const TrainK &k, int label, uint64_t fbc) {
    // two classes: u * (K - 1) < 1 whatever the draw, so it need not be
    // evaluated (the stream is random-access, core.py:7-10)
    if (k.K == 2) return label ^ 1;
    const double u = u01_from53(draw53(k.fb_seed, fbc));
    int neg = label + 1 + (int)(u * (double)(k.K - 1));  // < 2K
    return neg >= k.K ? neg - k.K : neg;
}

// Event bookkeeping of own clause j (kernels/_numba.py:101-125): window
// ordinal `ord` of its first event, event types, feedback-then-weight
// and the work list.  s.info[j] & I_OUT holds its output.
__device__ __forceinline__ void apply_events(const TrainK &k, const Smem &s, Counters &cn, int j,
                                             bool t_ev, bool n_ev, uint64_t ord, uint64_t bseed,
                                             int label, int neg) {
    int info = s.info[j] & I_OUT;
    if (t_ev || n_ev) {
        const bool out = info & I_OUT;
        int32_t *w = s.weights + j * k.K;
        const bool t1 = w[label] >= 0, n1 = w[neg] < 0;
        if (t_ev) {
            info |= I_TEV | (t1 ? I_T1 : 0);
            s.sk_t[j] = bseed + kGolden * ((ord << 32) + 1);
            ++cn.events;
            if (t1) ++cn.t1; else if (out) ++cn.t2;
        }
        if (n_ev) {
            const uint64_t o2 = ord + (t_ev ? 1 : 0);
            info |= I_NEV | (n1 ? I_N1 : 0);
            s.sk_n[j] = bseed + kGolden * ((o2 << 32) + 1);
            ++cn.events;
            if (n1) ++cn.t1; else if (out) ++cn.t2;
        }
        if (out) {
            if (t_ev) w[label] += 1;
            if (n_ev) w[neg] -= 1;
        }
        if ((t_ev && ((info & I_T1) || out)) || (n_ev && ((info & I_N1) || out)))
            s.work[atomicAdd(&s.misc[0], 1)] = j;
    }
    s.info[j] = info;
}

// Training-mode output of own clause j against literal row `lit` (warp-
// collective; kernels/_numba.py:36-50): no included literal false and the
// include count within the budget.
__device__ __forceinline__ bool clause_out(const TrainK &k, const Smem &s, int j,
                                           const uint32_t *lit) {
    uint32_t viol = 0;
    for (int w = (int)(threadIdx.x & 31); w < k.W; w += 32) viol |= s.masks[j * k.MW + w] & ~lit[w];
    viol = __reduce_or_sync(0xffffffffu, viol);
    return viol == 0 && s.cnt[j] <= k.budget;
}

__device__ __forceinline__ void cluster_arrive() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Phase profiling (k.phase != nullptr): thread 0 of every CTA accumulates
// clock64 deltas between consecutive PHASE marks.
#define PHASE(n)                                                          \
    do {                                                                  \
        if (prof && warp == 0) {                                          \
            const long long now = clock64();                              \
            ph[n] += (unsigned long long)(now - t_mark);                  \
            t_mark = now;                                                 \
        }                                                                 \
    } while (0)

// Grid-mode timeline (profiling): %globaltimer of thread 0 at arrival,
// all-reduce detection and step end for steps [64, 64 + kTimelineSteps),
// stored after the phase array as [kTimelineSteps][n_cta][3].
constexpr int kTimelineSteps = 1024;
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TIMELINE(i, q)                                                              \
    do {                                                                            \
        if (prof && warp == 0 && (i) >= 64 && (i) < 64 + kTimelineSteps) {                          \
            const unsigned long long g_ = gtimer();                                 \
            if (lane == 0) k.phase[n_cta * 8 + (((i) - 64) * n_cta + rank) * 3 + (q)] = g_; \
        }                                                                           \
    } while (0)

// One fused kernel, two synchronisation domains (see the header comment).
// NT: the CTA size the build is bounded for (1024: the HBM-state grid
// kernel with twice the warps to hide its feedback's dependency latency)
template <int MODE, bool SMEM_STATES, int NT = 512>
__global__ void __launch_bounds__(NT, 1) k_train(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, SMEM_STATES, MODE, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthr >> 5;
    int rank;
    if (MODE == MODE_CLUSTER) rank = (int)cg::this_cluster().block_rank();
    else rank = blockIdx.x;
    const int C = k.C, K = k.K, n_cta = k.n_cta;
    const int c0 = cta_begin(rank, C, n_cta), c1 = cta_begin(rank + 1, C, n_cta);
    const int cown = c1 - c0;
    const int b0 = block_of(c0, C, k.n_blocks), b1 = block_of(c1 - 1, C, k.n_blocks);
    const int fs = block_begin(b0, C, k.n_blocks), fe = block_begin(b1 + 1, C, k.n_blocks);
    const int fsa = fs & ~31;
    const int nfw = (fe - fsa + 31) >> 5;
    const bool pre = s.draw_t != nullptr;

    load_slice<SMEM_STATES>(k, s, c0, cown);
    for (int i = tid; i <= b1 - b0; i += nthr) {
        s.blk_ctr[i] = k.block_counters[b0 + i];
        s.blk_seed[i] = k.block_seeds[b0 + i];
    }
    prologue_ring(k, s);
    __syncthreads();
    if (MODE == MODE_CLUSTER) cg::this_cluster().sync();  // DSMEM peers resident

    Counters cn;
    const bool prof = k.phase != nullptr;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long t_mark = clock64();
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;

    const bool gbal = MODE == MODE_GRID && !SMEM_STATES && k.gbal;
    if (gbal) {
        // k.gmask mirrors every clause's include mask from the start (the
        // balanced feedback rewrites only the words whose include bits flip);
        // ordered before any peer's write by this CTA's first release arrival
        for (int q = tid; q < cown * k.W; q += nthr) {
            const int j = q / k.W, w = q - j * k.W;
            __stcg(&k.gmask[(int64_t)(c0 + j) * k.W + w], s.masks[j * k.MW + w]);
        }
        for (int j = tid; j < cown; j += nthr) __stcg(&k.gdirty[c0 + j], 0u);
        if (tid == 0) s.misc[2] = 0;
    }
    for (int64_t i = 0; i < k.n_steps; ++i) {
        const uint32_t *lit = (i & 1) ? s.lit1 : s.lit0;
        const int label = s.misc[8 + (int)(i % 3)];
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        const int neg = negative_class(k, label, fbc);
        Prefetch pf;
        prefetch_issue(k, s, i, pf);
        if (gbal && i > 0) {
            // all CTAs' feedback of step i-1 is done: pull the include masks
            // of the own clauses whose include bits it flipped, recount them
            grid_wait_step(&k.gsync[(i - 1) * 2 + 1], (unsigned)n_cta);  // arrived below
            PHASE(7);
            const int n_prev = s.misc[0];
            for (int q = warp; q < n_prev; q += nwarps) {
                const int j = s.work[q];
                if (__ldcg(&k.gdirty[c0 + j]) == 0u) continue;  // no include bit flipped
                __syncwarp();
                if (lane == 0) __stcg(&k.gdirty[c0 + j], 0u);
                const uint32_t *src = k.gmask + (int64_t)(c0 + j) * k.W;
                int cnt = 0;
                for (int w = lane; w < k.W; w += 32) {
                    const uint32_t m = __ldcg(src + w);
                    s.masks[j * k.MW + w] = m;
                    cnt += __popc(m);
                }
                cnt = __reduce_add_sync(0xffffffffu, cnt);
                if (lane == 0) s.cnt[j] = cnt;
            }
            __syncthreads();
        }
        // 1. training-mode outputs of own clauses (kernels/_numba.py:36-50);
        //    grid mode folds the two class sums the decision reads
        //    (dense.py:153 restricted to label / negative) into the same pass
        for (int j = warp; j < ((k.dbg & 2) ? 0 : cown); j += nwarps) {
            uint32_t viol = 0;
            for (int w = lane; w < k.W; w += 32) viol |= s.masks[j * k.MW + w] & ~lit[w];
            viol = __reduce_or_sync(0xffffffffu, viol);
            if (lane == 0) {
                const bool out = viol == 0 && s.cnt[j] <= k.budget;
                s.info[j] = out ? I_OUT : 0;
                if (MODE == MODE_GRID && out) {
                    atomicAdd(&s.vacc[0], (unsigned long long)(long long)s.weights[j * K + label]);
                    atomicAdd(&s.vacc[1], (unsigned long long)(long long)s.weights[j * K + neg]);
                }
            }
        }
        if (tid == 0) s.misc[0] = 0;
        __syncthreads();
        PHASE(0);
        // 2. all-reduce of the partial class sums
        const int buf = (int)(i & 1);
        if (MODE == MODE_CLUSTER) {
            if (warp < 2) {
                const int kk = warp == 0 ? label : neg;
                long long v = 0;
                for (int j = lane; j < cown; j += 32)
                    if (s.info[j] & I_OUT) v += s.weights[j * K + kk];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                // push into every CTA's inbox (DSMEM stores, no round trip)
                if (lane < n_cta) {
                    long long *dst = cg::this_cluster().map_shared_rank(s.vin, lane);
                    dst[(buf * 16 + rank) * 2 + warp] = v;
                }
            }
            cluster_arrive();
        } else if (tid == 0) {
            // fence-free arrival: one relaxed atomic per word carries the
            // arrival count (bits 40..63) and the biased partial (bits 0..39)
            const long long vl = (long long)s.vacc[0], vn = (long long)s.vacc[1];
            s.vacc[0] = 0;
            s.vacc[1] = 0;
            red_relaxed_add_u64(&k.rec[i * 2 + 0], (1ull << 40) + (unsigned long long)(vl + kVoteBias));
            red_relaxed_add_u64(&k.rec[i * 2 + 1], (1ull << 40) + (unsigned long long)(vn + kVoteBias));
            TIMELINE(i, 0);
        }
        PHASE(1);
        // while the all-reduce is pending: update-flag draws for [fs, fe)
        // (feedback.py:47-53; independent of the votes)
        if (pre) {
            for (int idx = tid; idx < nfw * 32; idx += nthr) {
                const int j = fsa + idx;
                s.draw_t[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)j);
                s.draw_n[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)j);
            }
        }
        PHASE(2);
        uint64_t t_t, t_n;
        if (MODE == MODE_CLUSTER) {
            cluster_wait();
            // every warp sums the inbox itself: no CTA-wide broadcast needed
            long long v = 0;
            if (lane < n_cta) v = s.vin[(buf * 16 + lane) * 2 + 0];
            else if (lane >= 16 && lane - 16 < n_cta) v = s.vin[(buf * 16 + lane - 16) * 2 + 1];
            long long vl = lane < 16 ? v : 0, vn = lane < 16 ? 0 : v;
            for (int o = 16; o; o >>= 1) {
                vl += __shfl_xor_sync(0xffffffffu, vl, o);
                vn += __shfl_xor_sync(0xffffffffu, vn, o);
            }
            decide(k, vl, vn, t_t, t_n);
            if (k.trace && rank == 0 && tid == 0) {
                k.trace[i * 4 + 0] = neg;
                k.trace[i * 4 + 1] = vl;
                k.trace[i * 4 + 2] = vn;
            }
        } else {
            // all-reduce complete when both words count n_cta arrivals;
            // thread 0 decides and broadcasts the two thresholds
            if (tid == 0) {
                const unsigned long long want = (unsigned long long)n_cta;
                ulonglong2 p;
                do {
                    p = ld_relaxed_v2u64(&k.rec[i * 2]);
                } while ((p.x >> 40) != want || (p.y >> 40) != want);
                TIMELINE(i, 1);
                const long long bias = (long long)n_cta * kVoteBias;
                const long long vl = (long long)(p.x & ((1ull << 40) - 1)) - bias;
                const long long vn = (long long)(p.y & ((1ull << 40) - 1)) - bias;
                decide(k, vl, vn, t_t, t_n);
                if (k.dbg & 4) t_t = t_n = 0;
                s.thr[0] = t_t;
                s.thr[1] = t_n;
                if (k.trace && rank == 0) {
                    k.trace[i * 4 + 0] = neg;
                    k.trace[i * 4 + 1] = vl;
                    k.trace[i * 4 + 2] = vn;
                }
            }
            __syncthreads();
            t_t = s.thr[0];
            t_n = s.thr[1];
        }
        PHASE(3);
        // 3. update flags over [fs, fe) as bitmaps
        for (int idx = tid; idx < nfw * 32; idx += nthr) {
            const int j = fsa + idx;
            const bool valid = j >= fs && j < fe;
            uint64_t mt, mn;
            if (pre) {
                mt = s.draw_t[idx];
                mn = s.draw_n[idx];
            } else {
                mt = draw53(k.fb_seed, fbc + 1 + (uint64_t)j);
                mn = draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)j);
            }
            const unsigned wt = __ballot_sync(0xffffffffu, valid && mt < t_t);
            const unsigned wn = __ballot_sync(0xffffffffu, valid && mn < t_n);
            if (lane == 0) {
                s.ut_bits[idx >> 5] = wt;
                s.un_bits[idx >> 5] = wn;
            }
        }
        __syncthreads();
        PHASE(4);
        // 4-5. warp 0: exclusive prefix of events per flag word, then
        //      window ordinals and the work list of the own clauses
        if (warp == 0) {
            int carry = 0;
            for (int base = 0; base < nfw; base += 32) {
                const int w = base + lane;
                const int v = w < nfw ? __popc(s.ut_bits[w]) + __popc(s.un_bits[w]) : 0;
                int x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (w < nfw) s.word_cum[w] = carry + x - v;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) {
                s.word_cum[nfw] = carry;
                if (k.trace && rank == 0 && fs == 0 && fe == C) k.trace[i * 4 + 3] = carry;
            }
            __syncwarp();
            auto cum = [&](int x) -> int {  // events over clauses [fsa, x)
                const int q = (x - fsa) >> 5, r = (x - fsa) & 31;
                int v = s.word_cum[q];
                if (r) {
                    const unsigned lo = (1u << r) - 1u;
                    v += __popc(s.ut_bits[q] & lo) + __popc(s.un_bits[q] & lo);
                }
                return v;
            };
            for (int j = lane; j < cown; j += 32) {
                const int c = c0 + j;
                const int q = (c - fsa) >> 5, r = (c - fsa) & 31;
                const bool t_ev = (s.ut_bits[q] >> r) & 1, n_ev = (s.un_bits[q] >> r) & 1;
                int bi = 0;
                uint64_t ord = 0;
                if (t_ev || n_ev) {
                    if (k.n_blocks == 1) {  // fs == 0: events before c in the block
                        ord = s.blk_ctr[0] + (uint64_t)cum(c);
                    } else {
                        bi = block_of(c, C, k.n_blocks) - b0;
                        ord = s.blk_ctr[bi] +
                              (uint64_t)(cum(c) - cum(block_begin(b0 + bi, C, k.n_blocks)));
                    }
                }
                apply_events(k, s, cn, j, t_ev, n_ev, ord, s.blk_seed[bi], label, neg);
            }
            __syncwarp();
            // one window per applied event (block counters)
            if (k.n_blocks == 1) {
                if (lane == 0) s.blk_ctr[0] += (uint64_t)s.word_cum[nfw];
            } else for (int bi = lane; bi <= b1 - b0; bi += 32) {
                const int bs = block_begin(b0 + bi, C, k.n_blocks);
                const int be = block_begin(b0 + bi + 1, C, k.n_blocks);
                s.blk_ctr[bi] += (uint64_t)(cum(be) - cum(bs));
            }
        }
        __syncthreads();
        PHASE(5);
        // 6. per-position Type I / II updates of the work list
        if (gbal) {
            // publish this CTA's work list, then take an even share of the
            // union's quads (work items in CTA order, quads in row order)
            const int n_work = s.misc[0];
            for (int q = tid; q < n_work; q += nthr) {
                const int j = s.work[q];
                const int64_t o = (int64_t)rank * k.cmax + q;
                __stcg(&k.gw_clause[o], c0 + j);
                __stcg(&k.gw_info[o], s.info[j]);
                __stcg(&k.gw_sk[2 * o], (unsigned long long)s.sk_t[j]);
                __stcg(&k.gw_sk[2 * o + 1], (unsigned long long)s.sk_n[j]);
            }
            {   // summed cost weight of the own work list
                int wsum = 0;
                for (int q = tid; q < n_work; q += nthr) wsum += gbal_weight(k, s.info[s.work[q]]);
                wsum = __reduce_add_sync(0xffffffffu, wsum);
                if (lane == 0 && wsum) atomicAdd(&s.misc[2], wsum);
            }
            __syncthreads();
            if (tid == 0) {
                __stcg(&k.gcount[rank], n_work);
                __stcg(&k.gcount[n_cta + rank], s.misc[2]);
                s.misc[2] = 0;
            }
            __syncthreads();
            grid_arrive_step(&k.gsync[i * 2]);
            grid_wait_step(&k.gsync[i * 2], (unsigned)n_cta);
            if (warp < 2) {  // warp 0: prefix of the counts, warp 1: of the cost weights
                int *pref = warp == 0 ? s.gpref : s.gwpref;
                int carry = 0;
                for (int base = 0; base < n_cta; base += 32) {
                    const int r = base + lane;
                    const int v = r < n_cta ? __ldcg(&k.gcount[warp * n_cta + r]) : 0;
                    int x = v;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const int y = __shfl_up_sync(0xffffffffu, x, o);
                        if (lane >= o) x += y;
                    }
                    if (r < n_cta) pref[r] = carry + x - v;
                    carry += __shfl_sync(0xffffffffu, x, 31);
                }
                if (lane == 0) pref[n_cta] = carry;
            }
            __syncthreads();
            // This CTA's share: the union's 32-quad units (work items in CTA
            // order, quads in row order), each unit weighted by its item's
            // cost, cut at the weighted positions X(rank), X(rank + 1) -- every
            // CTA computes the same cuts.  Warp 0 locates X(rank), warp 1
            // X(rank + 1): owner CTA by the weight prefix, item by a scan of
            // that CTA's published infos, unit = offset / item weight.
            const int QP = k.Ppad >> 2, U = QP >> 5;
            if (warp < 2) {
                const int64_t wt = (int64_t)s.gwpref[n_cta] * U;
                const int64_t X = wt * (rank + warp) / n_cta;
                int64_t q = (int64_t)s.gpref[n_cta] * QP;  // X == wt: the end
                if (X < wt) {
                    int lo = 0, hi = n_cta;  // owner: gwpref[lo] * U <= X < gwpref[lo + 1] * U
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if ((int64_t)s.gwpref[mid] * U <= X) lo = mid;
                        else hi = mid;
                    }
                    const int cnt = s.gpref[lo + 1] - s.gpref[lo];
                    int64_t off = X - (int64_t)s.gwpref[lo] * U;  // weighted offset inside the owner's list
                    int found = -1, unit = 0;
                    for (int base = 0; base < cnt && found < 0; base += 32) {
                        const int t = base + lane;
                        const int w = t < cnt ? gbal_weight(k, __ldcg(&k.gw_info[(int64_t)lo * k.cmax + t])) : 0;
                        int x = w;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int y = __shfl_up_sync(0xffffffffu, x, o);
                            if (lane >= o) x += y;
                        }
                        const int64_t before = (int64_t)(x - w) * U;  // weighted start of item t in this group
                        const bool here = t < cnt && off >= before && off < before + (int64_t)w * U;
                        const unsigned bal = __ballot_sync(0xffffffffu, here);
                        if (bal) {
                            const int src = __ffs(bal) - 1;
                            found = base + src;
                            unit = (int)((off - __shfl_sync(0xffffffffu, before, src)) /
                                         __shfl_sync(0xffffffffu, w, src));
                        } else {
                            off -= (int64_t)__shfl_sync(0xffffffffu, x, 31) * U;
                        }
                    }
                    if (found >= 0) q = ((int64_t)s.gpref[lo] + found) * QP + 32 * (int64_t)unit;
                }
                if (lane == 0) s.gcut[warp] = q;
            }
            __syncthreads();
            const int64_t q_begin = s.gcut[0], q_end = s.gcut[1];
            // the share's work items are staged cmax + 4 at a time (a share of
            // cheap items can hold more items than any CTA owns)
            const int rc_cap = k.cmax + 4;
            for (int64_t g_lo = q_begin / QP; g_lo * QP < q_end; g_lo += rc_cap) {
                const int64_t g_hi = (q_end - 1) / QP;  // last item of the share
                const int n_rc = (int)((g_hi - g_lo + 1) < rc_cap ? (g_hi - g_lo + 1) : rc_cap);
                for (int t = tid; t < n_rc; t += nthr) {
                    const int g = (int)(g_lo + t);
                    int lo = 0, hi = n_cta;  // owner r: gpref[r] <= g < gpref[r + 1]
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (s.gpref[mid] <= g) lo = mid;
                        else hi = mid;
                    }
                    const int64_t o = (int64_t)lo * k.cmax + (g - s.gpref[lo]);
                    s.rc_clause[t] = __ldcg(&k.gw_clause[o]);
                    const int info_t = __ldcg(&k.gw_info[o]);
                    s.rc_info[t] = info_t | (fb_class(info_t) << 8);  // event class decided once per item
                    // (a single-event row's key in slot 0, whichever event it is)
                    const bool neg_only = (info_t & (I_TEV | I_NEV)) == I_NEV;
                    s.rc_sk[2 * t] = __ldcg(&k.gw_sk[2 * o + (neg_only ? 1 : 0)]);
                    s.rc_sk[2 * t + 1] = __ldcg(&k.gw_sk[2 * o + 1]);
                }
                __syncthreads();
                const int64_t qa = q_begin > g_lo * QP ? q_begin : g_lo * QP;
                const int64_t qb = q_end < (g_lo + n_rc) * QP ? q_end : (g_lo + n_rc) * QP;
                if (!(k.dbg & 1))  // 1024 threads: half the words in flight per thread
                    feedback_quads_global<(NT > 512 ? TMB_GB_B : 4)>(k, s, lit, qa, qb, g_lo, cn);
                __syncthreads();
            }
            prefetch_commit(k, s, i, pf);
            __syncthreads();
            // feedback done: the next step waits on it
            grid_arrive_step(&k.gsync[i * 2 + 1]);
        } else {
            // shared-memory states: the byte-SIMD body; HBM states keep the
            // 4-word-in-flight body (its loads go to L2 / HBM)
            if (SMEM_STATES) feedback_simd<true>(k, s, c0, lit, (k.dbg & 1) ? 0 : s.misc[0], cn);
            else feedback_quads<false>(k, s, c0, lit, (k.dbg & 1) ? 0 : s.misc[0], cn);
            prefetch_commit(k, s, i, pf);
            __syncthreads();
        }
        PHASE(6);
        if (MODE == MODE_GRID) TIMELINE(i, 2);
    }
    if (prof && tid == 0)
        for (int q = 0; q < 8; ++q) k.phase[rank * 8 + q] = ph[q];
    if (MODE == MODE_CLUSTER) cg::this_cluster().sync();  // peers done with our inbox
    store_slice<SMEM_STATES>(k, s, c0, cown);
    for (int bi = tid; bi <= b1 - b0; bi += nthr) {
        const int b = b0 + bi;
        const int last = block_begin(b + 1, C, k.n_blocks) - 1;
        if (last >= c0 && last < c1) k.block_counters[b] = s.blk_ctr[bi];
    }
    flush_stats(k, cn, rank == 0);
}


// ------------------------------------------------------------- fast path --
// Step record (u32 words): [0..3] example, label, negative class, 0;
// [4, 4 + Wp) literal row; then u16 bucket starts [2][260] (stream 0 =
// target flags, 1 = negative flags; start[256] = C); then entries u32
// [2][Cp] = key << 16 | clause grouped by bucket key >> 8, key = draw53 >> 37
// (order inside a bucket arbitrary).  Flag of clause c in stream s is
// draw53(fb_seed, fbc + 1 + s*C + c) < t_s  <=>  key < t_s >> 37, or key equal
// and the exact draw below t_s (feedback.py:47-53).
__host__ __device__ inline int rec_buckets(const TrainK &k) { return 4 + k.Wp; }
__host__ __device__ inline int rec_entries(const TrainK &k) { return 4 + k.Wp + 260; }

// One CTA per (step, stream); dynamic shared memory: u16 keys [C].
__global__ void __launch_bounds__(256) k_step_records(TrainK k, uint32_t *out) {
    extern __shared__ uint16_t skey[];
    __shared__ unsigned hist[256], wsum[8];
    const int64_t i = blockIdx.x;
    const int str = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = k.C;
    uint32_t *r = out + i * (int64_t)k.R;
    const uint64_t fbc = k.fb_counter0 + (uint64_t)i * (1ull + 2ull * (uint64_t)C);
    if (str == 0) {
        const int ex = __ldg(&k.order[i]);
        if (tid == 0) {
            const int label = __ldg(&k.labels[ex]);
            r[0] = (uint32_t)ex;
            r[1] = (uint32_t)label;
            r[2] = (uint32_t)negative_class(k, label, fbc);
            r[3] = 0;
        }
        for (int w = tid; w < k.Wp; w += 256)
            r[4 + w] = w < k.W ? __ldg(&k.lit_words[(int64_t)ex * k.W + w]) : 0u;
    }
    hist[tid] = 0;
    __syncthreads();
    const uint64_t base = fbc + 1 + (str ? (uint64_t)C : 0);
    for (int j = tid; j < C; j += 256) {
        const unsigned key = (unsigned)(draw53(k.fb_seed, base + (uint64_t)j) >> 37);
        skey[j] = (uint16_t)key;
        atomicAdd(&hist[key >> 8], 1u);
    }
    __syncthreads();
    // exclusive scan of the 256 bucket sizes
    const unsigned h = hist[tid];
    unsigned x = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    unsigned wb = 0;
    for (int q = 0; q < warp; ++q) wb += wsum[q];
    const unsigned start = wb + x - h;
    uint16_t *off = reinterpret_cast<uint16_t *>(r + rec_buckets(k)) + str * 260;
    off[tid] = (uint16_t)start;
    if (tid == 0) off[256] = (uint16_t)C;
    __syncthreads();  // everyone read hist[] before it becomes the cursor
    hist[tid] = start;
    __syncthreads();
    uint32_t *ent = r + rec_entries(k) + str * k.Cp;
    for (int j = tid; j < C; j += 256) {
        const unsigned key = skey[j];
        const unsigned pos = atomicAdd(&hist[key >> 8], 1u);
        ent[pos] = (key << 16) | (unsigned)j;
    }
}

// Record of step i into ring slot i & 3 (cp.async, 16 B per copy).
__device__ __forceinline__ void rec_issue(const TrainK &k, const Smem &s, int64_t i, int t0,
                                          int nt) {
    const uint32_t *src = k.recs + i * (int64_t)k.R;
    uint32_t *dst = s.rec3 + (int)(i & 3) * k.R;
    for (int q = t0; q < k.R / 4; q += nt) cp_async16(dst + 4 * q, src + 4 * q);
    cp_async_commit();
}

// Two 64-bit warp sums from 32-bit reductions: low 24 bits unsigned, the rest
// signed (exact while |x| < 2^54 per lane).
__device__ __forceinline__ void warp_sum2(long long a, long long b, long long &sa, long long &sb) {
    const unsigned al = __reduce_add_sync(0xffffffffu, (unsigned)(a & 0xFFFFFF));
    const unsigned bl = __reduce_add_sync(0xffffffffu, (unsigned)(b & 0xFFFFFF));
    const int ah = __reduce_add_sync(0xffffffffu, (int)(a >> 24));
    const int bh = __reduce_add_sync(0xffffffffu, (int)(b >> 24));
    sa = (long long)ah * (1LL << 24) + (long long)al;
    sb = (long long)bh * (1LL << 24) + (long long)bl;
}

// Warp 0: outputs of example e (nout buffer e & 1) into info, and thread 0's
// partial class sums for its label and negative class (dense.py:153).
__device__ __forceinline__ void votes_pass(const TrainK &k, const Smem &s, int cown, int64_t e,
                                           long long &vl, long long &vn) {
    const int lane = threadIdx.x & 31;
    const uint32_t *rc = s.rec3 + (int)(e & 3) * k.R;
    const int label = (int)rc[1], neg = (int)rc[2];
    const int *no = s.nout + (int)(e & 1) * k.cmax;
    long long a = 0, b = 0;
    for (int j = lane; j < cown; j += 32) {
        const int o = no[j];
        s.info[j] = o ? I_OUT : 0;
        if (o) {
            a += s.weights[j * k.K + label];
            b += s.weights[j * k.K + neg];
        }
    }
    warp_sum2(a, b, vl, vn);
}

// Fast-path event application for own clause j (apply_events plus the class
// sum correction of example i+1): returns true when j joined the work list
// (its correction then comes with its re-evaluation).
__device__ __forceinline__ void fast_events(const TrainK &k, const Smem &s, Counters &cn, int j,
                                            bool t_ev, bool n_ev, uint64_t ord, int label,
                                            int neg, bool more, int par, int label1, int neg1) {
    const int n0 = s.misc[0];
    (void)n0;
    int info = s.info[j] & I_OUT;
    const bool out = info & I_OUT;
    int32_t *w = s.weights + j * k.K;
    const bool t1 = w[label] >= 0, n1 = w[neg] < 0;
    const uint64_t bseed = s.blk_seed[0];
    if (t_ev) {
        info |= I_TEV | (t1 ? I_T1 : 0);
        s.sk_t[j] = bseed + kGolden * ((ord << 32) + 1);
        ++cn.events;
        if (t1) ++cn.t1; else if (out) ++cn.t2;
    }
    if (n_ev) {
        const uint64_t o2 = ord + (t_ev ? 1 : 0);
        info |= I_NEV | (n1 ? I_N1 : 0);
        s.sk_n[j] = bseed + kGolden * ((o2 << 32) + 1);
        ++cn.events;
        if (n1) ++cn.t1; else if (out) ++cn.t2;
    }
    if (out) {
        if (t_ev) w[label] += 1;
        if (n_ev) w[neg] -= 1;
    }
    s.info[j] = info;
    if ((t_ev && ((info & I_T1) || out)) || (n_ev && ((info & I_N1) || out))) {
        s.work[atomicAdd(&s.misc[0], 1)] = j;
    } else if (more && out) {
        // weights moved, output unchanged: correct example i+1's sums now
        const bool o = s.nout[par * k.cmax + j] != 0;
        const long long *cl = s.clo + par * 2 * k.cmax;
        const long long dl = (o ? w[label1] : 0) - cl[j], dn = (o ? w[neg1] : 0) - cl[k.cmax + j];
        if (dl) atomicAdd(&s.vsh[par * 2 + 0], (unsigned long long)dl);
        if (dn) atomicAdd(&s.vsh[par * 2 + 1], (unsigned long long)dn);
    }
}

__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

constexpr int kRecRing = 4;  // step records in shared memory (i & 3)

// Largest CTA of the fast trainer (more warps: more shadow evaluation and
// feedback throughput per CTA, fewer registers per thread)
#ifndef TMB_FAST_MAX_THREADS
#define TMB_FAST_MAX_THREADS 512
#endif
constexpr int kFastMaxThreads = TMB_FAST_MAX_THREADS;

// PROF: the phase-profiling build (tools/phase_profile.py); its per-step
// accumulators cost registers the production build cannot spare
template <bool SMEM_STATES, bool PROF>
__global__ void __launch_bounds__(kFastMaxThreads, 1) k_train_fast(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, SMEM_STATES, MODE_GRID, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthr >> 5;
    const int rank = blockIdx.x;
    const int C = k.C, n_cta = k.n_cta;
    const int c0 = cta_begin(rank, C, n_cta), c1 = cta_begin(rank + 1, C, n_cta);
    const int cown = c1 - c0;
    const int64_t n = k.n_steps;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    auto REC = [&](int64_t e) { return s.rec3 + (int)(e & (kRecRing - 1)) * k.R; };

    load_slice<SMEM_STATES>(k, s, c0, cown);
    if (k.thr_smem)
        for (int64_t a = tid; a <= 2 * k.T; a += nthr) s.thr_tab[a] = k.thr_tab[a];
    if (tid == 0) {
        s.blk_ctr[0] = k.block_counters[0];
        s.blk_seed[0] = k.block_seeds[0];
        s.misc[0] = 0;
    }
    for (int j = tid; j < cown; j += nthr) s.oflag[j] = 0;
    if (tid < 4) s.vsh[tid] = 0;
    for (int64_t q = 0; q < 3 && q < n; ++q) rec_issue(k, s, q, tid, nthr);
    cp_async_wait_all();
    __syncthreads();
    for (int j = warp; j < cown; j += nwarps) {
        const bool o = clause_out(k, s, j, REC(0) + 4);
        if (lane == 0) s.nout[j] = o;
    }
    __syncthreads();
    // arrival of step 0: one relaxed atomic per word carries the arrival
    // count (bits 40..63) and the biased partial class sum (bits 0..39)
    if (warp == 0) {
        long long vl = 0, vn = 0;
        votes_pass(k, s, cown, 0, vl, vn);
        if (lane == 0 && n > 0) {
            red_relaxed_add_u64(&k.rec[0], (1ull << 40) + (unsigned long long)(vl + kVoteBias));
            red_relaxed_add_u64(&k.rec[1], (1ull << 40) + (unsigned long long)(vn + kVoteBias));
        }
    }

    Counters cn;
    const bool prof = PROF && k.phase != nullptr;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // per-step phase deltas, flushed into ph (empty / light steps) or phh
    // (steps with > 64 candidate flag entries) at the step's end
    unsigned long long cur[8] = {0, 0, 0, 0, 0, 0, 0, 0}, phh[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long n_heavy = 0;
#define PHASEF(n)                                                         \
    do {                                                                  \
        if (prof && warp == 0) {                                          \
            const long long now = clock64();                              \
            cur[n] += (unsigned long long)(now - t_mark);                 \
            t_mark = now;                                                 \
        }                                                                 \
    } while (0)
#define PHASE_FLUSH(heavy)                                                \
    do {                                                                  \
        if (prof && warp == 0) {                                          \
            for (int q_ = 0; q_ < 8; ++q_) {                              \
                if (heavy) phh[q_] += cur[q_]; else ph[q_] += cur[q_];    \
                cur[q_] = 0;                                              \
            }                                                             \
            n_heavy += (heavy) ? 1 : 0;                                   \
        }                                                                 \
    } while (0)
    // decision constants (loop-invariant, kept in registers): lane 0 of warp
    // 0 turns the label sum into T - v, lane 1 the negative sum into T + v
    const long long dec_bias = (long long)n_cta * kVoteBias;
    const long long dec_c0 = lane == 0 ? k.T + dec_bias : k.T - dec_bias;
    const long long dec_2T = 2 * k.T;
    const bool dec_tab = k.thr_smem != 0, dec_dbg = (k.dbg & 36) != 0;
    long long t_mark = clock64();
    for (int64_t i = 0; i < n; ++i) {
        uint32_t *rc = REC(i);
        const uint32_t *lit = rc + 4;
        const int label = (int)rc[1], neg = (int)rc[2];
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        const bool more = i + 1 < n;
        const int par = (int)((i + 1) & 1);
        const uint32_t *rn = REC(i + 1);
        const int label1 = more ? (int)rn[1] : 0, neg1 = more ? (int)rn[2] : 0;
        // 1. arrival (issued at the end of the previous step, or in the
        //    prologue for step 0)
        PHASEF(0);
        if (warp == 0) {
            // 2. all-reduce, then the decision (feedback.py:33-53): lane 0
            //    the target threshold, lane 1 the negative one.  The whole
            //    warp spins on the same 16 B (one request per iteration) so
            //    it stays converged.
            const unsigned long long want = (unsigned long long)n_cta;
            ulonglong2 p;
            do {
                p = ld_relaxed_v2u64(&k.rec[i * 2]);
            } while ((p.x >> 40) != want || (p.y >> 40) != want);
            TIMELINE(i, 1);
            PHASEF(1);
            // lane 0: a = T - clip(v_label), lane 1: a = T + clip(v_neg), as
            // one add on the biased 40-bit sum and one clamp to [0, 2T]
            // (the decision is on the critical path of every step)
            if (lane < 2) {
                const long long v40 = (long long)((lane == 0 ? p.x : p.y) & ((1ull << 40) - 1));
                long long a = lane == 0 ? dec_c0 - v40 : dec_c0 + v40;
                a = a < 0 ? 0 : (a > dec_2T ? dec_2T : a);
                uint64_t th = dec_tab ? s.thr_tab[a] : threshold_of(a, dec_2T >> 1);
                if (dec_dbg) th = (k.dbg & 4) ? 0 : (k.dbg & 32) ? (1ull << 50) : th;
                s.thr[lane] = th;
            }
            if (k.trace && rank == 0 && lane == 0) {
                const long long bias = (long long)n_cta * kVoteBias;
                const long long gl = (long long)(p.x & ((1ull << 40) - 1)) - bias;
                const long long gn = (long long)(p.y & ((1ull << 40) - 1)) - bias;
                k.trace[i * 4 + 0] = neg;
                k.trace[i * 4 + 1] = gl;
                k.trace[i * 4 + 2] = gn;
            }
            PHASEF(2);
        } else {
            // shadow of the all-reduce: record i+3 in flight; outputs of
            // example i into info (read by this step's events); outputs of
            // example i+1 with the current masks and their contributions to
            // its two class sums with the current weights (the clauses this
            // step touches are corrected later)
            if (i + 3 < n) rec_issue(k, s, i + 3, tid - 32, nthr - 32);
            else cp_async_commit();
            const int *nc = s.nout + (int)(i & 1) * k.cmax;
            int *no = s.nout + par * k.cmax;
            long long *cl = s.clo + par * 2 * k.cmax;
            const bool ev1 = more && !(k.dbg & 16);
            for (int j = warp - 1; j < cown; j += nwarps - 1) {
                bool o = false;
                if (ev1) o = clause_out(k, s, j, rn + 4);
                if (lane == 0) {
                    s.info[j] = nc[j] ? I_OUT : 0;
                    if (ev1) {
                        no[j] = o;
                        const long long a = o ? s.weights[j * k.K + label1] : 0;
                        const long long b = o ? s.weights[j * k.K + neg1] : 0;
                        cl[j] = a;
                        cl[k.cmax + j] = b;
                        if (a) atomicAdd(&s.vsh[par * 2 + 0], (unsigned long long)a);
                        if (b) atomicAdd(&s.vsh[par * 2 + 1], (unsigned long long)b);
                    }
                }
            }
            cp_async_wait_1();  // record i+2 landed (this thread's part); B1 publishes it
        }
        __syncthreads();
        PHASEF(3);
        const uint64_t tt = s.thr[0], tn = s.thr[1];
        if ((tt | tn) == 0) {
            // both update probabilities are 0 (the example is learned): no
            // events, nothing changes, the shadow's sums for example i+1 are
            // final -- arrive for it at once
            if (warp == 0) {
                if (lane < 2 && more) {
                    const long long v = (long long)s.vsh[par * 2 + lane];
                    s.vsh[par * 2 + lane] = 0;
                    red_relaxed_add_u64(&k.rec[(i + 1) * 2 + lane],
                                        (1ull << 40) + (unsigned long long)(v + kVoteBias));
                }
                if (k.trace && rank == 0 && lane == 0) k.trace[i * 4 + 3] = 0;
                TIMELINE(i, 2);
                if (more) TIMELINE(i + 1, 0);
            }
            PHASEF(7);
            PHASE_FLUSH(false);
            continue;
        }
        // 3. the step's events: every entry of the buckets up to the
        //    threshold's bucket whose key is below it (exact draw on a tie).
        //    Few entries: warp 0 alone, no extra barrier; else all warps.
        const uint32_t *ent = rc + rec_entries(k);
        const unsigned tbt = (unsigned)(tt >> 37), tbn = (unsigned)(tn >> 37);
        int hi_t, hi_n;
        {
            const uint16_t *off = reinterpret_cast<const uint16_t *>(rc + rec_buckets(k));
            hi_t = tbt >= 65536u ? C : off[(tbt >> 8) + 1];
            hi_n = tbn >= 65536u ? C : off[260 + (tbn >> 8) + 1];
        }
        const int ne = hi_t + hi_n;
        auto count_entries = [&](int t0, int nt, unsigned &pre, unsigned &tot) {
            for (int e = t0; e < ne; e += nt) {
                const int str = e >= hi_t ? 1 : 0;
                const uint32_t v = ent[str * k.Cp + e - str * hi_t];
                const unsigned key = v >> 16, c = v & 0xFFFFu;
                const unsigned tb = str ? tbn : tbt;
                bool q = key < tb;
                if (key == tb)
                    q = draw53(k.fb_seed, fbc + 1 + (str ? (uint64_t)C : 0) + c) < (str ? tn : tt);
                if (q) {
                    ++tot;
                    pre += c < (unsigned)c0 ? 1u : 0u;
                    if (c >= (unsigned)c0 && c < (unsigned)c1) atomicOr(&s.oflag[c - c0], 1 << str);
                }
            }
        };
        // 4-5. warp 0: window ordinals (events before c0 + own prefix),
        //      event types, weights, work list
        auto own_events = [&](unsigned pv, unsigned tv) {
            if (lane == 0) s.misc[0] = 0;
            __syncwarp();
            const uint64_t obase = s.blk_ctr[0] + pv;
            unsigned carry = 0;
            for (int jb = 0; jb < cown; jb += 32) {
                const int j = jb + lane;
                const int f = j < cown ? s.oflag[j] : 0;
                const unsigned v = (unsigned)(f & 1) + (unsigned)(f >> 1);
                unsigned x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (f) {
                    s.oflag[j] = 0;
                    fast_events(k, s, cn, j, f & 1, f & 2, obase + carry + (x - v), label, neg,
                                more, par, label1, neg1);
                }
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            __syncwarp();
            if (lane == 0) {
                s.blk_ctr[0] += (uint64_t)tv;
                if (k.trace && rank == 0) k.trace[i * 4 + 3] = tv;
            }
        };
        if (ne <= 64) {
            if (warp == 0) {
                unsigned pre = 0, tot = 0;
                count_entries(lane, 32, pre, tot);
                pre = __reduce_add_sync(0xffffffffu, pre);
                tot = __reduce_add_sync(0xffffffffu, tot);
                __syncwarp();
                own_events(pre, tot);
            }
        } else {
            unsigned pre = 0, tot = 0;
            count_entries(tid, nthr, pre, tot);
            pre = __reduce_add_sync(0xffffffffu, pre);
            tot = __reduce_add_sync(0xffffffffu, tot);
            if (lane == 0) {
                s.wcnt[warp] = pre;
                s.wcnt[32 + warp] = tot;
            }
            __syncthreads();
            if (warp == 0) {
                unsigned pv = lane < nwarps ? s.wcnt[lane] : 0u;
                unsigned tv = lane < nwarps ? s.wcnt[32 + lane] : 0u;
                pv = __reduce_add_sync(0xffffffffu, pv);
                tv = __reduce_add_sync(0xffffffffu, tv);
                own_events(pv, tv);
            }
        }
        __syncthreads();
        PHASEF(4);
        // 6. per-position Type I / II updates of the work list, then the
        //    re-evaluation for example i+1 of the clauses they changed (with
        //    the correction of its class sums)
        const int n_work = (k.dbg & 1) ? 0 : s.misc[0];
        if (n_work > 0) {
            if (SMEM_STATES) feedback_simd<true>(k, s, c0, lit, n_work, cn);
            else feedback_quads<false>(k, s, c0, lit, n_work, cn);
            __syncthreads();
            PHASEF(5);
            if (more) {
                int *no = s.nout + par * k.cmax;
                const long long *cl = s.clo + par * 2 * k.cmax;
                for (int q = warp; q < n_work; q += nwarps) {
                    const int j = s.work[q];
                    const bool o = clause_out(k, s, j, rn + 4);
                    if (lane == 0) {
                        no[j] = o;
                        const long long dl = (o ? s.weights[j * k.K + label1] : 0) - cl[j];
                        const long long dn = (o ? s.weights[j * k.K + neg1] : 0) - cl[k.cmax + j];
                        if (dl) atomicAdd(&s.vsh[par * 2 + 0], (unsigned long long)dl);
                        if (dn) atomicAdd(&s.vsh[par * 2 + 1], (unsigned long long)dn);
                    }
                }
                __syncthreads();
            }
            PHASEF(6);
        }
        TIMELINE(i, 2);
        // 7. thread 0: class sums of example i+1 -> its arrival
        //    (lane 0: label word, lane 1: negative word, one instruction)
        if (warp == 0 && lane < 2 && more) {
            const long long v = (long long)s.vsh[par * 2 + lane];
            s.vsh[par * 2 + lane] = 0;
            red_relaxed_add_u64(&k.rec[(i + 1) * 2 + lane], (1ull << 40) + (unsigned long long)(v + kVoteBias));
        }
        if (more) TIMELINE(i + 1, 0);
        PHASEF(7);
        PHASE_FLUSH(ne > 64);
    }
#undef PHASEF
#undef PHASE_FLUSH
    if (prof && tid == 0) {
        for (int q = 0; q < 8; ++q) k.phase[rank * 8 + q] = ph[q];
        // after the timeline: heavy-step phases [n_cta][8], then counts [n_cta]
        unsigned long long *hp = k.phase + n_cta * 8 + (size_t)kTimelineSteps * n_cta * 3;
        for (int q = 0; q < 8; ++q) hp[rank * 8 + q] = phh[q];
        hp[n_cta * 8 + rank] = n_heavy;
    }
    cp_async_wait_all();
    __syncthreads();
    store_slice<SMEM_STATES>(k, s, c0, cown);
    if (tid == 0 && rank == n_cta - 1) k.block_counters[0] = s.blk_ctr[0];
    flush_stats(k, cn, rank == 0);
}

// ------------------------------------------------- speculative windows --
// k_train_spec: the fast path's records and feedback, with the per-example
// grid exchange amortised over windows of up to k.spec consecutive steps.
//
// From epoch ~3 on, 80-90% of the steps are empty (both update probabilities
// 0, feedback.py:33-44): nothing changes, so the next example's class sums
// are already final.  Every CTA therefore evaluates a whole window of
// examples with its current clauses and publishes all of their partial sums
// at once; after ONE exchange every CTA knows the sums of every step of the
// window and finds (identically) its first non-empty step.  Steps before it
// are done; that step's events are applied exactly as in k_train_fast; the
// next window starts right after it.  While warp 0 waits for window w, the
// other warps already evaluate and publish window w+1 under the assumption
// that w is all-empty (true most of the time), so runs of empty steps cost
// max(exchange, evaluation) per window instead of one exchange per step.
// A window whose speculation failed is simply abandoned: window numbers are
// never reused (each has its own slots in k.rec), so stale partial sums can
// never be mistaken for current ones.
//
// Every evaluated step keeps, per CTA, its clause-output bitset and its two
// partial class sums (obs / vst, ring slot i % HR).  After a non-empty step
// only the clauses on the work list changed (states, masks, weights), so
// the next window -- which lies inside the two windows already evaluated --
// is published from the kept sums corrected by the work-list clauses alone.
// The result is bit-identical to the sequential loop (executor.py:275-340):
// every applied step sees exactly the states the steps before it produced.
// flag entries per stream staged with each head: k.spec_ent (the largest of
// 256, 224, ... 64 that fits next to everything else)
__host__ __device__ inline int spec_hsz(const TrainK &k) { return 4 + k.Wp + 260 + 2 * k.spec_ent; }

__device__ __forceinline__ int spec_wrap(int x, int HR) { return x >= HR ? x - HR : x; }

// Stage the heads of cnt <= HR steps from step `from` (ring slot fslot) --
// example, label, negative class, literal row, bucket starts and the first
// k.spec_ent flag entries of each stream -- one warp per step (warps wrel,
// wrel + nw, ...), 16-B cp.async units over the lanes.  k.dbg & 64 also
// prefetches the step's remaining flag entries into L2 (this CTA takes the
// 128-B lines l = rank - i mod n_cta).
__device__ __forceinline__ void spec_issue(const TrainK &k, const Smem &s, int64_t from, int fslot,
                                           int cnt, int wrel, int nw) {
    const int lane = threadIdx.x & 31;
    const int nh = (4 + k.Wp + 260) / 4;
    const int ne = min(k.spec_ent, k.Cp) / 4;
    const int per = nh + 2 * ne;
    const int HR = 3 * k.spec, HSZ = spec_hsz(k);
    for (int st = wrel; st < cnt; st += nw) {
        const int64_t i = from + st;
        const uint32_t *src = k.recs + i * (int64_t)k.R;
        uint32_t *dst = s.hring + spec_wrap(fslot + st, HR) * HSZ;
        for (int q = lane; q < per; q += 32) {
            if (q < nh) {
                cp_async16(dst + 4 * q, src + 4 * q);
            } else {
                const int r = q - nh, str = r >= ne ? 1 : 0, e = r - str * ne;
                cp_async16(dst + 4 * nh + str * k.spec_ent + 4 * e, src + rec_entries(k) + str * k.Cp + 4 * e);
            }
        }
        if ((k.dbg & 64) && lane == 0 && (int)(i % k.n_cta) == (int)blockIdx.x) {
            // one CTA per step: the step's flag entries into L2 (one bulk op)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         ::"l"(src + rec_entries(k)), "r"(8 * k.Cp) : "memory");
        }
    }
}

__device__ __forceinline__ void named_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void cp_async_wait_0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Fresh evaluation of a window: warp w (= wrel, wrel + nw, ...) takes own
// clauses 2w', 2w' + 1 against the kk <= 16 examples whose heads sit in ring
// slots sb, sb + 1, ...; lane c2 * 16 + q on (clause 2w' + c2, example q)
// ORs mask & ~literal over the row in 16-B shared loads (rows padded to Wp
// words; the mask is a 2-address broadcast).  A firing (clause, example)
// sets its bit in the example's output bitset obs[slot] (zeroed before);
// the lanes' label / negative weights are summed over the pair into
// part[warp][lane] (lane q: label sum of example q, lane 16 + q: negative).
__device__ __forceinline__ void spec_eval(const TrainK &k, const Smem &s, int wrel, int nw, int cown,
                                          int sb, int kk) {
    const int lane = threadIdx.x & 31, q = lane & 15, c2 = lane >> 4;
    const int HR = 3 * k.spec, HSZ = spec_hsz(k), MW = k.MW, CW = (k.cmax + 31) >> 5;
    const int slot = spec_wrap(sb + (q < kk ? q : 0), HR);
    const uint32_t *hd = s.hring + slot * HSZ;
    const uint4 *lit = reinterpret_cast<const uint4 *>(hd + 4);
    const int label = (int)hd[1], neg = (int)hd[2];
    const int n4 = MW >> 2;
    uint32_t *ob = s.obs + slot * CW;
    long long a = 0, b = 0;
    for (int jp = 2 * wrel; jp < cown; jp += 2 * nw) {
        const int j = jp + c2;
        const bool real = j < cown;
        const int jj = real ? j : jp;
        const uint4 *m = reinterpret_cast<const uint4 *>(s.masks + jj * MW);
        uint32_t v = 0;
#pragma unroll 4
        for (int u = 0; u < n4; ++u) {
            const uint4 mm = m[u], ll = lit[u];
            v |= (mm.x & ~ll.x) | (mm.y & ~ll.y) | (mm.z & ~ll.z) | (mm.w & ~ll.w);
        }
        if (real && q < kk && v == 0 && s.cnt[jj] <= k.budget) {
            atomicOr(&ob[j >> 5], 1u << (j & 31));
            a += s.weights[j * k.K + label];
            b += s.weights[j * k.K + neg];
        }
    }
    a += __shfl_xor_sync(0xffffffffu, a, 16);
    b += __shfl_xor_sync(0xffffffffu, b, 16);
    s.part[(threadIdx.x >> 5) * 32 + lane] = c2 ? b : a;
}

// After a non-empty step (label li, negative ni): the kk examples from ring
// slot sb were evaluated before it; only work-list clauses changed.  Warp w
// takes work items 2w', 2w' + 1: each (clause, example) lane re-tests the
// clause, flips its bit in obs[slot] if the output changed, and adds
// new - old contribution (old weights = new minus the step's +1 / -1 on li /
// ni when the clause fired on it, kernels/_numba.py:117-122) into part.
__device__ __forceinline__ void spec_correct(const TrainK &k, const Smem &s, int wrel, int nw,
                                             int n_work, int sb, int kk, int li, int ni) {
    const int lane = threadIdx.x & 31, q = lane & 15, c2 = lane >> 4;
    const int HR = 3 * k.spec, HSZ = spec_hsz(k), MW = k.MW, CW = (k.cmax + 31) >> 5;
    const int slot = spec_wrap(sb + (q < kk ? q : 0), HR);
    const uint32_t *hd = s.hring + slot * HSZ;
    const uint4 *lit = reinterpret_cast<const uint4 *>(hd + 4);
    const int label = (int)hd[1], neg = (int)hd[2];
    const int n4 = MW >> 2;
    uint32_t *ob = s.obs + slot * CW;
    long long a = 0, b = 0;
    for (int wp = 2 * wrel; wp < n_work; wp += 2 * nw) {
        const int idx = wp + c2;
        const bool real = idx < n_work;
        const int j = s.work[real ? idx : wp];
        const uint4 *m = reinterpret_cast<const uint4 *>(s.masks + j * MW);
        uint32_t v = 0;
#pragma unroll 4
        for (int u = 0; u < n4; ++u) {
            const uint4 mm = m[u], ll = lit[u];
            v |= (mm.x & ~ll.x) | (mm.y & ~ll.y) | (mm.z & ~ll.z) | (mm.w & ~ll.w);
        }
        if (real && q < kk) {
            const bool on = v == 0 && s.cnt[j] <= k.budget;
            const bool oo = (ob[j >> 5] >> (j & 31)) & 1u;
            const int info = s.info[j];
            const int fired = (info & I_OUT) ? 1 : 0;
            const int dt = (info & I_TEV) ? fired : 0, dn = (info & I_NEV) ? fired : 0;
            const int32_t *w = s.weights + j * k.K;
            const long long wl = w[label], wg = w[neg];
            const long long wl0 = wl - (label == li ? dt : 0) + (label == ni ? dn : 0);
            const long long wg0 = wg - (neg == li ? dt : 0) + (neg == ni ? dn : 0);
            a += (on ? wl : 0) - (oo ? wl0 : 0);
            b += (on ? wg : 0) - (oo ? wg0 : 0);
            if (on != oo) atomicXor(&ob[j >> 5], 1u << (j & 31));
        }
    }
    a += __shfl_xor_sync(0xffffffffu, a, 16);
    b += __shfl_xor_sync(0xffffffffu, b, 16);
    s.part[(threadIdx.x >> 5) * 32 + lane] = c2 ? b : a;
}

// Vote slot t of window wn: a window's 2 * spec words are contiguous (two
// 128-B lines).  Measured against one line per word (interleaved across
// windows, which spreads the atomics over L2 slices but makes every poll 32
// line reads): 3% faster per example.
__device__ __forceinline__ size_t spec_slot(const TrainK &k, int64_t wn, int t) {
    return (size_t)wn * 2 * k.spec + t;
}

// Thread t < 2kk publishes step t >> 1's label (t even) / negative (t odd)
// partial class sum of window wn: the kept sum (add_kept) plus the partials
// of warps w0 .. w0 + nw - 1; the result is kept for later corrections.
__device__ __forceinline__ void spec_push(const TrainK &k, const Smem &s, int t, int w0, int nw,
                                          int sb, bool add_kept, int64_t wn) {
    long long v = 0;
    for (int w = w0; w < w0 + nw; ++w) v += s.part[w * 32 + (t >> 1) + 16 * (t & 1)];
    long long *kept = s.vst + spec_wrap(sb + (t >> 1), 3 * k.spec) * 2 + (t & 1);
    if (add_kept) v += *kept;
    *kept = v;
    red_relaxed_add_u64(k.rec + spec_slot(k, wn, t), (1ull << 40) + (unsigned long long)(v + kVoteBias));
}

// Event bookkeeping of own clause j for the applied step (fast_events
// without the next-example correction).
// Returns whether the clause joins the work list (a state can move).
__device__ __forceinline__ bool spec_events(const TrainK &k, const Smem &s, Counters &cn, int j,
                                            bool t_ev, bool n_ev, uint64_t ord, int label, int neg) {
    int info = s.info[j] & I_OUT;
    const bool out = info & I_OUT;
    int32_t *w = s.weights + j * k.K;
    const bool t1 = w[label] >= 0, n1 = w[neg] < 0;
    const uint64_t bseed = s.blk_seed[0];
    if (t_ev) {
        info |= I_TEV | (t1 ? I_T1 : 0);
        s.sk_t[j] = bseed + kGolden * ((ord << 32) + 1);
        ++cn.events;
        if (t1) ++cn.t1; else if (out) ++cn.t2;
    }
    if (n_ev) {
        const uint64_t o2 = ord + (t_ev ? 1 : 0);
        info |= I_NEV | (n1 ? I_N1 : 0);
        s.sk_n[j] = bseed + kGolden * ((o2 << 32) + 1);
        ++cn.events;
        if (n1) ++cn.t1; else if (out) ++cn.t2;
    }
    if (out) {
        if (t_ev) w[label] += 1;
        if (n_ev) w[neg] -= 1;
    }
    s.info[j] = info | (fb_class(info) << 8);  // event class for feedback_simd<., true>
    return (t_ev && ((info & I_T1) || out)) || (n_ev && ((info & I_N1) || out));
}

__device__ __forceinline__ int mine_lane(int lane, int kk) { return lane < 2 * kk ? lane : 0; }

// PROF timeline: %globaltimer of this CTA's publication (thread 32) and poll
// completion (thread 0) of windows [kSpecTl0, kSpecTl0 + kSpecTlN), stored
// after the counters as [n_cta][kSpecTlN][2].
// Per polled window wn: [0] %globaltimer when the next window was published
// after wn's non-empty step, [1] %globaltimer at wn's poll completion, then
// clock64 at [2] poll completion, [3] events done, [4] feedback done, [5]
// publication, [6] work-list length, [7] flag entries of the step, [8]
// clock64 after the decision barrier, [9] after the preparation barrier,
// [10] after its warm repetition, [11] entries counted (warp 0), [12] own
// events assigned, [13] own flagged clauses (profiling build only); stored
// after the counters as [n_cta][kSpecTlN][kSpecTlQ].
constexpr int kSpecTl0 = 2000, kSpecTlN = 2048, kSpecTlQ = 14;
#define SPEC_TL(wn_, q_, v_)                                                                          \
    do {                                                                                              \
        if (PROF && (wn_) >= kSpecTl0 && (wn_) < kSpecTl0 + kSpecTlN)                                  \
            k.phase[n_cta * 16 + ((size_t)rank * kSpecTlN + ((wn_) - kSpecTl0)) * kSpecTlQ + (q_)] = \
                (unsigned long long)(v_);                                                             \
    } while (0)

// PROF: k.phase[rank * 16 + q] accumulates (thread 0, clock64) 0 poll, 1
// decision + barrier, 2 event preparation, 15 entries + own events, 3
// feedback, 13 next-window wait, 14 correction, 4 publication; counts 8
// windows, 9 non-empty steps, 10 steps with > 64 flag entries, 11 steps
// whose entries were staged, 12 whole loop
template <bool SMEM_STATES, bool PROF>
__global__ void __launch_bounds__(kFastMaxThreads, 1) k_train_spec(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, SMEM_STATES, MODE_GRID, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthr >> 5;
    const int rank = blockIdx.x;
    const int C = k.C, n_cta = k.n_cta;
    const int c0 = cta_begin(rank, C, n_cta), c1 = cta_begin(rank + 1, C, n_cta);
    const int cown = c1 - c0;
    const int64_t n = k.n_steps;
    const int KW = k.spec, HR = 3 * KW, HSZ = spec_hsz(k), CW = (k.cmax + 31) >> 5;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;

    load_slice<SMEM_STATES>(k, s, c0, cown);
    uint32_t *thr32 = reinterpret_cast<uint32_t *>(s.thr_tab);
    if (k.thr_smem)
        for (int64_t a = tid; a <= 2 * k.T; a += nthr) thr32[a] = k.thr32[a];
    if (tid == 0) {
        s.blk_ctr[0] = k.block_counters[0];
        s.blk_seed[0] = k.block_seeds[0];
        s.misc[0] = 0;
    }
    for (int j = tid; j < cown; j += nthr) s.oflag[j] = 0;
    for (int q = tid; q < HR * CW; q += nthr) s.obs[q] = 0;
    int64_t issued = n < (int64_t)HR ? n : (int64_t)HR;  // heads staged or in flight: [0, issued)
    int islot = spec_wrap((int)issued, HR);              // issued % HR
    spec_issue(k, s, 0, 0, (int)issued, warp, nwarps);
    cp_async_commit();
    cp_async_wait_0();
    __syncthreads();

    // window 0: every warp evaluates, then warp 1 publishes
    int64_t i0 = 0, wn = 0;
    int s0 = 0;  // i0 % HR
    {
        const int kk = (int)(n < (int64_t)KW ? n : (int64_t)KW);
        spec_eval(k, s, warp, nwarps, cown, 0, kk);
        __syncthreads();
        if (tid >= 32 && tid - 32 < 2 * kk) spec_push(k, s, tid - 32, 0, nwarps, 0, false, 0);
    }

    Counters cn;
    unsigned long long ph[16] = {0};
    long long t_mark = clock64();
    const long long t_loop0 = t_mark;
#define SPH(q)                                                   \
    do {                                                         \
        if (PROF && tid == 0) {                                  \
            const long long now_ = clock64();                    \
            ph[q] += (unsigned long long)(now_ - t_mark);        \
            t_mark = now_;                                       \
        }                                                        \
    } while (0)
    const long long dec_bias = (long long)n_cta * kVoteBias;
    const long long dec_2T = 2 * k.T;
    const bool dec_tab = k.thr_smem != 0;  // exact thresholds by table lookup (feedback.py:33-44)
    while (i0 < n) {
        const int kk = (int)(n - i0 < (int64_t)KW ? n - i0 : (int64_t)KW);
        const int64_t i1 = i0 + kk;
        const int s1 = spec_wrap(s0 + kk, HR);
        const int kk1 = (int)(n - i1 < (int64_t)KW ? n - i1 : (int64_t)KW);
        const int64_t want = i0 + HR < n ? i0 + HR : n;
        if (warp == 0) {
            // exchange of window wn: lane t < 2kk holds step t >> 1's label
            // (t even) or negative (t odd) class sum once all CTAs arrived
            const unsigned long long *slot = k.rec + spec_slot(k, wn, mine_lane(lane, kk));
            unsigned long long p = 0;
            const bool mine = lane < 2 * kk;
            for (;;) {
                if (mine) p = ld_relaxed_u64(slot);
                if (__all_sync(0xffffffffu, !mine || (p >> 40) == (unsigned long long)n_cta)) break;
            }
            SPH(0);
            if (lane == 0) {
                SPEC_TL(wn, 1, gtimer());
                SPEC_TL(wn, 2, clock64());
            }
            // decision (feedback.py:33-44) of every step of the window: the
            // update probability a / 2T is 0 iff a == 0; the exact threshold
            // ceil(p * 2^53) only for the first non-empty step
            long long a = 0;
            const long long v40 = (long long)(p & ((1ull << 40) - 1));
            if (mine) {
                a = (lane & 1) ? k.T - dec_bias + v40 : k.T + dec_bias - v40;
                a = a < 0 ? 0 : (a > dec_2T ? dec_2T : a);
            }
            const unsigned busy = __ballot_sync(0xffffffffu, a != 0);
            const int first = busy ? (__ffs(busy) - 1) >> 1 : kk;
            // the first non-empty step: its bucket (thresholds >> 37) from
            // the 32-bit table, a for the exact threshold on a key tie
            if (mine && (lane >> 1) == first) {
                s.thr[lane & 1] = (uint64_t)a;
                s.thr[2 + (lane & 1)] = a == dec_2T ? 65536u
                                        : dec_tab   ? (uint64_t)(thr32[a] >> 16)
                                                    : threshold_of(a, dec_2T >> 1) >> 37;
            }
            if (lane == 0) s.misc[1] = first;
            if (k.trace && rank == 0 && mine && (lane >> 1) <= first) {
                const int64_t i = i0 + (lane >> 1);
                const uint32_t *hd = s.hring + spec_wrap(s0 + (lane >> 1), HR) * HSZ;
                if ((lane & 1) == 0) k.trace[i * 4 + 0] = (long long)hd[2];
                k.trace[i * 4 + 1 + (lane & 1)] = v40 - dec_bias;
                if ((lane >> 1) < first) k.trace[i * 4 + 3] = 0;
            }
        } else {
            // speculative evaluation + publication of window wn + 1
            cp_async_wait_0();
            for (int q = tid - 32; q < kk1 * CW; q += nthr - 32) {
                const int st = q / CW;
                s.obs[spec_wrap(s1 + st, HR) * CW + (q - st * CW)] = 0;
            }
            named_bar(1, nthr - 32);
            if (kk1 > 0) {
                spec_eval(k, s, warp - 1, nwarps - 1, cown, s1, kk1);
                named_bar(1, nthr - 32);
                if (tid - 32 < 2 * kk1) spec_push(k, s, tid - 32, 1, nwarps - 1, s1, false, wn + 1);
            }
            if (want > issued) spec_issue(k, s, issued, islot, (int)(want - issued), warp - 1, nwarps - 1);
            cp_async_commit();
        }
        if (want > issued) {
            islot = spec_wrap(islot + (int)(want - issued), HR);
            issued = want;
        }
        __syncthreads();
        SPH(1);
        if (tid == 0) SPEC_TL(wn, 8, clock64());
        if (PROF && tid == 0) ph[8] += 1;
        const int first = s.misc[1];
        if (first >= kk) {  // all-empty window: the next one is already published
            i0 = i1;
            s0 = s1;
            wn += 1;
            continue;
        }
        if (PROF && tid == 0) ph[9] += 1;
        // the window's first non-empty step i: k_train_fast's steps 3-6
        const int64_t i = i0 + first;
        const int si = spec_wrap(s0 + first, HR);
        const uint32_t *rc = s.hring + si * HSZ;
        const uint32_t *lit = rc + 4;
        const int label = (int)rc[1], neg = (int)rc[2];
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        const long long at = (long long)s.thr[0], an = (long long)s.thr[1];
        const unsigned tbt = (unsigned)s.thr[2], tbn = (unsigned)s.thr[3];
        int hi_t = 0, hi_n = 0;
        // (the profiling build runs this block twice: cold vs warm code)
        for (int rep = 0; rep < (PROF ? 2 : 1); ++rep) {
            const uint32_t *ob = s.obs + si * CW;
            for (int j = tid; j < cown; j += nthr) s.info[j] = ((ob[j >> 5] >> (j & 31)) & 1u) ? I_OUT : 0;
            const uint16_t *off = reinterpret_cast<const uint16_t *>(rc + 4 + k.Wp);
            hi_t = tbt >= 65536u ? C : off[(tbt >> 8) + 1];
            hi_n = tbn >= 65536u ? C : off[260 + (tbn >> 8) + 1];
            // info[] of own clauses is read by warp 0 (own events) before the
            // next block barrier: a block barrier only when other warps wrote
            // part of it
            if (cown > 32) __syncthreads();
            else __syncwarp();
            if (tid == 0) SPEC_TL(wn, rep ? 10 : 9, clock64());
        }
        const bool staged = hi_t <= k.spec_ent && hi_n <= k.spec_ent;
        if (PROF && tid == 0) {
            ph[10] += (hi_t + hi_n > 64) ? 1 : 0;
            ph[11] += staged ? 1 : 0;
        }
        const uint32_t *ent = staged ? rc + 4 + k.Wp + 260 : k.recs + i * (int64_t)k.R + rec_entries(k);
        const int estr = staged ? k.spec_ent : k.Cp;
        const int ne = hi_t + hi_n;
        SPH(2);
        auto count_entries = [&](int t0, int nt, unsigned &pre, unsigned &tot) {
            for (int e = t0; e < ne; e += nt) {
                const int str = e >= hi_t ? 1 : 0;
                const uint32_t v = ent[str * estr + e - str * hi_t];
                const unsigned key = v >> 16, c = v & 0xFFFFu;
                const unsigned tb = str ? tbn : tbt;
                bool q = key < tb;
                if (key == tb)  // a tie on the 16-bit key: the exact draw and threshold
                    q = draw53(k.fb_seed, fbc + 1 + (str ? (uint64_t)C : 0) + c) <
                        threshold_of(str ? an : at, k.T);
                if (q) {
                    ++tot;
                    pre += c < (unsigned)c0 ? 1u : 0u;
                    if (c >= (unsigned)c0 && c < (unsigned)c1) atomicOr(&s.oflag[c - c0], 1 << str);
                }
            }
        };
        auto own_events = [&](unsigned pv, unsigned tv) {
            const uint64_t obase = s.blk_ctr[0] + pv;
            unsigned carry = 0;
            int n_wl = 0;  // work-list slots by ballot (no shared-memory atomics)
            for (int jb = 0; jb < cown; jb += 32) {
                const int j = jb + lane;
                const int f = j < cown ? s.oflag[j] : 0;
                // events before lane's clause within the chunk: two ballots
                const unsigned bt = __ballot_sync(0xffffffffu, f & 1);
                const unsigned bn = __ballot_sync(0xffffffffu, f & 2);
                const unsigned below = (1u << lane) - 1u;
                bool wk = false;
                if (f) {
                    s.oflag[j] = 0;
                    wk = spec_events(k, s, cn, j, f & 1, f & 2,
                                     obase + carry + (unsigned)(__popc(bt & below) + __popc(bn & below)),
                                     label, neg);
                }
                const unsigned wb = __ballot_sync(0xffffffffu, wk);
                if (wk) s.work[n_wl + __popc(wb & below)] = j;
                n_wl += __popc(wb);
                carry += (unsigned)(__popc(bt) + __popc(bn));
            }
            __syncwarp();
            if (lane == 0) {
                s.misc[0] = n_wl;
                s.blk_ctr[0] += (uint64_t)tv;
                if (k.trace && rank == 0) k.trace[i * 4 + 3] = tv;
            }
        };
        {
            // few entries: warp 0 alone; else all warps count, warp 0 assigns
            const bool few = ne <= 64;
            unsigned pre = 0, tot = 0;
            if (!few || warp == 0) count_entries(few ? lane : tid, few ? 32 : nthr, pre, tot);
            pre = __reduce_add_sync(0xffffffffu, pre);
            tot = __reduce_add_sync(0xffffffffu, tot);
            if (!few) {
                if (lane == 0) {
                    s.wcnt[warp] = pre;
                    s.wcnt[32 + warp] = tot;
                }
                __syncthreads();
                if (warp == 0) {
                    pre = __reduce_add_sync(0xffffffffu, lane < nwarps ? s.wcnt[lane] : 0u);
                    tot = __reduce_add_sync(0xffffffffu, lane < nwarps ? s.wcnt[32 + lane] : 0u);
                }
            }
            if (warp == 0) {
                __syncwarp();
                if (lane == 0) SPEC_TL(wn, 11, clock64());
                own_events(pre, tot);
                if (lane == 0) {
                    SPEC_TL(wn, 12, clock64());
                    SPEC_TL(wn, 13, s.misc[0]);
                }
            }
        }
        __syncthreads();
        SPH(15);
        if (tid == 0) SPEC_TL(wn, 3, clock64());
        const int n_work = (k.dbg & 1) ? 0 : s.misc[0];
        if (n_work > 0) {
            feedback_simd<SMEM_STATES, true>(k, s, c0, lit, n_work, cn);
            __syncthreads();
        }
        SPH(3);
        if (tid == 0) {
            SPEC_TL(wn, 4, clock64());
            SPEC_TL(wn, 6, n_work);
            SPEC_TL(wn, 7, ne);
        }
        // next window right after step i: the kept sums of its steps,
        // corrected by the work-list clauses
        i0 = i + 1;
        s0 = spec_wrap(si + 1, HR);
        wn += 2;
        if (i0 < n) {
            asm volatile("cp.async.wait_group 1;" ::: "memory");
            SPH(13);
            const int kn = (int)(n - i0 < (int64_t)KW ? n - i0 : (int64_t)KW);
            if (n_work > 0) {
                spec_correct(k, s, warp, nwarps, n_work, s0, kn, label, neg);
            } else if (tid < 64) {
                s.part[tid] = 0;  // warps 0-1: nothing to correct
            }
            __syncthreads();
            SPH(14);
            const int used = n_work > 0 ? nwarps : 2;  // warps whose partials count
            if (tid >= 32 && tid - 32 < 2 * kn) spec_push(k, s, tid - 32, 0, used, s0, true, wn);
            if (tid == 32) {
                SPEC_TL(wn - 2, 0, gtimer());
                SPEC_TL(wn - 2, 5, clock64());
            }
        }
        SPH(4);
    }
#undef SPH
    if (PROF && tid == 0) {
        ph[12] = (unsigned long long)(clock64() - t_loop0);
        for (int q = 0; q < 16; ++q) k.phase[rank * 16 + q] = ph[q];
    }
    cp_async_wait_all();
    __syncthreads();
    store_slice<SMEM_STATES>(k, s, c0, cown);
    if (tid == 0 && rank == n_cta - 1) k.block_counters[0] = s.blk_ctr[0];
    flush_stats(k, cn, rank == 0);
}

// --------------------------------------------------------- tiny banks --
// One warp trains the whole bank (C <= 32 clauses, P <= 1024 positions,
// K <= 32): lane c owns clause c (output, flag draws, event ordinals, event
// types, weights); the lanes sweep the positions of each event together.
// No block barrier, no exchange -- the per-example dependency chain of
// executor.py:326-330 is a handful of shuffles.  Same arithmetic as the
// other trainers (kernels/_numba.py:36-125, feedback.py:33-53).
constexpr int kWarpMaxC = 32, kWarpMaxW = 32;

__global__ void __launch_bounds__(32, 1) k_train_warp(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x;
    const int C = k.C, P = k.P, K = k.K, W = k.W, nb = k.n_blocks;
    const int Pp = (P + 3) & ~3;
    int8_t *st = reinterpret_cast<int8_t *>(smem_raw);                        // [C][Pp]
    uint32_t *masks = reinterpret_cast<uint32_t *>(st + align_up((size_t)C * Pp, 16));  // [C][W]
    int32_t *wts = reinterpret_cast<int32_t *>(masks + (size_t)C * W);        // [C][K]
    uint64_t *bctr = reinterpret_cast<uint64_t *>(
        align_up(reinterpret_cast<uintptr_t>(wts + (size_t)C * K), 8));       // [nb]
    for (int i = lane; i < C * P; i += 32) st[(i / P) * Pp + i % P] = k.states[i];
    for (int i = lane; i < C * K; i += 32) wts[i] = k.weights[i];
    for (int i = lane; i < nb; i += 32) bctr[i] = k.block_counters[i];
    __syncwarp();
    // include masks / counts of clause c from its states (warp-collective)
    auto rebuild = [&](int c) {
        int n = 0;
        for (int r = 0; r < W; ++r) {
            const int p = 32 * r + lane;
            const unsigned m = __ballot_sync(0xffffffffu, p < P && st[c * Pp + p] >= 0);
            if (lane == 0) masks[c * W + r] = m;
            n += __popc(m);
        }
        return n;
    };
    int cnt = 0;  // lane c: include count of clause c
    for (int c = 0; c < C; ++c) {
        const int n = rebuild(c);
        if (lane == c) cnt = n;
    }
    __syncwarp();
    const int c = lane;
    const bool real = c < C;
    const int b = real ? block_of(c, C, nb) : 0;
    const int bstart = block_begin(b, C, nb);
    const bool blast = real && (c == C - 1 || block_of(c + 1, C, nb) != b);
    const uint64_t bseed = real ? k.block_seeds[b] : 0;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    Counters cn;
    // the next example's index, label and literal row are loaded one step
    // ahead (the dependent global loads would otherwise open every step)
    int ex_n = k.n_steps > 0 ? __ldg(&k.order[0]) : 0;
    int label_n = k.n_steps > 0 ? __ldg(&k.labels[ex_n]) : 0;
    uint32_t litw_n = (k.n_steps > 0 && lane < W) ? __ldg(&k.lit_words[(int64_t)ex_n * W + lane]) : 0u;
    int ex_nn = k.n_steps > 1 ? __ldg(&k.order[1]) : 0;
    for (int64_t i = 0; i < k.n_steps; ++i) {
        const int label = label_n;
        const uint32_t litw = litw_n;
        if (i + 1 < k.n_steps) {
            label_n = __ldg(&k.labels[ex_nn]);
            litw_n = lane < W ? __ldg(&k.lit_words[(int64_t)ex_nn * W + lane]) : 0u;
            ex_nn = i + 2 < k.n_steps ? __ldg(&k.order[i + 2]) : 0;
        }
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        const int neg = negative_class(k, label, fbc);
        // 1. training-mode outputs (kernels/_numba.py:36-50)
        uint32_t viol = 0;
        for (int r = 0; r < W; ++r) {
            const uint32_t lw = __shfl_sync(0xffffffffu, litw, r);
            if (real) viol |= masks[c * W + r] & ~lw;
        }
        const bool out = real && viol == 0 && cnt <= k.budget;
        // 2. class sums of the label and the negative class (dense.py:153)
        long long vl, vn;
        warp_sum2(out ? wts[c * K + label] : 0, out ? wts[c * K + neg] : 0, vl, vn);
        // 3. decision and update flags (feedback.py:33-53)
        uint64_t tt, tn;
        if (k.thr_tab) {  // threshold_of(a, T) for a in [0, 2T], precomputed
            const long long T = k.T;
            const long long cl = vl < -T ? -T : (vl > T ? T : vl);
            const long long cv = vn < -T ? -T : (vn > T ? T : vn);
            tt = __ldg(&k.thr_tab[T - cl]);
            tn = __ldg(&k.thr_tab[T + cv]);
        } else {
            decide(k, vl, vn, tt, tn);
        }
        const bool ut = real && draw53(k.fb_seed, fbc + 1 + (uint64_t)c) < tt;
        const bool un = real && draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)c) < tn;
        // 4. event ordinals within the clause block (kernels/_numba.py:101-125)
        const int e = (ut ? 1 : 0) + (un ? 1 : 0);
        int incl = e;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int before_block = __shfl_sync(0xffffffffu, incl - e, bstart & 31);
        const uint64_t ord = real ? bctr[b] + (uint64_t)(incl - e - before_block) : 0;
        // 5. event types, weights (feedback first, then weight: SPEC.md:171)
        bool t1 = false, n1 = false;
        if (real && e) {
            int32_t *w = wts + c * K;
            t1 = w[label] >= 0;
            n1 = w[neg] < 0;
            if (ut) { ++cn.events; if (t1) ++cn.t1; else if (out) ++cn.t2; }
            if (un) { ++cn.events; if (n1) ++cn.t1; else if (out) ++cn.t2; }
            if (out) {
                if (ut) w[label] += 1;
                if (un) w[neg] -= 1;
            }
        }
        __syncwarp();
        if (blast) bctr[b] += (uint64_t)(incl - before_block);
        // 6. per-position feedback of the clauses whose states can move
        const bool work = (ut && (t1 || out)) || (un && (n1 || out));
        unsigned todo = __ballot_sync(0xffffffffu, work);
        unsigned nd = 0, nupd = 0;
        while (todo) {
            const int j = __ffs(todo) - 1;
            todo &= todo - 1;
            const int jo = __shfl_sync(0xffffffffu, out ? 1 : 0, j);
            const bool jt = __shfl_sync(0xffffffffu, ut, j), jn = __shfl_sync(0xffffffffu, un, j);
            const bool jt1 = __shfl_sync(0xffffffffu, t1, j), jn1 = __shfl_sync(0xffffffffu, n1, j);
            const uint64_t jord = __shfl_sync(0xffffffffu, ord, j);
            const uint64_t jseed = __shfl_sync(0xffffffffu, bseed, j);
            for (int r = 0; r < W; ++r) {
                const int p = 32 * r + lane;
                const uint32_t lw = __shfl_sync(0xffffffffu, litw, r);
                if (p >= P) continue;
                const int lit = (lw >> lane) & 1;
                int s0 = st[j * Pp + p], sv = s0;
                uint64_t d = 0;
                for (int ev = 0; ev < 2; ++ev) {
                    const bool has = ev == 0 ? jt : jn;
                    if (!has) continue;
                    const bool ti = ev == 0 ? jt1 : jn1;
                    if (ti) {
                        const uint64_t o = jord + (uint64_t)(ev == 1 && jt ? 1 : 0);
                        const uint64_t sk = jseed + kGolden * ((o << 32) + 1);
                        sv = type_i_stream(sv, lit, jo, k.fp, sk, (uint32_t)p, d);
                    } else {
                        sv = type_ii(sv, lit, jo);
                    }
                }
                nd += (unsigned)d;
                nupd += sv != s0 ? 1u : 0u;
                st[j * Pp + p] = (int8_t)sv;
            }
            __syncwarp();
            const int n = rebuild(j);
            if (lane == j) cnt = n;
            __syncwarp();
        }
        cn.draws += nd;
        cn.upd += nupd;
    }
    __syncwarp();
    for (int i = lane; i < C * P; i += 32) k.states[i] = st[(i / P) * Pp + i % P];
    for (int i = lane; i < C * K; i += 32) k.weights[i] = wts[i];
    for (int i = lane; i < nb; i += 32) k.block_counters[i] = bctr[i];
    flush_stats(k, cn, true);
}

// One warp per clause for the same tiny banks (C <= 32 clauses -> a CTA of C
// warps, K <= 32, literal rows <= 32 words), ONE block barrier per example.
// Warp c owns clause c: lane r keeps include-mask word r, lane kk the weight
// of class kk, the states live in the warp's own shared-memory row.  Per
// step every warp publishes its clause's contribution to the label / negative
// class sums (double-buffered by step parity), the barrier, then every warp
// derives -- redundantly, lane per clause -- the sums, the thresholds, all 2C
// update flags and the event ordinals (feedback.py:33-53,
// kernels/_numba.py:101-125) and applies its own clause's events over the
// lanes.  k_train_warp serialises the step's events (a dependent chain of
// ~5 000 instructions on one warp); here they run side by side.  Same
// arithmetic and draw addressing, bit-identical results.
__global__ void __launch_bounds__(32 * kWarpMaxC, 1) k_train_tiny(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
    const int C = k.C, P = k.P, K = k.K, W = k.W, nb = k.n_blocks;
    const int Pp = (P + 3) & ~3;
    int8_t *st = reinterpret_cast<int8_t *>(smem_raw) + (size_t)c * Pp;  // own row
    int2 *pub = reinterpret_cast<int2 *>(smem_raw + align_up((size_t)C * Pp, 16));  // [2][32]
    for (int p = lane; p < P; p += 32) st[p] = k.states[(int64_t)c * P + p];
    int wreg = lane < K ? k.weights[c * K + lane] : 0;
    __syncwarp();
    uint32_t mword = 0;  // lane r: include-mask word r
    int cnt = 0;
    auto rebuild = [&]() {
        int n = 0;
        for (int r = 0; r < W; ++r) {
            const int p = 32 * r + lane;
            const unsigned m = __ballot_sync(0xffffffffu, p < P && st[p] >= 0);
            if (lane == r) mword = m;
            n += __popc(m);
        }
        cnt = n;
    };
    rebuild();
    // lane c2 stands for clause c2: every warp derives every clause's flags
    // and the ordinals of its own block
    const bool real = lane < C;
    const int myb = block_of(c, C, nb);
    const int mybs = block_begin(myb, C, nb), mybe = block_begin(myb + 1, C, nb);
    const uint64_t bseed = k.block_seeds[myb];
    uint64_t myctr = k.block_counters[myb];  // event counter of the own clause's block
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    Counters cn;
    int ex_n = k.n_steps > 0 ? __ldg(&k.order[0]) : 0;
    int label_n = k.n_steps > 0 ? __ldg(&k.labels[ex_n]) : 0;
    uint32_t litw_n = (k.n_steps > 0 && lane < W) ? __ldg(&k.lit_words[(int64_t)ex_n * W + lane]) : 0u;
    int ex_nn = k.n_steps > 1 ? __ldg(&k.order[1]) : 0;
    for (int64_t i = 0; i < k.n_steps; ++i) {
        const int label = label_n;
        const uint32_t litw = litw_n;
        if (i + 1 < k.n_steps) {
            label_n = __ldg(&k.labels[ex_nn]);
            litw_n = lane < W ? __ldg(&k.lit_words[(int64_t)ex_nn * W + lane]) : 0u;
            ex_nn = i + 2 < k.n_steps ? __ldg(&k.order[i + 2]) : 0;
        }
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        const int neg = negative_class(k, label, fbc);
        // 1. own clause's training-mode output (kernels/_numba.py:36-50) and
        //    its contribution to the two class sums (dense.py:153)
        const bool out = !__any_sync(0xffffffffu, lane < W && (mword & ~litw) != 0u) && cnt <= k.budget;
        const int w_l = __shfl_sync(0xffffffffu, wreg, label), w_n = __shfl_sync(0xffffffffu, wreg, neg);
        int2 *pb = pub + (i & 1) * 32;
        if (lane == 0) pb[c] = make_int2(out ? w_l : 0, out ? w_n : 0);
        // the flag draws do not depend on the sums: before the barrier
        const uint64_t d_t = (k.dbg & 2) ? fbc * 0x9E3779B9ull >> 11 : real ? draw53(k.fb_seed, fbc + 1 + (uint64_t)lane) : ~0ull;
        const uint64_t d_n = (k.dbg & 2) ? fbc * 0x7F4A7C15ull >> 11 : real ? draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)lane) : ~0ull;
        if (!(k.dbg & 4)) __syncthreads();
        // 2. class sums, decision, every clause's flags (feedback.py:33-53)
        const int2 pv = real ? pb[lane] : make_int2(0, 0);
        long long vl, vn;
        warp_sum2(pv.x, pv.y, vl, vn);
        uint64_t tt, tn;
        if (k.thr_tab) {
            const long long T = k.T;
            const long long cl = vl < -T ? -T : (vl > T ? T : vl);
            const long long cv = vn < -T ? -T : (vn > T ? T : vn);
            tt = __ldg(&k.thr_tab[T - cl]);
            tn = __ldg(&k.thr_tab[T + cv]);
        } else {
            decide(k, vl, vn, tt, tn);
        }
        // 3. every clause's flags as two ballots; event ordinals within the
        //    clause block (kernels/_numba.py:101-125) by population counts
        const unsigned bt = __ballot_sync(0xffffffffu, real && d_t < tt);
        const unsigned bn = __ballot_sync(0xffffffffu, real && d_n < tn);
        const unsigned below_me = (1u << c) - 1u, below_blk = (1u << mybs) - 1u;
        const unsigned blk = (mybe >= 32 ? 0xFFFFFFFFu : (1u << mybe) - 1u) & ~below_blk;
        const uint64_t ord = myctr + (uint64_t)(__popc(bt & below_me & ~below_blk) +
                                                __popc(bn & below_me & ~below_blk));
        myctr += (uint64_t)(__popc(bt & blk) + __popc(bn & blk));
        const bool ut = (bt >> c) & 1u, un = (bn >> c) & 1u;
        if (!(ut || un)) continue;
        // 4. own clause's event types and weights (feedback first: SPEC.md:171)
        const bool t1 = w_l >= 0, n1 = w_n < 0;
        if (lane == 0) {
            if (ut) { ++cn.events; if (t1) ++cn.t1; else if (out) ++cn.t2; }
            if (un) { ++cn.events; if (n1) ++cn.t1; else if (out) ++cn.t2; }
        }
        if (out) {
            if (ut && lane == label) wreg += 1;
            if (un && lane == neg) wreg -= 1;
        }
        // 5. per-position feedback when a state can move
        if (!((ut && (t1 || out)) || (un && (n1 || out))) || (k.dbg & 1)) continue;
        unsigned nd = 0, nupd = 0;
        const int jo = out ? 1 : 0;
        for (int r = 0; r < W; ++r) {
            const int p = 32 * r + lane;
            const uint32_t lw = __shfl_sync(0xffffffffu, litw, r);
            if (p >= P) continue;
            const int lit = (lw >> lane) & 1;
            const int s0 = st[p];
            int sv = s0;
            uint64_t d = 0;
            // (branch-free Type I: the lanes hold different literals and
            // states, the mixer must not run once per diverged path)
            if (ut) {
                if (t1) sv = type_i_bf(sv, lit, jo, k.fp,
                                       bseed + kGolden * (((ord << 32) + 1) + (uint64_t)p), d);
                else sv = type_ii(sv, lit, jo);
            }
            if (un) {
                const uint64_t o2 = ord + (ut ? 1 : 0);
                if (n1) sv = type_i_bf(sv, lit, jo, k.fp,
                                       bseed + kGolden * (((o2 << 32) + 1) + (uint64_t)p), d);
                else sv = type_ii(sv, lit, jo);
            }
            nd += (unsigned)d;
            nupd += sv != s0 ? 1u : 0u;
            st[p] = (int8_t)sv;
        }
        __syncwarp();
        rebuild();
        cn.draws += nd;
        cn.upd += nupd;
    }
    __syncwarp();
    for (int p = lane; p < P; p += 32) k.states[(int64_t)c * P + p] = st[p];
    if (lane < K) k.weights[c * K + lane] = wreg;
    if (lane == 0 && c == mybe - 1) k.block_counters[myb] = myctr;
    flush_stats(k, cn, threadIdx.x == 0);
}

size_t tiny_kernel_smem(int C, int P) {
    return align_up((size_t)C * (size_t)((P + 3) & ~3), 16) + 2 * 32 * sizeof(int2);
}

size_t warp_kernel_smem(int C, int P, int K, int W, int nb) {
    const size_t Pp = (size_t)((P + 3) & ~3);
    return align_up(align_up((size_t)C * Pp, 16) + 4 * (size_t)C * W + 4 * (size_t)C * K, 8) +
           8 * (size_t)nb + 16;
}

}  // namespace tmb

using namespace tmb;

struct tmb_trainer {
    tmb_train_cfg cfg;
    int8_t *states;
    int32_t *weights;
    uint64_t *block_counters;
    int n_cta, threads, smem, smem_states, cluster;
    int warp = 0;  // tiny banks: 1 k_train_warp (one warp), 2 k_train_tiny (one warp per clause)
    uint64_t launches = 0;
    TrainK k;
    uint64_t *block_seeds_d = nullptr;
    unsigned long long *ring_d = nullptr;  // grid mode: per-example vote slots [cap][2]
    int64_t ring_cap = 0;
    uint32_t *recs_d = nullptr;  // fast path: step records [rec_cap][R]
    int64_t rec_cap = 0;
    unsigned *gsync_d = nullptr;  // gbal: [ring_cap][2] step arrival counters
    void *gbal_d = nullptr;       // gbal: gcount, gw_*, gmask in one allocation
    uint64_t *thr_d = nullptr;    // fast path: threshold table [2T + 1]
};

namespace {

void per_cta_maxima(TrainK &k) {
    int cmax = 0, fmax = 0, bmax = 0;
    for (int b = 0; b < k.n_cta; ++b) {
        int c0 = cta_begin(b, k.C, k.n_cta), c1 = cta_begin(b + 1, k.C, k.n_cta);
        cmax = std::max(cmax, c1 - c0);
        int b0 = block_of(c0, k.C, k.n_blocks), b1 = block_of(c1 - 1, k.C, k.n_blocks);
        int fs = block_begin(b0, k.C, k.n_blocks), fe = block_begin(b1 + 1, k.C, k.n_blocks);
        fmax = std::max(fmax, (fe - (fs & ~31) + 31) / 32);
        bmax = std::max(bmax, b1 - b0 + 1);
    }
    k.cmax = cmax;
    k.fmax_words = fmax;
    k.bmax = bmax;
}

const void *kernel_for(bool cluster, bool smem_states, bool fast, bool prof = false, bool spec = false,
                       int threads = 512) {
    if (fast && spec)
        return prof ? (smem_states ? (const void *)k_train_spec<true, true>
                                   : (const void *)k_train_spec<false, true>)
                    : (smem_states ? (const void *)k_train_spec<true, false>
                                   : (const void *)k_train_spec<false, false>);
    if (cluster)
        return smem_states ? (const void *)k_train<MODE_CLUSTER, true>
                           : (const void *)k_train<MODE_CLUSTER, false>;
    if (fast)
        return prof ? (smem_states ? (const void *)k_train_fast<true, true>
                                   : (const void *)k_train_fast<false, true>)
                    : (smem_states ? (const void *)k_train_fast<true, false>
                                   : (const void *)k_train_fast<false, false>);
    if (!smem_states && threads > 512) return (const void *)k_train<MODE_GRID, false, 1024>;
    return smem_states ? (const void *)k_train<MODE_GRID, true> : (const void *)k_train<MODE_GRID, false>;
}

// Fast-path step-record budget: longer runs are launched in chunks.
constexpr size_t kRecordBufferBytes = size_t(2) << 30;

}  // namespace

namespace tmb {
int64_t g_train_key_chunk = 0;  // tmb_set_option("train.key_chunk"): test override
int g_train_dbg = 0;            // tmb_set_option("train.debug_skip"): timing ablations
// tmb_set_option("train.spec_window"): examples per speculative window of the
// fast grid trainer (k_train_spec, 1..16), 0 = k_train_fast; read at create
int g_train_spec = 16;
// tmb_set_option("train.spec_entries"): flag entries staged per step head,
// 0 = as many as fit (256 measured no faster than 64: the entry loads are
// not what the non-empty path waits on)
int g_train_spec_ent = 64;
// tmb_set_option("train.hbm_threads"): CTA size of the HBM-state generic
// grid trainer when the caller leaves it to the library (512 | 1024, read at
// create); 1024 measured 9% faster on configs[3] (2.44 -> 2.65 k ex/s)
int g_train_hbm_threads = 1024;
int g_train_tiny = 1;  // tmb_set_option("train.tiny"): tiny banks on k_train_tiny (0: k_train_warp)
// tmb_set_option("train.gbal_weights"): cost weights of the balanced feedback's
// split, bytes 0..2 = Type II / Type I silent / Type I firing (0 = unweighted)
int g_train_gbw = 2 | (5 << 8) | (6 << 16);
}

namespace {

}  // namespace

extern "C" {

int tmb_trainer_create(const tmb_train_cfg *cfg, int8_t *states, int32_t *weights,
                       uint64_t *block_counters, int n_cta, int threads, tmb_trainer **out) {
    int rc = require_device();
    if (rc) return rc;
    if (!cfg || !states || !weights || !block_counters || !out)
        return fail(TMB_E_INVALID, "trainer_create: NULL argument");
    const tmb_train_cfg &c = *cfg;
    if (c.n_clauses < 1 || c.n_positions < 1 || c.n_classes < 2 || c.n_blocks < 1 ||
        c.n_blocks > c.n_clauses || c.threshold < 1 || !(c.s > 1.0))
        return fail(TMB_E_INVALID, "trainer_create: invalid configuration");
    if (c.n_clauses > (1LL << 30) || c.n_positions > (1LL << 30))
        return fail(TMB_E_UNSUPPORTED, "trainer_create: shape too large");
    const int C = (int)c.n_clauses, P = (int)c.n_positions, K = (int)c.n_classes;
    const int W = (P + 31) / 32;
    const int Ppad = ((P + 127) / 128) * 128;
    const int sms = sm_count();
    const int64_t work = (int64_t)C * Ppad;
    // auto: one CTA for tiny banks, else one CTA per SM (grid mode measured
    // faster than the 16-CTA cluster mode on the configs[1] shapes)
    if (n_cta <= 0) n_cta = work <= 65536 ? 1 : sms;
    n_cta = std::max(1, std::min(n_cta, C));
    if (n_cta > 16 && n_cta > sms) n_cta = sms;
    const bool cluster = n_cta <= 16;
    if (!cluster && n_cta >= 256)
        return fail(TMB_E_UNSUPPORTED, "trainer_create: grid mode supports < 256 CTAs");
    const bool auto_threads = threads <= 0;
    if (threads <= 0) threads = (n_cta == 1 && work <= 16384) ? 256 : 512;
    threads = std::max(64, std::min(std::max(512, kFastMaxThreads), threads / 32 * 32));
    if (threads > 512 && !(!cluster && c.n_blocks == 1 && !(c.flags & 2) && C <= 65535))
        threads = 512;  // only the fast grid kernel is built for more than 512 threads

    if (W > kRowRegs * threads)
        return fail(TMB_E_UNSUPPORTED, "trainer_create: literal rows wider than 4*threads words");
    TrainK k{};
    k.C = C; k.P = P; k.K = K; k.W = W; k.Ppad = Ppad;
    k.n_blocks = (int)c.n_blocks; k.n_cta = n_cta;
    k.vec4 = (P % 4 == 0) && (reinterpret_cast<uintptr_t>(states) % 4 == 0);
    k.budget = c.budget; k.T = c.threshold;
    k.fp = make_fb_params(c.s, c.boost, c.state_min, c.state_max);
    k.fb_seed = derive_stream(c.seed, 0xFEED);
    per_cta_maxima(k);
    // fast path: grid mode, one block, 16-bit clause ids (flags bit 1 forces
    // the generic grid kernel)
    k.Wp = (W + 3) / 4 * 4;
    k.Cp = (C + 3) / 4 * 4;
    k.R = 4 + k.Wp + 260 + 2 * k.Cp;
    k.fast = (!cluster && c.n_blocks == 1 && !(c.flags & 2) && C <= 65535) ? 1 : 0;
    // (window evaluation holds two literal words per lane: rows of <= 64 words)
    k.spec = (k.fast && W <= 64) ? std::max(0, std::min(16, g_train_spec)) : 0;
    k.MW = k.spec ? k.Wp : W;
    k.spec_ent = 64;
    k.gbal = (!cluster && !(c.flags & 4)) ? 1 : 0;  // used by the generic grid kernel, HBM states
    if (cluster && k.cmax > 32 * 1024)
        return fail(TMB_E_UNSUPPORTED, "trainer_create: too many clauses per CTA");

    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (k.spec && smem_layout(k, false, MODE_GRID, nullptr, nullptr) > (size_t)max_smem) {
        k.spec = 0;
        k.MW = W;
    }
    if (k.fast && smem_layout(k, false, MODE_GRID, nullptr, nullptr) > (size_t)max_smem) k.fast = 0;
    const size_t need_on = smem_layout(k, true, cluster ? MODE_CLUSTER : MODE_GRID, nullptr, nullptr);
    const size_t need_off = smem_layout(k, false, cluster ? MODE_CLUSTER : MODE_GRID, nullptr, nullptr);
    // flags bit 0 forces HBM-resident states (tests the streaming path)
    const int smem_states = (need_on <= (size_t)max_smem && !(c.flags & 1)) ? 1 : 0;
    size_t need = smem_states ? need_on : need_off;
    // fast path: the threshold table in shared memory if it fits next to
    // everything else (it never displaces resident states)
    if (k.fast && c.threshold <= 8192) {
        k.thr_smem = 1;
        const size_t with_tab = smem_layout(k, smem_states, MODE_GRID, nullptr, nullptr);
        if (with_tab <= (size_t)max_smem) need = with_tab;
        else k.thr_smem = 0;
    }
    // k_train_spec: stage as many flag entries per step head as fit
    // (tmb_set_option("train.spec_entries") fixes the count for A/B runs)
    if (k.spec && need <= (size_t)max_smem) {
        const int want[] = {256, 224, 192, 160, 128, 96, 64};
        for (int e : want) {
            if (g_train_spec_ent > 0 && e != g_train_spec_ent) continue;
            k.spec_ent = e;
            const size_t n2 = smem_layout(k, smem_states, MODE_GRID, nullptr, nullptr);
            if (n2 <= (size_t)max_smem) {
                need = n2;
                break;
            }
            k.spec_ent = 64;
        }
        need = smem_layout(k, smem_states, MODE_GRID, nullptr, nullptr);
    }
    if (need > (size_t)max_smem)
        return fail(TMB_E_UNSUPPORTED,
                    "trainer_create: per-CTA include masks exceed shared memory (" +
                        std::to_string(need) + " B); use more CTAs");
    // HBM-resident states on the generic grid kernel: optionally 1024 threads
    // (tmb_set_option("train.hbm_threads")), twice the warps to hide latency
    if (auto_threads && !smem_states && !cluster && !k.fast && g_train_hbm_threads > 512)
        threads = 1024;
    const void *fn = kernel_for(cluster, smem_states, k.fast, false, k.spec != 0, threads);
    if (k.fast && 2 * C > 48 * 1024)
        TMB_CUDA(cudaFuncSetAttribute((const void *)k_step_records,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * C));
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
    if (cluster) {
        if (n_cta > 8)
            TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = n_cta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(n_cta);
        lc.blockDim = dim3(threads);
        lc.dynamicSmemBytes = need;
        lc.attrs = at;
        lc.numAttrs = 1;
        int n_clusters = 0;
        TMB_CUDA(cudaOccupancyMaxActiveClusters(&n_clusters, fn, &lc));
        if (n_clusters < 1)
            return fail(TMB_E_UNSUPPORTED, "trainer_create: a cluster of " +
                                               std::to_string(n_cta) + " CTAs cannot be resident");
    } else {
        int per_sm = 0;
        TMB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, need));
        if (per_sm * sms < n_cta)
            return fail(TMB_E_UNSUPPORTED, "trainer_create: grid cannot be co-resident");
    }

    // tiny banks (C, K <= 32, literal rows of <= 32 words) on one CTA: the
    // single-warp trainer (flags bit 3 keeps the generic cluster kernel)
    const size_t warp_smem = warp_kernel_smem(C, P, K, W, (int)c.n_blocks);
    const bool warp_k = n_cta == 1 && C <= kWarpMaxC && K <= 32 && W <= kWarpMaxW &&
                        !(c.flags & 8) && warp_smem <= (size_t)max_smem;
    if (warp_k && warp_smem > 48 * 1024)
        TMB_CUDA(cudaFuncSetAttribute((const void *)k_train_warp,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)warp_smem));

    // ... by default with one warp per clause (k_train_tiny); train.tiny 0
    // keeps the single-warp kernel
    const bool tiny_k = warp_k && g_train_tiny && tiny_kernel_smem(C, P) <= (size_t)max_smem;
    if (tiny_k && tiny_kernel_smem(C, P) > 48 * 1024)
        TMB_CUDA(cudaFuncSetAttribute((const void *)k_train_tiny,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)tiny_kernel_smem(C, P)));

    tmb_trainer *t = new tmb_trainer();
    t->cfg = c;
    t->warp = tiny_k ? 2 : warp_k ? 1 : 0;
    t->states = states; t->weights = weights; t->block_counters = block_counters;
    t->n_cta = n_cta; t->threads = threads; t->smem = (int)need;
    t->smem_states = smem_states; t->cluster = cluster;
    std::vector<uint64_t> seeds(c.n_blocks);
    for (int64_t b = 0; b < c.n_blocks; ++b) seeds[b] = derive_stream(c.seed, (uint64_t)b);
    if ((rc = check_cuda(cudaMalloc(&t->block_seeds_d, 8 * c.n_blocks), "cudaMalloc")) ||

        (rc = check_cuda(cudaMemcpy(t->block_seeds_d, seeds.data(), 8 * c.n_blocks,
                                    cudaMemcpyHostToDevice), "cudaMemcpy"))) {
        tmb_trainer_destroy(t);
        return rc;
    }
    k.block_seeds = t->block_seeds_d;
    if (k.thr_smem || (t->warp && c.threshold <= (1 << 20))) {
        std::vector<uint64_t> tab((size_t)(2 * c.threshold + 1));
        for (int64_t a = 0; a <= 2 * c.threshold; ++a) tab[a] = threshold_of(a, c.threshold);
        // k_train_spec: 32-bit entries (threshold >> 21; a == 2T is p == 1)
        std::vector<uint32_t> tab32(tab.size());
        for (size_t a = 0; a < tab.size(); ++a)
            tab32[a] = (uint32_t)std::min<uint64_t>(tab[a] >> 21, 0xFFFFFFFFull);
        if ((rc = check_cuda(cudaMalloc(&t->thr_d, 12 * tab.size()), "cudaMalloc")) ||
            (rc = check_cuda(cudaMemcpy(t->thr_d, tab.data(), 8 * tab.size(),
                                        cudaMemcpyHostToDevice), "cudaMemcpy")) ||
            (rc = check_cuda(cudaMemcpy(reinterpret_cast<char *>(t->thr_d) + 8 * tab.size(),
                                        tab32.data(), 4 * tab.size(), cudaMemcpyHostToDevice),
                             "cudaMemcpy"))) {
            tmb_trainer_destroy(t);
            return rc;
        }
        k.thr_tab = t->thr_d;
        k.thr32 = reinterpret_cast<const uint32_t *>(reinterpret_cast<char *>(t->thr_d) +
                                                     8 * tab.size());
    }

    k.states = states; k.weights = weights; k.block_counters = block_counters;
    k.gbal = (k.gbal && !k.fast && !smem_states) ? 1 : 0;
    for (int q = 0; q < 3; ++q) k.gbw[q] = g_train_gbw ? ((g_train_gbw >> (8 * q)) & 255) : 1;
    for (int q = 0; q < 3; ++q) k.gbw[q] = k.gbw[q] > 0 ? k.gbw[q] : 1;
    if (k.gbal) {
        const size_t n_w = (size_t)n_cta * k.cmax;
        const size_t bytes = align_up(8 * (size_t)n_cta, 256) + 2 * align_up(4 * n_w, 256) +
                             align_up(16 * n_w, 256) + align_up(4 * (size_t)C, 256) + 4 * (size_t)C * W;
        if ((rc = check_cuda(cudaMalloc(&t->gbal_d, bytes), "cudaMalloc"))) {
            tmb_trainer_destroy(t);
            return rc;
        }
        char *b = (char *)t->gbal_d;
        k.gcount = (int *)b;
        b += align_up(8 * (size_t)n_cta, 256);
        k.gw_clause = (int *)b;
        b += align_up(4 * n_w, 256);
        k.gw_info = (int *)b;
        b += align_up(4 * n_w, 256);
        k.gw_sk = (uint64_t *)b;
        b += align_up(16 * n_w, 256);
        k.gdirty = (unsigned *)b;
        b += align_up(4 * (size_t)C, 256);
        k.gmask = (uint32_t *)b;
    }
    t->k = k;
    *out = t;
    return TMB_OK;
}

int tmb_trainer_set_profile(tmb_trainer *t, uint64_t *phase) {
    if (!t) return fail(TMB_E_INVALID, "trainer_set_profile: NULL trainer");
    t->k.phase = reinterpret_cast<unsigned long long *>(phase);
    return TMB_OK;
}

int tmb_trainer_set_trace(tmb_trainer *t, int64_t *trace) {
    if (!t) return fail(TMB_E_INVALID, "trainer_set_trace: NULL trainer");
    t->k.trace = reinterpret_cast<long long *>(trace);
    return TMB_OK;
}

int tmb_trainer_destroy(tmb_trainer *t) {
    if (!t) return TMB_OK;
    if (t->block_seeds_d) cudaFree(t->block_seeds_d);
    if (t->ring_d) cudaFree(t->ring_d);
    if (t->recs_d) cudaFree(t->recs_d);
    if (t->gsync_d) cudaFree(t->gsync_d);
    if (t->gbal_d) cudaFree(t->gbal_d);
    if (t->thr_d) cudaFree(t->thr_d);
    delete t;
    return TMB_OK;
}

int tmb_trainer_info(const tmb_trainer *t, int *n_cta, int *threads, int *smem_bytes,
                     int *states_in_smem) {
    if (!t) return fail(TMB_E_INVALID, "trainer_info: NULL");
    if (n_cta) *n_cta = t->n_cta;
    if (threads) *threads = t->warp == 2 ? 32 * t->k.C : t->warp ? 32 : t->threads;
    if (smem_bytes) *smem_bytes = t->smem;
    if (states_in_smem) *states_in_smem = t->smem_states;
    return TMB_OK;
}

int tmb_trainer_kernel(const tmb_trainer *t, int *kind, int *window) {
    if (!t) return fail(TMB_E_INVALID, "trainer_kernel: NULL");
    const int kd = t->warp == 2 ? 5 : t->warp ? 0 : t->cluster ? 1 : !t->k.fast ? 2 : t->k.spec ? 4 : 3;
    if (kind) *kind = kd;
    if (window) *window = kd == 4 ? t->k.spec : 0;
    return TMB_OK;
}

int tmb_trainer_run(tmb_trainer *t, const uint32_t *lit_words, const int32_t *labels,
                    const int32_t *order, int64_t n_steps, uint64_t fb_counter,
                    tmb_train_stats *stats, void *stream) {
    if (!t) return fail(TMB_E_INVALID, "trainer_run: NULL trainer");
    if (n_steps <= 0) return TMB_OK;
    if (!lit_words || !labels || !order) return fail(TMB_E_INVALID, "trainer_run: NULL data");

    cudaStream_t st = as_stream(stream);
    TrainK k = t->k;
    k.lit_words = lit_words; k.labels = labels; k.order = order;
    k.n_steps = n_steps; k.fb_counter0 = fb_counter; k.stats = stats;
    k.dbg = g_train_dbg;
    void *args[] = {&k};
    if (t->warp == 2) {
        const size_t sm = tiny_kernel_smem(k.C, k.P);
        if (sm > 48 * 1024)
            TMB_CUDA(cudaFuncSetAttribute((const void *)k_train_tiny,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_train_tiny<<<1, 32 * k.C, sm, st>>>(k);
        TMB_LAUNCHED();
        return TMB_OK;
    }
    if (t->warp) {
        const size_t sm = warp_kernel_smem(k.C, k.P, k.K, k.W, k.n_blocks);
        if (sm > 48 * 1024)
            TMB_CUDA(cudaFuncSetAttribute((const void *)k_train_warp,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_train_warp<<<1, 32, sm, st>>>(k);
        TMB_LAUNCHED();
        return TMB_OK;
    }
    const void *fn = kernel_for(t->cluster, t->smem_states, k.fast, k.phase != nullptr, k.spec != 0,
                                t->threads);
    // the dynamic shared-memory limit is a per-function attribute: another
    // trainer of a different shape may have lowered it since create
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, t->smem));
    if (k.fast && 2 * k.C > 48 * 1024)
        TMB_CUDA(cudaFuncSetAttribute((const void *)k_step_records,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * k.C));
    if (t->cluster) {
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = t->n_cta;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        lc.gridDim = dim3(t->n_cta);
        lc.blockDim = dim3(t->threads);
        lc.dynamicSmemBytes = (size_t)t->smem;
        lc.stream = st;
        lc.attrs = at;
        lc.numAttrs = 1;
        TMB_CUDA(cudaLaunchKernelExC(&lc, fn, args));
        TMB_LAUNCHED();
        return TMB_OK;
    }
    // grid mode; fast-path runs are split into chunks whose records fit
    int64_t chunk = n_steps;
    if (k.fast) {
        chunk = std::max<int64_t>(1, (int64_t)(kRecordBufferBytes / (4 * (size_t)k.R)));
        // k_train_spec's vote slots grow with the launch ((2n + 2) windows x
        // 2 * spec words): at most 2^18 steps per launch (128 MB of slots)
        if (k.spec) chunk = std::min<int64_t>(chunk, int64_t(1) << 18);
        if (g_train_key_chunk > 0) chunk = std::min(chunk, g_train_key_chunk);
    }
    const int64_t slots = std::min(n_steps, chunk);
    // vote slots: 2 per step, or (spec) 2 * spec per window number (< 2n + 2)
    auto ring_words = [&](int64_t nn) -> size_t {
        return k.spec ? (size_t)(2 * nn + 2) * 2 * (size_t)k.spec : 2 * (size_t)nn;
    };
    if (t->ring_cap < slots || (k.fast && t->rec_cap < slots)) {
        cudaStreamSynchronize(st);
        if (t->ring_d) cudaFree(t->ring_d);
        if (t->recs_d) cudaFree(t->recs_d);
        if (t->gsync_d) cudaFree(t->gsync_d);
        t->ring_d = nullptr; t->recs_d = nullptr; t->gsync_d = nullptr;
        t->ring_cap = 0; t->rec_cap = 0;
        TMB_CUDA(cudaMalloc(&t->ring_d, 8 * ring_words(slots)));
        if (k.gbal) TMB_CUDA(cudaMalloc(&t->gsync_d, 8 * (size_t)slots));
        t->ring_cap = slots;
        if (k.fast) {
            TMB_CUDA(cudaMalloc(&t->recs_d, 4 * (size_t)k.R * (size_t)slots));
            t->rec_cap = slots;
        }
    }
    const uint64_t step_draws = 1ull + 2ull * (uint64_t)k.C;
    for (int64_t off = 0; off < n_steps; off += chunk) {
        const int64_t n = std::min(chunk, n_steps - off);
        k.order = order + off;
        k.n_steps = n;
        k.fb_counter0 = fb_counter + (uint64_t)off * step_draws;
        k.rec = t->ring_d;
        TMB_CUDA(cudaMemsetAsync(t->ring_d, 0, 8 * ring_words(n), st));
        if (k.gbal) {
            k.gsync = t->gsync_d;
            TMB_CUDA(cudaMemsetAsync(t->gsync_d, 0, 8 * (size_t)n, st));
        }
        if (k.fast) {
            k.recs = t->recs_d;
            k_step_records<<<dim3((unsigned)n, 2), 256, 2 * (size_t)k.C, st>>>(k, t->recs_d);
            TMB_LAUNCHED();
        }
        TMB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(t->n_cta), dim3(t->threads), args,
                                             (size_t)t->smem, st));
        TMB_LAUNCHED();
    }
    return TMB_OK;
}

}  // extern "C"

// ------------------------------------------------- feedback microbench --
namespace tmb {
template <int VARIANT>
__global__ void __launch_bounds__(1024, 1) k_mb_feedback(TrainK k, int n_work, int two, int iters,
                                                          unsigned long long *cyc) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, true, MODE_GRID, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x;
    for (int i = tid; i < k.cmax * k.Ppad; i += nthr)
        s.states[i] = (int8_t)((int)(mix64((uint64_t)i) & 255) - 128);
    for (int i = tid; i < k.cmax * k.MW; i += nthr) s.masks[i] = 0;
    for (int j = tid; j < k.cmax; j += nthr) {
        s.work[j] = j;
        s.info[j] = ((two & 2) ? 0 : I_OUT) | I_TEV | I_T1 | ((two & 1) ? (I_NEV | I_N1) : 0);
        s.sk_t[j] = mix64(j);
        s.sk_n[j] = mix64(j + 100);
        s.cnt[j] = 0;
    }
    uint32_t *lit = s.lit0;
    for (int w = tid; w < k.W; w += nthr) lit[w] = (uint32_t)mix64(w + 7);
    __syncthreads();
    Counters cn;
    unsigned long long tot = 0;
    for (int it = 0; it < iters; ++it) {
        const long long t0 = clock64();
        if (VARIANT == 0) feedback_quads<true>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 1) feedback_compact<true>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 2) feedback_compact<true, 1>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 3) feedback_compact<true, 2>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 4) feedback_compact<true, 4>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 5) feedback_compact<true, 7>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 6) feedback_simd_v1<true>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 11) feedback_simd<true>(k, s, 0, lit, n_work, cn);
        else if (VARIANT == 7) feedback_wide<4, 1>(k, s, lit, n_work, cn);
        else if (VARIANT == 8) feedback_wide<4, 4>(k, s, lit, n_work, cn);
        else if (VARIANT == 9) feedback_wide<2, 1>(k, s, lit, n_work, cn);
        else feedback_wide<2, 2>(k, s, lit, n_work, cn);
        __syncthreads();
        tot += (unsigned long long)(clock64() - t0);
    }
    if (tid == 0) cyc[0] = tot + ((cn.draws + cn.t2) & 1);  // keep the work alive
}
}  // namespace tmb

extern "C" int tmb_microbench_feedback(int variant, int n_work, int two_events, int threads,
                                       int iters, double *cycles_per_call) {
    using namespace tmb;
    int rc = require_device();
    if (rc) return rc;
    if (n_work < 0 || n_work > 14 || iters < 1 || !cycles_per_call)
        return fail(TMB_E_INVALID, "microbench_feedback: bad arguments");
    TrainK k{};
    k.C = 2000; k.P = 1568; k.K = 10; k.W = 49; k.Ppad = 1664; k.n_blocks = 1; k.n_cta = 148;
    k.cmax = 14; k.fmax_words = 1; k.bmax = 1; k.vec4 = 1; k.fast = 1; k.Wp = 52; k.Cp = 2000;
    k.R = 4 + k.Wp + 260 + 2 * k.Cp; k.MW = 52; k.budget = 1 << 30; k.T = 5000;
    k.fp = make_fb_params(10.0, 0, -128, 127);
    const size_t sm = smem_layout(k, true, MODE_GRID, nullptr, nullptr);
    unsigned long long *cyc = nullptr;
    TMB_CUDA(cudaMalloc(&cyc, 8));
    const void *fns[12] = {(const void *)k_mb_feedback<0>, (const void *)k_mb_feedback<1>,
                           (const void *)k_mb_feedback<2>, (const void *)k_mb_feedback<3>,
                           (const void *)k_mb_feedback<4>, (const void *)k_mb_feedback<5>,
                           (const void *)k_mb_feedback<6>, (const void *)k_mb_feedback<7>,
                           (const void *)k_mb_feedback<8>, (const void *)k_mb_feedback<9>,
                           (const void *)k_mb_feedback<10>, (const void *)k_mb_feedback<11>};
    if (variant < 0 || variant > 11) return fail(TMB_E_INVALID, "microbench_feedback: variant 0..11");
    TMB_CUDA(cudaFuncSetAttribute(fns[variant], cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    void *args[] = {&k, &n_work, &two_events, &iters, &cyc};
    TMB_CUDA(cudaLaunchKernel(fns[variant], dim3(1), dim3(threads), args, sm, 0));
    rc = check_cuda(cudaGetLastError(), "microbench launch");
    unsigned long long c = 0;
    if (!rc) rc = check_cuda(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost), "cudaMemcpy");
    cudaFree(cyc);
    if (!rc) *cycles_per_call = (double)c / iters;
    return rc;
}
