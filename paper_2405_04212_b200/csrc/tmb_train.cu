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
//   GRID mode (n_cta > 16, cooperative launch, up to one CTA per SM): K int64
//     atomics + one global barrier per example; update-flag draws for the
//     CTA's block range are precomputed while the barrier is pending.
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
    int64_t budget, T;
    FbParams fp;
    uint64_t fb_seed, fb_counter0;
    int64_t n_steps;
    const uint32_t *lit_words;
    const int32_t *labels, *order;
    int8_t *states;
    int32_t *weights;
    uint64_t *block_counters;
    const uint64_t *block_seeds;
    unsigned long long *ring;  // [3][K] (grid mode)
    unsigned int *bar;
    tmb_train_stats *stats;
};

// executor.py:36-47 partition: block of clause c and block start.
__host__ __device__ __forceinline__ int block_of(int c, int C, int nb) {
    int base = C / nb, extra = C % nb;
    int big = extra * (base + 1);
    return c < big ? c / (base + 1) : extra + (c - big) / base;
}
__host__ __device__ __forceinline__ int block_begin(int b, int C, int nb) {
    int base = C / nb, extra = C % nb;
    return b * base + (b < extra ? b : extra);
}
__host__ __device__ __forceinline__ int cta_begin(int r, int C, int n_cta) {
    return (int)((int64_t)r * C / n_cta);
}
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

enum : int { I_TEV = 1, I_NEV = 2, I_T1 = 4, I_N1 = 8, I_OUT = 16 };

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct Smem {
    uint32_t *lit0, *lit1, *masks, *ut_bits, *un_bits;
    int32_t *word_cum, *weights, *work, *info, *lpref, *cta_pfx, *blk_lo, *blk_hi, *wsum;
    uint64_t *sk_t, *sk_n, *blk_ctr, *draw_t, *draw_n;
    int8_t *states;
    long long *votes;  // [K] partial (cluster) / total (single)
    int *misc;         // [0]=n_work [1]=negative [2]=label [3..5]=example ring
    uint64_t *thr;     // [0]=t_t [1]=t_n
};

// Shared-memory carve-up; identical on host (size) and device (pointers).
__host__ __device__ inline size_t smem_layout(const TrainK &k, bool smem_states, bool cluster,
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
    t.thr = (uint64_t *)take(8 * 2);
    t.votes = (long long *)take(8 * k.K);
    t.lit0 = (uint32_t *)take(4 * k.W);
    t.lit1 = (uint32_t *)take(4 * k.W);
    t.masks = (uint32_t *)take(4 * (size_t)k.cmax * k.W);
    t.weights = (int32_t *)take(4 * (size_t)k.cmax * k.K);
    t.work = (int32_t *)take(4 * k.cmax);
    t.info = (int32_t *)take(4 * k.cmax);
    t.misc = (int *)take(4 * 8);
    t.wsum = (int32_t *)take(4 * 32);
    if (cluster) {
        t.draw_t = (uint64_t *)take(8 * k.cmax);
        t.draw_n = (uint64_t *)take(8 * k.cmax);
        t.lpref = (int32_t *)take(4 * (k.cmax + 1));
        t.cta_pfx = (int32_t *)take(4 * 32);
        t.blk_lo = (int32_t *)take(4 * (k.bmax + 1));
        t.blk_hi = (int32_t *)take(4 * (k.bmax + 1));
        t.ut_bits = t.un_bits = nullptr;
        t.word_cum = nullptr;
    } else {
        t.ut_bits = (uint32_t *)take(4 * k.fmax_words);
        t.un_bits = (uint32_t *)take(4 * k.fmax_words);
        t.word_cum = (int32_t *)take(4 * (k.fmax_words + 1));
        t.draw_t = (uint64_t *)take(8 * 32 * k.fmax_words);
        t.draw_n = (uint64_t *)take(8 * 32 * k.fmax_words);
        t.lpref = t.cta_pfx = t.blk_lo = t.blk_hi = nullptr;
    }
    t.states = smem_states ? (int8_t *)take((size_t)k.cmax * k.Ppad) : nullptr;
    if (s) *s = t;
    return align_up(off, 16);
}

struct Counters {
    uint64_t draws = 0, upd = 0, events = 0, t1 = 0, t2 = 0;
};

// Per-position feedback over the CTA's work list, four positions per thread
// (one 32-bit state word), include masks rebuilt from the new states.
// kernels/_numba.py:71-98 semantics per position, target event then negative
// event.
template <bool SMEM_STATES>
__device__ __forceinline__ void feedback_quads(const TrainK &k, const Smem &s, int c0,
                                               const uint32_t *lit, int n_work, Counters &cn) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int QP = k.Ppad >> 2;  // quads per (padded) row; multiple of 32
    const int total = n_work * QP;
    int wc = tid / QP, q = tid - (tid / QP) * QP;
    for (int it = tid; it < total; it += nthr) {
        const int j = s.work[wc];
        const int info = s.info[j];
        const int out = (info & I_OUT) ? 1 : 0;
        const int p0 = q << 2;
        uint32_t word;
        int8_t *grow = k.states + (int64_t)(c0 + j) * k.P;
        if (SMEM_STATES) {
            word = *reinterpret_cast<const uint32_t *>(s.states + (size_t)j * k.Ppad + p0);
        } else if (k.vec4 && p0 + 4 <= k.P) {
            word = *reinterpret_cast<const uint32_t *>(grow + p0);
        } else {
            word = 0xFFFFFFFFu;
            for (int b = 0; b < 4; ++b)
                if (p0 + b < k.P) word = (word & ~(0xFFu << (8 * b))) | ((uint32_t)(uint8_t)grow[p0 + b] << (8 * b));
        }
        const uint32_t litn = p0 < k.P ? (lit[p0 >> 5] >> (p0 & 31)) & 0xFu : 0u;
        uint32_t nw = word, nib = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int p = p0 + b;
            int st = (int)(int8_t)(word >> (8 * b));
            if (p < k.P) {
                const int l = (litn >> b) & 1;
                int st0 = st;
                uint64_t nd = 0;
                if (info & I_TEV) {
                    if (info & I_T1) st = type_i_stream(st, l, out, k.fp, s.sk_t[j], (uint32_t)p, nd);
                    else st = type_ii(st, l, out);
                }
                if (info & I_NEV) {
                    if (info & I_N1) st = type_i_stream(st, l, out, k.fp, s.sk_n[j], (uint32_t)p, nd);
                    else st = type_ii(st, l, out);
                }
                cn.draws += nd;
                if (st != st0) {
                    ++cn.upd;
                    nw = (nw & ~(0xFFu << (8 * b))) | ((uint32_t)(uint8_t)st << (8 * b));
                }
                nib |= (uint32_t)(st >= 0) << b;
            }
        }
        if (nw != word) {
            if (SMEM_STATES) {
                *reinterpret_cast<uint32_t *>(s.states + (size_t)j * k.Ppad + p0) = nw;
            } else if (k.vec4 && p0 + 4 <= k.P) {
                *reinterpret_cast<uint32_t *>(grow + p0) = nw;
            } else {
                for (int b = 0; b < 4; ++b)
                    if (p0 + b < k.P) grow[p0 + b] = (int8_t)(nw >> (8 * b));
            }
        }
        // mask word for positions 32*w .. : lanes 8g..8g+7 hold its 8 nibbles
        uint32_t m = nib << ((lane & 7) * 4);
        m |= __shfl_xor_sync(0xffffffffu, m, 1);
        m |= __shfl_xor_sync(0xffffffffu, m, 2);
        m |= __shfl_xor_sync(0xffffffffu, m, 4);
        if ((lane & 7) == 0) {
            const int w = p0 >> 5;
            if (w < k.W) s.masks[j * k.W + w] = m;
        }
        q += nthr;
        while (q >= QP) {
            q -= QP;
            ++wc;
        }
    }
}

// Load the model slice into shared memory and build the include masks.
template <bool SMEM_STATES>
__device__ __forceinline__ void load_slice(const TrainK &k, const Smem &s, int c0, int cown) {
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31;
    const int warp = tid >> 5, nwarps = nthr >> 5;
    for (int i = tid; i < cown * k.K; i += nthr) s.weights[i] = k.weights[(int64_t)c0 * k.K + i];
    if (SMEM_STATES) {
        for (int i = tid; i < cown * k.Ppad; i += nthr) {
            int j = i / k.Ppad, p = i - j * k.Ppad;
            s.states[i] = p < k.P ? k.states[(int64_t)(c0 + j) * k.P + p] : (int8_t)-1;
        }
        __syncthreads();
    }
    for (int it = warp; it < cown * k.W; it += nwarps) {
        int j = it / k.W, w = it - j * k.W;
        int p = w * 32 + lane;
        int st;
        if (SMEM_STATES) st = s.states[j * k.Ppad + p];
        else st = p < k.P ? k.states[(int64_t)(c0 + j) * k.P + p] : -1;
        unsigned m = __ballot_sync(0xffffffffu, st >= 0);
        if (lane == 0) s.masks[j * k.W + w] = m;
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

// Example ring in shared memory: misc[3 + (i % 3)] = order[i]; rows of
// example i live in lit[i & 1].  Issued one/two examples ahead so the
// dependent global loads overlap the current example.
__device__ __forceinline__ void prefetch(const TrainK &k, const Smem &s, int64_t i) {
    // order index two ahead
    if (threadIdx.x == 0 && i + 2 < k.n_steps) s.misc[3 + (int)((i + 2) % 3)] = __ldg(&k.order[i + 2]);
    // literal row one ahead (its index arrived one iteration ago)
    if (i + 1 < k.n_steps) {
        const int ex = s.misc[3 + (int)((i + 1) % 3)];
        uint32_t *dst = ((i + 1) & 1) ? s.lit1 : s.lit0;
        for (int w = threadIdx.x; w < k.W; w += blockDim.x)
            dst[w] = __ldg(&k.lit_words[(int64_t)ex * k.W + w]);
    }
}

__device__ __forceinline__ void prologue_ring(const TrainK &k, const Smem &s) {
    if (threadIdx.x == 0) {
        s.misc[3] = __ldg(&k.order[0]);
        if (k.n_steps > 1) s.misc[4] = __ldg(&k.order[1]);
    }
    __syncthreads();
    const int ex = s.misc[3];
    for (int w = threadIdx.x; w < k.W; w += blockDim.x)
        s.lit0[w] = __ldg(&k.lit_words[(int64_t)ex * k.W + w]);
}

// training-mode clause outputs (kernels/_numba.py:36-50) -> info[j] = I_OUT|0
__device__ __forceinline__ void eval_own(const TrainK &k, const Smem &s, const uint32_t *lit,
                                         int cown) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int j = warp; j < cown; j += nwarps) {
        uint32_t viol = 0;
        int cnt = 0;
        for (int w = lane; w < k.W; w += 32) {
            uint32_t m = s.masks[j * k.W + w];
            viol |= m & ~lit[w];
            cnt += __popc(m);
        }
        viol = __reduce_or_sync(0xffffffffu, viol);
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) s.info[j] = (viol == 0 && cnt <= k.budget) ? I_OUT : 0;
    }
}

// partial class sums of own clauses (dense.py:153): warp per class
__device__ __forceinline__ void partial_votes(const TrainK &k, const Smem &s, int cown) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int kk = warp; kk < k.K; kk += nwarps) {
        long long v = 0;
        for (int j = lane; j < cown; j += 32)
            if (s.info[j] & I_OUT) v += s.weights[j * k.K + kk];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) s.votes[kk] = v;
    }
}

// feedback.py:33-44 given the summed votes of the label / negative classes.
__device__ __forceinline__ void decide(const TrainK &k, long long vl, long long vn, uint64_t *thr) {
    const long long T = k.T;
    long long cl = vl < -T ? -T : (vl > T ? T : vl);
    long long cn = vn < -T ? -T : (vn > T ? T : vn);
    double pt = (double)(T - cl) / (2.0 * (double)T);
    double pn = (double)(T + cn) / (2.0 * (double)T);
    thr[0] = prob_threshold(pt);
    thr[1] = prob_threshold(pn);
}

__device__ __forceinline__ int negative_class(const TrainK &k, int label, uint64_t fbc) {
    double u = u01_from53(draw53(k.fb_seed, fbc));
    return (int)((label + 1 + (int64_t)(u * (double)(k.K - 1))) % k.K);
}

// Event bookkeeping for own clause j given its window ordinal (events of its
// block before it, plus the block counter).  Updates weights (feedback first,
// then weight) and appends to the work list.
__device__ __forceinline__ void clause_events(const TrainK &k, const Smem &s, int j, int c,
                                              bool t_ev, bool n_ev, uint64_t ord, int label,
                                              int neg, Counters &cn) {
    int info = s.info[j] & I_OUT;
    if (t_ev || n_ev) {
        const uint64_t bseed = k.block_seeds[block_of(c, k.C, k.n_blocks)];
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
        const bool work = (t_ev && ((info & I_T1) || out)) || (n_ev && ((info & I_N1) || out));
        if (work) s.work[atomicAdd(&s.misc[0], 1)] = j;
    }
    s.info[j] = info;
}

// ============================================================ CLUSTER mode
template <bool SMEM_STATES>
__global__ void __launch_bounds__(512, 1) k_train_cluster(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    Smem s;
    smem_layout(k, SMEM_STATES, true, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int rank = (int)cluster.block_rank();
    const int n_cta = k.n_cta, C = k.C, K = k.K;
    const int c0 = cta_begin(rank, C, n_cta), c1 = cta_begin(rank + 1, C, n_cta);
    const int cown = c1 - c0;
    const int b0 = block_of(c0, C, k.n_blocks), b1 = block_of(c1 - 1, C, k.n_blocks);

    load_slice<SMEM_STATES>(k, s, c0, cown);
    for (int i = tid; i <= b1 - b0; i += nthr) s.blk_ctr[i] = k.block_counters[b0 + i];
    prologue_ring(k, s);
    __syncthreads();
    cluster.sync();  // every CTA of the cluster is resident before DSMEM use

    Counters cn;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    for (int64_t i = 0; i < k.n_steps; ++i) {
        const uint32_t *lit = (i & 1) ? s.lit1 : s.lit0;
        const int ex = s.misc[3 + (int)(i % 3)];
        const int label = __ldg(&k.labels[ex]);
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        // 1. outputs of own clauses; update-flag draws of own clauses (they do
        //    not depend on the votes); prefetch the next example
        eval_own(k, s, lit, cown);
        for (int j = tid; j < cown; j += nthr) {
            s.draw_t[j] = draw53(k.fb_seed, fbc + 1 + (uint64_t)(c0 + j));
            s.draw_n[j] = draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)(c0 + j));
        }
        if (tid == 0) s.misc[0] = 0;
        prefetch(k, s, i);
        const int neg = negative_class(k, label, fbc);
        __syncthreads();
        // 2. partial class sums
        partial_votes(k, s, cown);
        cluster.sync();  // #1: partial votes visible cluster-wide
        // 3. decision from the cluster's summed votes
        if (warp == 0) {
            long long v = 0;
            if (lane < n_cta) {
                const long long *rv = cluster.map_shared_rank(s.votes, lane);
                v = rv[label];
            } else if (lane >= 16 && lane - 16 < n_cta) {
                const long long *rv = cluster.map_shared_rank(s.votes, lane - 16);
                v = rv[neg];
            }
            long long vl = v, vn = v;
            if (lane >= 16) vl = 0; else vn = 0;
            for (int o = 16; o; o >>= 1) {
                vl += __shfl_xor_sync(0xffffffffu, vl, o);
                vn += __shfl_xor_sync(0xffffffffu, vn, o);
            }
            if (lane == 0) decide(k, vl, vn, s.thr);
        }
        __syncthreads();
        // 4. own update flags and their exclusive prefix (block-wide scan)
        {
            const uint64_t t_t = s.thr[0], t_n = s.thr[1];
            int carry = 0;
            for (int base = 0; base < cown; base += nthr) {
                const int j = base + tid;
                int f = 0;
                if (j < cown) {
                    const bool te = s.draw_t[j] < t_t, ne = s.draw_n[j] < t_n;
                    f = (int)te + (int)ne;
                    s.info[j] |= (te ? I_TEV : 0) | (ne ? I_NEV : 0);
                }
                int x = f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                int *wsum = s.wsum;
                if (lane == 31) wsum[warp] = x;
                __syncthreads();
                if (warp == 0) {
                    int v = lane < (nthr >> 5) ? wsum[lane] : 0;
                    for (int o = 1; o < 32; o <<= 1) {
                        int y = __shfl_up_sync(0xffffffffu, v, o);
                        if (lane >= o) v += y;
                    }
                    wsum[lane] = v;
                }
                __syncthreads();
                const int excl = carry + (warp ? wsum[warp - 1] : 0) + x - f;
                if (j < cown) s.lpref[j] = excl;
                carry += wsum[(nthr >> 5) - 1];
                __syncthreads();
            }
            if (tid == 0) s.lpref[cown] = carry;
        }
        cluster.sync();  // #2: event prefixes visible cluster-wide
        // 5. CTA prefixes (events over clauses [0, cta_begin(r)))
        if (warp == 0) {
            int v = 0;
            if (lane < n_cta) {
                const int r_own = cta_begin(lane + 1, C, n_cta) - cta_begin(lane, C, n_cta);
                const int *rp = cluster.map_shared_rank(s.lpref, lane);
                v = rp[r_own];
            }
            int x = v;
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            s.cta_pfx[lane] = x - v;  // exclusive
        }
        __syncthreads();
        // Pfx(x): events over clauses [0, x) (x may belong to another CTA)
        auto pfx = [&](int x) -> int {
            if (x >= C) return s.cta_pfx[n_cta];  // total events of the cluster
            if (x >= c0 && x < c1) return s.cta_pfx[rank] + s.lpref[x - c0];
            const int r = cta_of(x, C, n_cta);
            const int *rp = cluster.map_shared_rank(s.lpref, r);
            return s.cta_pfx[r] + rp[x - cta_begin(r, C, n_cta)];
        };
        for (int bi = tid; bi <= b1 - b0; bi += nthr) {
            s.blk_lo[bi] = pfx(block_begin(b0 + bi, C, k.n_blocks));
            s.blk_hi[bi] = pfx(block_begin(b0 + bi + 1, C, k.n_blocks));
        }
        __syncthreads();
        // 6. window ordinals, event types, weights, work list
        for (int j = tid; j < cown; j += nthr) {
            const int c = c0 + j;
            const int inf = s.info[j];
            const bool t_ev = inf & I_TEV, n_ev = inf & I_NEV;
            uint64_t ord = 0;
            if (t_ev || n_ev) {
                const int bi = block_of(c, C, k.n_blocks) - b0;
                ord = s.blk_ctr[bi] + (uint64_t)(s.cta_pfx[rank] + s.lpref[j] - s.blk_lo[bi]);
            }
            s.info[j] = inf & I_OUT;
            clause_events(k, s, j, c, t_ev, n_ev, ord, label, neg, cn);
        }
        __syncthreads();
        for (int bi = tid; bi <= b1 - b0; bi += nthr)
            s.blk_ctr[bi] += (uint64_t)(s.blk_hi[bi] - s.blk_lo[bi]);
        // 7. per-position Type I / II on the work list
        feedback_quads<SMEM_STATES>(k, s, c0, lit, s.misc[0], cn);
        __syncthreads();
    }
    cluster.sync();  // no CTA leaves while others may still read its DSMEM
    store_slice<SMEM_STATES>(k, s, c0, cown);
    for (int bi = tid; bi <= b1 - b0; bi += nthr) {
        const int b = b0 + bi;
        const int last = block_begin(b + 1, C, k.n_blocks) - 1;
        if (last >= c0 && last < c1) k.block_counters[b] = s.blk_ctr[bi];
    }
    flush_stats(k, cn, rank == 0);
    (void)K;
}

// =============================================================== GRID mode
template <bool SMEM_STATES>
__global__ void __launch_bounds__(512, 1) k_train_grid(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, SMEM_STATES, false, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int cta = blockIdx.x;
    const int C = k.C, K = k.K;
    const int c0 = cta_begin(cta, C, k.n_cta), c1 = cta_begin(cta + 1, C, k.n_cta);
    const int cown = c1 - c0;
    const int b0 = block_of(c0, C, k.n_blocks), b1 = block_of(c1 - 1, C, k.n_blocks);
    const int fs = block_begin(b0, C, k.n_blocks), fe = block_begin(b1 + 1, C, k.n_blocks);
    const int fsa = fs & ~31;
    const int nfw = (fe - fsa + 31) >> 5;

    load_slice<SMEM_STATES>(k, s, c0, cown);
    for (int i = tid; i <= b1 - b0; i += nthr) s.blk_ctr[i] = k.block_counters[b0 + i];
    prologue_ring(k, s);
    __syncthreads();

    Counters cn;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    for (int64_t i = 0; i < k.n_steps; ++i) {
        const uint32_t *lit = (i & 1) ? s.lit1 : s.lit0;
        const int ex = s.misc[3 + (int)(i % 3)];
        const int label = __ldg(&k.labels[ex]);
        const int slot = (int)(i % 3);
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        eval_own(k, s, lit, cown);
        if (tid == 0) s.misc[0] = 0;
        const int neg = negative_class(k, label, fbc);
        __syncthreads();
        partial_votes(k, s, cown);
        __syncthreads();
        // arrive: K relaxed atomics then a release increment (one thread)
        if (tid == 0) {
            for (int kk = 0; kk < K; ++kk)
                if (s.votes[kk]) atomicAdd(&k.ring[slot * K + kk], (unsigned long long)s.votes[kk]);
            red_release_add(k.bar, 1u);
        }
        // while the barrier is pending: update-flag draws for [fs, fe)
        for (int idx = tid; idx < nfw * 32; idx += nthr) {
            const int j = fsa + idx;
            s.draw_t[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)j);
            s.draw_n[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)j);
        }
        prefetch(k, s, i);
        if (tid == 0) {
            const unsigned target = (unsigned)((i + 1) * k.n_cta);
            while ((int)(ld_acquire_u32(k.bar) - target) < 0) {
            }
            const long long vl = (long long)__ldcg(&k.ring[slot * K + label]);
            const long long vn = (long long)__ldcg(&k.ring[slot * K + neg]);
            decide(k, vl, vn, s.thr);
            // slot (i+2)%3 == (i-1)%3: every CTA read it before arriving here
            if (cta == 0)
                for (int kk = 0; kk < K; ++kk) k.ring[((i + 2) % 3) * K + kk] = 0ull;
        }
        __syncthreads();
        const uint64_t t_t = s.thr[0], t_n = s.thr[1];
        for (int idx = tid; idx < nfw * 32; idx += nthr) {
            const int j = fsa + idx;
            const bool valid = j >= fs && j < fe;
            const unsigned wt = __ballot_sync(0xffffffffu, valid && s.draw_t[idx] < t_t);
            const unsigned wn = __ballot_sync(0xffffffffu, valid && s.draw_n[idx] < t_n);
            if (lane == 0) {
                s.ut_bits[idx >> 5] = wt;
                s.un_bits[idx >> 5] = wn;
            }
        }
        __syncthreads();
        if (warp == 0) {
            int carry = 0;
            for (int base = 0; base < nfw; base += 32) {
                const int w = base + lane;
                const int v = w < nfw ? __popc(s.ut_bits[w]) + __popc(s.un_bits[w]) : 0;
                int x = v;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, x, o);
                    if (lane >= o) x += y;
                }
                if (w < nfw) s.word_cum[w] = carry + x - v;
                carry += __shfl_sync(0xffffffffu, x, 31);
            }
            if (lane == 0) s.word_cum[nfw] = carry;
        }
        __syncthreads();
        auto cum = [&](int x) -> int {  // events over clauses [fsa, x)
            const int q = (x - fsa) >> 5, r = (x - fsa) & 31;
            int v = s.word_cum[q];
            if (r) {
                const unsigned lo = (1u << r) - 1u;
                v += __popc(s.ut_bits[q] & lo) + __popc(s.un_bits[q] & lo);
            }
            return v;
        };
        for (int j = tid; j < cown; j += nthr) {
            const int c = c0 + j;
            const int q = (c - fsa) >> 5, r = (c - fsa) & 31;
            const bool t_ev = (s.ut_bits[q] >> r) & 1, n_ev = (s.un_bits[q] >> r) & 1;
            uint64_t ord = 0;
            if (t_ev || n_ev) {
                const int b = block_of(c, C, k.n_blocks);
                ord = s.blk_ctr[b - b0] + (uint64_t)(cum(c) - cum(block_begin(b, C, k.n_blocks)));
            }
            clause_events(k, s, j, c, t_ev, n_ev, ord, label, neg, cn);
        }
        __syncthreads();
        for (int bi = tid; bi <= b1 - b0; bi += nthr) {
            const int bs = block_begin(b0 + bi, C, k.n_blocks);
            const int be = block_begin(b0 + bi + 1, C, k.n_blocks);
            s.blk_ctr[bi] += (uint64_t)(cum(be) - cum(bs));
        }
        feedback_quads<SMEM_STATES>(k, s, c0, lit, s.misc[0], cn);
        __syncthreads();
    }
    store_slice<SMEM_STATES>(k, s, c0, cown);
    for (int bi = tid; bi <= b1 - b0; bi += nthr) {
        const int b = b0 + bi;
        const int last = block_begin(b + 1, C, k.n_blocks) - 1;
        if (last >= c0 && last < c1) k.block_counters[b] = s.blk_ctr[bi];
    }
    flush_stats(k, cn, cta == 0);
}

}  // namespace tmb

using namespace tmb;

struct tmb_trainer {
    tmb_train_cfg cfg;
    int8_t *states;
    int32_t *weights;
    uint64_t *block_counters;
    int n_cta, threads, smem, smem_states, cluster;
    TrainK k;
    uint64_t *block_seeds_d = nullptr;
    unsigned long long *ring_d = nullptr;  // ring [3K] + barrier word
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

const void *kernel_for(bool cluster, bool smem_states) {
    if (cluster) return smem_states ? (const void *)k_train_cluster<true> : (const void *)k_train_cluster<false>;
    return smem_states ? (const void *)k_train_grid<true> : (const void *)k_train_grid<false>;
}

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
    if (n_cta <= 0) n_cta = work <= 65536 ? 1 : (work <= (64LL << 20) ? 16 : sms);
    n_cta = std::max(1, std::min(n_cta, C));
    if (n_cta > 16 && n_cta > sms) n_cta = sms;
    const bool cluster = n_cta <= 16;
    if (threads <= 0) threads = (n_cta == 1 && work <= 16384) ? 256 : 512;
    threads = std::max(64, std::min(512, threads / 32 * 32));

    TrainK k{};
    k.C = C; k.P = P; k.K = K; k.W = W; k.Ppad = Ppad;
    k.n_blocks = (int)c.n_blocks; k.n_cta = n_cta;
    k.vec4 = (P % 4 == 0) && (reinterpret_cast<uintptr_t>(states) % 4 == 0);
    k.budget = c.budget; k.T = c.threshold;
    k.fp = make_fb_params(c.s, c.boost, c.state_min, c.state_max);
    k.fb_seed = derive_stream(c.seed, 0xFEED);
    per_cta_maxima(k);
    if (cluster && k.cmax > 32 * 1024)
        return fail(TMB_E_UNSUPPORTED, "trainer_create: too many clauses per CTA");

    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t need_on = smem_layout(k, true, cluster, nullptr, nullptr);
    const size_t need_off = smem_layout(k, false, cluster, nullptr, nullptr);
    // flags bit 0 forces HBM-resident states (tests the streaming path)
    const int smem_states = (need_on <= (size_t)max_smem && !(c.flags & 1)) ? 1 : 0;
    const size_t need = smem_states ? need_on : need_off;
    if (need > (size_t)max_smem)
        return fail(TMB_E_UNSUPPORTED,
                    "trainer_create: per-CTA include masks exceed shared memory (" +
                        std::to_string(need) + " B); use more CTAs");
    const void *fn = kernel_for(cluster, smem_states);
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

    tmb_trainer *t = new tmb_trainer();
    t->cfg = c;
    t->states = states; t->weights = weights; t->block_counters = block_counters;
    t->n_cta = n_cta; t->threads = threads; t->smem = (int)need;
    t->smem_states = smem_states; t->cluster = cluster;
    std::vector<uint64_t> seeds(c.n_blocks);
    for (int64_t b = 0; b < c.n_blocks; ++b) seeds[b] = derive_stream(c.seed, (uint64_t)b);
    if ((rc = check_cuda(cudaMalloc(&t->block_seeds_d, 8 * c.n_blocks), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&t->ring_d, 8 * (3 * K + 2)), "cudaMalloc")) ||
        (rc = check_cuda(cudaMemcpy(t->block_seeds_d, seeds.data(), 8 * c.n_blocks,
                                    cudaMemcpyHostToDevice), "cudaMemcpy"))) {
        tmb_trainer_destroy(t);
        return rc;
    }
    k.block_seeds = t->block_seeds_d;
    k.ring = t->ring_d;
    k.bar = reinterpret_cast<unsigned *>(t->ring_d + 3 * K);
    k.states = states; k.weights = weights; k.block_counters = block_counters;
    t->k = k;
    *out = t;
    return TMB_OK;
}

int tmb_trainer_destroy(tmb_trainer *t) {
    if (!t) return TMB_OK;
    if (t->block_seeds_d) cudaFree(t->block_seeds_d);
    if (t->ring_d) cudaFree(t->ring_d);
    delete t;
    return TMB_OK;
}

int tmb_trainer_info(const tmb_trainer *t, int *n_cta, int *threads, int *smem_bytes,
                     int *states_in_smem) {
    if (!t) return fail(TMB_E_INVALID, "trainer_info: NULL");
    if (n_cta) *n_cta = t->n_cta;
    if (threads) *threads = t->threads;
    if (smem_bytes) *smem_bytes = t->smem;
    if (states_in_smem) *states_in_smem = t->smem_states;
    return TMB_OK;
}

int tmb_trainer_run(tmb_trainer *t, const uint32_t *lit_words, const int32_t *labels,
                    const int32_t *order, int64_t n_steps, uint64_t fb_counter,
                    tmb_train_stats *stats, void *stream) {
    if (!t) return fail(TMB_E_INVALID, "trainer_run: NULL trainer");
    if (n_steps <= 0) return TMB_OK;
    if (!lit_words || !labels || !order) return fail(TMB_E_INVALID, "trainer_run: NULL data");
    if (n_steps > (int64_t)(0xFFFFFFFFu / (unsigned)t->n_cta) - 1)
        return fail(TMB_E_UNSUPPORTED, "trainer_run: split runs longer than 2^32/n_cta steps");
    cudaStream_t st = as_stream(stream);
    TrainK k = t->k;
    k.lit_words = lit_words; k.labels = labels; k.order = order;
    k.n_steps = n_steps; k.fb_counter0 = fb_counter; k.stats = stats;
    void *args[] = {&k};
    const void *fn = kernel_for(t->cluster, t->smem_states);
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
    } else {
        TMB_CUDA(cudaMemsetAsync(t->ring_d, 0, 8 * (3 * k.K + 2), st));
        TMB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(t->n_cta), dim3(t->threads), args,
                                             (size_t)t->smem, st));
    }
    TMB_LAUNCHED();
    return TMB_OK;
}

}  // extern "C"
