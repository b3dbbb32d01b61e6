// tmb_train.cu -- the fused, persistent Coalesced-TM training kernel.
//
// One cooperative launch runs a whole epoch (or any run of consecutive
// examples) of executor.train's per-example loop (executor.py:275-340):
//
//   eval_block   (dense.py:147-154, kernels/_numba.py:36-58)  -> per-CTA clause
//                outputs + partial class sums
//   grid-wide vote all-reduce (votes summed over ALL blocks, executor.py:303)
//   decide       (feedback.py:33-53) -- recomputed redundantly by every CTA
//                from random-access feedback-stream draws; no second sync
//   update_block (kernels/_numba.py:101-125) -- event windows from an
//                on-chip scan of the update flags, Type I / II per literal
//                position, weights +-1
//
// Layout: CTA b owns a contiguous clause range [c0, c1).  Its include
// bitmasks (and, when they fit, its int8 TA states) live in shared memory for
// the whole launch; weights are in shared memory.  Literal rows are
// pre-packed bit vectors in HBM (L2-resident).  The only cross-CTA traffic
// per example is K int64 atomics + one barrier arrival.
#include <algorithm>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"

namespace tmb {

struct TrainK {
    int C, P, K, W, Ppad, n_blocks, n_cta, cmax, fmax_words, bmax;
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
    unsigned long long *ring;  // [3][K]
    unsigned int *bar;
    tmb_train_stats *stats;
};

// executor.py:36-47 partition: block of clause c and block start.
__device__ __forceinline__ int block_of(int c, int C, int nb) {
    int base = C / nb, extra = C % nb;
    int big = extra * (base + 1);
    return c < big ? c / (base + 1) : extra + (c - big) / base;
}
__device__ __forceinline__ int block_begin(int b, int C, int nb) {
    int base = C / nb, extra = C % nb;
    return b * base + min(b, extra);
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while ((int)(ld_acquire_u32(bar) - target) < 0) {
        }
        __threadfence();
    }
    __syncthreads();
}

struct Smem {
    uint32_t *lit, *masks, *ut_bits, *un_bits;
    int32_t *word_cum, *weights, *work, *info;
    uint64_t *sk_t, *sk_n, *blk_ctr;
    int8_t *states;
    long long *votes;  // [K] (single-CTA mode) / scratch
    int *misc;         // [0]=n_work [1]=negative
    uint64_t *thr;     // [0]=t_t [1]=t_n
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Shared-memory carve-up; identical on host (size) and device (pointers).
__host__ __device__ inline size_t smem_layout(const TrainK &k, bool smem_states, char *base,
                                              Smem *s) {
    size_t off = 0;
    auto take = [&](size_t bytes, size_t al) -> char * {
        off = align_up(off, al);
        char *p = base ? base + off : nullptr;
        off += bytes;
        return p;
    };
    Smem t;
    t.sk_t = (uint64_t *)take(8 * k.cmax, 16);
    t.sk_n = (uint64_t *)take(8 * k.cmax, 16);
    t.blk_ctr = (uint64_t *)take(8 * (k.bmax + 1), 16);
    t.thr = (uint64_t *)take(8 * 2, 16);
    t.votes = (long long *)take(8 * k.K, 16);
    t.lit = (uint32_t *)take(4 * k.W, 16);
    t.masks = (uint32_t *)take(4 * (size_t)k.cmax * k.W, 16);
    t.ut_bits = (uint32_t *)take(4 * k.fmax_words, 16);
    t.un_bits = (uint32_t *)take(4 * k.fmax_words, 16);
    t.word_cum = (int32_t *)take(4 * (k.fmax_words + 1), 16);
    t.weights = (int32_t *)take(4 * (size_t)k.cmax * k.K, 16);
    t.work = (int32_t *)take(4 * k.cmax, 16);
    t.info = (int32_t *)take(4 * k.cmax, 16);
    t.misc = (int *)take(4 * 4, 16);
    t.states = smem_states ? (int8_t *)take((size_t)k.cmax * k.Ppad, 16) : nullptr;
    if (s) *s = t;
    return align_up(off, 16);
}

enum : int { I_TEV = 1, I_NEV = 2, I_T1 = 4, I_N1 = 8, I_OUT = 16 };

template <bool SMEM_STATES>
__global__ void __launch_bounds__(1024, 1) k_train(TrainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    Smem s;
    smem_layout(k, SMEM_STATES, smem_raw, &s);
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
    const int cta = blockIdx.x;
    const int c0 = (int)((int64_t)cta * k.C / k.n_cta);
    const int c1 = (int)((int64_t)(cta + 1) * k.C / k.n_cta);
    const int cown = c1 - c0;
    const int W = k.W, Ppad = k.Ppad, P = k.P, K = k.K, C = k.C;
    // flag range: whole blocks overlapping [c0, c1)
    const int b0 = block_of(c0, C, k.n_blocks);
    const int b1 = block_of(c1 - 1, C, k.n_blocks);  // inclusive
    const int fs = block_begin(b0, C, k.n_blocks);
    const int fe = block_begin(b1 + 1, C, k.n_blocks);
    const int fsa = fs & ~31;
    const int nfw = (fe - fsa + 31) >> 5;
    const bool single = (k.n_cta == 1);

    // ---- load model slice
    for (int i = tid; i < cown * K; i += nthr) s.weights[i] = k.weights[(int64_t)c0 * K + i];
    if (SMEM_STATES) {
        for (int i = tid; i < cown * Ppad; i += nthr) {
            int j = i / Ppad, p = i - j * Ppad;
            s.states[i] = p < P ? k.states[(int64_t)(c0 + j) * P + p] : (int8_t)-1;
        }
    }
    for (int i = tid; i <= b1 - b0; i += nthr) s.blk_ctr[i] = k.block_counters[b0 + i];
    __syncthreads();
    // include masks from states: one warp per (clause, word) via ballot
    for (int it = warp; it < cown * W; it += nwarps) {
        int j = it / W, w = it - j * W;
        int p = w * 32 + lane;
        int st;
        if (SMEM_STATES) st = s.states[j * Ppad + p];
        else st = p < P ? k.states[(int64_t)(c0 + j) * P + p] : -1;
        unsigned m = __ballot_sync(0xffffffffu, st >= 0);
        if (lane == 0) s.masks[j * W + w] = m;
    }
    __syncthreads();

    uint64_t n_draws = 0, n_upd = 0, n_events = 0, n_t1 = 0, n_t2 = 0;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;

    for (int64_t i = 0; i < k.n_steps; ++i) {
        const int ex = k.order[i];
        const int label = k.labels[ex];
        const int slot = (int)(i % 3);
        const uint64_t fbc = k.fb_counter0 + (uint64_t)i * step_draws;
        // 1. literal row
        for (int w = tid; w < W; w += nthr) s.lit[w] = __ldg(&k.lit_words[(int64_t)ex * W + w]);
        if (single && tid < K) s.votes[tid] = 0;
        __syncthreads();
        // 2. training-mode outputs (kernels/_numba.py:36-50); packed into info
        for (int j = warp; j < cown; j += nwarps) {
            uint32_t viol = 0;
            int cnt = 0;
            for (int w = lane; w < W; w += 32) {
                uint32_t m = s.masks[j * W + w];
                viol |= m & ~s.lit[w];
                cnt += __popc(m);
            }
            viol = __reduce_or_sync(0xffffffffu, viol);
            cnt = __reduce_add_sync(0xffffffffu, cnt);
            if (lane == 0) s.info[j] = (viol == 0 && cnt <= k.budget) ? I_OUT : 0;
        }
        __syncthreads();
        // 3. partial class sums (dense.py:153)
        for (int kk = tid; kk < K; kk += nthr) {
            long long v = 0;
            for (int j = 0; j < cown; ++j)
                if (s.info[j] & I_OUT) v += s.weights[j * K + kk];
            if (single) s.votes[kk] = v;
            else if (v) atomicAdd(&k.ring[slot * K + kk], (unsigned long long)v);
        }
        // 4. grid-wide all-reduce point
        if (!single) grid_sync(k.bar, (unsigned)((i + 1) * k.n_cta));
        else __syncthreads();
        // 5. decision (feedback.py:33-44), identical in every CTA
        if (tid == 0) {
            double u = u01_from53(draw53(k.fb_seed, fbc));
            int neg = (int)((label + 1 + (int64_t)(u * (double)(K - 1))) % K);
            long long vl, vn;
            if (single) {
                vl = s.votes[label];
                vn = s.votes[neg];
            } else {
                vl = (long long)__ldcg(&k.ring[slot * K + label]);
                vn = (long long)__ldcg(&k.ring[slot * K + neg]);
            }
            long long T = k.T;
            long long cl = vl < -T ? -T : (vl > T ? T : vl);
            long long cn = vn < -T ? -T : (vn > T ? T : vn);
            double pt = (double)(T - cl) / (2.0 * (double)T);
            double pn = (double)(T + cn) / (2.0 * (double)T);
            s.thr[0] = prob_threshold(pt);
            s.thr[1] = prob_threshold(pn);
            s.misc[1] = neg;
            s.misc[0] = 0;
        }
        if (!single && cta == 0 && tid < K) k.ring[((i + 2) % 3) * K + tid] = 0ull;
        __syncthreads();
        const int neg = s.misc[1];
        const uint64_t t_t = s.thr[0], t_n = s.thr[1];
        // 6. update flags for the clause range [fs, fe) (feedback.py:47-53)
        for (int idx = tid; idx < nfw * 32; idx += nthr) {
            int j = fsa + idx;
            bool valid = j >= fs && j < fe;
            bool bt = valid && draw53(k.fb_seed, fbc + 1 + (uint64_t)j) < t_t;
            bool bn = valid && draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)j) < t_n;
            unsigned wt = __ballot_sync(0xffffffffu, bt);
            unsigned wn = __ballot_sync(0xffffffffu, bn);
            if (lane == 0) {
                s.ut_bits[idx >> 5] = wt;
                s.un_bits[idx >> 5] = wn;
            }
        }
        __syncthreads();
        // 7. exclusive prefix of events per flag word
        if (warp == 0) {
            int carry = 0;
            for (int base = 0; base < nfw; base += 32) {
                int w = base + lane;
                int v = w < nfw ? __popc(s.ut_bits[w]) + __popc(s.un_bits[w]) : 0;
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
            int q = (x - fsa) >> 5, r = (x - fsa) & 31;
            int v = s.word_cum[q];
            if (r) {
                unsigned lo = (1u << r) - 1u;
                v += __popc(s.ut_bits[q] & lo) + __popc(s.un_bits[q] & lo);
            }
            return v;
        };
        // 8. per own clause: window ordinals, event types, weights
        for (int j = tid; j < cown; j += nthr) {
            int c = c0 + j;
            int q = (c - fsa) >> 5, r = (c - fsa) & 31;
            bool t_ev = (s.ut_bits[q] >> r) & 1, n_ev = (s.un_bits[q] >> r) & 1;
            int info = s.info[j] & I_OUT;
            if (t_ev || n_ev) {
                int b = block_of(c, C, k.n_blocks);
                int bs = block_begin(b, C, k.n_blocks);
                uint64_t ord = s.blk_ctr[b - b0] + (uint64_t)(cum(c) - cum(bs));
                uint64_t bseed = k.block_seeds[b];
                bool out = info & I_OUT;
                int32_t *w = s.weights + j * K;
                bool t1 = w[label] >= 0, n1 = w[neg] < 0;
                if (t_ev) {
                    info |= I_TEV | (t1 ? I_T1 : 0);
                    s.sk_t[j] = bseed + kGolden * ((ord << 32) + 1);
                    ++n_events;
                    if (t1) ++n_t1; else if (out) ++n_t2;
                }
                if (n_ev) {
                    uint64_t o2 = ord + (t_ev ? 1 : 0);
                    info |= I_NEV | (n1 ? I_N1 : 0);
                    s.sk_n[j] = bseed + kGolden * ((o2 << 32) + 1);
                    ++n_events;
                    if (n1) ++n_t1; else if (out) ++n_t2;
                }
                if (out) {
                    if (t_ev) w[label] += 1;
                    if (n_ev) w[neg] -= 1;
                }
                bool work = (t_ev && ((info & I_T1) || out)) || (n_ev && ((info & I_N1) || out));
                if (work) {
                    int slotw = atomicAdd(&s.misc[0], 1);
                    s.work[slotw] = j;
                }
            }
            s.info[j] = info;
        }
        __syncthreads();
        // 9a. advance the local block counters (one window per applied event)
        for (int bi = tid; bi <= b1 - b0; bi += nthr) {
            int bs = block_begin(b0 + bi, C, k.n_blocks);
            int be = block_begin(b0 + bi + 1, C, k.n_blocks);
            s.blk_ctr[bi] += (uint64_t)(cum(be) - cum(bs));
        }
        // 9b. per-position Type I / II (kernels/_numba.py:71-98), masks by ballot
        const int n_work = s.misc[0];
        const int total = n_work * Ppad;
        int wc = tid / Ppad, p = tid - (tid / Ppad) * Ppad;
        for (int it = tid; it < total; it += nthr) {
            const int j = s.work[wc];
            const int info = s.info[j];
            const int out = (info & I_OUT) ? 1 : 0;
            int st, st0;
            int8_t *gp = nullptr;
            if (SMEM_STATES) {
                st = s.states[j * Ppad + p];
            } else {
                gp = k.states + (int64_t)(c0 + j) * P + p;
                st = p < P ? *gp : -1;
            }
            st0 = st;
            if (p < P) {
                const int lit = (s.lit[p >> 5] >> (p & 31)) & 1;
                if (info & I_TEV) {
                    if (info & I_T1) st = type_i_stream(st, lit, out, k.fp, s.sk_t[j], (uint32_t)p, n_draws);
                    else st = type_ii(st, lit, out);
                }
                if (info & I_NEV) {
                    if (info & I_N1) st = type_i_stream(st, lit, out, k.fp, s.sk_n[j], (uint32_t)p, n_draws);
                    else st = type_ii(st, lit, out);
                }
                if (st != st0) {
                    ++n_upd;
                    if (SMEM_STATES) s.states[j * Ppad + p] = (int8_t)st;
                    else *gp = (int8_t)st;
                }
            }
            unsigned m = __ballot_sync(0xffffffffu, p < P && st >= 0);
            if (lane == 0) s.masks[j * W + (p >> 5)] = m;
            p += nthr;
            while (p >= Ppad) {
                p -= Ppad;
                ++wc;
            }
        }
        __syncthreads();
    }

    // ---- write back the model slice and counters
    for (int i = tid; i < cown * K; i += nthr) k.weights[(int64_t)c0 * K + i] = s.weights[i];
    if (SMEM_STATES) {
        for (int i = tid; i < cown * Ppad; i += nthr) {
            int j = i / Ppad, p = i - j * Ppad;
            if (p < P) k.states[(int64_t)(c0 + j) * P + p] = s.states[i];
        }
    }
    for (int bi = tid; bi <= b1 - b0; bi += nthr) {
        int b = b0 + bi;
        int last = block_begin(b + 1, C, k.n_blocks) - 1;
        if (last >= c0 && last < c1) k.block_counters[b] = s.blk_ctr[bi];
    }
    if (k.stats) {
        // warp-aggregate then one atomic per warp
        for (int o = 16; o; o >>= 1) {
            n_draws += __shfl_xor_sync(0xffffffffu, n_draws, o);
            n_upd += __shfl_xor_sync(0xffffffffu, n_upd, o);
            n_events += __shfl_xor_sync(0xffffffffu, n_events, o);
            n_t1 += __shfl_xor_sync(0xffffffffu, n_t1, o);
            n_t2 += __shfl_xor_sync(0xffffffffu, n_t2, o);
        }
        if (lane == 0) {
            atomicAdd((unsigned long long *)&k.stats->draws, (unsigned long long)n_draws);
            atomicAdd((unsigned long long *)&k.stats->state_updates, (unsigned long long)n_upd);
            atomicAdd((unsigned long long *)&k.stats->events, (unsigned long long)n_events);
            atomicAdd((unsigned long long *)&k.stats->type_i, (unsigned long long)n_t1);
            atomicAdd((unsigned long long *)&k.stats->type_ii, (unsigned long long)n_t2);
        }
        if (cta == 0 && tid == 0)
            atomicAdd((unsigned long long *)&k.stats->examples, (unsigned long long)k.n_steps);
    }
}

}  // namespace tmb

using namespace tmb;

struct tmb_trainer {
    tmb_train_cfg cfg;
    int8_t *states;
    int32_t *weights;
    uint64_t *block_counters;
    int n_cta, threads, smem, smem_states;
    TrainK k;
    uint64_t *block_seeds_d = nullptr;
    unsigned long long *ring_d = nullptr;  // ring [3K] + barrier word
};

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
    const int W = (P + 31) / 32, Ppad = W * 32;
    int sms = sm_count();
    if (n_cta <= 0) {
        int64_t work = (int64_t)C * Ppad;
        n_cta = work <= 65536 ? 1 : std::min<int64_t>(sms, C);
    }
    n_cta = std::max(1, std::min(n_cta, C));
    if (threads <= 0) threads = (n_cta == 1 && (int64_t)C * Ppad <= 16384) ? 256 : 512;
    threads = std::max(32, std::min(1024, threads / 32 * 32));

    TrainK k{};
    k.C = C; k.P = P; k.K = K; k.W = W; k.Ppad = Ppad;
    k.n_blocks = (int)c.n_blocks; k.n_cta = n_cta;
    k.budget = c.budget; k.T = c.threshold;
    k.fp = make_fb_params(c.s, c.boost, c.state_min, c.state_max);
    k.fb_seed = derive_stream(c.seed, 0xFEED);
    // per-CTA maxima (clause count, flag words, overlapping blocks)
    int cmax = 0, fmax = 0, bmax = 0;
    auto blk_of = [&](int cc) {
        int base = C / k.n_blocks, extra = C % k.n_blocks, big = extra * (base + 1);
        return cc < big ? cc / (base + 1) : extra + (cc - big) / base;
    };
    auto blk_begin = [&](int b) {
        int base = C / k.n_blocks, extra = C % k.n_blocks;
        return b * base + std::min(b, extra);
    };
    for (int b = 0; b < n_cta; ++b) {
        int c0 = (int)((int64_t)b * C / n_cta), c1 = (int)((int64_t)(b + 1) * C / n_cta);
        cmax = std::max(cmax, c1 - c0);
        int b0 = blk_of(c0), b1 = blk_of(c1 - 1);
        int fs = blk_begin(b0), fe = blk_begin(b1 + 1);
        fmax = std::max(fmax, (fe - (fs & ~31) + 31) / 32);
        bmax = std::max(bmax, b1 - b0 + 1);
    }
    k.cmax = cmax; k.fmax_words = fmax; k.bmax = bmax;

    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    size_t need_smem_states = smem_layout(k, true, nullptr, nullptr);
    size_t need_global = smem_layout(k, false, nullptr, nullptr);
    // cfg.reserved bit 0 forces HBM-resident states (tests the streaming path)
    int smem_states = (need_smem_states <= (size_t)max_smem && !(c.flags & 1)) ? 1 : 0;
    size_t need = smem_states ? need_smem_states : need_global;
    if (need > (size_t)max_smem)
        return fail(TMB_E_UNSUPPORTED,
                    "trainer_create: per-CTA include masks exceed shared memory (" +
                        std::to_string(need) + " B); use more CTAs");
    const void *fn = smem_states ? (const void *)k_train<true> : (const void *)k_train<false>;
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
    int per_sm = 0;
    TMB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, need));
    if (per_sm * sms < n_cta)
        return fail(TMB_E_UNSUPPORTED, "trainer_create: grid cannot be co-resident");

    tmb_trainer *t = new tmb_trainer();
    t->cfg = c;
    t->states = states; t->weights = weights; t->block_counters = block_counters;
    t->n_cta = n_cta; t->threads = threads; t->smem = (int)need; t->smem_states = smem_states;
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
    TMB_CUDA(cudaMemsetAsync(t->ring_d, 0, 8 * (3 * k.K + 2), st));
    void *args[] = {&k};
    const void *fn = t->smem_states ? (const void *)k_train<true> : (const void *)k_train<false>;
    if (t->n_cta > 1) {
        TMB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(t->n_cta), dim3(t->threads), args,
                                             (size_t)t->smem, st));
    } else {
        TMB_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(t->threads), args, (size_t)t->smem, st));
    }
    TMB_LAUNCHED();
    return TMB_OK;
}

}  // extern "C"
