// tmb_sparse.cu -- SparseTM (sparse.py:78-256) on the device.
//
// Model: per clause a sorted list of (literal int32, state int8) pairs in a
// fixed-capacity slab (double-buffered: an event writes the other buffer),
// weights int32 [C, K], per-block event counters.  Documents are CSR
// (indptr int64 [N+1], indices int32 sorted per row).
//
// Training (executor.py:275-340 with the sparse banks): one cooperative grid
// launch per run of examples with the dense trainer's fence-free vote
// exchange and flag scan (tmb_train.cu), and per event a warp-parallel merge:
//   Type I  over stored U active     (sparse.py:162-190), draw per literal INDEX
//   Type II over stored U candidates (sparse.py:192-210), output 1 only
//   keep rule (sparse.py:212-220): drop st <= floor; an insertion (literal not
//   stored) is dropped iff >= capacity pairs were emitted before it.  Every
//   condition-true element before position i is emitted unless it is a
//   dropped insertion, and insertions are only dropped once that count has
//   reached the capacity, so the sequential rule equals the parallel prefix
//   rule  keep_i = cond_i && (stored_i || #cond_true_before_i < capacity).
// Inference: inverted index literal -> clauses, one warp per document.
#include <algorithm>
#include <cstring>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"

namespace tmb {

constexpr int kMaxActive = 4096;  // active literals of one document held in smem
constexpr int kMaxIns = 512;      // Type II insertions per event (per-warp smem)
constexpr int kCandStage = 1024;  // leading candidates held in smem (every Type II walk
                                  // starts at candidate 0 and stops at the capacity)
constexpr int kStage = 1024;      // per-warp shared staging of a clause list (longer: global)
constexpr int kPfRegs = 8;        // next document's active ids per thread (prefetch)

struct SparseK {
    int C, K, n_blocks, n_cta, cmax, fmax_words, bmax, slab;
    int64_t budget, T;
    int floor_, smax, capacity;  // capacity < 0: None
    FbParams fp;
    uint64_t fb_seed, fb_counter0;
    int64_t n_steps;
    const int64_t *indptr;
    const int32_t *indices;
    const int32_t *labels, *order;
    const int32_t *cands;
    int64_t n_cand;
    int32_t *lits0, *lits1;  // [C][slab]
    int8_t *sts0, *sts1;
    int32_t *len;
    uint8_t *cur;
    int32_t *weights;
    uint64_t *block_counters;
    const uint64_t *block_seeds;
    unsigned long long *rec;  // [n_steps][2]
    unsigned int *overflow;
    tmb_train_stats *stats;
    // explicit-flag single-example mode (SparseClauseBank.apply_feedback)
    const uint8_t *x_ut, *x_un, *x_out;
    int x_label, x_neg;
    uint64_t x_counter, x_seed;
    unsigned long long *phase;  // optional [n_cta][16] clock64 profile (see kPh* below)
};

__device__ __forceinline__ int32_t *lits_of(const SparseK &k, int c, int which) {
    return (which ? k.lits1 : k.lits0) + (size_t)c * k.slab;
}
__device__ __forceinline__ int8_t *sts_of(const SparseK &k, int c, int which) {
    return (which ? k.sts1 : k.sts0) + (size_t)c * k.slab;
}

// number of elements < v in sorted a[0..n), when the answer is usually 0:
// one probe, then a binary search (warp-uniform v: broadcast loads)
__device__ __forceinline__ int count_below_gallop(const int32_t *a, int n, int32_t v) {
    if (n <= 0 || a[0] >= v) return 0;
    int lo = 1, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// number of elements < v in sorted a[0..n)
__device__ __forceinline__ int count_below(const int32_t *a, int n, int32_t v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] < v) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ bool contains(const int32_t *a, int n, int32_t v) {
    const int p = count_below(a, n, v);
    return p < n && a[p] == v;
}

// warp-wide exclusive scan of a 0/1 flag; *tot = warp total (one ballot)
__device__ __forceinline__ int warp_excl(int f, int lane, int *tot) {
    const unsigned b = __ballot_sync(0xffffffffu, f != 0);
    *tot = __popc(b);
    return __popc(b & ((1u << lane) - 1u));
}

// Type I on clause c (one warp): domain = stored U active, merged by a merge
// path (stored first on ties; the active duplicate of a stored literal is
// skipped).  Returns the new length in the other buffer, -1 on slab overflow.
// Copy the clause's list into the warp's shared staging buffers (the merge
// path's binary searches then hit shared memory, not L2); returns the
// pointers to use.
__device__ __forceinline__ void stage_list(const int32_t *L, const int8_t *S, int n, int32_t *sL,
                                           int8_t *sS, int lane, const int32_t *&Lp,
                                           const int8_t *&Sp) {
    if (n <= kStage) {
        for (int q = lane; q < n; q += 32) {
            sL[q] = L[q];
            sS[q] = S[q];
        }
        __syncwarp();
        Lp = sL;
        Sp = sS;
    } else {
        Lp = L;
        Sp = S;
    }
}

// Warp-wide ranks in a sorted 32-window held one value per lane (v): the
// number of lanes whose v is < x (or <= x), by binary lifting over shuffles.
__device__ __forceinline__ int window_rank_lt(int32_t v, int32_t x) {
    int r = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1)
        if (__shfl_sync(0xffffffffu, v, r + step - 1) < x) r += step;
    if (__shfl_sync(0xffffffffu, v, r) < x) r += 1;
    return r;
}
__device__ __forceinline__ int window_rank_le(int32_t v, int32_t x) {
    int r = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1)
        if (__shfl_sync(0xffffffffu, v, r + step - 1) <= x) r += step;
    if (__shfl_sync(0xffffffffu, v, r) <= x) r += 1;
    return r;
}

// L/S: the clause's current list (n pairs), DL/DS: the other buffer;
// scratch: 32 x u64 of warp-private shared memory.
//
// The merged sequence (stored first on ties) is walked 32 positions per
// round.  A round's positions come from the next 32 stored and the next 32
// active elements (windows loaded one per lane); each element's position in
// the round is its window index plus its rank in the other window (two
// interleaved 6-step shuffle searches), and the elements that land in
// [0, 32) are scattered through `scratch` to the lane of their position.
__device__ __forceinline__ int event_type_i(const SparseK &k, const int32_t *L, const int8_t *S,
                                            int n, int32_t *DL, int8_t *DS, const int32_t *act,
                                            int n_act, int out, uint64_t sk, int lane,
                                            uint64_t &ndraws, uint64_t *scratch) {
    constexpr int32_t kInf = 0x7fffffff;
    const int total = n + n_act;
    int emitted = 0, cond_before = 0;
    if (out == 0) {
        // Type Ib: every element can only move down, so an active literal that
        // is not stored (state = floor) is never kept and its draw cannot
        // matter; the merge reduces to a pass over the stored pairs, in
        // order, each kept iff it stays above the floor.
        for (int base = 0; base < n; base += 32) {
            const int i = base + lane;
            bool keep = false;
            int32_t lit = 0;
            int st = 0;
            if (i < n) {
                lit = L[i];
                st = S[i];
                const uint64_t m = mix64(sk + kGolden * (uint64_t)(uint32_t)lit) >> 11;
                ++ndraws;
                if (m < k.fp.t_dec && st > k.floor_) st -= 1;
                keep = st > k.floor_;
            }
            int ktot;
            const int kpre = warp_excl(keep ? 1 : 0, lane, &ktot) + emitted;
            if (keep && kpre < k.slab) {
                DL[kpre] = lit;
                DS[kpre] = (int8_t)st;
            }
            emitted += ktot;
        }
        return emitted <= k.slab ? emitted : -1;
    }
    // 64 merged positions per round: stored / active windows of 64 held as two
    // registers per lane (A = window[lane], B = window[32 + lane]); the rank of
    // a value in a 64-window is the sum of its ranks in the two halves, so the
    // eight shuffle searches of a round are independent and overlap.
    int i0 = 0, a0 = 0;
    int32_t prev_stored = -1;  // last stored literal consumed by earlier rounds
    const unsigned lt = (1u << lane) - 1u;
    for (int base = 0; base < total; base += 64) {
        const int lim = min(64, total - base);
        int32_t lw[2], aw[2];
        int sw[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int li = i0 + 32 * h + lane, ai = a0 + 32 * h + lane;
            lw[h] = li < n ? L[li] : kInf;
            sw[h] = li < n ? (int)S[li] : 0;
            aw[h] = ai < n_act ? act[ai] : kInf;
        }
        int pl[2], pa[2];
        bool l_act[2], a_dup[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int ra = window_rank_lt(aw[0], lw[h]) + window_rank_lt(aw[1], lw[h]);
            const int rl = window_rank_le(lw[0], aw[h]) + window_rank_le(lw[1], aw[h]);
            const int32_t a0v = __shfl_sync(0xffffffffu, aw[0], ra & 31);
            const int32_t a1v = __shfl_sync(0xffffffffu, aw[1], ra & 31);
            const int32_t l0v = __shfl_sync(0xffffffffu, lw[0], (rl - 1) & 31);
            const int32_t l1v = __shfl_sync(0xffffffffu, lw[1], (rl - 1) & 31);
            l_act[h] = ra < 64 && (ra < 32 ? a0v : a1v) == lw[h];
            a_dup[h] = (rl == 0 ? prev_stored : (rl <= 32 ? l0v : l1v)) == aw[h];
            pl[h] = 32 * h + lane + ra;
            pa[h] = 32 * h + lane + rl;
        }
        // entry: lit << 32 | flags << 8 | (u8)state; flags 1 stored, 2 active, 4 duplicate
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (pl[h] < lim)
                scratch[pl[h]] = ((uint64_t)(uint32_t)lw[h] << 32) |
                                 ((1u | (l_act[h] ? 2u : 0u)) << 8) | (uint32_t)(sw[h] & 0xff);
            if (pa[h] < lim)
                scratch[pa[h]] = ((uint64_t)(uint32_t)aw[h] << 32) | ((2u | (a_dup[h] ? 4u : 0u)) << 8);
        }
        const int nl = __popc(__ballot_sync(0xffffffffu, pl[0] < lim)) +
                       __popc(__ballot_sync(0xffffffffu, pl[1] < lim));
        const int na = __popc(__ballot_sync(0xffffffffu, pa[0] < lim)) +
                       __popc(__ballot_sync(0xffffffffu, pa[1] < lim));
        {
            const int32_t p0 = __shfl_sync(0xffffffffu, lw[0], (nl - 1) & 31);
            const int32_t p1 = __shfl_sync(0xffffffffu, lw[1], (nl - 1) & 31);
            if (nl > 0) prev_stored = nl <= 32 ? p0 : p1;
        }
        __syncwarp();
        int32_t lit[2];
        int st[2];
        bool stored[2];
        unsigned cm[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int pos = 32 * h + lane;
            bool valid = pos < lim, active = false;
            lit[h] = 0;
            st[h] = k.floor_;
            stored[h] = false;
            if (valid) {
                const uint64_t e = scratch[pos];
                const unsigned fl = (unsigned)(e >> 8) & 0xffu;
                lit[h] = (int32_t)(e >> 32);
                stored[h] = fl & 1u;
                active = fl & 2u;
                if (stored[h]) st[h] = (int)(int8_t)(e & 0xffu);
                if (fl & 4u) valid = false;  // active duplicate of a stored literal
            }
            bool cond = false;
            if (valid) {
                const uint64_t m = mix64(sk + kGolden * (uint64_t)(uint32_t)lit[h]) >> 11;
                ++ndraws;
                if (active) {  // output 1
                    if ((k.fp.boost || m < k.fp.t_inc) && st[h] < k.smax) st[h] += 1;
                } else if (m < k.fp.t_dec && st[h] > k.floor_) {
                    st[h] -= 1;
                }
                cond = st[h] > k.floor_;
            }
            cm[h] = __ballot_sync(0xffffffffu, cond);
        }
        __syncwarp();
        i0 += nl;
        a0 += na;
        // keep_i = cond_i && (stored_i || #cond_true_before_i < capacity)
        int cpre = cond_before, kpre = emitted;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const bool cond = (cm[h] >> lane) & 1u;
            const int my_c = cpre + __popc(cm[h] & lt);
            const bool keep = cond && (stored[h] || k.capacity < 0 || my_c < k.capacity);
            const unsigned km = __ballot_sync(0xffffffffu, keep);
            const int my_k = kpre + __popc(km & lt);
            if (keep && my_k < k.slab) {
                DL[my_k] = lit[h];
                DS[my_k] = (int8_t)st[h];
            }
            cpre += __popc(cm[h]);
            kpre += __popc(km);
        }
        emitted = kpre;
        cond_before = cpre;
    }
    return emitted <= k.slab ? emitted : -1;
}

// Type II, output 1 (one warp): every stored pair survives (states only move
// up from above the floor); inserted = the first non-stored, non-active
// candidates x with #stored(<x) + #inserted(<x) < capacity, at floor + 1.
//
// Candidates, stored literals and active literals are all sorted, so each
// round of 32 candidates finds its place in L and act with one uniform
// (broadcast) binary search for the round's first candidate plus
// shuffle ranks inside the 32-wide windows that follow; a lane whose
// candidate lies beyond its window (more than 32 stored / active literals
// inside one candidate round) falls back to a binary search.
__device__ __forceinline__ int event_type_ii(const SparseK &k, const int32_t *L, const int8_t *S,
                                             int n, int32_t *DL, int8_t *DS, const int32_t *act,
                                             int n_act, int32_t *ins_buf, int ins_cap,
                                             const int32_t *cand_s, int lane,
                                             unsigned long long *pc) {
    constexpr int32_t kInf = 0x7fffffff;
    const int cap = k.capacity;
    int ins = 0;
    bool overflow = false;
    long long t0 = pc ? clock64() : 0;
    int i_lo = 0, a_lo = 0;  // stored / active literals below the round's first candidate
    for (int64_t cb = 0; cb < k.n_cand; cb += 32) {
        const int64_t ci = cb + lane;
        const bool real = ci < k.n_cand;
        const int32_t x = real ? (ci < kCandStage ? cand_s[ci] : __ldg(&k.cands[ci])) : kInf;
        const int32_t x0 = __shfl_sync(0xffffffffu, x, 0);
        i_lo += count_below_gallop(L + i_lo, n - i_lo, x0);
        a_lo += count_below_gallop(act + a_lo, n_act - a_lo, x0);
        const int32_t lw = i_lo + lane < n ? L[i_lo + lane] : kInf;
        const int32_t aw = a_lo + lane < n_act ? act[a_lo + lane] : kInf;
        const int rl = window_rank_lt(lw, x), ra = window_rank_lt(aw, x);
        const int32_t l_at = __shfl_sync(0xffffffffu, lw, rl & 31);
        const int32_t a_at = __shfl_sync(0xffffffffu, aw, ra & 31);
        int below = i_lo + rl;
        bool stored_eq = rl < 32 && l_at == x, in_act = ra < 32 && a_at == x;
        if (real && rl == 32) {
            below += count_below(L + below, n - below, x);
            stored_eq = below < n && L[below] == x;
        }
        if (real && ra == 32) in_act = contains(act + a_lo + 32, n_act - a_lo - 32, x);
        const bool cand = real && !stored_eq && !in_act;
        int ctot, ktot;
        const int cpre = warp_excl(cand ? 1 : 0, lane, &ctot) + ins;
        const bool keep = cand && (cap < 0 || below + cpre < cap);
        const unsigned fail = __ballot_sync(0xffffffffu, cand && !keep);
        const int kpre = warp_excl(keep ? 1 : 0, lane, &ktot) + ins;
        if (keep) {
            if (kpre < ins_cap) ins_buf[kpre] = x;
            else overflow = true;
        }
        ins += ktot;
        if (pc) pc[0] += 1;
        if (fail) break;  // monotone: every later candidate fails as well
        // the next round starts past this round's last candidate (lower bounds)
        i_lo = __shfl_sync(0xffffffffu, below + (stored_eq ? 1 : 0), 31);
        a_lo = __shfl_sync(0xffffffffu, a_lo + ra + (in_act ? 1 : 0), 31);
    }
    if (pc) {
        const long long t1 = clock64();
        pc[1] += n;
        pc[2] += ins;
        pc[3] += t1 - t0;
    }
    __syncwarp();
    if (__any_sync(0xffffffffu, overflow) || n + ins > k.slab) return -1;
    // stored pairs: shifted by the insertions below them (window ranks as above)
    const int32_t iw = lane < ins ? ins_buf[lane] : kInf;
    a_lo = 0;
    for (int base = 0; base < n; base += 32) {
        const int i = base + lane;
        const bool real = i < n;
        const int32_t lit = real ? L[i] : kInf;
        const int32_t l0 = L[base];
        a_lo += count_below_gallop(act + a_lo, n_act - a_lo, l0);
        const int32_t aw = a_lo + lane < n_act ? act[a_lo + lane] : kInf;
        const int ra = window_rank_lt(aw, lit);
        const int32_t a_at = __shfl_sync(0xffffffffu, aw, ra & 31);
        bool in_act = ra < 32 && a_at == lit;
        if (real && ra == 32) in_act = contains(act + a_lo + 32, n_act - a_lo - 32, lit);
        const int ib = ins <= 32 ? window_rank_lt(iw, lit) : 0;
        if (real) {
            int st = S[i];
            if (st < 0 && !in_act) st += 1;
            const int pos = i + (ins <= 32 ? ib : count_below(ins_buf, ins, lit));
            DL[pos] = lit;
            DS[pos] = (int8_t)st;
        }
    }
    // insertions: shifted by the stored pairs below them
    for (int m = lane; m < ins; m += 32) {
        const int32_t x = ins_buf[m];
        const int pos = m + count_below(L, n, x);
        DL[pos] = x;
        DS[pos] = (int8_t)(k.floor_ + 1);
    }
    __syncwarp();
    return n + ins;
}

struct SSmem {
    int32_t *act;       // [2][kMaxActive] current / next document
    int32_t *cand;      // [kCandStage] leading candidates
    int32_t *stL;       // [nwarps][kStage] staged clause literals (global-list mode)
    int8_t *stS;        // [nwarps][kStage] staged clause states
    int32_t *resL;      // [cmax][2][slab] resident clause lists (resident mode)
    int8_t *resS;       // [cmax][2][slab]
    int32_t *rlen;      // [cmax]
    int32_t *rcur;      // [cmax]
    int64_t *meta;      // [3][4] prefetched document: a0, a1, label, -
    uint64_t *mscr;     // [nwarps][64] Type I merge scatter
    int32_t *ins;       // [nwarps][kMaxIns] (global-list mode; resident mode uses the
                        // source list's free tail, whose size is exactly the room left)
    uint32_t *ut_bits, *un_bits;
    int32_t *word_cum, *info, *work, *misc;
    uint64_t *sk_t, *sk_n, *blk_ctr, *blk_seed, *draw_t, *draw_n;
    long long *vsum;
};

__host__ __device__ inline size_t salign(size_t x) { return (x + 15) / 16 * 16; }

// res: every owned clause's two list buffers live in shared memory for the
// whole launch (loaded at entry, written back at exit); otherwise the lists
// stay in global memory and events stage the source list per warp.
__host__ __device__ inline size_t sparse_smem(const SparseK &k, int nwarps, bool res, char *base,
                                              SSmem *s) {
    size_t off = 0;
    auto take = [&](size_t bytes) -> char * {
        off = salign(off);
        char *p = base ? base + off : nullptr;
        off += bytes;
        return p;
    };
    SSmem t;
    t.act = (int32_t *)take(4 * 2 * kMaxActive);
    t.cand = (int32_t *)take(4 * kCandStage);
    const size_t stage = res ? 0 : (size_t)kStage * nwarps;
    const size_t rsz = res ? (size_t)k.cmax * 2 * k.slab : 0;
    t.stL = (int32_t *)take(4 * stage);
    t.stS = (int8_t *)take(stage);
    t.resL = (int32_t *)take(4 * rsz);
    t.resS = (int8_t *)take(rsz);
    t.rlen = (int32_t *)take(4 * (size_t)(res ? k.cmax : 0));
    t.rcur = (int32_t *)take(4 * (size_t)(res ? k.cmax : 0));
    t.meta = (int64_t *)take(8 * 12);
    t.mscr = (uint64_t *)take(8 * 64 * (size_t)nwarps);
    t.ins = (int32_t *)take(res ? 0 : 4 * (size_t)kMaxIns * nwarps);
    t.ut_bits = (uint32_t *)take(4 * k.fmax_words);
    t.un_bits = (uint32_t *)take(4 * k.fmax_words);
    t.word_cum = (int32_t *)take(4 * (k.fmax_words + 1));
    t.info = (int32_t *)take(4 * k.cmax);
    t.work = (int32_t *)take(4 * k.cmax);
    t.misc = (int32_t *)take(4 * 8);
    t.sk_t = (uint64_t *)take(8 * k.cmax);
    t.sk_n = (uint64_t *)take(8 * k.cmax);
    t.blk_ctr = (uint64_t *)take(8 * (k.bmax + 1));
    t.blk_seed = (uint64_t *)take(8 * (k.bmax + 1));
    t.draw_t = (uint64_t *)take(8 * 32 * (size_t)k.fmax_words);
    t.draw_n = (uint64_t *)take(8 * 32 * (size_t)k.fmax_words);
    t.vsum = (long long *)take(8 * 2);
    if (s) *s = t;
    return salign(off);
}

enum : int { SI_TEV = 1, SI_NEV = 2, SI_T1 = 4, SI_N1 = 8, SI_OUT = 16 };

// One cooperative grid; CTA b owns clauses [c0, c1).  k.x_ut != nullptr runs
// a single example with explicit outputs / flags / counter (bank-level API).
template <bool RES>
__global__ void __launch_bounds__(512, 1) k_sparse_train(SparseK k) {
    extern __shared__ __align__(16) char smem_raw[];
    SSmem s;
    const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = nthr >> 5;
    sparse_smem(k, nwarps, RES, smem_raw, &s);
    const int rank = blockIdx.x, n_cta = k.n_cta, C = k.C, K = k.K;
    const int c0 = cta_begin(rank, C, n_cta), c1 = cta_begin(rank + 1, C, n_cta);
    const int cown = c1 - c0;
    const int b0 = block_of(c0, C, k.n_blocks), b1 = block_of(c1 - 1, C, k.n_blocks);
    const int fs = block_begin(b0, C, k.n_blocks), fe = block_begin(b1 + 1, C, k.n_blocks);
    const int fsa = fs & ~31;
    const int nfw = (fe - fsa + 31) >> 5;
    const bool explicit_flags = k.x_ut != nullptr;
    for (int i = tid; i <= b1 - b0; i += nthr) {
        s.blk_ctr[i] = explicit_flags ? k.x_counter : k.block_counters[b0 + i];
        s.blk_seed[i] = explicit_flags ? k.x_seed : k.block_seeds[b0 + i];
    }
    if (tid == 0) s.misc[2] = s.misc[3] = 0;
    for (int q = tid; q < kCandStage && q < k.n_cand; q += nthr) s.cand[q] = __ldg(&k.cands[q]);  // profile: slowest warp's event cycles this step
    // clause list accessors: (literals, states, length) of local clause j's
    // current list, and the other buffer
    const int slab = k.slab;
    if (RES) {
        for (int j = warp; j < cown; j += nwarps) {
            const int c = c0 + j, src = k.cur[c], n = k.len[c];
            const int32_t *gL = lits_of(k, c, src);
            const int8_t *gS = sts_of(k, c, src);
            int32_t *rL = s.resL + (size_t)j * 2 * slab;
            int8_t *rS = s.resS + (size_t)j * 2 * slab;
            for (int q = lane; q < n; q += 32) {
                rL[q] = gL[q];
                rS[q] = gS[q];
            }
            if (lane == 0) {
                s.rlen[j] = n;
                s.rcur[j] = 0;
            }
        }
    }
    __syncthreads();
    uint64_t n_draws = 0, n_events = 0, n_t1 = 0, n_t2 = 0;
    const unsigned long long step_draws = 1ull + 2ull * (unsigned long long)C;
    const bool prof = k.phase != nullptr;
    unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // profile slots: 0-5 phases (thread 0; 15: the part of phase 0 up to the
    // next document's prefetch issue), 6 Type I (output 0) / 7 Type II /
    // 8 Type I (output 1) event cycles summed over warps, 9 output-1 Type I
    // events, 10 sum over steps of the slowest warp's event cycles
    unsigned long long ev_clk[4] = {0, 0, 0, 0};
    long long step_ev = 0;
    unsigned long long crit = 0;
    unsigned long long pc2[4] = {0, 0, 0, 0};
    long long t_mark = clock64();
#define SPH(n)                                                            \
    do {                                                                  \
        if (prof && tid == 0) {                                           \
            const long long now = clock64();                              \
            ph[n] += (unsigned long long)(now - t_mark);                  \
            t_mark = now;                                                 \
        }                                                                 \
    } while (0)
    // document pipeline: meta (range, label) two steps ahead, active ids one
    // step ahead (registers, committed to act[(it+1)&1] at the step's end)
    auto load_meta = [&](int64_t d, int slot) {
        const int ex = explicit_flags ? 0 : __ldg(&k.order[d]);
        s.meta[slot * 4 + 0] = __ldg(&k.indptr[ex]);
        s.meta[slot * 4 + 1] = __ldg(&k.indptr[ex + 1]);
        s.meta[slot * 4 + 2] = explicit_flags ? k.x_label : __ldg(&k.labels[ex]);
    };
    if (tid == 0) {
        load_meta(0, 0);
        if (k.n_steps > 1) load_meta(1, 1);
        if (k.n_steps > 2) s.meta[2 * 4 + 3] = __ldg(&k.order[2]);  // example of step 2
    }
    __syncthreads();
    {
        const int64_t a0 = s.meta[0], a1 = s.meta[1];
        const int n0 = (int)(a1 - a0 < kMaxActive ? a1 - a0 : kMaxActive);
        for (int q = tid; q < n0; q += nthr) s.act[q] = __ldg(&k.indices[a0 + q]);
    }
    for (int64_t it = 0; it < k.n_steps; ++it) {
        const int cur = (int)(it & 1);
        const int64_t a0 = s.meta[(it % 3) * 4 + 0], a1 = s.meta[(it % 3) * 4 + 1];
        // a document longer than the shared-memory stage is read in place
        // (its CSR row is sorted, like the staged copy)
        const int n_act = (int)(a1 - a0);
        const int32_t *act = n_act > kMaxActive ? k.indices + a0 : s.act + cur * kMaxActive;
        // next document's ids into registers; meta of the one after
        int32_t pf[kPfRegs];
        int n_next = 0;
        if (it + 1 < k.n_steps) {
            const int64_t b0 = s.meta[((it + 1) % 3) * 4 + 0], b1 = s.meta[((it + 1) % 3) * 4 + 1];
            n_next = (int)(b1 - b0 < kMaxActive ? b1 - b0 : kMaxActive);
#pragma unroll
            for (int r = 0; r < kPfRegs; ++r) {
                const int q = tid + r * nthr;
                if (q < n_next) pf[r] = __ldg(&k.indices[b0 + q]);
            }
        }
        // three-stage meta pipeline, no dependent load inside a step: the
        // example of step it+3, and the range / label of step it+2 (whose
        // example index was fetched one step earlier)
        int64_t nm0 = 0, nm1 = 0, nm2 = 0, nx3 = 0;
        if (tid == nthr - 1) {
            if (it + 2 < k.n_steps) {
                const int ex2 = (int)s.meta[((it + 2) % 3) * 4 + 3];
                nm0 = __ldg(&k.indptr[ex2]);
                nm1 = __ldg(&k.indptr[ex2 + 1]);
                nm2 = __ldg(&k.labels[ex2]);
            }
            if (it + 3 < k.n_steps) nx3 = __ldg(&k.order[it + 3]);
        }
        if (prof && tid == 0) {  // loop top up to here (prefetch issue) -> slot 15
            const long long now = clock64();
            ph[6] += (unsigned long long)(now - t_mark);
        }
        const uint64_t fbc = k.fb_counter0 + (uint64_t)it * step_draws;
        int label, neg;
        if (explicit_flags) {
            label = k.x_label;
            neg = k.x_neg;
        } else {
            label = (int)s.meta[(it % 3) * 4 + 2];
            const double u = u01_from53(draw53(k.fb_seed, fbc));
            neg = label + 1 + (int)(u * (double)(K - 1));
            if (neg >= K) neg -= K;
        }
        if (tid == 0) s.misc[0] = 0;
        __syncthreads();
        SPH(0);
        // 1. training-mode outputs of own clauses (sparse.py:123-138), warp
        //    per clause: included = stored with state >= 0, all must be active
        for (int j = warp; j < cown; j += nwarps) {
            const int c = c0 + j;
            int outv;
            if (explicit_flags) {
                outv = k.x_out[c];
            } else {
                const int32_t *L;
                const int8_t *S;
                int n;
                if (RES) {
                    const int b = s.rcur[j];
                    L = s.resL + ((size_t)j * 2 + b) * slab;
                    S = s.resS + ((size_t)j * 2 + b) * slab;
                    n = s.rlen[j];
                } else {
                    const int src = k.cur[c];
                    L = lits_of(k, c, src);
                    S = sts_of(k, c, src);
                    n = k.len[c];
                }
                int n_inc = 0;
                bool viol = false;
                for (int q = lane; q < n; q += 32) {
                    if (S[q] >= 0) {
                        ++n_inc;
                        if (!contains(act, n_act, L[q])) viol = true;
                    }
                }
                n_inc = __reduce_add_sync(0xffffffffu, n_inc);
                viol = __any_sync(0xffffffffu, viol);
                outv = n_inc == 0 ? 1 : ((n_inc > k.budget || viol) ? 0 : 1);
            }
            if (lane == 0) s.info[j] = outv ? SI_OUT : 0;
        }
        __syncthreads();
        SPH(1);
        uint64_t t_t = 0, t_n = 0;
        if (!explicit_flags) {
            // 2. partial sums of the label / negative class, fence-free exchange
            if (warp < 2) {
                const int kk = warp == 0 ? label : neg;
                long long v = 0;
                for (int j = lane; j < cown; j += 32)
                    if (s.info[j] & SI_OUT) v += k.weights[(size_t)(c0 + j) * K + kk];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0)
                    red_relaxed_add_u64(&k.rec[it * 2 + warp],
                                        (1ull << 40) + (unsigned long long)(v + kVoteBias));
            }
            for (int idx = tid; idx < nfw * 32; idx += nthr) {
                const int j = fsa + idx;
                s.draw_t[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)j);
                s.draw_n[idx] = draw53(k.fb_seed, fbc + 1 + (uint64_t)C + (uint64_t)j);
            }
            if (tid == 0) {
                const unsigned long long want = (unsigned long long)n_cta;
                ulonglong2 p;
                do {
                    p = ld_relaxed_v2u64(&k.rec[it * 2]);
                } while ((p.x >> 40) != want || (p.y >> 40) != want);
                const long long bias = (long long)n_cta * kVoteBias;
                s.vsum[0] = (long long)(p.x & ((1ull << 40) - 1)) - bias;
                s.vsum[1] = (long long)(p.y & ((1ull << 40) - 1)) - bias;
            }
            __syncthreads();
            SPH(2);
            const long long T = k.T, vl = s.vsum[0], vn = s.vsum[1];
            const long long cl = vl < -T ? -T : (vl > T ? T : vl);
            const long long cn2 = vn < -T ? -T : (vn > T ? T : vn);
            t_t = threshold_of(T - cl, T);
            t_n = threshold_of(T + cn2, T);
        }
        // 3. update-flag bitmaps over [fs, fe)
        for (int idx = tid; idx < nfw * 32; idx += nthr) {
            const int j = fsa + idx;
            const bool valid = j >= fs && j < fe;
            bool bt, bn;
            if (explicit_flags) {
                bt = valid && k.x_ut[j];
                bn = valid && k.x_un[j];
            } else {
                bt = valid && s.draw_t[idx] < t_t;
                bn = valid && s.draw_n[idx] < t_n;
            }
            const unsigned wt = __ballot_sync(0xffffffffu, bt);
            const unsigned wn = __ballot_sync(0xffffffffu, bn);
            if (lane == 0) {
                s.ut_bits[idx >> 5] = wt;
                s.un_bits[idx >> 5] = wn;
            }
        }
        __syncthreads();
        SPH(3);
        // 4. warp 0: event prefix, ordinals, types, weights, work list
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
            if (lane == 0) s.word_cum[nfw] = carry;
            __syncwarp();
            auto cum = [&](int x) -> int {
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
                int info = s.info[j] & SI_OUT;
                if (t_ev || n_ev) {
                    const int bi = block_of(c, C, k.n_blocks) - b0;
                    const uint64_t ord =
                        s.blk_ctr[bi] + (uint64_t)(cum(c) - cum(block_begin(b0 + bi, C, k.n_blocks)));
                    const uint64_t bseed = s.blk_seed[bi];
                    const bool out = info & SI_OUT;
                    int32_t *w = k.weights + (size_t)c * K;
                    const bool t1 = w[label] >= 0, n1 = w[neg] < 0;
                    if (t_ev) {
                        info |= SI_TEV | (t1 ? SI_T1 : 0);
                        s.sk_t[j] = bseed + kGolden * ((ord << 32) + 1);
                        ++n_events;
                        if (t1) ++n_t1; else if (out) ++n_t2;
                    }
                    if (n_ev) {
                        const uint64_t o2 = ord + (t_ev ? 1 : 0);
                        info |= SI_NEV | (n1 ? SI_N1 : 0);
                        s.sk_n[j] = bseed + kGolden * ((o2 << 32) + 1);
                        ++n_events;
                        if (n1) ++n_t1; else if (out) ++n_t2;
                    }
                    if (out) {
                        if (t_ev) w[label] += 1;
                        if (n_ev) w[neg] -= 1;
                    }
                    if ((t_ev && ((info & SI_T1) || out)) || (n_ev && ((info & SI_N1) || out)))
                        s.work[atomicAdd(&s.misc[0], 1)] = j;
                }
                s.info[j] = info;
            }
            __syncwarp();
            for (int bi = lane; bi <= b1 - b0; bi += 32) {
                const int bs = block_begin(b0 + bi, C, k.n_blocks);
                const int be = block_begin(b0 + bi + 1, C, k.n_blocks);
                s.blk_ctr[bi] += (uint64_t)(cum(be) - cum(bs));
            }
        }
        __syncthreads();
        SPH(4);
        // 5. events: warp per clause of the work list, target then negative
        const int n_work = s.misc[0];
        for (int wi = warp; wi < n_work; wi += nwarps) {
            const int j = s.work[wi];
            const int c = c0 + j;
            const int info = s.info[j];
            const int out = (info & SI_OUT) ? 1 : 0;
            int src = RES ? s.rcur[j] : k.cur[c];
            int n = RES ? s.rlen[j] : k.len[c];
            for (int ev = 0; ev < 2; ++ev) {
                const bool has = ev == 0 ? (info & SI_TEV) : (info & SI_NEV);
                if (!has) continue;
                const bool t1 = ev == 0 ? (info & SI_T1) : (info & SI_N1);
                if (!t1 && !out) continue;  // Type II on output 0: no-op (window still consumed)
                int nl;
                const long long e_t0 = prof ? clock64() : 0;
                const int32_t *L;
                const int8_t *S;
                int32_t *DL;
                int8_t *DS;
                if (RES) {
                    L = s.resL + ((size_t)j * 2 + src) * slab;
                    S = s.resS + ((size_t)j * 2 + src) * slab;
                    DL = s.resL + ((size_t)j * 2 + (src ^ 1)) * slab;
                    DS = s.resS + ((size_t)j * 2 + (src ^ 1)) * slab;
                } else {
                    stage_list(lits_of(k, c, src), sts_of(k, c, src), n,
                               s.stL + (size_t)warp * kStage, s.stS + (size_t)warp * kStage, lane,
                               L, S);
                    DL = lits_of(k, c, src ^ 1);
                    DS = sts_of(k, c, src ^ 1);
                }
                if (t1) {
                    nl = event_type_i(k, L, S, n, DL, DS, act, n_act, out,
                                      ev == 0 ? s.sk_t[j] : s.sk_n[j], lane, n_draws,
                                      s.mscr + (size_t)warp * 64);
                } else {
                    // insertion buffer: resident lists use their own slab's
                    // free tail; with a capacity <= kMaxIns the warp's shared
                    // buffer; unbounded insertions (sparse_capacity None) the
                    // unused tail of the source list's global slab.  One call
                    // site: the merge is inlined once (its code is fetched
                    // for every document)
                    int32_t *ib;
                    int icap;
                    if (RES) {
                        ib = const_cast<int32_t *>(L) + n;
                        icap = slab - n;
                    } else if (k.capacity >= 0 && k.capacity <= kMaxIns) {
                        ib = s.ins + (size_t)warp * kMaxIns;
                        icap = kMaxIns;
                    } else {
                        ib = lits_of(k, c, src) + n;
                        icap = slab - n;
                    }
                    nl = event_type_ii(k, L, S, n, DL, DS, act, n_act, ib, icap, s.cand, lane,
                                       prof ? pc2 : nullptr);
                }
                if (prof) {
                    const long long dt = clock64() - e_t0;
                    ev_clk[t1 ? (out ? 2 : 0) : 1] += (unsigned long long)dt;
                    if (t1 && out) ev_clk[3] += 1;
                    step_ev += dt;
                }
                if (nl < 0) {
                    if (lane == 0) atomicOr(k.overflow, 1u);
                    nl = 0;
                }
                __syncwarp();
                src ^= 1;
                n = nl;
                if (lane == 0) {
                    if (RES) {
                        s.rlen[j] = nl;
                        s.rcur[j] = src;
                    } else {
                        k.len[c] = nl;
                        k.cur[c] = (uint8_t)src;
                    }
                }
                __syncwarp();
            }
        }
        if (prof && lane == 0 && step_ev) atomicMax((unsigned long long *)&s.misc[2], (unsigned long long)step_ev);
        step_ev = 0;
        // commit the prefetched document (read after the next step's first
        // barrier)
#pragma unroll
        for (int r = 0; r < kPfRegs; ++r) {
            const int q = tid + r * nthr;
            if (q < n_next) s.act[(cur ^ 1) * kMaxActive + q] = pf[r];
        }
        if (tid == nthr - 1) {
            if (it + 2 < k.n_steps) {
                s.meta[((it + 2) % 3) * 4 + 0] = nm0;
                s.meta[((it + 2) % 3) * 4 + 1] = nm1;
                s.meta[((it + 2) % 3) * 4 + 2] = nm2;
            }
            // slot (it+3)%3 == it%3: this step's meta is no longer read
            if (it + 3 < k.n_steps) s.meta[((it + 3) % 3) * 4 + 3] = nx3;
        }
        __syncthreads();
        SPH(5);
        if (prof && tid == 0) {
            unsigned long long *mx = (unsigned long long *)&s.misc[2];
            crit += *mx;
            *mx = 0;
        }
    }
#undef SPH
    if (prof && tid == 0)
    {
        for (int q = 0; q < 6; ++q) k.phase[rank * 16 + q] = ph[q];
        k.phase[rank * 16 + 10] = crit;
        k.phase[rank * 16 + 15] = ph[6];
    }
    if (RES) {  // resident lists back to their global buffers (k.cur unchanged)
        for (int j = warp; j < cown; j += nwarps) {
            const int c = c0 + j, n = s.rlen[j], b = s.rcur[j], dst = k.cur[c];
            const int32_t *rL = s.resL + ((size_t)j * 2 + b) * slab;
            const int8_t *rS = s.resS + ((size_t)j * 2 + b) * slab;
            int32_t *gL = lits_of(k, c, dst);
            int8_t *gS = sts_of(k, c, dst);
            for (int q = lane; q < n; q += 32) {
                gL[q] = rL[q];
                gS[q] = rS[q];
            }
            if (lane == 0) k.len[c] = n;
        }
    }
    if (prof && lane == 0) {
        atomicAdd(&k.phase[rank * 16 + 6], ev_clk[0]);
        atomicAdd(&k.phase[rank * 16 + 7], ev_clk[1]);
        atomicAdd(&k.phase[rank * 16 + 8], ev_clk[2]);
        atomicAdd(&k.phase[rank * 16 + 9], ev_clk[3]);
        for (int q = 0; q < 4; ++q) atomicAdd(&k.phase[rank * 16 + 11 + q], pc2[q]);
    }
    for (int bi = tid; bi <= b1 - b0; bi += nthr) {
        const int b = b0 + bi;
        const int last = block_begin(b + 1, C, k.n_blocks) - 1;
        if (last >= c0 && last < c1) k.block_counters[b] = s.blk_ctr[bi];
    }
    if (k.stats) {
        for (int o = 16; o; o >>= 1) {
            n_draws += __shfl_xor_sync(0xffffffffu, n_draws, o);
            n_events += __shfl_xor_sync(0xffffffffu, n_events, o);
            n_t1 += __shfl_xor_sync(0xffffffffu, n_t1, o);
            n_t2 += __shfl_xor_sync(0xffffffffu, n_t2, o);
        }
        if (lane == 0) {
            atomicAdd((unsigned long long *)&k.stats->draws, (unsigned long long)n_draws);
            atomicAdd((unsigned long long *)&k.stats->events, (unsigned long long)n_events);
            atomicAdd((unsigned long long *)&k.stats->type_i, (unsigned long long)n_t1);
            atomicAdd((unsigned long long *)&k.stats->type_ii, (unsigned long long)n_t2);
        }
        if (rank == 0 && tid == 0)
            atomicAdd((unsigned long long *)&k.stats->examples, (unsigned long long)k.n_steps);
    }
}

// ---------------------------------------------------------- inference --
// Key-literal index (sparse.py:123-147 semantics: a clause fires in
// inference iff it has >= 1 included literal and all of them are active).
// Every clause with includes is filed under ONE of its included literals,
// its key (the one the query documents contain least often, estimated on a
// sample of them), so a document's candidates are the clauses keyed by its
// own tokens -- each clause at most once -- and each candidate is verified
// include by include against the document's sorted ids (binary search in
// global memory, L1-resident).  No per-document hit buffer, no limit on
// document length, hits or classes.  One warp per document.
struct SparseInferK {
    const int64_t *indptr;
    const int32_t *indices;
    int64_t N;
    const int32_t *key_ptr;     // [n_literals + 1]
    const int32_t *key_clause;  // clauses by key literal
    const int32_t *inc_ptr;     // [C + 1]
    const int32_t *inc_lits;    // included literals per clause, sorted
    int64_t n_literals;
    const int32_t *weights;
    int C, K;
    int64_t *votes, *pred;
    uint8_t *outputs;  // optional [N, C] inference-mode outputs
    // counting variant: the full inverted index and include counts
    const int32_t *post_ptr;     // [n_literals + 1]
    const int32_t *post_clause;  // clauses including each literal
    const int32_t *n_inc;        // [C]
    // K <= 2: the same postings as {clause, include count, w0, w1} -- one
    // 16-byte load per posting instead of three dependent gathers
    const int4 *post_ent;
    int cnt8;  // every include count <= 255: byte counters (4x the warps per SM)
};

// votes (argmax ties to the lowest class, np.argmax) of document d from the
// warp's int64 class sums; lanes stripe the classes
__device__ __forceinline__ void finish_doc(const SparseInferK &k, int64_t d, const long long *vacc,
                                           int lane) {
    long long bv = 0;
    int best = 0x7FFFFFFF;
    for (int kk = lane; kk < k.K; kk += 32) {
        const long long v = vacc[kk];
        if (k.votes) k.votes[d * k.K + kk] = v;
        if (best == 0x7FFFFFFF || v > bv) {
            bv = v;
            best = kk;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const long long ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int ob = __shfl_xor_sync(0xffffffffu, best, o);
        if (ob != 0x7FFFFFFF && (best == 0x7FFFFFFF || ov > bv || (ov == bv && ob < best))) {
            bv = ov;
            best = ob;
        }
    }
    if (lane == 0 && k.pred) k.pred[d] = best;
}

// Counting variant (clause count small enough for a per-warp counter array
// in shared memory): every (token, including clause) posting of the
// document increments the clause's counter; the posting that brings it to
// the clause's include count fires it.  Linear in the postings, no buffer.
// Class sums of fired clauses: KR > 0 (K <= KR) accumulates per lane in
// registers and reduces once per document -- a clause fires on most
// postings of a trained configs[4] model (1.2 includes per clause), and
// shared atomics from all lanes onto the same K sums serialise; KR = 0 keeps
// per-warp shared int64 sums.
template <int KR>
struct VoteAcc {
    long long r[KR > 0 ? KR : 1];
    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int kk = 0; kk < (KR > 0 ? KR : 1); ++kk) r[kk] = 0;
    }
    __device__ __forceinline__ void add(const SparseInferK &k, int c, long long *vacc) {
        const int32_t *wr = k.weights + (size_t)c * k.K;
        if (KR > 0) {
#pragma unroll
            for (int kk = 0; kk < KR; ++kk)
                if (kk < k.K) r[kk] += __ldg(&wr[kk]);
        } else {
            for (int kk = 0; kk < k.K; ++kk) {
                const int32_t wv = __ldg(&wr[kk]);
                if (wv) atomicAdd((unsigned long long *)&vacc[kk], (unsigned long long)(long long)wv);
            }
        }
    }
    // lane sums -> vacc (KR > 0); call with the whole warp
    __device__ __forceinline__ void flush(const SparseInferK &k, long long *vacc, int lane) {
        if (KR > 0) {
#pragma unroll
            for (int kk = 0; kk < KR; ++kk) {
                long long v = r[kk];
#pragma unroll
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && kk < k.K) vacc[kk] = v;
            }
        }
    }
};

template <int KR>
__global__ void __launch_bounds__(256) k_sparse_infer_count(SparseInferK k) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // counter words per warp: one per clause, or (cnt8) one byte per clause
    const int Cp = k.cnt8 ? ((k.C + 15) & ~15) / 4 : (k.C + 3) & ~3;
    uint32_t *cnt = reinterpret_cast<uint32_t *>(smem_raw) + (size_t)warp * Cp;
    long long *vacc = reinterpret_cast<long long *>(
        reinterpret_cast<uint32_t *>(smem_raw) + (size_t)nwarps * Cp) + (size_t)warp * k.K;
    auto bump = [&](int c) -> int {  // this posting's count before it
        if (k.cnt8) {
            const uint32_t sh = 8u * (uint32_t)(c & 3);
            return (int)((atomicAdd(&cnt[c >> 2], 1u << sh) >> sh) & 0xFFu);
        }
        return (int)atomicAdd(&cnt[c], 1u);
    };
    for (int64_t d = (int64_t)blockIdx.x * nwarps + warp; d < k.N; d += (int64_t)gridDim.x * nwarps) {
        const int64_t a0 = k.indptr[d], a1 = k.indptr[d + 1];
        const int32_t *doc = k.indices + a0;
        const int n = (int)(a1 - a0);
        for (int q = lane; q < Cp / 4; q += 32) reinterpret_cast<uint4 *>(cnt)[q] = make_uint4(0, 0, 0, 0);
        for (int kk = lane; kk < k.K; kk += 32) vacc[kk] = 0;
        VoteAcc<KR> acc;
        acc.clear();
        __syncwarp();
        for (int base = 0; base < n; base += 32) {
            int p0 = 0, np = 0;
            if (base + lane < n) {
                const int32_t lit = __ldg(&doc[base + lane]);
                const bool dup = base + lane > 0 && __ldg(&doc[base + lane - 1]) == lit;
                if (lit >= 0 && lit < k.n_literals && !dup) {
                    p0 = __ldg(&k.post_ptr[lit]);
                    np = __ldg(&k.post_ptr[lit + 1]) - p0;
                }
            }
            int incl = np;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            for (int s0 = 0; s0 < total; s0 += 32) {
                const int slot = s0 + lane;
                int lo = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
                    if (v <= slot) lo += step;
                }
                const int pj = __shfl_sync(0xffffffffu, p0, lo & 31);
                const int ej = __shfl_sync(0xffffffffu, incl - np, lo & 31);
                if (slot >= total) continue;
                if (KR == 2 && k.post_ent) {
                    const int4 e = __ldg(&k.post_ent[pj + slot - ej]);
                    if (bump(e.x) + 1 == e.y) {
                        acc.r[0] += e.z;
                        acc.r[KR > 1 ? 1 : 0] += e.w;
                        if (k.outputs) k.outputs[d * k.C + e.x] = 1;
                    }
                    continue;
                }
                const int c = __ldg(&k.post_clause[pj + slot - ej]);
                if (bump(c) + 1 == __ldg(&k.n_inc[c])) {
                    acc.add(k, c, vacc);
                    if (k.outputs) k.outputs[d * k.C + c] = 1;
                }
            }
        }
        __syncwarp();
        acc.flush(k, vacc, lane);
        __syncwarp();
        finish_doc(k, d, vacc, lane);
        __syncwarp();
    }
}

__device__ __forceinline__ bool doc_has(const int32_t *doc, int n, int32_t v) {
    int lo = 0, hi = n;  // first index with doc[i] >= v
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(&doc[mid]) < v) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && __ldg(&doc[lo]) == v;
}

template <int KR>
__global__ void __launch_bounds__(256) k_sparse_infer(SparseInferK k) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    long long *vacc = reinterpret_cast<long long *>(smem_raw) + (size_t)warp * k.K;
    for (int64_t d = (int64_t)blockIdx.x * nwarps + warp; d < k.N; d += (int64_t)gridDim.x * nwarps) {
        const int64_t a0 = k.indptr[d], a1 = k.indptr[d + 1];
        const int32_t *doc = k.indices + a0;
        const int n = (int)(a1 - a0);
        for (int kk = lane; kk < k.K; kk += 32) vacc[kk] = 0;
        VoteAcc<KR> acc;
        acc.clear();
        __syncwarp();
        for (int base = 0; base < n; base += 32) {
            int p0 = 0, cnt = 0;
            if (base + lane < n) {
                const int32_t lit = __ldg(&doc[base + lane]);
                // (a repeated id would make its clauses candidates twice)
                const bool dup = base + lane > 0 && __ldg(&doc[base + lane - 1]) == lit;
                if (lit >= 0 && lit < k.n_literals && !dup) {
                    p0 = __ldg(&k.key_ptr[lit]);
                    cnt = __ldg(&k.key_ptr[lit + 1]) - p0;
                }
            }
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            for (int s0 = 0; s0 < total; s0 += 32) {
                const int slot = s0 + lane;
                // owner token: the first lane whose inclusive count exceeds slot
                int lo = 0;
#pragma unroll
                for (int step = 16; step; step >>= 1) {
                    const int v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
                    if (v <= slot) lo += step;
                }
                const int j = lo;
                const int pj = __shfl_sync(0xffffffffu, p0, j & 31);
                const int ej = __shfl_sync(0xffffffffu, incl - cnt, j & 31);
                if (slot >= total) continue;
                const int c = __ldg(&k.key_clause[pj + slot - ej]);
                bool fire = true;
                for (int q = __ldg(&k.inc_ptr[c]), qe = __ldg(&k.inc_ptr[c + 1]); q < qe && fire; ++q)
                    fire = doc_has(doc, n, __ldg(&k.inc_lits[q]));
                if (fire) {
                    acc.add(k, c, vacc);
                    if (k.outputs) k.outputs[d * k.C + c] = 1;
                }
            }
        }
        __syncwarp();
        acc.flush(k, vacc, lane);
        __syncwarp();
        finish_doc(k, d, vacc, lane);
        __syncwarp();
    }
}

int g_sparse_infer_key = 0;  // tmb_set_option("sparse.infer_key"): force the key-literal kernel
int g_sparse_cnt32 = 0;      // tmb_set_option("sparse.counters32"): 32-bit clause counters
unsigned long long *g_sparse_phase = nullptr;  // tmb_set_option("sparse.phase_buffer")
int g_sparse_resident = 1;                      // tmb_set_option("sparse.resident")

}  // namespace tmb

using namespace tmb;

// compiled inference index (device arrays), see build_infer_index
struct SparseIndex {
    uint64_t version = ~0ull;
    bool counting = false;
    int cnt_warps = 0;
    int32_t *pptr = nullptr, *pcl = nullptr, *ninc = nullptr;             // counting
    int4 *pent = nullptr;                                                 // counting, K <= 2
    bool cnt8 = false;                                                    // max include count <= 255
    int32_t *kptr = nullptr, *kcl = nullptr, *iptr = nullptr, *ilit = nullptr;  // key literal
    void release() {
        for (int32_t **p : {&pptr, &pcl, &ninc, &kptr, &kcl, &iptr, &ilit}) {
            if (*p) cudaFree(*p);
            *p = nullptr;
        }
        if (pent) cudaFree(pent);
        pent = nullptr;
        version = ~0ull;
    }
    void release_after(cudaStream_t st) {  // after the kernels queued on st
        cudaStreamSynchronize(st);
        release();
    }
};

struct tmb_sparse {
    tmb_sparse_cfg cfg;
    uint64_t version = 0;  // bumped whenever the model changes (train / feedback / set)
    SparseIndex ix;
    int n_cta = 0, threads = 512;
    size_t smem = 0;
    bool resident = false;  // clause lists held in shared memory by the trainer
    int32_t *lits[2] = {nullptr, nullptr};
    int8_t *sts[2] = {nullptr, nullptr};
    int32_t *len = nullptr;
    uint8_t *cur = nullptr;
    int32_t *weights = nullptr;
    uint64_t *block_counters = nullptr, *block_seeds = nullptr;
    int32_t *cands = nullptr;
    int64_t n_cand = 0;
    unsigned long long *rec = nullptr;
    int64_t rec_cap = 0;
    unsigned int *overflow = nullptr;
    SparseK k{};
};

namespace {

int sparse_fill_k(tmb_sparse *sp) {
    const tmb_sparse_cfg &c = sp->cfg;
    SparseK &k = sp->k;
    k.C = (int)c.n_clauses;
    k.K = (int)c.n_classes;
    k.n_blocks = (int)c.n_blocks;
    k.n_cta = sp->n_cta;
    k.slab = (int)c.slab;
    k.budget = c.budget;
    k.T = c.threshold;
    k.floor_ = c.floor_;
    k.smax = c.state_max;
    k.capacity = c.capacity;
    k.fp = make_fb_params(c.s, c.boost, c.floor_, c.state_max);
    k.fb_seed = derive_stream(c.seed, 0xFEED);
    int cmax = 0, fmax = 0, bmax = 0;
    for (int b = 0; b < k.n_cta; ++b) {
        const int c0 = cta_begin(b, k.C, k.n_cta), c1 = cta_begin(b + 1, k.C, k.n_cta);
        cmax = std::max(cmax, c1 - c0);
        const int b0 = block_of(c0, k.C, k.n_blocks), b1 = block_of(c1 - 1, k.C, k.n_blocks);
        const int fs = block_begin(b0, k.C, k.n_blocks), fe = block_begin(b1 + 1, k.C, k.n_blocks);
        fmax = std::max(fmax, (fe - (fs & ~31) + 31) / 32);
        bmax = std::max(bmax, b1 - b0 + 1);
    }
    k.cmax = cmax;
    k.fmax_words = fmax;
    k.bmax = bmax;
    k.lits0 = sp->lits[0];
    k.lits1 = sp->lits[1];
    k.sts0 = sp->sts[0];
    k.sts1 = sp->sts[1];
    k.len = sp->len;
    k.cur = sp->cur;
    k.weights = sp->weights;
    k.block_counters = sp->block_counters;
    k.block_seeds = sp->block_seeds;
    k.cands = sp->cands;
    k.n_cand = sp->n_cand;
    k.overflow = sp->overflow;
    return TMB_OK;
}


int sparse_launch(tmb_sparse *sp, SparseK &k, cudaStream_t st) {
    k.phase = g_sparse_phase;
    void *args[] = {&k};
    const void *fn = sp->resident ? (const void *)k_sparse_train<true>
                                  : (const void *)k_sparse_train<false>;
    // per-function limit: another bank of a different shape may have set it
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp->smem));
    TMB_CUDA(cudaLaunchCooperativeKernel(fn, dim3(sp->n_cta),
                                         dim3(sp->threads), args, sp->smem, st));
    TMB_LAUNCHED();
    return TMB_OK;
}

int sparse_check_overflow(tmb_sparse *sp, cudaStream_t st) {
    unsigned v = 0;
    TMB_CUDA(cudaMemcpyAsync(&v, sp->overflow, 4, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaStreamSynchronize(st));
    if (v) {
        cudaMemsetAsync(sp->overflow, 0, 4, st);
        return fail(TMB_E_UNSUPPORTED,
                    std::string("sparse: ") +
                        ((v & 1) ? "a clause list exceeded the device slab (pass a larger "
                                   "slab= to the training session)" :
                                   "a document has more than 4096 active literals"));
    }
    return TMB_OK;
}

}  // namespace

extern "C" {

int tmb_sparse_create(const tmb_sparse_cfg *cfg, const int32_t *candidates, int64_t n_candidates,
                      tmb_sparse **out) {
    int rc = require_device();
    if (rc) return rc;
    if (!cfg || !out || cfg->n_clauses < 1 || cfg->n_classes < 2 || cfg->n_blocks < 1 ||
        cfg->n_blocks > cfg->n_clauses || !(cfg->s > 1.0) || cfg->slab < 8 ||
        cfg->slab > (1 << 20) || cfg->floor_ >= 0 || n_candidates < 0 ||
        (n_candidates > 0 && !candidates) || cfg->n_literals >= (1LL << 31))
        return fail(TMB_E_INVALID, "sparse_create: bad arguments");
    tmb_sparse *sp = new tmb_sparse();
    sp->cfg = *cfg;
    sp->cfg.slab = (cfg->slab + 15) / 16 * 16;
    const int64_t C = cfg->n_clauses, K = cfg->n_classes, slab = sp->cfg.slab;
    const int sms = sm_count();
    sp->n_cta = (int)std::min<int64_t>(C, sms);
    sp->threads = 512;
    auto cleanup = [&](int code) {
        tmb_sparse_destroy(sp);
        return code;
    };
    for (int b = 0; b < 2; ++b) {
        if ((rc = check_cuda(cudaMalloc(&sp->lits[b], 4 * C * slab), "cudaMalloc")) ||
            (rc = check_cuda(cudaMalloc(&sp->sts[b], C * slab), "cudaMalloc")))
            return cleanup(rc);
    }
    if ((rc = check_cuda(cudaMalloc(&sp->len, 4 * C), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->cur, C), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->weights, 4 * C * K), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->block_counters, 8 * cfg->n_blocks), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->block_seeds, 8 * cfg->n_blocks), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->cands, 4 * std::max<int64_t>(n_candidates, 1)), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&sp->overflow, 4), "cudaMalloc")))
        return cleanup(rc);
    cudaMemset(sp->len, 0, 4 * C);
    cudaMemset(sp->cur, 0, C);
    cudaMemset(sp->weights, 0, 4 * C * K);
    cudaMemset(sp->block_counters, 0, 8 * cfg->n_blocks);
    cudaMemset(sp->overflow, 0, 4);
    std::vector<uint64_t> seeds(cfg->n_blocks);
    for (int64_t b = 0; b < cfg->n_blocks; ++b) seeds[b] = derive_stream(cfg->seed, (uint64_t)b);
    cudaMemcpy(sp->block_seeds, seeds.data(), 8 * cfg->n_blocks, cudaMemcpyHostToDevice);
    if (n_candidates)
        cudaMemcpy(sp->cands, candidates, 4 * n_candidates, cudaMemcpyHostToDevice);
    sp->n_cand = n_candidates;
    if ((rc = check_cuda(cudaGetLastError(), "sparse_create"))) return cleanup(rc);
    sparse_fill_k(sp);
    int max_smem = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // resident clause lists when every CTA's share (2 buffers x slab) fits
    const size_t smem_res = sparse_smem(sp->k, sp->threads / 32, true, nullptr, nullptr);
    sp->resident = g_sparse_resident && smem_res <= (size_t)max_smem;
    sp->smem = sp->resident ? smem_res : sparse_smem(sp->k, sp->threads / 32, false, nullptr, nullptr);
    if (sp->smem > (size_t)max_smem) return cleanup(fail(TMB_E_UNSUPPORTED, "sparse: smem"));
    const void *fn = sp->resident ? (const void *)k_sparse_train<true>
                                  : (const void *)k_sparse_train<false>;
    if ((rc = check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)sp->smem), "cudaFuncSetAttribute")))
        return cleanup(rc);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, sp->threads, sp->smem);
    if (per_sm * sms < sp->n_cta) return cleanup(fail(TMB_E_UNSUPPORTED, "sparse: co-residency"));
    *out = sp;
    return TMB_OK;
}

int tmb_sparse_layout(const tmb_sparse *sp, int64_t *out4) {
    if (!sp || !out4) return fail(TMB_E_INVALID, "sparse_layout: NULL");
    out4[0] = sp->resident ? 1 : 0;
    out4[1] = sp->n_cta;
    out4[2] = sp->threads;
    out4[3] = (int64_t)sp->smem;
    return TMB_OK;
}

int tmb_sparse_destroy(tmb_sparse *sp) {
    if (sp) sp->ix.release();
    if (!sp) return TMB_OK;
    for (int b = 0; b < 2; ++b) {
        if (sp->lits[b]) cudaFree(sp->lits[b]);
        if (sp->sts[b]) cudaFree(sp->sts[b]);
    }
    for (void *p : {(void *)sp->len, (void *)sp->cur, (void *)sp->weights,
                    (void *)sp->block_counters, (void *)sp->block_seeds, (void *)sp->cands,
                    (void *)sp->rec, (void *)sp->overflow})
        if (p) cudaFree(p);
    delete sp;
    return TMB_OK;
}

int tmb_sparse_train(tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                     const int32_t *labels, const int32_t *order, int64_t n_steps,
                     uint64_t fb_counter, tmb_train_stats *stats, void *stream) {
    if (sp) ++sp->version;  // the compiled inference index is stale
    if (!sp) return fail(TMB_E_INVALID, "sparse_train: NULL");
    if (n_steps <= 0) return TMB_OK;
    if (!indptr || !indices || !labels || !order) return fail(TMB_E_INVALID, "sparse_train: NULL data");
    cudaStream_t st = as_stream(stream);
    if (sp->rec_cap < n_steps) {
        if (sp->rec) {
            cudaStreamSynchronize(st);
            cudaFree(sp->rec);
        }
        sp->rec = nullptr;
        sp->rec_cap = 0;
        TMB_CUDA(cudaMalloc(&sp->rec, 16 * (size_t)n_steps));
        sp->rec_cap = n_steps;
    }
    TMB_CUDA(cudaMemsetAsync(sp->rec, 0, 16 * (size_t)n_steps, st));
    SparseK k = sp->k;
    k.indptr = indptr; k.indices = indices; k.labels = labels; k.order = order;
    k.n_steps = n_steps; k.fb_counter0 = fb_counter; k.stats = stats; k.rec = sp->rec;
    k.x_ut = k.x_un = k.x_out = nullptr;
    int rc = sparse_launch(sp, k, st);
    if (rc) return rc;
    return sparse_check_overflow(sp, st);
}

int tmb_sparse_feedback(tmb_sparse *sp, const int32_t *active, int64_t n_active,
                        const uint8_t *outputs, int64_t label, int64_t negative,
                        const uint8_t *ut, const uint8_t *un, uint64_t stream_seed,
                        uint64_t counter, uint64_t *counter_out, void *stream) {
    if (sp) ++sp->version;  // the compiled inference index is stale
    if (!sp) return fail(TMB_E_INVALID, "sparse_feedback: NULL");
    if (sp->cfg.n_blocks != 1) return fail(TMB_E_UNSUPPORTED, "sparse_feedback: one block only");
    if (!outputs || !ut || !un || (n_active > 0 && !active) || label < 0 ||
        label >= sp->cfg.n_classes || negative < 0 || negative >= sp->cfg.n_classes)
        return fail(TMB_E_INVALID, "sparse_feedback: bad arguments");
    cudaStream_t st = as_stream(stream);
    int64_t *dptr = nullptr;
    TMB_CUDA(cudaMallocAsync(&dptr, 16, st));
    int64_t hptr[2] = {0, n_active};
    TMB_CUDA(cudaMemcpyAsync(dptr, hptr, 16, cudaMemcpyHostToDevice, st));
    SparseK k = sp->k;
    k.indptr = dptr;
    k.indices = active ? active : sp->cands;
    k.n_steps = 1;
    k.x_ut = ut; k.x_un = un; k.x_out = outputs;
    k.x_label = (int)label; k.x_neg = (int)negative; k.x_counter = counter;
    k.x_seed = stream_seed;
    k.stats = nullptr;
    uint64_t *bc = nullptr;
    TMB_CUDA(cudaMallocAsync(&bc, 8, st));
    k.block_counters = bc;  // the counter comes from x_counter, result lands here
    int rc = sparse_launch(sp, k, st);
    uint64_t res = 0;
    if (!rc) rc = check_cuda(cudaMemcpyAsync(&res, bc, 8, cudaMemcpyDeviceToHost, st), "copy");
    if (!rc) rc = sparse_check_overflow(sp, st);
    cudaFreeAsync(dptr, st);
    cudaFreeAsync(bc, st);
    cudaStreamSynchronize(st);
    if (!rc && counter_out) *counter_out = res;
    return rc;
}

int tmb_sparse_get(const tmb_sparse *sp, int32_t *lens, int32_t *lits, int8_t *states,
                   int32_t *weights, uint64_t *block_counters, void *stream) {
    if (!sp) return fail(TMB_E_INVALID, "sparse_get: NULL");
    cudaStream_t st = as_stream(stream);
    const int64_t C = sp->cfg.n_clauses, slab = sp->cfg.slab, K = sp->cfg.n_classes;
    std::vector<uint8_t> cur(C);
    std::vector<int32_t> len(C);
    TMB_CUDA(cudaMemcpyAsync(cur.data(), sp->cur, C, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaMemcpyAsync(len.data(), sp->len, 4 * C, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaStreamSynchronize(st));
    if (lens) TMB_CUDA(cudaMemcpyAsync(lens, sp->len, 4 * C, cudaMemcpyDeviceToDevice, st));
    for (int64_t c = 0; c < C; ++c) {
        const int b = cur[c];
        if (lits && len[c])
            TMB_CUDA(cudaMemcpyAsync(lits + c * slab, sp->lits[b] + c * slab, 4 * len[c],
                                     cudaMemcpyDeviceToDevice, st));
        if (states && len[c])
            TMB_CUDA(cudaMemcpyAsync(states + c * slab, sp->sts[b] + c * slab, len[c],
                                     cudaMemcpyDeviceToDevice, st));
    }
    if (weights) TMB_CUDA(cudaMemcpyAsync(weights, sp->weights, 4 * C * K, cudaMemcpyDeviceToDevice, st));
    if (block_counters)
        TMB_CUDA(cudaMemcpyAsync(block_counters, sp->block_counters, 8 * sp->cfg.n_blocks,
                                 cudaMemcpyDeviceToDevice, st));
    return TMB_OK;
}

int tmb_sparse_set(tmb_sparse *sp, const int32_t *lens, const int32_t *lits, const int8_t *states,
                   const int32_t *weights, const uint64_t *block_counters, void *stream) {
    if (sp) ++sp->version;  // the compiled inference index is stale
    if (!sp) return fail(TMB_E_INVALID, "sparse_set: NULL");
    cudaStream_t st = as_stream(stream);
    const int64_t C = sp->cfg.n_clauses, slab = sp->cfg.slab, K = sp->cfg.n_classes;
    if (lens) {
        TMB_CUDA(cudaMemcpyAsync(sp->len, lens, 4 * C, cudaMemcpyDeviceToDevice, st));
        TMB_CUDA(cudaMemsetAsync(sp->cur, 0, C, st));
    }
    if (lits) TMB_CUDA(cudaMemcpyAsync(sp->lits[0], lits, 4 * C * slab, cudaMemcpyDeviceToDevice, st));
    if (states) TMB_CUDA(cudaMemcpyAsync(sp->sts[0], states, C * slab, cudaMemcpyDeviceToDevice, st));
    if (weights) TMB_CUDA(cudaMemcpyAsync(sp->weights, weights, 4 * C * K, cudaMemcpyDeviceToDevice, st));
    if (block_counters)
        TMB_CUDA(cudaMemcpyAsync(sp->block_counters, block_counters, 8 * sp->cfg.n_blocks,
                                 cudaMemcpyDeviceToDevice, st));
    return TMB_OK;
}

// Compiled inference index of a sparse model (the included literals of
// every clause), kept in the handle and rebuilt only when the model changed
// (tmb_sparse::version) -- except the key-literal form, whose keys depend
// on the query's id frequencies and are rebuilt per call.
static int build_infer_index(tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                             int64_t N, cudaStream_t st) {
    SparseIndex &ix = sp->ix;
    const int64_t C = sp->cfg.n_clauses, slab = sp->cfg.slab, K = sp->cfg.n_classes;
    const int64_t L = sp->cfg.n_literals;
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t per_warp_cnt = 4 * (size_t)((C + 3) & ~3LL) + 8 * (size_t)K;
    const int cnt_warps =
        (int)std::min<size_t>(8, (size_t)std::min(max_smem, 200 * 1024) / per_warp_cnt);
    const bool counting = cnt_warps >= 2 && !g_sparse_infer_key;
    ix.release();
    std::vector<uint8_t> cur(C);
    std::vector<int32_t> len(C);
    TMB_CUDA(cudaMemcpyAsync(cur.data(), sp->cur, C, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaMemcpyAsync(len.data(), sp->len, 4 * C, cudaMemcpyDeviceToHost, st));
    std::vector<int32_t> sample;
    if (!counting) {  // a sample of the query's ids (up to 2^20) estimates frequencies
        int64_t ends[2] = {0, 0};
        TMB_CUDA(cudaMemcpyAsync(&ends[0], indptr, 8, cudaMemcpyDeviceToHost, st));
        TMB_CUDA(cudaMemcpyAsync(&ends[1], indptr + N, 8, cudaMemcpyDeviceToHost, st));
        TMB_CUDA(cudaStreamSynchronize(st));
        const int64_t n_sample = std::max<int64_t>(0, std::min<int64_t>(ends[1] - ends[0], 1 << 20));
        sample.resize((size_t)n_sample);
        if (n_sample)
            TMB_CUDA(cudaMemcpyAsync(sample.data(), indices + ends[0], 4 * n_sample,
                                     cudaMemcpyDeviceToHost, st));
    }
    TMB_CUDA(cudaStreamSynchronize(st));
    std::vector<int32_t> inc_ptr(C + 1, 0), inc_lits;
    {
        std::vector<int32_t> tl[2];
        std::vector<int8_t> ts[2];
        for (int b = 0; b < 2; ++b) {
            tl[b].resize(C * slab);
            ts[b].resize(C * slab);
            TMB_CUDA(cudaMemcpyAsync(tl[b].data(), sp->lits[b], 4 * C * slab, cudaMemcpyDeviceToHost, st));
            TMB_CUDA(cudaMemcpyAsync(ts[b].data(), sp->sts[b], C * slab, cudaMemcpyDeviceToHost, st));
        }
        TMB_CUDA(cudaStreamSynchronize(st));
        for (int64_t c = 0; c < C; ++c) {
            const int b = cur[c];
            for (int q = 0; q < len[c]; ++q)
                if (ts[b][c * slab + q] >= 0) inc_lits.push_back(tl[b][c * slab + q]);
            inc_ptr[c + 1] = (int32_t)inc_lits.size();
        }
    }
    int rc = TMB_OK;
    auto up = [&](int32_t **dst, const std::vector<int32_t> &v) {
        if (rc) return;
        rc = check_cuda(cudaMalloc(dst, 4 * std::max<size_t>(v.size(), 1)), "cudaMalloc");
        if (!rc && !v.empty())
            rc = check_cuda(cudaMemcpyAsync(*dst, v.data(), 4 * v.size(), cudaMemcpyHostToDevice, st), "H2D");
    };
    if (counting) {
        std::vector<int32_t> post_ptr(L + 1, 0), n_inc(C, 0);
        for (int64_t c = 0; c < C; ++c) {
            n_inc[c] = inc_ptr[c + 1] - inc_ptr[c];
            for (int32_t q = inc_ptr[c]; q < inc_ptr[c + 1]; ++q) ++post_ptr[inc_lits[q] + 1];
        }
        for (int64_t l = 0; l < L; ++l) post_ptr[l + 1] += post_ptr[l];
        std::vector<int32_t> post_clause(inc_lits.size()), fillp(post_ptr.begin(), post_ptr.end() - 1);
        for (int64_t c = 0; c < C; ++c)
            for (int32_t q = inc_ptr[c]; q < inc_ptr[c + 1]; ++q)
                post_clause[fillp[inc_lits[q]]++] = (int32_t)c;
        up(&ix.pptr, post_ptr);
        up(&ix.pcl, post_clause);
        up(&ix.ninc, n_inc);
        ix.cnt8 = C == 0 || *std::max_element(n_inc.begin(), n_inc.end()) <= 255;
        if (K <= 2) {  // packed postings {clause, include count, weights}
            std::vector<int32_t> w(C * K);
            if (!rc) rc = check_cuda(cudaMemcpyAsync(w.data(), sp->weights, 4 * C * K,
                                                     cudaMemcpyDeviceToHost, st), "D2H");
            if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "weights");
            std::vector<int4> ent(post_clause.size());
            for (size_t q = 0; q < post_clause.size(); ++q) {
                const int32_t c = post_clause[q];
                ent[q] = make_int4(c, n_inc[c], w[(size_t)c * K], K > 1 ? w[(size_t)c * K + 1] : 0);
            }
            if (!rc) rc = check_cuda(cudaMalloc(&ix.pent, 16 * std::max<size_t>(ent.size(), 1)),
                                     "cudaMalloc");
            if (!rc && !ent.empty())
                rc = check_cuda(cudaMemcpyAsync(ix.pent, ent.data(), 16 * ent.size(),
                                                cudaMemcpyHostToDevice, st), "H2D");
        }
    } else {
        // key = the included literal the sample contains least often (ties:
        // the one fewest clauses include)
        std::vector<int32_t> ids(inc_lits);
        std::sort(ids.begin(), ids.end());
        ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
        std::vector<uint32_t> freq(ids.size(), 0), n_clauses_of(ids.size(), 0);
        auto idx = [&](int32_t lit) {
            return (size_t)(std::lower_bound(ids.begin(), ids.end(), lit) - ids.begin());
        };
        for (int32_t lit : inc_lits) ++n_clauses_of[idx(lit)];
        for (int32_t v : sample) {
            const size_t i = idx(v);
            if (i < ids.size() && ids[i] == v) ++freq[i];
        }
        std::vector<std::pair<int32_t, int32_t>> keyed;
        for (int64_t c = 0; c < C; ++c) {
            if (inc_ptr[c + 1] == inc_ptr[c]) continue;  // no includes: never fires
            int32_t key = -1;
            size_t best = 0;
            for (int32_t q = inc_ptr[c]; q < inc_ptr[c + 1]; ++q) {
                const size_t i = idx(inc_lits[q]);
                if (key < 0 || freq[i] < freq[best] ||
                    (freq[i] == freq[best] && n_clauses_of[i] < n_clauses_of[best])) {
                    key = inc_lits[q];
                    best = i;
                }
            }
            keyed.emplace_back(key, (int32_t)c);
        }
        std::vector<int32_t> key_ptr(L + 1, 0), key_clause(keyed.size());
        for (auto &kc : keyed) ++key_ptr[kc.first + 1];
        for (int64_t l = 0; l < L; ++l) key_ptr[l + 1] += key_ptr[l];
        std::vector<int32_t> fillp(key_ptr.begin(), key_ptr.end() - 1);
        for (auto &kc : keyed) key_clause[fillp[kc.first]++] = kc.second;
        up(&ix.kptr, key_ptr);
        up(&ix.kcl, key_clause);
        up(&ix.iptr, inc_ptr);
        up(&ix.ilit, inc_lits);
    }
    if (!rc) rc = check_cuda(cudaStreamSynchronize(st), "index upload");
    if (rc) {
        ix.release();
        return rc;
    }
    ix.counting = counting;
    ix.cnt_warps = cnt_warps;
    ix.version = counting ? sp->version : ~0ull;
    return TMB_OK;
}

static int sparse_infer_impl(const tmb_sparse *csp, const int64_t *indptr, const int32_t *indices,
                             int64_t N, int64_t *votes, int64_t *pred, uint8_t *outputs,
                             void *stream) {
    if (!csp) return fail(TMB_E_INVALID, "sparse_infer: NULL");
    if (N < 0 || (N > 0 && (!indptr || !indices))) return fail(TMB_E_INVALID, "sparse_infer: bad args");
    if (N == 0) return TMB_OK;
    tmb_sparse *sp = const_cast<tmb_sparse *>(csp);  // the index cache only
    cudaStream_t st = as_stream(stream);
    const int64_t C = sp->cfg.n_clauses, K = sp->cfg.n_classes;
    int rc = TMB_OK;
    if (!(sp->ix.counting && sp->ix.version == sp->version && !g_sparse_infer_key))
        if ((rc = build_infer_index(sp, indptr, indices, N, st))) return rc;
    const SparseIndex &ix = sp->ix;
    SparseInferK k{};
    k.indptr = indptr; k.indices = indices; k.N = N;
    k.key_ptr = ix.kptr; k.key_clause = ix.kcl; k.inc_ptr = ix.iptr; k.inc_lits = ix.ilit;
    k.post_ptr = ix.pptr; k.post_clause = ix.pcl; k.n_inc = ix.ninc; k.post_ent = ix.pent;
    k.cnt8 = ix.counting && ix.cnt8 && !g_sparse_cnt32 ? 1 : 0;
    k.n_literals = sp->cfg.n_literals; k.weights = sp->weights; k.C = (int)C; k.K = (int)K;
    k.votes = votes; k.pred = pred; k.outputs = outputs;
    if (outputs) TMB_CUDA(cudaMemsetAsync(outputs, 0, (size_t)N * C, st));
    const bool counting = ix.counting;
    const int threads = counting ? 32 * ix.cnt_warps : 256;
    const size_t cnt_bytes = k.cnt8 ? (size_t)((C + 15) & ~15LL) : 4 * (size_t)((C + 3) & ~3LL);
    const size_t smem = counting ? (cnt_bytes + 8 * (size_t)K) * ix.cnt_warps
                                 : 8 * (size_t)K * (threads / 32);
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem > (size_t)max_smem) return fail(TMB_E_UNSUPPORTED, "sparse_infer: too many classes");
    const void *fn = counting ? (K <= 2 ? (const void *)k_sparse_infer_count<2>
                                 : K <= 8 ? (const void *)k_sparse_infer_count<8>
                                          : (const void *)k_sparse_infer_count<0>)
                              : (K <= 2 ? (const void *)k_sparse_infer<2>
                                 : K <= 8 ? (const void *)k_sparse_infer<8>
                                          : (const void *)k_sparse_infer<0>);
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t per_cta = threads / 32;
    const int64_t per_sm = counting ? std::max<int64_t>(1, std::min<int64_t>(64 / ix.cnt_warps,
                                                                              (220 * 1024) / (int64_t)smem))
                                    : 8;
    const int64_t grid = std::min<int64_t>((N + per_cta - 1) / per_cta, (int64_t)sm_count() * per_sm);
    void *args[] = {&k};
    TMB_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(threads), args, smem, st));
    TMB_LAUNCHED();
    if (!counting) sp->ix.release_after(st);  // key-literal index: per call
    return TMB_OK;
}

int tmb_sparse_infer(const tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                     int64_t N, int64_t *votes, int64_t *pred, void *stream) {
    return sparse_infer_impl(sp, indptr, indices, N, votes, pred, nullptr, stream);
}

}  // extern "C"

namespace tmb {
namespace {
// One warp per event: lists at [0, 3n) step 3 (stored) and [1, 2n_act) step 2
// (active) so they interleave; states alternate around the floor.
__global__ void k_sparse_event_bench(SparseK k, int which, int n, int n_act, int reps,
                                     unsigned long long *cyc) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int slab = k.slab;
    int32_t *act = (int32_t *)smem_raw;
    int32_t *cand = act + kMaxActive;
    char *wb = (char *)(cand + kCandStage) + (size_t)warp * (slab * 10 + 64 * 8 + 16);
    int32_t *L = (int32_t *)wb, *DL = L + slab;
    int8_t *S = (int8_t *)(DL + slab), *DS = S + slab;
    uint64_t *scr = (uint64_t *)(((uintptr_t)(DS + slab) + 15) & ~(uintptr_t)15);
    for (int q = threadIdx.x; q < n_act; q += blockDim.x) act[q] = 1 + 2 * q;
    for (int q = threadIdx.x; q < kCandStage; q += blockDim.x) cand[q] = q;
    for (int q = lane; q < n; q += 32) {
        L[q] = 3 * q;
        S[q] = (int8_t)(q & 1 ? k.floor_ + 1 : -1);
    }
    __syncthreads();
    uint64_t nd = 0;
    int acc = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        int nl;
        const uint64_t sk = 0x9E37ull * (uint64_t)(r + 1);
        if (which == 2)
            nl = event_type_ii(k, L, S, n, DL, DS, act, n_act, L + n, slab - n, cand, lane, nullptr);
        else
            nl = event_type_i(k, L, S, n, DL, DS, act, n_act, which, sk, lane, nd, scr);
        acc += nl;
        __syncwarp();
    }
    const long long t1 = clock64();
    if (lane == 0) {
        atomicAdd(cyc, (unsigned long long)(t1 - t0));
        if (acc == -12345) cyc[1] = nd;  // keep the work
    }
}
}  // namespace
}  // namespace tmb

extern "C" int tmb_microbench_sparse_event(int which, int n, int n_act, int reps, int n_cta,
                                           int n_warps, double *us_per_event) {
    int rc = require_device();
    if (rc) return rc;
    if (which < 0 || which > 2 || n < 1 || n > 512 || n_act < 1 || n_act > kMaxActive ||
        reps < 1 || n_cta < 1 || n_warps < 1 || n_warps > 16 || !us_per_event)
        return fail(TMB_E_INVALID, "microbench_sparse_event: bad arguments");
    SparseK k{};
    k.slab = 1024;
    k.floor_ = -15;
    k.smax = 127;
    k.capacity = 64;
    k.fp = make_fb_params(5.0, 0, -15, 127);
    k.n_cand = kCandStage;
    const size_t smem = 4 * (kMaxActive + kCandStage) + (size_t)n_warps * (k.slab * 10 + 64 * 8 + 16);
    unsigned long long *cyc = nullptr;
    TMB_CUDA(cudaMalloc(&cyc, 16));
    cudaMemset(cyc, 0, 16);
    cudaFuncSetAttribute((const void *)k_sparse_event_bench,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_sparse_event_bench<<<n_cta, 32 * n_warps, smem>>>(k, which, n, n_act, reps, cyc);
    TMB_LAUNCHED();
    unsigned long long h[2] = {0, 0};
    cudaMemcpy(h, cyc, 16, cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    cudaFree(cyc);
    if (e != cudaSuccess) return fail(TMB_E_CUDA, cudaGetErrorString(e));
    int clk_khz = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    *us_per_event = (double)h[0] / ((double)n_cta * n_warps * reps) / (clk_khz * 1e-3);
    return TMB_OK;
}

extern "C" {

int tmb_sparse_outputs(const tmb_sparse *sp, const int64_t *indptr, const int32_t *indices,
                       int64_t N, uint8_t *outputs, void *stream) {
    if (!outputs) return fail(TMB_E_INVALID, "sparse_outputs: NULL outputs");
    return sparse_infer_impl(sp, indptr, indices, N, nullptr, nullptr, outputs, stream);
}

}  // extern "C"
