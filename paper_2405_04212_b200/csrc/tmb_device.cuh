// tmb_device.cuh -- per-literal-position Type I / Type II automaton updates
// shared by the plugin feedback kernel and the fused trainer.
#pragma once

#include "tmb_common.cuh"

namespace tmb {

struct FbParams {
    uint64_t t_inc;   // ceil(((s-1)/s) * 2^53): increment iff draw53 < t_inc
    uint64_t t_dec;   // ceil((1/s) * 2^53)
    double p_inc;     // (s-1)/s  (explicit-draws hook compares doubles)
    double p_dec;     // 1/s
    int boost;
    int smin;
    int smax;
};

inline FbParams make_fb_params(double s, int boost, int smin, int smax) {
    FbParams f;
    f.p_inc = (s - 1.0) / s;  // kernels/_numba.py:73-74
    f.p_dec = 1.0 / s;
    f.t_inc = prob_threshold(f.p_inc);
    f.t_dec = prob_threshold(f.p_dec);
    f.boost = boost;
    f.smin = smin;
    f.smax = smax;
    return f;
}

// Type I at one position (kernels/_numba.py:71-90).  `sk` = seed + G*(base+1)
// so the draw for position p is mix64(sk + G*p).  Draws whose outcome cannot
// change the state (clamped automaton, boosted increment) are skipped: the
// stream is random-access, so skipping is bit-exact (core.py:7-10).
__device__ __forceinline__ int type_i_stream(int st, int lit, int out, const FbParams &fp,
                                             uint64_t sk, uint32_t p, uint64_t &ndraws) {
    if (out && lit) {
        if (st < fp.smax) {
            if (fp.boost) return st + 1;
            ++ndraws;
            if ((mix64(sk + kGolden * (uint64_t)p) >> 11) < fp.t_inc) return st + 1;
        }
    } else if (st > fp.smin) {
        ++ndraws;
        if ((mix64(sk + kGolden * (uint64_t)p) >> 11) < fp.t_dec) return st - 1;
    }
    return st;
}

// type_i_stream without data-dependent branches, for warps whose lanes hold
// different states / literals: the draw mix64(z) (z = sk + G*p) is computed
// for every position and used only where the reference consumes one, so a
// warp never runs the mixer twice on diverged paths.  Bit-identical.
__device__ __forceinline__ int type_i_bf(int st, int lit, int out, const FbParams &fp, uint64_t z,
                                         uint64_t &ndraws) {
    const bool inc = out && lit;
    const bool room = st < fp.smax;
    const bool need = inc ? (room && !fp.boost) : (st > fp.smin);
    const bool hit = (mix64(z) >> 11) < (inc ? fp.t_inc : fp.t_dec);
    ndraws += need ? 1u : 0u;
    const int up = (inc && room && (fp.boost || hit)) ? 1 : 0;
    const int down = (!inc && need && hit) ? 1 : 0;
    return st + up - down;
}

// Same with an explicit uniform draw u (test hook).
__device__ __forceinline__ int type_i_explicit(int st, int lit, int out, const FbParams &fp,
                                               double u) {
    if (out && lit) {
        if ((fp.boost || u < fp.p_inc) && st < fp.smax) return st + 1;
    } else if (u < fp.p_dec && st > fp.smin) {
        return st - 1;
    }
    return st;
}

// Type II at one position (kernels/_numba.py:93-98): output 1 only.
__device__ __forceinline__ int type_ii(int st, int lit, int out) {
    return (out && !lit && st < 0) ? st + 1 : st;
}

// feedback.py:33-44: update probability (a / 2T, a in [0, 2T]) -> integer
// threshold.  The saturated ends are common once the class sums reach T and
// would take the division's slow path (zero numerator), so they are exact
// constants here.
__host__ __device__ __forceinline__ uint64_t threshold_of(long long a, long long T) {
    if (a <= 0) return 0;
    if (a >= 2 * T) return 1ull << 53;
    return prob_threshold((double)a / (2.0 * (double)T));
}

// ---- partitions (executor.py:36-47): block of clause c, block start, CTA ranges
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

// ---- fence-free cross-CTA vote all-reduce (see tmb_train.cu)
constexpr long long kVoteBias = 1LL << 31;  // |partial votes of one CTA| < 2^31
__device__ __forceinline__ void red_relaxed_add_u64(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_acquire() {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ ulonglong2 ld_relaxed_v2u64(const unsigned long long *p) {
    ulonglong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                 : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
    return r;
}



int dev_pack_literals(const uint8_t *x, int64_t N, int64_t cols, int negations, int64_t P,
                      uint32_t *out, cudaStream_t st);
int dev_build_masks(const int8_t *states, int64_t C, int64_t P, uint32_t *masks,
                    int32_t *counts, cudaStream_t st);

}  // namespace tmb
