// tmb_microbench.cu -- latency microbenchmarks of the per-example all-reduce
// candidates used by the fused trainer (design evidence, not product code).
#include <cooperative_groups.h>

#include "tmb_common.cuh"

namespace cg = cooperative_groups;

namespace tmb {

__device__ __forceinline__ void mb_red(unsigned long long *p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long mb_ld(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// mode 0: one relaxed red per CTA into a fresh per-iteration word, thread 0
//         polls until the count reaches n_cta, __syncthreads.
// mode 1: same with __nanosleep(64) backoff between polls.
// mode 2: every CTA's red goes to one of 8 words 256 B apart; warp 0 polls
//         all 8 in parallel.
// mode 3: cooperative_groups grid.sync().
// mode 4: the trainer's protocol -- two words in one 16 B slot, both red by
//         thread 0, warp 0 spins on a 16 B load.
// mode 5: the two words in different 128 B lines (two loads per spin).
// mode 6: all-gather, no atomics: every CTA stores a tagged 16 B slot
//         (ring of 4 steps x n_cta slots); warp 0 polls all slots (lane l
//         reads slots l, l+32, ...) until every tag matches, then sums them.
// mode 7: mode 6 with 8 B slots (one tagged word per CTA).
// mode 8+q: mode 4 with q in {2, 3, 4} polling loads in flight, staggered by
//         `spacing` cycles (a poll samples the slot ~L/2 after issue; q
//         loads spaced L/q apart cut the detection delay from ~L to ~L/2 + L/2q).
__global__ void k_mb_allreduce(unsigned long long *slots, int iters, int mode,
                               unsigned long long *cycles) {
    const int n = gridDim.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 3) {
            cg::this_grid().sync();
            continue;
        }
        if (mode == 4 || mode == 5) {
            unsigned long long *w0 = slots + (size_t)i * 32;
            unsigned long long *w1 = w0 + (mode == 4 ? 1 : 16);
            if (threadIdx.x < 2) mb_red(threadIdx.x == 0 ? w0 : w1, 1ull);
            if (threadIdx.x < 32) {
                unsigned long long a, b;
                do {
                    if (mode == 4) {
                        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                                     : "=l"(a), "=l"(b) : "l"(w0) : "memory");
                    } else {
                        a = mb_ld(w0);
                        b = mb_ld(w1);
                    }
                } while (a < (unsigned long long)n || b < (unsigned long long)n);
            }
            __syncthreads();
            continue;
        }
        if (mode >= 10 && mode <= 12) {
            const int q = mode - 8;
            const long long spacing = 700 / q;
            unsigned long long *w0 = slots + (size_t)i * 32;
            if (threadIdx.x < 2) mb_red(threadIdx.x == 0 ? w0 : w0 + 1, 1ull);
            if (threadIdx.x < 32) {
                ulonglong2 v[4];
                auto ld2 = [&](ulonglong2 &r) {
                    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                                 : "=l"(r.x), "=l"(r.y) : "l"(w0) : "memory");
                };
                auto done = [&](const ulonglong2 &r) {
                    return r.x >= (unsigned long long)n && r.y >= (unsigned long long)n;
                };
                for (int u = 0; u < q; ++u) {
                    ld2(v[u]);
                    if (u + 1 < q) {
                        const long long t = clock64();
                        while (clock64() - t < spacing) {}
                    }
                }
                bool fin = false;
                while (!fin) {
                    for (int u = 0; u < q && !fin; ++u) {
                        if (done(v[u])) fin = true;
                        else ld2(v[u]);
                    }
                }
            }
            __syncthreads();
            continue;
        }
        if (mode == 6 || mode == 7) {
            // slots: [4][n] x (mode 6: 2 words, mode 7: 1 word)
            const int ws = mode == 6 ? 2 : 1;
            unsigned long long *ring = slots + (size_t)(i & 3) * n * ws;
            const unsigned long long tag = (unsigned long long)(i + 1) << 40;
            if (threadIdx.x == 0) {
                unsigned long long *me = ring + (size_t)blockIdx.x * ws;
                if (ws == 2)
                    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(me), "l"(tag | 5),
                                 "l"(tag | 7) : "memory");
                else
                    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(me), "l"(tag | 5) : "memory");
            }
            if (threadIdx.x < 32) {
                unsigned long long acc = 0;
                bool done;
                do {
                    bool ok = true;
                    acc = 0;
                    for (int c = threadIdx.x; c < n; c += 32) {
                        unsigned long long a, b = tag;
                        if (ws == 2)
                            asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                                         : "=l"(a), "=l"(b) : "l"(ring + 2 * c) : "memory");
                        else
                            a = mb_ld(ring + c);
                        ok = ok && (a >> 40) == (tag >> 40) && (b >> 40) == (tag >> 40);
                        acc += (a & 0xFFFFFFFFFFull) + (b & 0xFFFFFFFFFFull);
                    }
                    done = __all_sync(0xffffffffu, ok);
                } while (!done);
                for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
                if (threadIdx.x == 0 && acc == 0) slots[0] = 1;  // keep the sum live
            }
            __syncthreads();
            continue;
        }
        if (mode == 2) {
            unsigned long long *base = slots + (size_t)i * 8 * 32;
            if (threadIdx.x == 0) mb_red(base + (blockIdx.x & 7) * 32, 1ull);
            if (threadIdx.x < 32) {
                const int g = threadIdx.x;
                const unsigned long long want = (g < 8) ? (unsigned long long)((n - g + 7) / 8) : 0;
                bool done;
                do {
                    const unsigned long long v = g < 8 ? mb_ld(base + g * 32) : 0;
                    done = __all_sync(0xffffffffu, v >= want);
                } while (!done);
            }
            __syncthreads();
            continue;
        }
        unsigned long long *w = slots + (size_t)i * 32;
        if (threadIdx.x == 0) {
            mb_red(w, 1ull);
            while (mb_ld(w) < (unsigned long long)n) {
                if (mode == 1) __nanosleep(64);
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = (unsigned long long)(clock64() - t0);
}

}  // namespace tmb

using namespace tmb;

extern "C" int tmb_microbench_allreduce(int n_cta, int threads, int iters, int mode,
                                        double *us_per_iter) {
    int rc = require_device();
    if (rc) return rc;
    unsigned long long *slots = nullptr, *cyc = nullptr;
    size_t words = (mode == 6 || mode == 7) ? (size_t)8 * n_cta : (size_t)iters * (mode == 2 ? 8 * 32 : 32);
    TMB_CUDA(cudaMalloc(&slots, 8 * words));
    TMB_CUDA(cudaMalloc(&cyc, 8));
    TMB_CUDA(cudaMemset(slots, 0, 8 * words));
    void *args[] = {&slots, &iters, &mode, &cyc};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    rc = check_cuda(cudaLaunchCooperativeKernel((const void *)k_mb_allreduce, dim3(n_cta),
                                                dim3(threads), args, 0, 0),
                    "microbench launch");
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (!rc) *us_per_iter = (double)ms * 1e3 / iters;
    cudaFree(slots);
    cudaFree(cyc);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc;
}
