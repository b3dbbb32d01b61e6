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
        if (mode >= 20 && mode < 64) {
            // mode 20 + G: the trainer's packed (count << 40 | biased sum)
            // arrival, spread over G groups (CTA r -> group r % G), each a
            // 16 B slot in its own 256 B line; lanes 0..G-1 poll one slot
            // each, the warp reduces the G partial words
            const int G = mode - 20;
            unsigned long long *base = slots + (size_t)i * G * 32;
            if (threadIdx.x < 2)
                mb_red(base + (blockIdx.x % G) * 32 + threadIdx.x, (1ull << 40) + 12345ull);
            if (threadIdx.x < 32) {
                const int g = threadIdx.x;
                const unsigned long long want = g < G ? (unsigned long long)((n - g + G - 1) / G) : 0;
                unsigned long long a = 0, b = 0;
                bool done;
                do {
                    if (g < G)
                        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];"
                                     : "=l"(a), "=l"(b) : "l"(base + g * 32) : "memory");
                    done = __all_sync(0xffffffffu, (a >> 40) == want && (b >> 40) == want);
                } while (!done);
                unsigned long long sa = a & 0xFFFFFFFFFFull, sb = b & 0xFFFFFFFFFFull;
                for (int o = 16; o; o >>= 1) {
                    sa += __shfl_xor_sync(0xffffffffu, sa, o);
                    sb += __shfl_xor_sync(0xffffffffu, sb, o);
                }
                if (threadIdx.x == 0 && sa + sb == 1) slots[0] = 1;  // keep the sums live
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


// ---------------------------------------------------------------------------
// Integer-pipe issue rates (roofline denominators, measured on the box).
// Every thread runs 8 interleaved dependent chains of ONE SASS opcode
// (chains feed each other so nothing folds); 64 ops per loop trip.  One CTA
// per SM; clock64 gives the SM clocks the CTA ran for.
//   op 0 LOP3   1 IADD3   2 SHF   3 IMAD   4 IMAD.WIDE   5 POPC   6 PRMT
//   op 7 LOP3 + IMAD interleaved (ALU and FMA pipes issuing together)
//   op 8 one SplitMix64 draw + threshold compare per "op" (the trainers'
//        per-literal unit of work)
template <int OP>
__global__ void k_mb_pipe(int iters, unsigned seed, unsigned long long *sink,
                          unsigned long long *cycles) {
    unsigned x[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = seed * (threadIdx.x + 1) + c * 0x9E3779B9u + blockIdx.x;
    const unsigned y = seed ^ threadIdx.x, sel = 0x3210u + (seed & 0x1111u);
    unsigned long long w[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) w[c] = x[c];
    unsigned long long acc = 0;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const unsigned o = x[(c + 1) & 7];
                if (OP == 0) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(o), "r"(y));
                if (OP == 1) asm volatile("{.reg .u32 t; add.u32 t, %0, %1; add.u32 %0, t, %2;}" : "+r"(x[c]) : "r"(o), "r"(y));
                if (OP == 2) asm volatile("shf.l.wrap.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(o), "r"(y));
                if (OP == 3) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(o), "r"(y));
                if (OP == 4) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(w[c]) : "r"((unsigned)w[(c + 1) & 7]), "r"(y));
                if (OP == 5) asm volatile("popc.b32 %0, %1;" : "=r"(x[c]) : "r"(o));
                if (OP == 6) asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(o), "r"(sel));
                if (OP == 7) {
                    if (c & 1) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[c]) : "r"(o), "r"(y));
                    else asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(o), "r"(y));
                }
                if (OP == 8) {
                    w[c] += 0x9E3779B97F4A7C15ull;
                    acc += (mix64(w[c]) >> 11) < 0x1999999999999ull;
                }
            }
        }
    }
    const long long t1 = clock64();
    unsigned long long r = acc;
#pragma unroll
    for (int c = 0; c < 8; ++c) r += x[c] + w[c];
    if (r == 0x1234567ull) sink[0] = r;
    if (threadIdx.x == 0) cycles[blockIdx.x] = (unsigned long long)(t1 - t0);
}

// Cross-SM signal latency through L2 (the hardware floor under any
// per-example grid exchange): CTA 0 and CTA 1 (different SMs) bounce a
// counter through one global word: each waits for its turn with
// ld.relaxed.gpu polls and answers with st.relaxed.gpu (mode 0) or
// red.relaxed.gpu.add (mode 1).  One hop = one write observed by the peer.
__global__ void k_mb_pingpong(unsigned long long *word, int hops, int mode,
                              unsigned long long *cycles) {
    if (threadIdx.x != 0) return;
    const unsigned long long me = blockIdx.x;
    const long long t0 = clock64();
    for (unsigned long long h = me; h < (unsigned long long)hops; h += 2) {
        while (mb_ld(word) != h) {}
        if (mode == 0)
            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(word), "l"(h + 1) : "memory");
        else
            mb_red(word, 1ull);
    }
    if (me == 0) *cycles = (unsigned long long)(clock64() - t0);
}

}  // namespace tmb

using namespace tmb;

extern "C" int tmb_microbench_allreduce(int n_cta, int threads, int iters, int mode,
                                        double *us_per_iter) {
    int rc = require_device();
    if (rc) return rc;
    unsigned long long *slots = nullptr, *cyc = nullptr;
    size_t words = (mode == 6 || mode == 7) ? (size_t)8 * n_cta
                   : (mode >= 20 && mode < 64) ? (size_t)iters * (mode - 20) * 32
                   : (size_t)iters * (mode == 2 ? 8 * 32 : 32);
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

template <int OP>
static int run_pipe(int n_cta, int threads, int iters, double *ops_per_clk_per_sm, double *sm_mhz) {
    unsigned long long *buf = nullptr;
    TMB_CUDA(cudaMalloc(&buf, 8 * (size_t)(n_cta + 1)));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int rc = 0;
    float ms = 0;
    for (int rep = 0; rep < 2 && !rc; ++rep) {  // rep 0 warms up
        cudaEventRecord(a);
        k_mb_pipe<OP><<<n_cta, threads>>>(iters, 0x2545F491u, buf, buf + 1);
        cudaEventRecord(b);
        rc = check_cuda(cudaEventSynchronize(b), "pipe microbench");
        cudaEventElapsedTime(&ms, a, b);
    }
    if (!rc) {
        unsigned long long *cyc = (unsigned long long *)malloc(8 * (size_t)n_cta);
        rc = check_cuda(cudaMemcpy(cyc, buf + 1, 8 * (size_t)n_cta, cudaMemcpyDeviceToHost), "copy");
        double mean = 0;
        for (int i = 0; i < n_cta; ++i) mean += (double)cyc[i];
        mean /= n_cta;
        const double ops_per_cta = (double)threads * iters * 64;
        *ops_per_clk_per_sm = ops_per_cta / mean;
        *sm_mhz = mean / ((double)ms * 1e3);  // cycles per us, the busy SMs' clock
        free(cyc);
    }
    cudaFree(buf);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc;
}

extern "C" int tmb_microbench_pipe(int op, int n_cta, int threads, int iters,
                                   double *ops_per_clk_per_sm, double *sm_mhz) {
    int rc = require_device();
    if (rc) return rc;
    switch (op) {
        case 0: return run_pipe<0>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 1: return run_pipe<1>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 2: return run_pipe<2>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 3: return run_pipe<3>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 4: return run_pipe<4>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 5: return run_pipe<5>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 6: return run_pipe<6>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 7: return run_pipe<7>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        case 8: return run_pipe<8>(n_cta, threads, iters, ops_per_clk_per_sm, sm_mhz);
        default: return fail(TMB_E_INVALID, "tmb_microbench_pipe: op must be 0..8");
    }
}

extern "C" int tmb_microbench_pingpong(int mode, int hops, double *ns_per_hop,
                                       double *cycles_per_hop) {
    int rc = require_device();
    if (rc) return rc;
    unsigned long long *buf = nullptr;
    TMB_CUDA(cudaMalloc(&buf, 16));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0;
    for (int rep = 0; rep < 2 && !rc; ++rep) {
        cudaMemset(buf, 0, 16);
        void *args[] = {&buf, &hops, &mode, (void *)nullptr};
        unsigned long long *cyc = buf + 1;
        args[3] = &cyc;
        cudaEventRecord(a);
        // cooperative launch: both CTAs are guaranteed co-resident
        rc = check_cuda(cudaLaunchCooperativeKernel((const void *)k_mb_pingpong, dim3(2), dim3(32),
                                                    args, 0, 0), "pingpong launch");
        cudaEventRecord(b);
        if (!rc) rc = check_cuda(cudaEventSynchronize(b), "pingpong");
        cudaEventElapsedTime(&ms, a, b);
    }
    if (!rc) {
        unsigned long long cyc = 0;
        rc = check_cuda(cudaMemcpy(&cyc, buf + 1, 8, cudaMemcpyDeviceToHost), "copy");
        *ns_per_hop = (double)ms * 1e6 / hops;
        *cycles_per_hop = (double)cyc / hops;
    }
    cudaFree(buf);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc;
}

// ------------------------------------------------ instruction fetch --
// Straight-line blocks of N independent IADDs (16 B of SASS each, 8
// rotating registers so the chain never stalls) looped `iters` times by
// `warps` warps of one CTA: cycles per instruction show where the block
// stops fitting the instruction caches and what a refetch costs.
namespace tmb {
template <int N>
__global__ void __launch_bounds__(1024, 1) k_mb_icache(int iters, unsigned long long *out) {
    unsigned r0 = threadIdx.x, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3, r4 = r0 + 4, r5 = r0 + 5,
             r6 = r0 + 6, r7 = r0 + 7;
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < N / 8; ++i) {
            // register-only xor / add ring: nothing for ptxas to fold
            asm volatile(
                "xor.b32 %0, %0, %1;\n\tadd.u32 %1, %1, %2;\n\txor.b32 %2, %2, %3;\n\tadd.u32 %3, %3, %4;\n\t"
                "xor.b32 %4, %4, %5;\n\tadd.u32 %5, %5, %6;\n\txor.b32 %6, %6, %7;\n\tadd.u32 %7, %7, %0;"
                : "+r"(r0), "+r"(r1), "+r"(r2), "+r"(r3), "+r"(r4), "+r"(r5), "+r"(r6), "+r"(r7));
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    if ((r0 ^ r1 ^ r2 ^ r3 ^ r4 ^ r5 ^ r6 ^ r7) == 0xFFFFFFFFu) out[1] = 1;  // keep the chains
}
}  // namespace tmb

extern "C" int tmb_microbench_icache(int kbytes, int warps, int iters, double *cycles_per_instr) {
    using namespace tmb;
    int rc = require_device();
    if (rc) return rc;
    const void *fn = nullptr;
    int n = 0;
    switch (kbytes) {
        case 8: fn = (const void *)k_mb_icache<512>; n = 512; break;
        case 16: fn = (const void *)k_mb_icache<1024>; n = 1024; break;
        case 32: fn = (const void *)k_mb_icache<2048>; n = 2048; break;
        case 64: fn = (const void *)k_mb_icache<4096>; n = 4096; break;
        case 96: fn = (const void *)k_mb_icache<6144>; n = 6144; break;
        case 128: fn = (const void *)k_mb_icache<8192>; n = 8192; break;
        case 192: fn = (const void *)k_mb_icache<12288>; n = 12288; break;
        case 256: fn = (const void *)k_mb_icache<16384>; n = 16384; break;
        default: return fail(TMB_E_INVALID, "microbench_icache: kbytes in 8,16,32,64,96,128,192,256");
    }
    if (warps < 1 || warps > 32 || iters < 1 || !cycles_per_instr)
        return fail(TMB_E_INVALID, "microbench_icache: bad arguments");
    unsigned long long *out = nullptr;
    TMB_CUDA(cudaMalloc(&out, 16));
    void *args[] = {&iters, &out};
    rc = check_cuda(cudaLaunchKernel(fn, dim3(1), dim3(32 * warps), args, 0, 0), "icache launch");
    unsigned long long c = 0;
    if (!rc) rc = check_cuda(cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost), "copy");
    cudaFree(out);
    if (!rc) *cycles_per_instr = (double)c / ((double)iters * n);
    return rc;
}
