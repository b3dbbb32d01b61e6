// tmb_infer_solo.cu -- batched inference with one INDEPENDENT CTA per SM
// (predictor.py:79-96 / dense.py:171-174 / executor.py:355-383).
//
// Every CTA owns whole tiles of 128 examples: its transposer warps turn the
// tile's raw feature bytes (HBM) into X^T [F+2][4] uint32 in shared memory
// (one 16-byte row per feature = 128 examples; row F all ones, row F+1 all
// zeros), double-buffered, while its evaluator warps run EVERY rule over the
// previous tile.  Rules are not resident: their 16-slot heads (32 B per rule,
// 320 KB for configs[2]) stream from L2 -- each warp prefetches the next
// 64-rule chunk's heads into registers while it evaluates the current one --
// so no CTA depends on another: no cluster, no DSMEM exchange of X^T
// quarters, and all SMs run (the 4-CTA cluster kernel fits only 33 clusters
// = 132 SMs).
//
// Head slots come in (positive, negated) pairs of X^T row indices (padding:
// the all-ones / all-zeros rows), so one LOP3 per word tests two includes:
//     acc &= X^T[p] & ~X^T[n]
// and a pair costs two 16-bit extractions, two LDS.128 and four LOP3 for 128
// examples.  Slots 8..15 of rules already dead for all 128 examples skip
// their loads; the warp leaves a 64-rule chunk when all its rules are dead
// (checked after 12 includes).  The rare survivors of all 16 head slots run
// their CSR tail (generic (feature << 1 | negated) codes) and add their
// weights into the tile's int32 partial sums in shared memory; a finalizer
// warp takes the argmax (ties -> lowest class, np.argmax) and writes
// predictions (and int64 votes when asked).
//
// Hand-offs (mbarriers, CTA scope):
//   full[b]  transposer warps -> evaluators   (X^T buffer b holds tile it)
//   efree[b] evaluator warps  -> finalizer    (tile it evaluated)
//   empty[b] finalizer        -> transposers  (buffer b and its partials free)
#include <algorithm>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_infer.cuh"

namespace tmb {

int g_infer_solo = 1;

constexpr int kSoTG = 4;  // 32-example groups per tile (128 examples)
#ifndef TMB_SOLO_T
#define TMB_SOLO_T 7
#endif
#ifndef TMB_SOLO_THREADS
#define TMB_SOLO_THREADS 512
#endif
constexpr int kSoThreads = TMB_SOLO_THREADS;
#ifndef TMB_SOLO_PD
#define TMB_SOLO_PD 3
#endif
constexpr int kSoPD = TMB_SOLO_PD;  // transposer L2 prefetch distance (items)
// evaluator load predication of slots 8..15: 0 none, 1 liveness before
// every pair, 2 liveness before each group of two pairs
#ifndef TMB_SOLO_PRED
#define TMB_SOLO_PRED 1
#endif
constexpr int kSoPred = TMB_SOLO_PRED;
// > 512 threads: warpgroups 0-1 (the transposers; warps 0..7) re-allocated
// to TMB_SOLO_REGS_T registers per thread, the rest share what is left
#ifndef TMB_SOLO_REGS_T
#define TMB_SOLO_REGS_T 104
#endif
constexpr int kSoRegsT = TMB_SOLO_REGS_T;
constexpr int kSoRegsE = kSoThreads <= 512 ? 128
    : ((65536 / kSoThreads / 8 * 8) * kSoThreads - 256 * kSoRegsT) / (kSoThreads - 256) / 8 * 8;

struct InferSK {
    const uint8_t *x;    // raw features [N][F] (uint8 path)
    const uint64_t *xb;  // bit-packed [N][W64] (packed path)
    int64_t W64;
    int xb_vec16;
    int64_t N, F;
    const uint4 *heads;  // [R_pad][2]: 16 uint16 slots
    const int32_t *tail_ptr;
    const uint16_t *tails;
    const int32_t *w;
    int R, R_pad, K;
    int64_t *votes, *pred;
    const int64_t *labels;
    unsigned long long *correct;
    unsigned int *bad_input;
    int vec_ok;
    int dbg;  // timing experiments only (wrong results): bit0 skip eval, bit1 skip transpose
};

__device__ __forceinline__ uint4 ldg_heads(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// X^T row addresses of the two 16-bit row indices of a head word: one
// extraction + one LEA each (written out: left to itself the compiler spends
// three instructions per index)
__device__ __forceinline__ uint32_t row_lo(uint32_t w, uint32_t base) {
    uint32_t a;
    asm("{\n .reg .u32 t;\n and.b32 t, %1, 0xFFFF;\n mad.lo.u32 %0, t, 16, %2;\n}"
        : "=r"(a) : "r"(w), "r"(base));
    return a;
}
__device__ __forceinline__ uint32_t row_hi(uint32_t w, uint32_t base) {
    uint32_t a;
    asm("{\n .reg .u32 t;\n shr.u32 t, %1, 16;\n mad.lo.u32 %0, t, 16, %2;\n}"
        : "=r"(a) : "r"(w), "r"(base));
    return a;
}

template <bool PACKED>
__global__ void __launch_bounds__(kSoThreads, 1) k_infer_solo(InferSK k) {
#ifndef TMB_SOLO_TP
#define TMB_SOLO_TP 6
#endif
    constexpr int kT = PACKED ? TMB_SOLO_TP : TMB_SOLO_T;  // transposer warps
    extern __shared__ __align__(16) char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int nE = nwarps - kT - 1;  // evaluator warps (the last warp finalizes)
    const int K = k.K;
    const int64_t F = k.F;
    const int xrows = (int)F + 2;
    uint32_t *xt0 = reinterpret_cast<uint32_t *>(smem_raw);
    uint32_t *xt1 = xt0 + (size_t)xrows * kSoTG;
    int32_t *part2 = reinterpret_cast<int32_t *>(xt1 + (size_t)xrows * kSoTG);  // [2][128][K]
    int32_t *dirty2 = part2 + 2 * 32 * kSoTG * K;                              // [2][4]
    uint64_t *mb = reinterpret_cast<uint64_t *>(
        (reinterpret_cast<uintptr_t>(dirty2 + 2 * kSoTG) + 7) & ~(uintptr_t)7);
    uint64_t *full = mb, *empty = mb + 2, *efree = mb + 4;
    uint32_t *ectr = reinterpret_cast<uint32_t *>(mb + 6);  // [2] next rule chunk

    for (int i = tid; i < kSoTG; i += blockDim.x) {
        xt0[(size_t)F * kSoTG + i] = 0xFFFFFFFFu;
        xt1[(size_t)F * kSoTG + i] = 0xFFFFFFFFu;
        xt0[(size_t)(F + 1) * kSoTG + i] = 0u;
        xt1[(size_t)(F + 1) * kSoTG + i] = 0u;
    }
    for (int i = tid; i < 2 * 32 * kSoTG * K; i += blockDim.x) part2[i] = 0;
    if (tid < 2 * kSoTG) dirty2[tid] = 0;
    if (tid < 2) ectr[tid] = 0;
    if (tid == 0) {
        mbar_init(&full[0], kT);
        mbar_init(&full[1], kT);
        mbar_init(&empty[0], 1);
        mbar_init(&empty[1], 1);
        mbar_init(&efree[0], nE);
        mbar_init(&efree[1], nE);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (kSoThreads > 512) {
        static_assert(kSoThreads <= 512 || (kSoRegsE >= 24 && kSoRegsE <= 256), "register split");
        if (warp < 8)
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kSoRegsT));
        else
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kSoRegsE));
    }
    const int64_t tile_n = 32 * kSoTG;
    const int64_t n_tiles = (k.N + tile_n - 1) / tile_n;
    const int64_t n_my = blockIdx.x < n_tiles
                             ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto tile_of = [&](int64_t it) { return (int64_t)blockIdx.x + it * gridDim.x; };

    if (warp < kT) {
        // ======================= transposer warps =======================
        uint32_t bad = 0;
        auto tile_begin = [&](int64_t it) {
            if (it >= 2) mbar_wait(&empty[it & 1], (uint32_t)(((it >> 1) + 1) & 1));
        };
        auto tile_end = [&](int64_t it) {
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&full[it & 1]);
        };
        if (PACKED) {
            // unit = 32 examples x 256 features: lane l holds 256 feature bits
            // of example 32g + l; eight 32x32 warp bit transposes leave lane j
            // with the X^T words of features fb + 32q + j
            const int units = (int)((F + 255) / 256) * kSoTG;
            const int nq = (k.dbg & 2) ? 0 : units > warp ? (units - warp + kT - 1) / kT : 0;
            auto ug = [&](int q) { return (warp + q * kT) % kSoTG; };
            auto ufb = [&](int q) { return (int64_t)((warp + q * kT) / kSoTG) * 256; };
            auto load_p = [&](int64_t itx, int q, uint32_t (&w)[8]) {
                const int64_t e = tile_of(itx) * tile_n + 32 * ug(q) + lane;
                const int64_t fb = ufb(q);
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = 0;
                if (e >= k.N) return;
                const uint32_t *row = reinterpret_cast<const uint32_t *>(k.xb + e * k.W64);
                const int64_t u0 = fb >> 5, nu = 2 * k.W64;
                if (k.xb_vec16 && (u0 & 3) == 0 && u0 + 8 <= nu) {
                    const uint4 a = __ldcs(reinterpret_cast<const uint4 *>(row + u0));
                    const uint4 b = __ldcs(reinterpret_cast<const uint4 *>(row + u0 + 4));
                    w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
                    w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
                } else {
#pragma unroll
                    for (int h = 0; h < 8; ++h)
                        if (u0 + h < nu) w[h] = __ldcs(row + u0 + h);
                }
            };
            auto finish_p = [&](const uint32_t (&w)[8], int q, uint32_t *mine) {
                const int64_t fb = ufb(q);
                const int g = ug(q);
#pragma unroll
                for (int qq = 0; qq < 8; ++qq) {
                    const uint32_t xv = warp_transpose32(w[qq], lane);
                    const int64_t f = fb + 32 * qq + lane;
                    if (f < F) mine[(size_t)f * kSoTG + g] = xv;
                }
            };
            uint32_t wa[8], wb[8];
            for (int64_t it = 0; it < n_my; ++it) {
                uint32_t *mine = (it & 1) ? xt1 : xt0;
                tile_begin(it);
                int q = 0;
                for (; q + 1 < nq; q += 2) {
                    load_p(it, q, wa);
                    load_p(it, q + 1, wb);
                    finish_p(wa, q, mine);
                    finish_p(wb, q + 1, mine);
                }
                if (q < nq) {
                    load_p(it, q, wa);
                    finish_p(wa, q, mine);
                }
                tile_end(it);
            }
        } else {
            // unit = 32 examples x 128 features; lane (j, c16) loads 16 feature
            // bytes of 8 example rows.  Bytes are 0/1 (anything else is
            // flagged and fails the call), so OR-ing row i shifted by i builds
            // the 8 row bits of each feature in place; a 4-lane shuffle and a
            // 4x4 byte transpose finish the X^T words (see k_infer_ws).
            const int j = lane >> 3, c16 = lane & 7;
            const int nblk = (int)((F + 127) / 128);
            const int units = nblk * kSoTG;
            const int nq = units > warp ? (units - warp + kT - 1) / kT : 0;
            auto ug = [&](int q) { return (warp + q * kT) % kSoTG; };
            auto ufb = [&](int q) { return (int64_t)((warp + q * kT) / kSoTG) * 128 + 16 * c16; };
            const uint32_t psel = (uint32_t)(j | ((1 ^ j) << 4) | ((2 ^ j) << 8) | ((3 ^ j) << 12));
            auto load_item = [&](int64_t itx, int q, uint4 (&w)[8]) {
                const int64_t er = tile_of(itx) * tile_n + 32 * ug(q) + 8 * j;
                const int64_t fb = ufb(q);
                if (k.vec_ok && fb + 16 <= F && er + 7 < k.N) {
                    const uint8_t *src = k.x + er * F + fb;
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        w[i] = __ldcs(reinterpret_cast<const uint4 *>(src + i * F));
                    return;
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int64_t e = er + i;
                    w[i] = make_uint4(0, 0, 0, 0);
                    if (e < k.N && fb < F) {
                        const uint8_t *src = k.x + e * F + fb;
                        uint32_t bw[4] = {0, 0, 0, 0};
                        for (int bb = 0; bb < 16 && fb + bb < F; ++bb)
                            bw[bb >> 2] |= (uint32_t)src[bb] << (8 * (bb & 3));
                        w[i] = make_uint4(bw[0], bw[1], bw[2], bw[3]);
                    }
                }
            };
            auto finish_item = [&](const uint4 (&w)[8], int q, uint32_t *mine) {
                const int64_t fb = ufb(q);
                const int g = ug(q);
                uint32_t R[4], ob = 0;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    uint32_t acc = 0;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const uint32_t xv = d == 0 ? w[i].x : d == 1 ? w[i].y : d == 2 ? w[i].z : w[i].w;
                        ob |= xv;
                        acc |= xv << i;
                    }
                    R[d] = acc;
                }
                bad |= ob & 0xFEFEFEFEu;
                {
                    const uint32_t m1 = 0u - (uint32_t)(j & 1), m2 = 0u - (uint32_t)((j >> 1) & 1);
                    uint32_t t0 = (R[0] ^ R[1]) & m1, t1 = (R[2] ^ R[3]) & m1;
                    R[0] ^= t0; R[1] ^= t0; R[2] ^= t1; R[3] ^= t1;
                    t0 = (R[0] ^ R[2]) & m2; t1 = (R[1] ^ R[3]) & m2;
                    R[0] ^= t0; R[2] ^= t0; R[1] ^= t1; R[3] ^= t1;
                }
                uint32_t recv[4];
                recv[0] = R[0];
#pragma unroll
                for (int sft = 1; sft < 4; ++sft) recv[sft] = __shfl_xor_sync(0xffffffffu, R[sft], 8 * sft);
                const uint32_t t0 = __byte_perm(recv[0], recv[1], 0x5140);
                const uint32_t t1 = __byte_perm(recv[2], recv[3], 0x5140);
                const uint32_t t2 = __byte_perm(recv[0], recv[1], 0x7362);
                const uint32_t t3 = __byte_perm(recv[2], recv[3], 0x7362);
                uint32_t wq[4];
                wq[0] = __byte_perm(__byte_perm(t0, t1, 0x5410), 0, psel);
                wq[1] = __byte_perm(__byte_perm(t0, t1, 0x7632), 0, psel);
                wq[2] = __byte_perm(__byte_perm(t2, t3, 0x5410), 0, psel);
                wq[3] = __byte_perm(__byte_perm(t2, t3, 0x7632), 0, psel);
                {
                    const uint32_t m1 = 0u - (uint32_t)(c16 & 1), m2 = 0u - (uint32_t)((c16 >> 1) & 1);
                    const uint32_t a0 = (wq[0] & ~m1) | (wq[1] & m1), a1 = (wq[1] & ~m1) | (wq[2] & m1);
                    const uint32_t a2 = (wq[2] & ~m1) | (wq[3] & m1), a3 = (wq[3] & ~m1) | (wq[0] & m1);
                    wq[0] = (a0 & ~m2) | (a2 & m2);
                    wq[1] = (a1 & ~m2) | (a3 & m2);
                    wq[2] = (a2 & ~m2) | (a0 & m2);
                    wq[3] = (a3 & ~m2) | (a1 & m2);
                }
                uint32_t *dst0 = mine + (size_t)(fb + 4 * j) * kSoTG + g;
#pragma unroll
                for (int r = 0; r < 4; ++r) {
                    const int kq = (r + c16) & 3;
                    if (fb + 4 * j + kq < F) dst0[kq * kSoTG] = wq[r];
                }
            };
            if (nq == 0 || (k.dbg & 2)) {
                for (int64_t it = 0; it < n_my; ++it) {
                    tile_begin(it);
                    tile_end(it);
                }
            } else {
                // items in order (it, q); A / B alternate, the next item's
                // loads go out before the current item is transposed
                uint4 wa[8], wb[8];
                int64_t ia = 0, ib = 0;
                int qa = 0, qb = 0;
                auto next_of = [&](int64_t itx, int q, int64_t &itn, int &qn) {
                    qn = q + 1;
                    itn = itx;
                    if (qn == nq) {
                        qn = 0;
                        ++itn;
                    }
                };
                // L2 prefetch kSoPD items beyond the one in registers: the
                // register loads then hit L2 instead of waiting out the HBM
                // latency (bytes in flight without registers or smem)
                int64_t ipf = 0;
                int qpf = 0;
                auto prefetch_next = [&]() {
                    if (ipf >= n_my) return;
                    const int64_t e = tile_of(ipf) * tile_n + 32 * ug(qpf) + lane;
                    const int64_t f0 = (int64_t)((warp + qpf * kT) / kSoTG) * 128;
                    if (e < k.N && f0 < F)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(k.x + e * F + f0));
                    next_of(ipf, qpf, ipf, qpf);
                };
                for (int d = 0; d <= kSoPD && n_my > 0; ++d) prefetch_next();
                if (n_my > 0) load_item(0, 0, wa);
                while (ia < n_my) {
                    next_of(ia, qa, ib, qb);
                    if (ib < n_my) {
                        load_item(ib, qb, wb);
                        prefetch_next();
                    }
                    if (qa == 0) tile_begin(ia);
                    finish_item(wa, qa, (ia & 1) ? xt1 : xt0);
                    if (qa == nq - 1) tile_end(ia);
                    if (ib >= n_my) break;
                    next_of(ib, qb, ia, qa);
                    if (ia < n_my) {
                        load_item(ia, qa, wa);
                        prefetch_next();
                    }
                    if (qb == 0) tile_begin(ib);
                    finish_item(wb, qb, (ib & 1) ? xt1 : xt0);
                    if (qb == nq - 1) tile_end(ib);
                }
            }
        }
        if (bad) atomicOr(k.bad_input, 1u);
    } else if (warp == nwarps - 1) {
        // ========================= finalizer warp =========================
        unsigned long long hits = 0;
        for (int64_t it = 0; it < n_my; ++it) {
            const int buf = (int)(it & 1);
            mbar_wait(&efree[buf], (uint32_t)((it >> 1) & 1));
            int32_t *part = part2 + buf * 32 * kSoTG * K;
            int32_t *dirty = dirty2 + buf * kSoTG;
            const int64_t e0 = tile_of(it) * tile_n;
#pragma unroll 1
            for (int gq = 0; gq < kSoTG; ++gq) {
                const bool dg = dirty[gq] != 0;
                const int64_t e = e0 + 32 * gq + lane;
                int32_t *pe = part + (32 * gq + lane) * K;
                int best = 0;
                if (dg || k.votes) {
                    int32_t bv = 0;
                    for (int kk = 0; kk < K; ++kk) {
                        const int32_t v = dg ? pe[kk] : 0;
                        if (kk == 0 || v > bv) {
                            bv = v;
                            best = kk;
                        }
                        if (k.votes && e < k.N) k.votes[e * K + kk] = (int64_t)v;
                        if (dg) pe[kk] = 0;
                    }
                }
                if (e < k.N) {
                    if (k.pred) k.pred[e] = best;  // all sums 0 -> class 0 (np.argmax)
                    if (k.labels) hits += (k.labels[e] == best);
                }
            }
            __syncwarp();
            if (lane < kSoTG) dirty[lane] = 0;
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&empty[buf]);
        }
        if (k.correct) {
            for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
            if (lane == 0 && hits) atomicAdd(k.correct, hits);
        }
    } else {
        // ========================= evaluator warps =========================
        const int ew = warp - kT;
        const int n_chunks = k.R_pad / 64;
        const uint32_t xb0 = smem_u32(xt0), xb1 = smem_u32(xt1);
        for (int64_t it = 0; it < n_my; ++it) {
            const int buf = (int)(it & 1);
            mbar_wait(&full[buf], (uint32_t)((it >> 1) & 1));
            const uint32_t xaddr = buf ? xb1 : xb0;
            int32_t *part = part2 + buf * 32 * kSoTG * K;
            int32_t *dirty = dirty2 + buf * kSoTG;
            // a surviving rule's tail (generic codes) and its votes into part
            auto finish_rule = [&](int r, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
                for (int q = __ldg(&k.tail_ptr[r]), qe = __ldg(&k.tail_ptr[r + 1]);
                     q < qe && (a0 | a1 | a2 | a3); ++q) {
                    const uint32_t c = __ldg(&k.tails[q]);
                    const uint4 xv = lds128(xaddr + (c >> 1) * 16);
                    const uint32_t m = 0u - (c & 1u);
                    a0 &= xv.x ^ m;
                    a1 &= xv.y ^ m;
                    a2 &= xv.z ^ m;
                    a3 &= xv.w ^ m;
                }
                const int32_t *wr = k.w + (size_t)r * K;
#pragma unroll
                for (int gq = 0; gq < kSoTG; ++gq) {
                    uint32_t acc = gq == 0 ? a0 : gq == 1 ? a1 : gq == 2 ? a2 : a3;
                    if (acc) dirty[gq] = 1;
                    while (acc) {
                        const int b = __ffs(acc) - 1;
                        acc &= acc - 1;
                        int32_t *dst = part + (gq * 32 + b) * K;
                        for (int kk = 0; kk < K; ++kk) {
                            const int32_t wv = __ldg(&wr[kk]);
                            if (wv) atomicAdd(&dst[kk], wv);
                        }
                    }
                }
            };
            // chunks 0..nE-1 static, then one shared-memory atomic per
            // evaluated chunk hands out the next; ectr[buf] is never reset
            // (use u = it >> 1 numbers its chunks from u * n_chunks)
            const uint32_t ebase = (uint32_t)(it >> 1) * (uint32_t)n_chunks;
            int rc = (k.dbg & 1) ? n_chunks : ew;
            uint4 hA0 = make_uint4(0, 0, 0, 0), hA1 = hA0, hB0 = hA0, hB1 = hA0;
            if (rc < n_chunks) {
                const uint4 *hp = k.heads + (size_t)(rc * 64 + lane) * 2;
                hA0 = ldg_heads(hp);
                hA1 = ldg_heads(hp + 1);
                hB0 = ldg_heads(hp + 64);
                hB1 = ldg_heads(hp + 65);
            }
            while (rc < n_chunks) {
                int nx = 0;
                if (lane == 0) nx = nE + (int)(atom_add_shared(&ectr[buf], 1u) - ebase);
                nx = __shfl_sync(0xffffffffu, nx, 0);
                // the next chunk's heads are in flight while this one runs
                uint4 nA0 = make_uint4(0, 0, 0, 0), nA1 = nA0, nB0 = nA0, nB1 = nA0;
                if (nx < n_chunks) {
                    const uint4 *hp = k.heads + (size_t)(nx * 64 + lane) * 2;
                    nA0 = ldg_heads(hp);
                    nA1 = ldg_heads(hp + 1);
                    nB0 = ldg_heads(hp + 64);
                    nB1 = ldg_heads(hp + 65);
                }
                const int rA = rc * 64 + lane, rB = rA + 32;
                const uint32_t lA = rA < k.R ? 0xFFFFFFFFu : 0u, lB = rB < k.R ? 0xFFFFFFFFu : 0u;
                uint32_t A0 = lA, A1 = lA, A2 = lA, A3 = lA, B0 = lB, B1 = lB, B2 = lB, B3 = lB;
                uint4 pa = make_uint4(0, 0, 0, 0), na = pa, pb = pa, nb = pa;
                // slot pair q: slots 8..15 of a rule dead for all 128 examples
                // skip their loads (its accumulator stays 0 whatever stale
                // registers it is ANDed with)
                // la / lb: load predicates (liveness sampled before a group
                // of pairs, so the group's loads issue back to back)
                auto pair = [&](const uint32_t ha, const uint32_t hb, const bool la, const bool lb) {
                    lds128_if(pa, la, row_lo(ha, xaddr));
                    lds128_if(na, la, row_hi(ha, xaddr));
                    lds128_if(pb, lb, row_lo(hb, xaddr));
                    lds128_if(nb, lb, row_hi(hb, xaddr));
                    A0 &= pa.x & ~na.x;
                    A1 &= pa.y & ~na.y;
                    A2 &= pa.z & ~na.z;
                    A3 &= pa.w & ~na.w;
                    B0 &= pb.x & ~nb.x;
                    B1 &= pb.y & ~nb.y;
                    B2 &= pb.z & ~nb.z;
                    B3 &= pb.w & ~nb.w;
                };
                auto alive_a = [&]() { return kSoPred == 0 || (A0 | A1 | A2 | A3) != 0; };
                auto alive_b = [&]() { return kSoPred == 0 || (B0 | B1 | B2 | B3) != 0; };
                pair(hA0.x, hB0.x, true, true);
                pair(hA0.y, hB0.y, true, true);
                pair(hA0.z, hB0.z, true, true);
                pair(hA0.w, hB0.w, true, true);
                if (kSoPred == 1) {
                    pair(hA1.x, hB1.x, alive_a(), alive_b());
                    pair(hA1.y, hB1.y, alive_a(), alive_b());
                } else {
                    const bool la = alive_a(), lb = alive_b();
                    pair(hA1.x, hB1.x, la, lb);
                    pair(hA1.y, hB1.y, la, lb);
                }
                if (__any_sync(0xffffffffu, A0 | A1 | A2 | A3 | B0 | B1 | B2 | B3)) {
                    if (kSoPred == 1) {
                        pair(hA1.z, hB1.z, alive_a(), alive_b());
                        pair(hA1.w, hB1.w, alive_a(), alive_b());
                    } else {
                        const bool la = alive_a(), lb = alive_b();
                        pair(hA1.z, hB1.z, la, lb);
                        pair(hA1.w, hB1.w, la, lb);
                    }
                }
                if (A0 | A1 | A2 | A3) finish_rule(rA, A0, A1, A2, A3);
                if (B0 | B1 | B2 | B3) finish_rule(rB, B0, B1, B2, B3);
                hA0 = nA0; hA1 = nA1; hB0 = nB0; hB1 = nB1;
                rc = nx;
            }
            // this warp's share of tile it is evaluated (its lanes' partial-sum
            // atomics ordered before lane 0's releasing arrival)
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&efree[buf]);
        }
    }
}

// ------------------------------------------------------------------ host --

// Paired head slots for every rule (see tmb_rules::sheads).  Within each
// aligned 8-rule group (8 lanes of one 16-byte shared load = one wavefront
// when their rows hit distinct bank quads; row f occupies quad f mod 8) the
// include placed at each slot is chosen greedily from the rule's remaining
// includes of that slot's polarity to spread the quads; a rule with no
// include of a polarity left repeats one it has (AND is idempotent) or reads
// the padding row.  Includes that do not fit the 8 + 8 slots form the tail.
int build_solo_heads(const std::vector<int64_t> &ptr, const std::vector<uint32_t> &inc,
                     int64_t R, int64_t F, tmb_rules *r) {
    if (R < 1 || F + 2 > 65535) return TMB_OK;
    const int64_t R_pad = (R + 63) / 64 * 64;
    std::vector<uint16_t> heads((size_t)R_pad * 16, 0);
    std::vector<int32_t> tptr((size_t)R + 1, 0);
    std::vector<uint16_t> tails;
    std::vector<std::vector<uint32_t>> pool[2], orig[2];
    for (int p = 0; p < 2; ++p) {
        pool[p].resize((size_t)R);
        orig[p].resize((size_t)R);
    }
    for (int64_t i = 0; i < R; ++i)
        for (int64_t q = ptr[i]; q < ptr[i + 1]; ++q) {
            const uint32_t c = inc[q];
            pool[c & 1][i].push_back(c >> 1);
            orig[c & 1][i].push_back(c >> 1);
        }
    for (int64_t g0 = 0; g0 < R; g0 += 8) {
        const int64_t g1 = std::min<int64_t>(g0 + 8, R);
        for (int s = 0; s < 16; ++s) {
            const int pol = s & 1;
            int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            std::vector<int64_t> order;
            for (int64_t i = g0; i < g1; ++i) order.push_back(i);
            std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
                return pool[pol][a].size() < pool[pol][b].size();
            });
            for (int64_t i : order) {
                auto &L = pool[pol][i];
                uint32_t row;
                if (!L.empty()) {
                    size_t best = 0;
                    int bc = 1 << 30;
                    for (size_t j = 0; j < L.size(); ++j)
                        if (cnt[L[j] & 7] < bc) { bc = cnt[L[j] & 7]; best = j; }
                    row = L[best];
                    L[best] = L.back();
                    L.pop_back();
                } else if (!orig[pol][i].empty()) {
                    const auto &O = orig[pol][i];
                    size_t best = 0;
                    int bc = 1 << 30;
                    for (size_t j = 0; j < O.size(); ++j)
                        if (cnt[O[j] & 7] < bc) { bc = cnt[O[j] & 7]; best = j; }
                    row = O[best];
                } else {
                    row = (uint32_t)(pol ? F + 1 : F);  // all-zeros / all-ones row
                }
                cnt[row & 7]++;
                heads[(size_t)i * 16 + s] = (uint16_t)row;
            }
        }
    }
    for (int64_t i = 0; i < R; ++i) {
        std::vector<uint32_t> rest;
        for (int p = 0; p < 2; ++p)
            for (uint32_t f : pool[p][i]) rest.push_back((f << 1) | (uint32_t)p);
        std::sort(rest.begin(), rest.end());
        for (uint32_t c : rest) tails.push_back((uint16_t)c);
        tptr[i + 1] = (int32_t)tails.size();
    }
    if (F * 2 + 1 >= 65536 && !tails.empty()) return TMB_OK;  // tail codes must fit 16 bits
    int rc;
    if ((rc = check_cuda(cudaMalloc(&r->sheads, 2 * heads.size()), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&r->stail_ptr, 4 * tptr.size()), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&r->stails, 2 * std::max<size_t>(tails.size(), 1)), "cudaMalloc")))
        return rc;
    TMB_CUDA(cudaMemcpy(r->sheads, heads.data(), 2 * heads.size(), cudaMemcpyHostToDevice));
    TMB_CUDA(cudaMemcpy(r->stail_ptr, tptr.data(), 4 * tptr.size(), cudaMemcpyHostToDevice));
    if (!tails.empty())
        TMB_CUDA(cudaMemcpy(r->stails, tails.data(), 2 * tails.size(), cudaMemcpyHostToDevice));
    r->R_pad = R_pad;
    r->sheads_ok = 1;
    return TMB_OK;
}

int launch_infer_solo(const tmb_rules *r, const uint8_t *x, const uint64_t *xb, int64_t W64,
                      int64_t N, int64_t *votes, int64_t *pred, const int64_t *labels,
                      unsigned long long *correct, unsigned int *bad_flag, cudaStream_t st,
                      bool *launched) {
    *launched = false;
    if (!g_infer_solo || !r->sheads_ok || r->K > 32 || N == 0) return TMB_OK;
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t smem = 2 * 16 * (size_t)(r->F + 2) + 2 * 4 * (size_t)32 * kSoTG * r->K +
                        4 * 2 * kSoTG + 8 + 8 * 6 + 8;
    if (smem > (size_t)max_smem) return TMB_OK;
    InferSK k;
    k.x = x; k.xb = xb; k.W64 = W64;
    k.xb_vec16 = xb && (W64 % 2 == 0) && (reinterpret_cast<uintptr_t>(xb) % 16 == 0);
    k.N = N; k.F = r->F;
    k.heads = reinterpret_cast<const uint4 *>(r->sheads);
    k.tail_ptr = r->stail_ptr; k.tails = r->stails; k.w = r->weights;
    k.R = (int)r->R; k.R_pad = (int)r->R_pad; k.K = (int)r->K;
    k.votes = votes; k.pred = pred; k.labels = labels; k.correct = correct;
    k.bad_input = bad_flag;
    k.vec_ok = (r->F % 16 == 0) && x && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
    k.dbg = g_infer_dbg;
    const void *fn = xb ? (const void *)k_infer_solo<true> : (const void *)k_infer_solo<false>;
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t tiles = (N + 32 * kSoTG - 1) / (32 * kSoTG);
    const int64_t grid = std::min<int64_t>(tiles, sm_count());
    void *args[] = {&k};
    TMB_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(kSoThreads), args, smem, st));
    TMB_LAUNCHED();
    *launched = true;
    return TMB_OK;
}

}  // namespace tmb
