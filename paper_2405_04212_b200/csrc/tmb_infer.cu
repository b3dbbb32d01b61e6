// tmb_infer.cu -- batched inference over compiled include lists
// (predictor.py:45-96 / dense.py:171-174 / executor.py:355-383).
//
// Bit-sliced evaluation: a CTA transposes a tile of 32*G examples' raw
// feature bytes into shared memory as X^T[feature][group] (one 32-bit word =
// one feature over 32 examples), then evaluates rules with
//     acc &= neg ? ~X^T[f][g] : X^T[f][g]
// so one LDS + one LOP3 tests one include literal for 32 examples at once,
// with early exit once all 32 examples violated the rule.  Votes of firing
// (rule, example) pairs accumulate in shared memory; the epilogue does the
// argmax (ties -> lowest class, np.argmax) and writes votes / predictions.
// HBM traffic is the raw input (F bytes per example) plus the outputs.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"
#include "tmb_infer.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace tmb {

struct InferK {
    const uint8_t *x;
    int64_t N, F;
    const uint32_t *inc;
    const int64_t *ptr;
    const int32_t *w;
    int R, K;
    int64_t *votes, *pred;
    const int64_t *labels;
    unsigned long long *correct;
    unsigned int *bad_input;
    int vec_ok;
};

template <int G>
__global__ void __launch_bounds__(512) k_infer(InferK k) {
    extern __shared__ __align__(16) char smem_raw[];
    uint32_t *xt = reinterpret_cast<uint32_t *>(smem_raw);                 // [F][G]
    int32_t *vt = reinterpret_cast<int32_t *>(xt + ((k.F * G + 3) & ~3LL));  // [32G][K]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int64_t tile_n = 32 * G;
    const int64_t n_tiles = (k.N + tile_n - 1) / tile_n;
    const int64_t nch = (k.F + 31) / 32;
    const int K = k.K;
    uint32_t bad = 0;
    unsigned long long hits = 0;
    for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        const int64_t e0 = tile * tile_n;
        // ---- transpose raw bytes -> X^T (one ballot per feature column)
        for (int64_t u = warp; u < nch * G; u += nwarps) {
            const int g = (int)(u % G);
            const int64_t c = (u / G) * 32;
            const int64_t e = e0 + 32 * g + lane;
            uint32_t v[8];
            if (e < k.N && k.vec_ok && c + 32 <= k.F) {
                const uint4 *src = reinterpret_cast<const uint4 *>(k.x + e * k.F + c);
                uint4 a = __ldcs(src), b = __ldcs(src + 1);
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
                v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
            } else {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    uint32_t word = 0;
                    for (int bb = 0; bb < 4; ++bb) {
                        int64_t col = c + q * 4 + bb;
                        uint32_t byte = (e < k.N && col < k.F) ? k.x[e * k.F + col] : 0u;
                        word |= byte << (8 * bb);
                    }
                    v[q] = word;
                }
            }
            uint32_t mine = 0;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                bad |= v[q] & 0xFEFEFEFEu;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                    uint32_t m = __ballot_sync(0xffffffffu, (v[q] >> (8 * bb)) & 1u);
                    if (lane == q * 4 + bb) mine = m;
                }
            }
            if (c + lane < k.F) xt[(c + lane) * G + g] = mine;
        }
        for (int i = tid; i < tile_n * K; i += blockDim.x) vt[i] = 0;
        __syncthreads();
        // ---- evaluate rules: lane = (rule slot, group)
        constexpr int S = 32 / G;
        const int slot = lane / G, g = lane % G;
        for (int rc = warp; rc * S < k.R; rc += nwarps) {
            const int r = rc * S + slot;
            if (r < k.R) {
                uint32_t acc = 0xffffffffu;
                int64_t q = __ldg(&k.ptr[r]);
                const int64_t qe = __ldg(&k.ptr[r + 1]);
                for (; q < qe; ++q) {
                    const uint32_t code = __ldg(&k.inc[q]);
                    const uint32_t xw = xt[(code >> 1) * G + g];
                    acc &= (code & 1u) ? ~xw : xw;
                    if (!acc) break;
                }
                if (acc) {
                    const int32_t *wr = k.w + (int64_t)r * K;
                    while (acc) {
                        const int b = __ffs(acc) - 1;
                        acc &= acc - 1;
                        int32_t *dst = vt + (g * 32 + b) * K;
                        for (int kk = 0; kk < K; ++kk) {
                            int32_t wv = __ldg(&wr[kk]);
                            if (wv) atomicAdd(&dst[kk], wv);
                        }
                    }
                }
            }
        }
        __syncthreads();
        // ---- epilogue: argmax (ties -> lowest class), outputs
        for (int t = tid; t < tile_n; t += blockDim.x) {
            const int64_t e = e0 + t;
            if (e >= k.N) continue;
            const int32_t *v = vt + t * K;
            int best = 0;
            int32_t bv = v[0];
            for (int kk = 1; kk < K; ++kk)
                if (v[kk] > bv) { bv = v[kk]; best = kk; }
            if (k.votes)
                for (int kk = 0; kk < K; ++kk) k.votes[e * K + kk] = (int64_t)v[kk];
            if (k.pred) k.pred[e] = best;
            if (k.labels) hits += (k.labels[e] == best);
        }
        __syncthreads();
    }
    if (k.correct) {
        for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
        if (lane == 0 && hits) atomicAdd(k.correct, hits);
    }
    if (bad) atomicOr(k.bad_input, 1u);
}

// ---------------------------------------------------------------------------
// Cluster kernel: CS = 4 CTAs per cluster split the rule set (each keeps the
// 16-code heads of its quarter resident in shared memory) and share one
// bit-transposed tile of TG*32 examples: CTA r transposes feature chunks
// [r*nch/4, (r+1)*nch/4) of the raw bytes and stores the X^T words into all
// four CTAs' shared memory (DSMEM).  Tiles are double-buffered so the next
// tile's HBM reads overlap the current tile's rule evaluation; partial class
// sums are pushed to the CTA that owns each 32-example block, which sums the
// four partials and writes votes / predictions.  One cluster barrier per tile.
constexpr int kCS = 4;   // CTAs per cluster
constexpr int kTG = 4;   // 32-example groups per tile

struct InferCK {
    const uint8_t *x;
    int64_t N, F;
    const uint16_t *heads;
    const int32_t *tail_ptr;
    const uint16_t *tails;
    const int32_t *w;
    int R, K;
    int64_t *votes, *pred;
    const int64_t *labels;
    unsigned long long *correct;
    unsigned int *bad_input;
    int vec_ok;
    int rloc_max;
    int dbg;  // bit0: skip eval, bit1: skip transpose (timing experiments only)
    unsigned long long *phase;  // optional [grid][8] clock64 per phase (thread 0)
    const uint64_t *xb;  // bit-packed input [N][W64] (feature f = bit f%64 of word f/64), or null
    int64_t W64;
    int xb_vec16;        // 16-byte loads legal (W64 even, base 16-B aligned)
    int eval_mode;       // k_infer_ws evaluators: 2 = loads of dead rules skipped from code
                         // 8 on (default), 3 = same without early-exit votes, 0 = plain
};

__global__ void __launch_bounds__(512, 1) k_infer_cluster(InferCK k) {
    extern __shared__ __align__(16) char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int K = k.K;
    const int64_t F = k.F;
    const int xrows = (int)F + 1;  // + all-ones row for padding codes
    // shared layout: heads | xt[2] | part | inbox[2][kCS][32][K]
    uint4 *heads = reinterpret_cast<uint4 *>(smem_raw);                       // [rloc][2]
    uint32_t *xt0 = reinterpret_cast<uint32_t *>(heads + 2 * (size_t)k.rloc_max);
    uint32_t *xt1 = xt0 + (size_t)xrows * kTG;
    int32_t *part = reinterpret_cast<int32_t *>(xt1 + (size_t)xrows * kTG);   // [32*kTG][K]
    int32_t *inbox = part + 32 * kTG * K;                                     // [2][kCS][32][K]
    int32_t *iflag = inbox + 2 * kCS * 32 * K;                                // [2][kCS]
    int32_t *dirty = iflag + 2 * kCS;                                         // [kTG]
    uint64_t *mbar = reinterpret_cast<uint64_t *>(
        reinterpret_cast<uintptr_t>(dirty + kTG + 3) & ~(uintptr_t)7);       // [2]

    const int r0 = (int)((int64_t)rank * k.R / kCS), r1 = (int)((int64_t)(rank + 1) * k.R / kCS);
    const int rloc = r1 - r0;
    for (int i = tid; i < rloc * 2; i += blockDim.x)
        heads[i] = reinterpret_cast<const uint4 *>(k.heads)[(size_t)r0 * 2 + i];
    // all-ones padding row in both buffers
    if (tid < kTG) {
        xt0[(size_t)F * kTG + tid] = 0xFFFFFFFFu;
        xt1[(size_t)F * kTG + tid] = 0xFFFFFFFFu;
    }

    const int64_t tile_n = 32 * kTG;
    const int64_t n_tiles = (k.N + tile_n - 1) / tile_n;
    const int n_clusters = gridDim.x / kCS;
    const int cid = blockIdx.x / kCS;
    const int nch = (int)((F + 31) / 32);
    const int ch0 = (int)((int64_t)rank * nch / kCS), ch1 = (int)((int64_t)(rank + 1) * nch / kCS);
    uint32_t bad = 0;
    unsigned long long hits = 0;

    // transpose this CTA's feature quarter of tile `t` into buffer `buf` of
    // every CTA in the cluster.  Unit = 32 examples (one group) x 128
    // features: 8 coalesced 16-byte loads per lane (4 rows x 128 B per
    // instruction), byte->bit packing, two in-register 8x8 bit transposes and
    // a 4-lane byte exchange leave each lane with 4 finished X^T words.
    const int64_t qf0 = (int64_t)ch0 * 32;
    const int64_t qf1 = std::min<int64_t>((int64_t)ch1 * 32, F);
    const int nblk = (int)((qf1 - qf0 + 127) / 128);
    auto transpose = [&](int64_t t, int buf) {
        const int64_t e0 = t * tile_n;
        uint32_t *mine = buf ? xt1 : xt0;
        const int j = lane >> 3, c16 = lane & 7;
        const int units = nblk * kTG;
        auto load_unit = [&](int u, uint4 (&w)[8], int64_t &fb_out) {
            const int g = u % kTG;
            const int64_t fb = qf0 + (int64_t)(u / kTG) * 128 + 16 * c16;  // my 16 features
            fb_out = fb;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t e = e0 + 32 * g + 8 * j + i;
                w[i] = make_uint4(0, 0, 0, 0);
                if (u < units && e < k.N && fb < qf1) {
                    const uint8_t *src = k.x + e * F + fb;
                    if (k.vec_ok && fb + 16 <= F) {
                        w[i] = *reinterpret_cast<const uint4 *>(src);
                    } else {
                        uint32_t b0 = 0, b1 = 0, b2 = 0, b3 = 0;
                        for (int bb = 0; bb < 16; ++bb) {
                            if (fb + bb >= F) break;
                            const uint32_t byte = (uint32_t)src[bb] << (8 * (bb & 3));
                            if (bb < 4) b0 |= byte;
                            else if (bb < 8) b1 |= byte;
                            else if (bb < 12) b2 |= byte;
                            else b3 |= byte;
                        }
                        w[i] = make_uint4(b0, b1, b2, b3);
                    }
                }
            }
        };
        auto finish_unit = [&](int u, const uint4 (&w)[8], int64_t fb) {
            const int g = u % kTG;
            uint32_t v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                bad |= (w[i].x | w[i].y | w[i].z | w[i].w) & 0xFEFEFEFEu;
                v[i] = pack4(w[i].x) | (pack4(w[i].y) << 4) | (pack4(w[i].z) << 8) |
                       (pack4(w[i].w) << 12);
            }
            unsigned long long lo = 0, hi = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                lo |= (unsigned long long)(v[i] & 0xFFu) << (8 * i);
                hi |= (unsigned long long)(v[i] >> 8) << (8 * i);
            }
            lo = transpose8x8(lo);
            hi = transpose8x8(hi);
            const uint32_t R0 = (uint32_t)lo, R1 = (uint32_t)(lo >> 32);
            const uint32_t R2 = (uint32_t)hi, R3 = (uint32_t)(hi >> 32);
            uint32_t recv[4];
#pragma unroll
            for (int sft = 0; sft < 4; ++sft) {
                const int d = j ^ sft;
                const uint32_t send = d == 0 ? R0 : d == 1 ? R1 : d == 2 ? R2 : R3;
                recv[sft] = sft ? __shfl_xor_sync(0xffffffffu, send, 8 * sft) : send;
            }
#pragma unroll
            for (int kq = 0; kq < 4; ++kq) {
                uint32_t word = 0;
#pragma unroll
                for (int sft = 0; sft < 4; ++sft)
                    word |= ((recv[sft] >> (8 * kq)) & 0xFFu) << (8 * (j ^ sft));
                const int64_t f = fb + 4 * j + kq;
                if (f < qf1) mine[(size_t)f * kTG + g] = word;
            }
        };
        for (int u = warp; u < units; u += 2 * nwarps) {
            uint4 wa[8], wb[8];
            int64_t fa, fbb;
            const int u2 = u + nwarps;
            load_unit(u, wa, fa);
            load_unit(u2, wb, fbb);  // both units' 16 loads in flight together
            finish_unit(u, wa, fa);
            if (u2 < units) finish_unit(u2, wb, fbb);
        }
    };

    // bulk L2 prefetch of this CTA's feature quarter of tile `t` (one TMA
    // bulk-prefetch per example row; no registers, no shared memory)
    auto prefetch_l2 = [&](int64_t t) {
        if (t >= n_tiles || !k.vec_ok || !(k.dbg & 8)) return;  // opt-in (measured no gain)
        const int64_t e0 = t * tile_n;
        const int64_t off = (int64_t)ch0 * 32;
        const int64_t len = std::min<int64_t>((int64_t)(ch1 - ch0) * 32, F - off);
        if (len <= 0) return;
        const unsigned bytes = (unsigned)(len & ~15LL);
        for (int i = tid; i < tile_n; i += blockDim.x) {
            const int64_t e = e0 + i;
            if (e < k.N && bytes)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(k.x + e * F + off),
                             "r"(bytes) : "memory");
        }
    };

    // rows [0, F) of every tile come from the four quarters; my peers send
    // (F - my quarter) rows x 16 B into each of my buffers per use
    const uint32_t my_bytes = (uint32_t)((qf1 > qf0 ? qf1 - qf0 : 0) * 16);
    const uint32_t expect_bytes = (uint32_t)(F * 16) - my_bytes;
    uint32_t parity[2] = {0, 0};
    // share this CTA's freshly transposed quarter of buffer `buf` with peers
    auto publish = [&](int buf) {
        __syncthreads();
        if (tid == 0 && my_bytes) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            const uint32_t src = smem_u32((buf ? xt1 : xt0) + (size_t)qf0 * kTG);
            for (int p = 0; p < kCS; ++p) {
                if (p == rank) continue;
                bulk_copy_to_peer(mapa_u32(src, p), src, my_bytes, mapa_u32(smem_u32(&mbar[buf]), p));
            }
        }
    };
    auto await_tile = [&](int buf) {
        if (expect_bytes) mbar_wait(&mbar[buf], parity[buf]);
        parity[buf] ^= 1u;
        __syncthreads();
        // re-arm for this buffer's next use (before the cluster barrier that
        // lets peers write into it again)
        if (tid == 0 && expect_bytes) mbar_arm(&mbar[buf], expect_bytes);
    };
    if (tid == 0) {
        mbar_init(&mbar[0], 1);
        mbar_init(&mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (expect_bytes) {
            mbar_arm(&mbar[0], expect_bytes);
            mbar_arm(&mbar[1], expect_bytes);
        }
    }
    cluster.sync();

    unsigned long long iph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long imark = clock64();
#define IPH(n)                                                            \
    do {                                                                  \
        if (k.phase && tid == 0) {                                        \
            const long long now = clock64();                              \
            iph[n] += (unsigned long long)(now - imark);                  \
            imark = now;                                                  \
        }                                                                 \
    } while (0)
    int64_t it = 0;
    int64_t t = cid;
    prefetch_l2(t);
    prefetch_l2(t + n_clusters);
    if (t < n_tiles) {
        transpose(t, 0);
        publish(0);
        await_tile(0);
    }
    for (; t < n_tiles; t += n_clusters, ++it) {
        const int buf = (int)(it & 1);
        const uint32_t *xt = buf ? xt1 : xt0;
        IPH(7);
        prefetch_l2(t + 2 * (int64_t)n_clusters);
        IPH(0);
        for (int i = tid; i < 32 * kTG * K; i += blockDim.x) part[i] = 0;
        if (tid < kTG) dirty[tid] = 0;
        __syncthreads();
        // ---- evaluate the local rules: one lane per rule; an include code
        //      reads the 16-byte X^T row of its feature = 128 examples
        const uint32_t xaddr = smem_u32(xt);  // explicit shared-window loads
        const uint32_t haddr = smem_u32(heads);
        for (int rc = warp; rc * 32 < rloc && !(k.dbg & 1); rc += nwarps) {
            const int r = rc * 32 + lane;
            const int rr = r < rloc ? r : 0;  // idle lanes still join the votes
            const uint32_t live = r < rloc ? 0xFFFFFFFFu : 0u;
            uint32_t a0 = live, a1 = live, a2 = live, a3 = live;
            const uint4 h0 = lds128(haddr + rr * 32), h1 = lds128(haddr + rr * 32 + 16);
            const uint32_t hw[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t c = hh ? (hw[q] >> 16) : (hw[q] & 0xFFFFu);
                    const uint4 x = lds128(xaddr + (c >> 1) * 16);
                    const uint32_t m = 0u - (c & 1u);
                    a0 &= x.x ^ m;
                    a1 &= x.y ^ m;
                    a2 &= x.z ^ m;
                    a3 &= x.w ^ m;
                }
                if (!__any_sync(0xffffffffu, a0 | a1 | a2 | a3)) break;
            }
            if ((a0 | a1 | a2 | a3) && r < rloc) {
                const int rg = r0 + r;
                for (int q = __ldg(&k.tail_ptr[rg]), qe = __ldg(&k.tail_ptr[rg + 1]);
                     q < qe && (a0 | a1 | a2 | a3); ++q) {
                    const uint32_t c = __ldg(&k.tails[q]);
                    const uint4 x = lds128(xaddr + (c >> 1) * 16);
                    const uint32_t m = 0u - (c & 1u);
                    a0 &= x.x ^ m;
                    a1 &= x.y ^ m;
                    a2 &= x.z ^ m;
                    a3 &= x.w ^ m;
                }
                const int32_t *wr = k.w + (size_t)rg * K;
#pragma unroll
                for (int gq = 0; gq < kTG; ++gq) {
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
            }
        }
        __syncthreads();
        IPH(1);
        // ---- push partial sums of example block b to CTA b's inbox; blocks
        //      where no local rule fired only send their (zero) flag
        for (int i = tid; i < 32 * kTG * K; i += blockDim.x) {
            const int b = i / (32 * K);  // example block == owning CTA
            if (!dirty[b]) continue;
            const int rem = i - b * 32 * K;
            int32_t *dst = cluster.map_shared_rank(inbox, b);
            dst[((buf * kCS + rank) * 32) * K + rem] = part[i];
        }
        if (tid < kCS) cluster.map_shared_rank(iflag, tid)[buf * kCS + rank] = dirty[tid];
        IPH(2);
        // ---- next tile's X^T (its raw rows were prefetched into L2)
        const int64_t tn = t + n_clusters;
        if (tn < n_tiles && !(k.dbg & 2)) {
            transpose(tn, buf ^ 1);
            IPH(3);
            publish(buf ^ 1);
        }
        IPH(4);
        cluster.sync();
        IPH(5);
        if (tn < n_tiles && !(k.dbg & 2)) await_tile(buf ^ 1);
        IPH(6);
        // ---- finalize the 32 examples of block `rank`
        if (warp == 0) {
            const int64_t e = t * tile_n + 32 * rank + lane;
            if (e < k.N) {
                int best = 0;
                int32_t bv = 0;
                for (int kk = 0; kk < K; ++kk) {
                    int32_t sum = 0;
#pragma unroll
                    for (int p = 0; p < kCS; ++p)
                        if (iflag[buf * kCS + p]) sum += inbox[((buf * kCS + p) * 32 + lane) * K + kk];
                    if (kk == 0 || sum > bv) { bv = sum; best = kk; }
                    if (k.votes) k.votes[e * K + kk] = (int64_t)sum;
                }
                if (k.pred) k.pred[e] = best;
                if (k.labels) hits += (k.labels[e] == best);
            }
        }
    }
    if (k.phase && tid == 0)
        for (int q = 0; q < 8; ++q) k.phase[blockIdx.x * 8 + q] = iph[q];
    cluster.sync();  // peers may still write into our buffers until here
    if (k.correct) {
        for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
        if (lane == 0 && hits) atomicAdd(k.correct, hits);
    }
    if (bad) atomicOr(k.bad_input, 1u);
}

// ---------------------------------------------------------------------------
// Warp-specialised cluster kernel (same cluster / tile / rule split as
// k_infer_cluster, same results): warps [0, 8) of every CTA only transpose
// (HBM -> X^T), warps [8, 16) only evaluate, so the HBM reads of tile t+1
// overlap the rule evaluation of tile t instead of alternating with it.
// Hand-offs are mbarriers, no cluster-wide barrier per tile:
//   full[b]   (per CTA)  local transposers arrive + 3 peers' bulk copies (tx)
//   empty[b]  (per CTA)  the 4 CTAs' evaluator groups are done with buffer b
//   vfull[b]  (owner)    the 4 CTAs pushed their partial sums for block b
//   vempty[b] (writer)   the 4 owners consumed this CTA's partials of slot b
// 5 warpgroups: warpgroups 0-1 re-allocated to 128 registers per thread
// (setmaxnreg) -- 7 transposer warps, whose loads in flight live in
// registers, and 1 evaluator warp -- and warpgroups 2-4 to 72 (11 more
// evaluators and the finalizer).  12 evaluator warps instead of 7 at a
// uniform 128.  Transposer warps measured per 2^22 configs[2] examples with
// the evaluators' tile barrier: 4: 8.74 ms, 5: 7.44, 6: 7.15, 7: 7.29,
// 8: 7.88; after the push moved to the finalizer and the barrier went:
// 6: 7.06, 7: 7.01, 8: 7.16.
#ifndef TMB_WS_THREADS
#define TMB_WS_THREADS 640
#endif
constexpr int kWsThreads = TMB_WS_THREADS;
#ifndef TMB_WS_REGS_T
#define TMB_WS_REGS_T 128
#endif
constexpr int kWsRegsT = TMB_WS_REGS_T;
// the rest of the 640 x 96 pool (warpgroups 2-4)
constexpr int kWsRegsE = kWsThreads == 768 ? 56
                       : kWsThreads == 640 ? ((61440 - 2 * 128 * kWsRegsT) / (3 * 128)) / 8 * 8
                                           : 128;

template <bool PACKED>
__global__ void __launch_bounds__(kWsThreads, 1) k_infer_ws(InferCK k) {
    // transposer warps per CTA (a multiple of kTG); the last warp finalizes,
    // the rest evaluate (11 evaluators for bit-packed input measured slower)
#ifndef TMB_WS_T
#define TMB_WS_T 7
#endif
    // bit-packed input: the transposer's 32x32 warp bit transposes cost more
    // per byte, 8 transposer warps measured best (6.8 vs 7.0 ms with 6)
    constexpr int kWsT = PACKED ? 8 : TMB_WS_T;
    static_assert(kWsT <= 8, "transposer warps must fit the two 128-register warpgroups");
    extern __shared__ __align__(16) char smem_raw[];
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int nE = nwarps - kWsT - 1;
    const int K = k.K;
    const int64_t F = k.F;
    const int xrows = (int)F + 1;
    // shared layout: heads | xt[2] | part | inbox[2][kCS][32][K] | iflag[2][kCS] | dirty | mbar[8]
    uint4 *heads = reinterpret_cast<uint4 *>(smem_raw);
    uint32_t *xt0 = reinterpret_cast<uint32_t *>(heads + 2 * (size_t)k.rloc_max);
    uint32_t *xt1 = xt0 + (size_t)xrows * kTG;
    // partial class sums, one set per X^T buffer: the evaluators of tile
    // it+1 accumulate while the finalizer warp pushes tile it's
    int32_t *part2 = reinterpret_cast<int32_t *>(xt1 + (size_t)xrows * kTG);  // [2][32*kTG][K]
    int32_t *inbox = part2 + 2 * 32 * kTG * K;                                // [2][kCS][32][K]
    int32_t *iflag = inbox + 2 * kCS * 32 * K;                               // [2][kCS]
    int32_t *dirty2 = iflag + 2 * kCS;                                       // [2][kTG]
    uint64_t *mb = reinterpret_cast<uint64_t *>(
        reinterpret_cast<uintptr_t>(dirty2 + 2 * kTG + 3) & ~(uintptr_t)7);  // [8]
    uint64_t *full = mb, *empty = mb + 2, *vfull = mb + 4, *vempty = mb + 6;
    uint64_t *efree = mb + 8;  // local: evaluators -> finalizer (tile evaluated)
    uint64_t *pfree = mb + 10; // local: finalizer -> evaluators (partials of the buffer pushed)
    int32_t *ectr = reinterpret_cast<int32_t *>(mb + 12);  // [2] next rule chunk (dynamic)

    const int r0 = (int)((int64_t)rank * k.R / kCS), r1 = (int)((int64_t)(rank + 1) * k.R / kCS);
    const int rloc = r1 - r0;
    for (int i = tid; i < rloc * 2; i += blockDim.x)
        heads[i] = reinterpret_cast<const uint4 *>(k.heads)[(size_t)r0 * 2 + i];
    if (tid < kTG) {
        xt0[(size_t)F * kTG + tid] = 0xFFFFFFFFu;
        xt1[(size_t)F * kTG + tid] = 0xFFFFFFFFu;
    }
    for (int i = tid; i < 2 * 32 * kTG * K; i += blockDim.x) part2[i] = 0;
    if (tid < 2 * kTG) dirty2[tid] = 0;
    if (tid < 2 * kCS) iflag[tid] = 0;
    if (tid < 2) ectr[tid] = 0;  // (mbarrier area is initialised below, before the cluster sync)

    const int64_t tile_n = 32 * kTG;
    const int64_t n_tiles = (k.N + tile_n - 1) / tile_n;
    const int n_clusters = gridDim.x / kCS;
    const int cid = blockIdx.x / kCS;
    const int nch = (int)((F + 31) / 32);
    const int ch0 = (int)((int64_t)rank * nch / kCS), ch1 = (int)((int64_t)(rank + 1) * nch / kCS);
    const int64_t qf0 = (int64_t)ch0 * 32;
    const int64_t qf1 = std::min<int64_t>((int64_t)ch1 * 32, F);
    const int nblk = (int)((qf1 - qf0 + 127) / 128);
    // debug bit 64 (timing experiment only, wrong results): no peer copies
    const uint32_t my_bytes = (k.dbg & 64) ? 0u : (uint32_t)((qf1 > qf0 ? qf1 - qf0 : 0) * 16);
    const uint32_t expect_bytes = (k.dbg & 64) ? 0u : (uint32_t)(F * 16) - my_bytes;
    if (tid == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&empty[0], kCS);
        mbar_init(&empty[1], kCS);
        mbar_init(&vfull[0], kCS);
        mbar_init(&vfull[1], kCS);
        mbar_init(&vempty[0], kCS);
        mbar_init(&vempty[1], kCS);
        mbar_init(&efree[0], nE);  // every evaluator warp arrives when its chunks are done
        mbar_init(&efree[1], nE);
        mbar_init(&pfree[0], 1);
        mbar_init(&pfree[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster.sync();
    const int64_t n_my = cid < n_tiles ? (n_tiles - cid + n_clusters - 1) / n_clusters : 0;
    uint32_t bad = 0;
    unsigned long long hits = 0;
    // phase profile (k.phase): thread 0 = transposer slots 0..3, thread
    // 32*kWsT = evaluator slots 4..7
    const bool prof = k.phase && (tid == 0 || tid == 32 * kWsT);
    unsigned long long wph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long wmark = clock64();
#define WPH(n)                                                            \
    do {                                                                  \
        if (prof) {                                                       \
            const long long now = clock64();                              \
            wph[n] += (unsigned long long)(now - wmark);                  \
            wmark = now;                                                  \
        }                                                                 \
    } while (0)

    if (kWsThreads > 512) {
        if (warp < 8)  // warpgroups 0-1 (transposers; evaluators if kWsT < 8)
            asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kWsRegsT));
        else
            asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kWsRegsE));
    }
    if (PACKED && warp < kWsT) {
        // ========== transposer group, bit-packed input ==========
        // unit = 32 examples x 256 features: lane l holds 256 feature bits
        // of example 32g + l (two 16-byte loads); eight 32x32 warp bit
        // transposes leave lane j with the X^T words of features fb+32q+j.
        const int units = (int)((qf1 - qf0 + 255) / 256) * kTG;
        const int nq = units > warp ? (units - warp + kWsT - 1) / kWsT : 0;
        // unit U = warp + q*kWsT: example group U % kTG, feature block U / kTG
        auto ug = [&](int q) { return (warp + q * kWsT) % kTG; };
        auto ufb = [&](int q) { return qf0 + (int64_t)((warp + q * kWsT) / kTG) * 256; };
        auto load_p = [&](int64_t itx, int q, uint32_t (&w)[8]) {
            const int64_t e = (cid + itx * n_clusters) * tile_n + 32 * ug(q) + lane;
            const int64_t fb = ufb(q);
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = 0;
            if (e >= k.N || fb >= qf1) return;
            // the row as little-endian 32-bit words: word fb/32 holds
            // features fb..fb+31 (quarter starts are multiples of 32)
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
                const uint32_t x = warp_transpose32(w[qq], lane);
                const int64_t f = fb + 32 * qq + lane;
                if (f < qf1) mine[(size_t)f * kTG + g] = x;
            }
        };
        auto tile_end_p = [&](int64_t it) {
            const int buf = (int)(it & 1);
            uint32_t *mine = buf ? xt1 : xt0;
            named_sync(1, 32 * kWsT);
            if (tid == 0) {
                if (my_bytes) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const uint32_t src = smem_u32(mine + (size_t)qf0 * kTG);
                    for (int p = 0; p < kCS; ++p) {
                        if (p == rank) continue;
                        bulk_copy_to_peer(mapa_u32(src, p), src, my_bytes,
                                          mapa_u32(smem_u32(&full[buf]), p));
                    }
                }
                if (expect_bytes) mbar_arm(&full[buf], expect_bytes);
                else mbar_arrive_local(&full[buf]);
            }
        };
        uint32_t wa[8], wb[8];
        for (int64_t it = 0; it < n_my; ++it) {
            const int buf = (int)(it & 1);
            uint32_t *mine = buf ? xt1 : xt0;
            if (it >= 2) mbar_wait(&empty[buf], (uint32_t)(((it >> 1) + 1) & 1));
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
            tile_end_p(it);
        }
    } else if (!PACKED && warp < kWsT) {
        const int j = lane >> 3, c16 = lane & 7;
        const int units = nblk * kTG;
        const int nq = units > warp ? (units - warp + kWsT - 1) / kWsT : 0;
        // unit U = warp + q*kWsT: example group U % kTG, feature block U / kTG
        auto ug = [&](int q) { return (warp + q * kWsT) % kTG; };
        auto ufb = [&](int q) {
            return qf0 + (int64_t)((warp + q * kWsT) / kTG) * 128 + 16 * c16;
        };
        const uint32_t psel = (uint32_t)(j | ((1 ^ j) << 4) | ((2 ^ j) << 8) | ((3 ^ j) << 12));
        const bool do_t = !(k.dbg & 2);
        // item (tile itx, unit q): my 8 rows x 16 bytes
        auto load_item = [&](int64_t itx, int q, uint4 (&w)[8]) {
            const int64_t er = (cid + itx * n_clusters) * tile_n + 32 * ug(q) + 8 * j;
            const int64_t fb = ufb(q);
            if (k.vec_ok && fb + 16 <= qf1 && er + 7 < k.N) {
                const uint8_t *src = k.x + er * F + fb;
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = __ldcs(reinterpret_cast<const uint4 *>(src + i * F));
                return;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int64_t e = er + i;
                w[i] = make_uint4(0, 0, 0, 0);
                if (e < k.N && fb < qf1) {
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
            // bytes are 0/1 (anything else is flagged and aborts the call),
            // so OR-ing row i shifted by i builds, in byte b of R_d, the 8
            // row bits of feature 4d + b: the byte -> bit transpose is 7
            // shift-adds per word
            uint32_t R[4], ob = 0;
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                uint32_t acc = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint32_t x = d == 0 ? w[i].x : d == 1 ? w[i].y : d == 2 ? w[i].z : w[i].w;
                    ob |= x;
                    acc |= x << i;
                }
                R[d] = acc;
            }
            bad |= ob & 0xFEFEFEFEu;
            // R[d] <- R[d ^ j] by two masked swap stages (a select chain on
            // the lane-dependent index compiles to divergent branches)
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
            // 4x4 byte transpose (word kq gathers byte kq of recv[0..3]),
            // then byte p <- byte p^j (recv[s] came from lane j^s)
            const uint32_t t0 = __byte_perm(recv[0], recv[1], 0x5140);
            const uint32_t t1 = __byte_perm(recv[2], recv[3], 0x5140);
            const uint32_t t2 = __byte_perm(recv[0], recv[1], 0x7362);
            const uint32_t t3 = __byte_perm(recv[2], recv[3], 0x7362);
            uint32_t wq[4];
            wq[0] = __byte_perm(__byte_perm(t0, t1, 0x5410), 0, psel);
            wq[1] = __byte_perm(__byte_perm(t0, t1, 0x7632), 0, psel);
            wq[2] = __byte_perm(__byte_perm(t2, t3, 0x5410), 0, psel);
            wq[3] = __byte_perm(__byte_perm(t2, t3, 0x7632), 0, psel);
            // store round r writes feature 4j + ((r + c16) & 3): the 32
            // lanes of one store then cover all 8 bank quads of the 16-byte
            // rows (4-way instead of 16-way bank conflicts).  wq is rotated
            // by c16 & 3 with masked selects (no lane-dependent indexing).
            {
                const uint32_t m1 = 0u - (uint32_t)(c16 & 1), m2 = 0u - (uint32_t)((c16 >> 1) & 1);
                const uint32_t a0 = (wq[0] & ~m1) | (wq[1] & m1), a1 = (wq[1] & ~m1) | (wq[2] & m1);
                const uint32_t a2 = (wq[2] & ~m1) | (wq[3] & m1), a3 = (wq[3] & ~m1) | (wq[0] & m1);
                wq[0] = (a0 & ~m2) | (a2 & m2);
                wq[1] = (a1 & ~m2) | (a3 & m2);
                wq[2] = (a2 & ~m2) | (a0 & m2);
                wq[3] = (a3 & ~m2) | (a1 & m2);
            }
            uint32_t *dst0 = mine + (size_t)(fb + 4 * j) * kTG + g;
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int kq = (r + c16) & 3;
                if (fb + 4 * j + kq < qf1) dst0[kq * kTG] = wq[r];
            }
        };
        auto tile_begin = [&](int64_t it) {
            WPH(3);
            // empty[] arrivals publish nothing: a CTA-scope wait (a cluster-
            // scope acquire would invalidate L1 on every tile)
            if (it >= 2) mbar_wait(&empty[it & 1], (uint32_t)(((it >> 1) + 1) & 1));
            WPH(0);
        };
        auto tile_end = [&](int64_t it) {
            const int buf = (int)(it & 1);
            uint32_t *mine = buf ? xt1 : xt0;
            WPH(1);
            named_sync(1, 32 * kWsT);
            if (tid == 0) {
                // my quarter to the 3 peers (complete_tx on their full[buf]),
                // then my own arrival (+ the bytes the peers will send me).
                // (Copying each feature block as soon as a round of units
                // completes it needs a transposer barrier per round, which
                // stalls the load pipeline: 9.1 vs 7.0 ms, measured.)
                if (my_bytes) {
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                    const uint32_t src = smem_u32(mine + (size_t)qf0 * kTG);
                    for (int p = 0; p < kCS; ++p) {
                        if (p == rank) continue;
                        bulk_copy_to_peer(mapa_u32(src, p), src, my_bytes,
                                          mapa_u32(smem_u32(&full[buf]), p));
                    }
                }
                if (expect_bytes) mbar_arm(&full[buf], expect_bytes);
                else mbar_arrive_local(&full[buf]);
            }
            WPH(2);
        };
        if (!do_t || nq == 0) {
            for (int64_t it = 0; it < n_my; ++it) {
                tile_begin(it);
                tile_end(it);
            }
        } else {
            // items in order (it, q); A / B alternate, the next item's loads
            // go out before the current item is transposed
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
            if (n_my > 0) load_item(0, 0, wa);
            while (ia < n_my) {
                next_of(ia, qa, ib, qb);
                if (ib < n_my) load_item(ib, qb, wb);
                if (qa == 0) tile_begin(ia);
                finish_item(wa, qa, (ia & 1) ? xt1 : xt0);
                if (qa == nq - 1) tile_end(ia);
                if (ib >= n_my) break;
                next_of(ib, qb, ia, qa);
                if (ia < n_my) load_item(ia, qa, wa);
                if (qb == 0) tile_begin(ib);
                finish_item(wb, qb, (ib & 1) ? xt1 : xt0);
                if (qb == nq - 1) tile_end(ib);
            }
        }
    } else if (warp == nwarps - 1) {
        // ================= finalizer warp =================
        // the 32 examples of block `rank` of every tile: wait for the four
        // CTAs' partials (slot = tile parity), sum, argmax, write, release
        for (int64_t it = 0; it < n_my; ++it) {
            const int64_t t = cid + it * n_clusters;
            const int buf = (int)(it & 1);
            const uint32_t par = (uint32_t)((it >> 1) & 1);
            // the evaluators are done with tile it (part / dirty of buffer buf
            // are final): push the partial sums of example block b to owner
            // b's inbox slot `buf` once the owners consumed that slot (tile
            // it-2) -- the evaluators move on to tile it+1 meanwhile
            mbar_wait(&efree[buf], par);
            // X^T buffer `buf` is free as far as this CTA is concerned:
            // forward to all four transposer groups at once (the partials
            // have their own release, pfree, below)
            if (lane < kCS) mbar_arrive_remote_relaxed(mapa_u32(smem_u32(&empty[buf]), lane));
            int32_t *pbuf = part2 + buf * 32 * kTG * K;
            int32_t *dbuf = dirty2 + buf * kTG;
            const int pm = dbuf[0] | (dbuf[1] << 1) | (dbuf[2] << 2) | (dbuf[3] << 3);
            if (it >= 2) mbar_wait(&vempty[buf], (uint32_t)(((it >> 1) + 1) & 1));
            if (pm) {
                for (int i = lane; i < 32 * kTG * K; i += 32) {
                    const int b = i / (32 * K);
                    if (!((pm >> b) & 1)) continue;
                    const int rem = i - b * 32 * K;
                    int32_t *dst = cluster.map_shared_rank(inbox, b);
                    dst[((buf * kCS + rank) * 32) * K + rem] = pbuf[i];
                    pbuf[i] = 0;
                }
                if (lane < kCS && ((pm >> lane) & 1))
                    cluster.map_shared_rank(iflag, lane)[buf * kCS + rank] = (int)(it + 1);  // tile tag
            }
            if (lane < kTG) dbuf[lane] = 0;  // next used by tile it+2
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&pfree[buf]);  // tile it+2's evaluators may accumulate
            // forward "partials pushed" to the 4 owners; blocks that received
            // partials need a releasing arrival (this warp's DSMEM stores)
            if (lane < kCS) {
                const uint32_t vb = mapa_u32(smem_u32(&vfull[buf]), lane);
                if ((pm >> lane) & 1) mbar_arrive_remote(vb);
                else mbar_arrive_remote_relaxed(vb);
            }
            // the partials are DSMEM stores into this CTA's shared memory,
            // performed before the writers' releasing arrivals: a CTA-scope
            // wait sees them (a cluster-scope acquire adds an L1 invalidate
            // per tile).  iflag slots carry the tile's tag (it + 1), so they
            // are never reset and need no release on the way back.
            mbar_wait(&vfull[buf], par);
            const int tag = (int)(it + 1);
            const int64_t e = t * tile_n + 32 * rank + lane;
            const bool any = iflag[buf * kCS + 0] == tag || iflag[buf * kCS + 1] == tag ||
                             iflag[buf * kCS + 2] == tag || iflag[buf * kCS + 3] == tag;
            if (e < k.N) {
                int best = 0;
                if (any || k.votes) {
                    int32_t bv = 0;
                    for (int kk = 0; kk < K; ++kk) {
                        int32_t sum = 0;
#pragma unroll
                        for (int p = 0; p < kCS; ++p)
                            if (iflag[buf * kCS + p] == tag)
                                sum += inbox[((buf * kCS + p) * 32 + lane) * K + kk];
                        if (kk == 0 || sum > bv) {
                            bv = sum;
                            best = kk;
                        }
                        if (k.votes) k.votes[e * K + kk] = (int64_t)sum;
                    }
                }
                if (k.pred) k.pred[e] = best;  // all sums 0 -> class 0 (np.argmax)
                if (k.labels) hits += (k.labels[e] == best);
            }
            __syncwarp();
            if (lane < kCS) mbar_arrive_remote_relaxed(mapa_u32(smem_u32(&vempty[buf]), lane));
        }
    } else {
        // ================= evaluator group =================
        const int ew = warp - kWsT;
        const uint32_t haddr = smem_u32(heads);
        for (int64_t it = 0; it < n_my; ++it) {
            const int buf = (int)(it & 1);
            const uint32_t *xt = buf ? xt1 : xt0;
            int32_t *dirty = dirty2 + buf * kTG;
            int32_t *part = part2 + buf * 32 * kTG * K;
            WPH(6);
            // the peers' quarters arrive by bulk copy (complete_tx), so the
            // phase completion makes them visible: CTA-scope wait
            mbar_wait(&full[buf], (uint32_t)((it >> 1) & 1));
            // the finalizer has pushed (and zeroed) tile it-2's partials of
            // this buffer -- normally long before the transposers are done
            if (it >= 2) mbar_wait(&pfree[buf], (uint32_t)(((it >> 1) + 1) & 1));
            WPH(4);
            const uint32_t xaddr = smem_u32(xt);
            // a rule's tail codes (CSR, global) and its votes into part[]
            auto finish_rule = [&](int r, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3) {
                const int rg = r0 + r;
                for (int q = __ldg(&k.tail_ptr[rg]), qe = __ldg(&k.tail_ptr[rg + 1]);
                     q < qe && (a0 | a1 | a2 | a3); ++q) {
                    const uint32_t c = __ldg(&k.tails[q]);
                    const uint4 x = lds128(xaddr + (c >> 1) * 16);
                    const uint32_t m = 0u - (c & 1u);
                    a0 &= x.x ^ m;
                    a1 &= x.y ^ m;
                    a2 &= x.z ^ m;
                    a3 &= x.w ^ m;
                }
                const int32_t *wr = k.w + (size_t)rg * K;
#pragma unroll
                for (int gq = 0; gq < kTG; ++gq) {
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
            // two rules per lane (rc*64 + lane and +32): two independent
            // shared-memory chains, early-exit vote every 4 codes
            // 64-rule chunks handed out dynamically: early exits make chunk
            // costs uneven, and a static split left the evaluator barrier
            // waiting ~0.7 us per tile for the slowest warp
            const int n_chunks = (rloc + 63) / 64;
            const uint32_t ebase = (uint32_t)(it >> 1) * (uint32_t)n_chunks;
            for (int rc = ew;;) {
                if (rc * 64 >= rloc || (k.dbg & 1)) break;
                const int rA = rc * 64 + lane, rB = rA + 32;
                const uint32_t lA = rA < rloc ? 0xFFFFFFFFu : 0u, lB = rB < rloc ? 0xFFFFFFFFu : 0u;
                uint32_t A0 = lA, A1 = lA, A2 = lA, A3 = lA, B0 = lB, B1 = lB, B2 = lB, B3 = lB;
                const uint32_t hA = haddr + (rA < rloc ? rA : 0) * 32;
                const uint32_t hB = haddr + (rB < rloc ? rB : 0) * 32;
                const uint4 ha0 = lds128(hA), ha1 = lds128(hA + 16);
                const uint4 hb0 = lds128(hB), hb1 = lds128(hB + 16);
                const uint32_t wa[8] = {ha0.x, ha0.y, ha0.z, ha0.w, ha1.x, ha1.y, ha1.z, ha1.w};
                const uint32_t wb[8] = {hb0.x, hb0.y, hb0.z, hb0.w, hb1.x, hb1.y, hb1.z, hb1.w};
                // mode 2: rules already dead for all 128 examples skip their
                // loads from code 8 on (fewer shared-memory wavefronts), and
                // the first exit check is after code 8
                const bool pred2 = k.eval_mode >= 2;
                const bool no_exit = k.eval_mode == 3;  // all 16 head codes, no warp vote
                uint4 xa_prev = make_uint4(0, 0, 0, 0), xb_prev = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int grp = 0; grp < 4; ++grp) {
                    const bool la = !pred2 || grp < 2 || (A0 | A1 | A2 | A3);
                    const bool lb = !pred2 || grp < 2 || (B0 | B1 | B2 | B3);
#pragma unroll
                    for (int q = 2 * grp; q < 2 * grp + 2; ++q) {
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const uint32_t ca = hh ? (wa[q] >> 16) : (wa[q] & 0xFFFFu);
                            const uint32_t cb = hh ? (wb[q] >> 16) : (wb[q] & 0xFFFFu);
                            // a dead rule's accumulator stays 0 whatever it is
                            // ANDed with: its load is skipped, stale registers reused
                            uint4 xa = xa_prev, xb = xb_prev;
                            lds128_if(xa, la, xaddr + (ca >> 1) * 16);
                            lds128_if(xb, lb, xaddr + (cb >> 1) * 16);
                            xa_prev = xa;
                            xb_prev = xb;
                            const uint32_t ma = 0u - (ca & 1u), mb2 = 0u - (cb & 1u);
                            A0 &= xa.x ^ ma;
                            A1 &= xa.y ^ ma;
                            A2 &= xa.z ^ ma;
                            A3 &= xa.w ^ ma;
                            B0 &= xb.x ^ mb2;
                            B1 &= xb.y ^ mb2;
                            B2 &= xb.z ^ mb2;
                            B3 &= xb.w ^ mb2;
                        }
                    }
                    if ((!pred2 || grp > 0) && !no_exit &&
                        !__any_sync(0xffffffffu, A0 | A1 | A2 | A3 | B0 | B1 | B2 | B3))
                        break;
                    if ((k.dbg & 32) && grp == 1) break;  // timing experiment only
                }
                if ((A0 | A1 | A2 | A3) && rA < rloc) finish_rule(rA, A0, A1, A2, A3);
                if ((B0 | B1 | B2 | B3) && rB < rloc) finish_rule(rB, B0, B1, B2, B3);
                int nx = 0;
                // ectr[buf] is never reset: each use of the buffer advances it
                // by exactly n_chunks (one atomic per evaluated chunk), so use
                // u = it >> 1 numbers its chunks from u * n_chunks
                if (lane == 0) nx = nE + (int)(atom_add_shared(&ectr[buf], 1u) - ebase);
                rc = __shfl_sync(0xffffffffu, nx, 0);
            }
            WPH(5);
            // this warp's share of tile it is evaluated: arrive (releasing its
            // lanes' partial-sum atomics, ordered by the warp barrier) and go
            // on to tile it+1 without waiting for the other evaluator warps.
            // When all have arrived, the finalizer warp pushes the partials
            // and forwards the buffer to the transposers (a remote arrival
            // stalls the issuing warp ~0.7 us).
            __syncwarp();
            if (lane == 0) mbar_arrive_local(&efree[buf]);
            WPH(7);
        }
    }
    if (prof && tid == 0)
        for (int q = 0; q < 4; ++q) k.phase[blockIdx.x * 8 + q] = wph[q];
    if (prof && tid == 32 * kWsT)
        for (int q = 4; q < 8; ++q) k.phase[blockIdx.x * 8 + q] = wph[q];
#undef WPH
    cluster.sync();  // peers may still copy into / signal this CTA until here
    if (k.correct) {
        for (int o = 16; o; o >>= 1) hits += __shfl_xor_sync(0xffffffffu, hits, o);
        if (lane == 0 && hits) atomicAdd(k.correct, hits);
    }
    if (bad) atomicOr(k.bad_input, 1u);
}


// ---------------------------------------------------------------------------
// Batched predict_and_explain (predictor.py:99-124): one warp per example.
// Pass 1: lane per rule tests the includes against the example's feature
// bytes (staged in shared memory), marks firing rules and adds their weights
// to the class sums; argmax (ties -> lowest).  Pass 2: every firing rule adds
// its weight for the explained class to each literal position it includes
// (int64 atomics into the example's score row, zeroed first).
struct ExplainK {
    const uint8_t *x;
    int64_t N, F;
    const uint32_t *inc;
    const int64_t *ptr;
    const int32_t *w;
    int R, K, negations, for_class;
    int64_t *votes, *pred, *scores;
};

__global__ void __launch_bounds__(256) k_explain(ExplainK k) {
    extern __shared__ __align__(16) char smem_raw[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t F = k.F, P = k.negations ? 2 * F : F;
    const int fire_words = (k.R + 31) / 32;
    // per warp: votes [K] int64 | fire bits [fire_words] | feature bytes [F]
    const size_t per = 8 * (size_t)k.K + 4 * (size_t)fire_words + (size_t)((F + 15) & ~15LL);
    char *mine = smem_raw + (size_t)wib * ((per + 15) & ~(size_t)15);
    long long *sv = reinterpret_cast<long long *>(mine);
    unsigned *fire = reinterpret_cast<unsigned *>(mine + 8 * (size_t)k.K);
    uint8_t *xr = reinterpret_cast<uint8_t *>(mine + 8 * (size_t)k.K + 4 * (size_t)fire_words);
    for (int64_t e = (int64_t)blockIdx.x * nw + wib; e < k.N; e += (int64_t)gridDim.x * nw) {
        for (int q = lane; q < k.K; q += 32) sv[q] = 0;
        for (int q = lane; q < fire_words; q += 32) fire[q] = 0;
        for (int64_t f = lane; f < F; f += 32) xr[f] = k.x[e * F + f];
        int64_t *srow = k.scores ? k.scores + e * P : nullptr;
        if (srow)
            for (int64_t p = lane; p < P; p += 32) srow[p] = 0;
        __syncwarp();
        for (int r = lane; r < k.R; r += 32) {
            const int64_t q0 = k.ptr[r], q1 = k.ptr[r + 1];
            bool f = q1 > q0;  // inference: a rule without includes never fires
            for (int64_t q = q0; q < q1 && f; ++q) {
                const uint32_t c = k.inc[q];
                const uint8_t v = xr[c >> 1];
                f = (c & 1u) ? v == 0 : v != 0;
            }
            if (f) {
                atomicOr(&fire[r >> 5], 1u << (r & 31));
                for (int kk = 0; kk < k.K; ++kk) {
                    const int32_t wv = k.w[(size_t)r * k.K + kk];
                    if (wv) atomicAdd(reinterpret_cast<unsigned long long *>(&sv[kk]),
                                      (unsigned long long)(long long)wv);
                }
            }
        }
        __syncwarp();
        int best = 0;
        long long bv = sv[0];
        for (int kk = 1; kk < k.K; ++kk)
            if (sv[kk] > bv) {
                bv = sv[kk];
                best = kk;
            }
        if (lane == 0 && k.pred) k.pred[e] = best;
        if (k.votes)
            for (int kk = lane; kk < k.K; kk += 32) k.votes[e * k.K + kk] = sv[kk];
        const int cls = k.for_class >= 0 ? k.for_class : best;
        if (srow) {
            for (int r = lane; r < k.R; r += 32) {
                if (!((fire[r >> 5] >> (r & 31)) & 1u)) continue;
                const long long wv = k.w[(size_t)r * k.K + cls];
                if (!wv) continue;
                for (int64_t q = k.ptr[r]; q < k.ptr[r + 1]; ++q) {
                    const uint32_t c = k.inc[q];
                    const int64_t p = (c & 1u) ? F + (c >> 1) : (int64_t)(c >> 1);
                    atomicAdd(reinterpret_cast<unsigned long long *>(&srow[p]),
                              (unsigned long long)wv);
                }
            }
        }
        __syncwarp();
    }
}

static unsigned int *g_bad_flag = nullptr;

static int pick_g(int64_t F, int64_t K, int max_smem, int *G_out, size_t *smem_out) {
    for (int G : {8, 4, 2, 1}) {
        size_t bytes = 4 * (size_t)((F * G + 3) & ~3LL) + 4 * (size_t)(32 * G) * K;
        if (bytes <= (size_t)max_smem) {
            *G_out = G;
            *smem_out = bytes;
            return TMB_OK;
        }
    }
    return fail(TMB_E_UNSUPPORTED, "infer: feature width too large for one tile in shared memory");
}

static int launch_infer_cluster(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes,
                                int64_t *pred, const int64_t *labels,
                                unsigned long long *correct, cudaStream_t st, bool *launched,
                                const uint64_t *xb = nullptr, int64_t W64 = 0);

int g_force_generic_infer = 0;
int g_infer_dbg = 0;
int g_infer_ws = 1;  // tmb_set_option("infer.warp_specialized", 0|1)
int g_infer_eval = 2;  // tmb_set_option("infer.eval_mode", 0|2|3): k_infer_ws evaluator
extern unsigned long long *g_sparse_phase;  // tmb_sparse.cu
extern int g_sparse_resident;                // tmb_sparse.cu
extern int g_sparse_infer_key;               // tmb_sparse.cu
extern int g_sparse_cnt32;                   // tmb_sparse.cu
unsigned long long *g_infer_phase = nullptr;

int launch_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes, int64_t *pred,
                 const int64_t *labels, unsigned long long *correct, cudaStream_t st) {
    if (N == 0) return TMB_OK;
    if (!g_bad_flag) {
        TMB_CUDA(cudaMalloc(&g_bad_flag, sizeof(unsigned)));
        TMB_CUDA(cudaMemset(g_bad_flag, 0, sizeof(unsigned)));
    }
    if (!g_force_generic_infer && r->sheads_ok) {
        bool launched = false;
        int rc = launch_infer_solo(r, x, nullptr, 0, N, votes, pred, labels, correct, g_bad_flag,
                                   st, &launched);
        if (rc || launched) return rc;
    }
    if (!g_force_generic_infer && r->heads_ok) {
        bool launched = false;
        int rc = launch_infer_cluster(r, x, N, votes, pred, labels, correct, st, &launched);
        if (rc || launched) return rc;
    }
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    int G;
    size_t smem;
    int rc = pick_g(r->F, r->K, std::min(max_smem, 200 * 1024), &G, &smem);
    if (rc) return rc;
    InferK k;
    k.x = x; k.N = N; k.F = r->F; k.inc = r->inc; k.ptr = r->ptr; k.w = r->weights;
    k.R = (int)r->R; k.K = (int)r->K; k.votes = votes; k.pred = pred; k.labels = labels;
    k.correct = correct; k.bad_input = g_bad_flag;
    k.vec_ok = (r->F % 16 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
    const int threads = 512;
    int64_t tiles = (N + 32 * G - 1) / (32 * G);
    const void *fn = G == 8 ? (const void *)k_infer<8> : G == 4 ? (const void *)k_infer<4>
                   : G == 2 ? (const void *)k_infer<2> : (const void *)k_infer<1>;
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    TMB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem));
    int64_t grid = std::min<int64_t>(tiles, (int64_t)sm_count() * std::max(per_sm, 1));
    void *args[] = {&k};
    TMB_CUDA(cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(threads), args, smem, st));
    TMB_LAUNCHED();
    return TMB_OK;
}

static int launch_infer_cluster(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes,
                                int64_t *pred, const int64_t *labels,
                                unsigned long long *correct, cudaStream_t st, bool *launched,
                                const uint64_t *xb, int64_t W64) {
    *launched = false;
    if (r->K > 32 || r->R < 1) return TMB_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const int64_t rloc_max = (r->R + kCS - 1) / kCS;
    const bool ws_kernel = xb || g_infer_ws;
    const size_t smem = 32 * (size_t)rloc_max + 2 * 4 * (size_t)(r->F + 1) * kTG +
                        (ws_kernel ? 2 : 1) * 4 * (size_t)32 * kTG * r->K +
                        4 * (size_t)2 * kCS * 32 * r->K + 4 * (2 * kCS + 2 * kTG) + 176;
    if (smem > (size_t)max_smem) return TMB_OK;  // generic kernel instead
    InferCK k;
    k.x = x; k.N = N; k.F = r->F; k.heads = r->heads; k.tail_ptr = r->tail_ptr; k.tails = r->tails;
    k.w = r->weights; k.R = (int)r->R; k.K = (int)r->K; k.votes = votes; k.pred = pred;
    k.labels = labels; k.correct = correct; k.bad_input = g_bad_flag;
    k.vec_ok = (r->F % 16 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0);
    k.rloc_max = (int)rloc_max;
    k.dbg = g_infer_dbg;
    k.phase = g_infer_phase;
    k.xb = xb;
    k.W64 = W64;
    k.xb_vec16 = xb && (W64 % 2 == 0) && (reinterpret_cast<uintptr_t>(xb) % 16 == 0);
    k.eval_mode = g_infer_eval;
    const bool ws = k.xb || g_infer_ws;
    const void *fn = k.xb ? (const void *)k_infer_ws<true>
                   : g_infer_ws ? (const void *)k_infer_ws<false> : (const void *)k_infer_cluster;
    TMB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = ws ? kWsThreads : 512;
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.gridDim = dim3(kCS);
    int max_clusters = 0;
    if (cudaOccupancyMaxActiveClusters(&max_clusters, fn, &lc) != cudaSuccess || max_clusters < 1) {
        cudaGetLastError();
        return TMB_OK;
    }
    const int64_t tiles = (N + 32 * kTG - 1) / (32 * kTG);
    const int64_t n_clusters = std::min<int64_t>(tiles, max_clusters);
    lc.gridDim = dim3((unsigned)(n_clusters * kCS));
    void *args[] = {&k};
    TMB_CUDA(cudaLaunchKernelExC(&lc, fn, args));
    TMB_LAUNCHED();
    *launched = true;
    return TMB_OK;
}

int check_bad_input(cudaStream_t st) {
    if (!g_bad_flag) return TMB_OK;
    unsigned v = 0;
    TMB_CUDA(cudaMemcpyAsync(&v, g_bad_flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaStreamSynchronize(st));
    if (v) {
        cudaMemsetAsync(g_bad_flag, 0, sizeof(unsigned), st);
        return fail(TMB_E_INVALID, "infer: input features must be 0/1 bytes");
    }
    return TMB_OK;
}

}  // namespace tmb

using namespace tmb;


// Build the 16-code heads (and CSR tails) of every rule.  A conjunction is
// order-independent, so within every 32-rule chunk that one warp of the
// cluster kernel evaluates together (chunks restart at each CTA's rule-slice
// boundary), the includes placed at head position q are chosen greedily so
// the 32 X^T rows read at that step spread over the 8 shared-memory bank
// quads (row f occupies quad f mod 8): fewer bank conflicts, same result.
static void balance_heads(const std::vector<int64_t> &ptr, const std::vector<uint32_t> &inc,
                          int64_t R, int64_t F, std::vector<uint16_t> &heads,
                          std::vector<int32_t> &tptr, std::vector<uint16_t> &tails) {
    std::vector<std::vector<uint32_t>> left((size_t)R);
    for (int64_t i = 0; i < R; ++i) left[i].assign(inc.begin() + ptr[i], inc.begin() + ptr[i + 1]);
    for (int rank = 0; rank < kCS; ++rank) {
        const int64_t s0 = rank * R / kCS, s1 = (rank + 1) * R / kCS;
        for (int64_t c0 = s0; c0 < s1; c0 += 32) {
            const int64_t c1 = std::min<int64_t>(c0 + 32, s1);
            for (int q = 0; q < 16; ++q) {
                // a 16-byte shared load is served a quarter-warp (8 lanes) at a
                // time: balance the bank quads within each 8-lane group
                for (int64_t g0 = c0; g0 < c1; g0 += 8) {
                    const int64_t g1 = std::min<int64_t>(g0 + 8, c1);
                    int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    // rules with fewer remaining choices pick first
                    std::vector<int64_t> order;
                    for (int64_t i = g0; i < g1; ++i) order.push_back(i);
                    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
                        return left[a].size() < left[b].size();
                    });
                    for (int64_t i : order) {
                        auto &L = left[i];
                        if (L.empty()) {  // padding code reads the all-ones row F
                            cnt[(F) & 7]++;
                            continue;
                        }
                        size_t best = 0;
                        int bc = 1 << 30;
                        for (size_t j = 0; j < L.size(); ++j) {
                            const int qd = (int)((L[j] >> 1) & 7);
                            if (cnt[qd] < bc) { bc = cnt[qd]; best = j; }
                        }
                        heads[(size_t)i * 16 + q] = (uint16_t)L[best];
                        cnt[(L[best] >> 1) & 7]++;
                        L[best] = L.back();
                        L.pop_back();
                    }
                }
            }
        }
    }
    for (int64_t i = 0; i < R; ++i) {
        std::sort(left[i].begin(), left[i].end());
        for (uint32_t c : left[i]) tails.push_back((uint16_t)c);
        tptr[i + 1] = (int32_t)tails.size();
    }
}

static int upload_rules(const std::vector<int64_t> &ptr, const std::vector<uint32_t> &inc,
                        const std::vector<int32_t> &w, int64_t K, int64_t F, int negations,
                        tmb_rules **out) {
    tmb_rules *r = new tmb_rules();
    r->R = (int64_t)ptr.size() - 1;
    r->K = K;
    r->F = F;
    r->n_inc = (int64_t)inc.size();
    r->negations = negations;
    // worst-case |vote| must fit the int32 shared-memory accumulators
    long double worst = 0;
    for (int64_t i = 0; i < r->R; ++i) {
        int64_t m = 0;
        for (int64_t kk = 0; kk < K; ++kk) m = std::max<int64_t>(m, std::llabs(w[i * K + kk]));
        worst += m;
    }
    if (worst >= 2147483647.0L) {
        delete r;
        return fail(TMB_E_UNSUPPORTED, "rules: |votes| could overflow int32 accumulators");
    }
    int rc;
    if ((rc = check_cuda(cudaMalloc(&r->ptr, 8 * ptr.size()), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&r->inc, 4 * std::max<size_t>(inc.size(), 1)), "cudaMalloc")) ||
        (rc = check_cuda(cudaMalloc(&r->weights, 4 * std::max<size_t>(w.size(), 1)), "cudaMalloc"))) {
        tmb_rules_destroy(r);
        return rc;
    }
    // head / tail form (uint16 codes) for the cluster kernel
    if (F + 1 < 32768 && r->R > 0) {
        std::vector<uint16_t> heads((size_t)r->R * 16, (uint16_t)(F << 1));
        std::vector<int32_t> tptr((size_t)r->R + 1, 0);
        std::vector<uint16_t> tails;
        balance_heads(ptr, inc, r->R, F, heads, tptr, tails);
        if ((rc = check_cuda(cudaMalloc(&r->heads, 2 * heads.size()), "cudaMalloc")) ||
            (rc = check_cuda(cudaMalloc(&r->tail_ptr, 4 * tptr.size()), "cudaMalloc")) ||
            (rc = check_cuda(cudaMalloc(&r->tails, 2 * std::max<size_t>(tails.size(), 1)), "cudaMalloc"))) {
            tmb_rules_destroy(r);
            return rc;
        }
        cudaMemcpy(r->heads, heads.data(), 2 * heads.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(r->tail_ptr, tptr.data(), 4 * tptr.size(), cudaMemcpyHostToDevice);
        if (!tails.empty()) cudaMemcpy(r->tails, tails.data(), 2 * tails.size(), cudaMemcpyHostToDevice);
        r->heads_ok = 1;
    }
    if ((rc = build_solo_heads(ptr, inc, r->R, F, r))) {
        tmb_rules_destroy(r);
        return rc;
    }
    cudaMemcpy(r->ptr, ptr.data(), 8 * ptr.size(), cudaMemcpyHostToDevice);
    if (!inc.empty()) cudaMemcpy(r->inc, inc.data(), 4 * inc.size(), cudaMemcpyHostToDevice);
    if (!w.empty()) cudaMemcpy(r->weights, w.data(), 4 * w.size(), cudaMemcpyHostToDevice);
    if ((rc = check_cuda(cudaGetLastError(), "rules upload"))) {
        tmb_rules_destroy(r);
        return rc;
    }
    *out = r;
    return TMB_OK;
}

static void host_pipe_free(HostPipe *hp) {
    if (!hp) return;
    if (hp->ks) cudaStreamSynchronize(hp->ks);
    if (hp->cs) cudaStreamSynchronize(hp->cs);
    for (int b = 0; b < kPipe; ++b) {
        if (hp->dx[b]) cudaFree(hp->dx[b]);
        if (hp->dp[b]) cudaFree(hp->dp[b]);
        if (hp->dv[b]) cudaFree(hp->dv[b]);
        if (hp->hp[b]) cudaFreeHost(hp->hp[b]);
        if (hp->hv[b]) cudaFreeHost(hp->hv[b]);
        if (hp->kdone[b]) cudaEventDestroy(hp->kdone[b]);
        if (hp->copied[b]) cudaEventDestroy(hp->copied[b]);
        if (hp->done[b]) cudaEventDestroy(hp->done[b]);
    }
    if (hp->cs) cudaStreamDestroy(hp->cs);
    if (hp->ks) cudaStreamDestroy(hp->ks);
    delete hp;
}

static inline uint32_t encode_inc(int64_t p, int64_t F, int negations) {
    if (negations && p >= F) return (uint32_t)(((p - F) << 1) | 1);
    return (uint32_t)(p << 1);
}

extern "C" {

int tmb_rules_from_bank(const int8_t *states, const int32_t *weights, int64_t C, int64_t P,
                        int64_t K, int64_t n_features, int negations, tmb_rules **out,
                        void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (!states || !weights || !out || C < 1 || P < 1 || K < 2 ||
        P != (negations ? 2 * n_features : n_features) || n_features >= (1LL << 31))
        return fail(TMB_E_INVALID, "rules_from_bank: bad arguments");
    cudaStream_t st = as_stream(stream);
    std::vector<int8_t> hs((size_t)(C * P));
    std::vector<int32_t> hw((size_t)(C * K));
    TMB_CUDA(cudaMemcpyAsync(hs.data(), states, C * P, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaMemcpyAsync(hw.data(), weights, 4 * C * K, cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaStreamSynchronize(st));
    // predictor.py:45-68: include = state >= 0; drop empty / all-zero-weight
    std::vector<int64_t> ptr{0};
    std::vector<uint32_t> inc;
    std::vector<int32_t> w;
    for (int64_t c = 0; c < C; ++c) {
        bool any_w = false;
        for (int64_t kk = 0; kk < K; ++kk) any_w |= hw[c * K + kk] != 0;
        if (!any_w) continue;
        size_t before = inc.size();
        const int8_t *row = hs.data() + c * P;
        for (int64_t p = 0; p < P; ++p)
            if (row[p] >= 0) inc.push_back(encode_inc(p, n_features, negations));
        if (inc.size() == before) continue;
        ptr.push_back((int64_t)inc.size());
        w.insert(w.end(), hw.begin() + c * K, hw.begin() + (c + 1) * K);
    }
    return upload_rules(ptr, inc, w, K, n_features, negations, out);
}

int tmb_rules_from_csr(const int64_t *inc_ptr, const int64_t *inc_idx, int64_t R,
                       const int32_t *weights, int64_t K, int64_t n_features, int negations,
                       tmb_rules **out) {
    int rc = require_device();
    if (rc) return rc;
    if (!inc_ptr || !out || R < 0 || K < 2 || (R > 0 && (!inc_idx || !weights)))
        return fail(TMB_E_INVALID, "rules_from_csr: bad arguments");
    int64_t P = negations ? 2 * n_features : n_features;
    std::vector<int64_t> ptr{0};
    std::vector<uint32_t> inc;
    std::vector<int32_t> w;
    for (int64_t r = 0; r < R; ++r) {
        if (inc_ptr[r + 1] <= inc_ptr[r]) continue;  // an empty rule never fires
        for (int64_t q = inc_ptr[r]; q < inc_ptr[r + 1]; ++q) {
            int64_t p = inc_idx[q];
            if (p < 0 || p >= P) return fail(TMB_E_INVALID, "rules_from_csr: index out of range");
            inc.push_back(encode_inc(p, n_features, negations));
        }
        ptr.push_back((int64_t)inc.size());
        w.insert(w.end(), weights + r * K, weights + (r + 1) * K);
    }
    return upload_rules(ptr, inc, w, K, n_features, negations, out);
}

int tmb_rules_destroy(tmb_rules *r) {
    if (!r) return TMB_OK;
    if (r->ptr) cudaFree(r->ptr);
    if (r->inc) cudaFree(r->inc);
    if (r->weights) cudaFree(r->weights);
    if (r->heads) cudaFree(r->heads);
    if (r->tail_ptr) cudaFree(r->tail_ptr);
    if (r->tails) cudaFree(r->tails);
    if (r->pipe) host_pipe_free(r->pipe);
    if (r->sheads) cudaFree(r->sheads);
    if (r->stail_ptr) cudaFree(r->stail_ptr);
    if (r->stails) cudaFree(r->stails);
    delete r;
    return TMB_OK;
}

int tmb_rules_info(const tmb_rules *r, int64_t *n_rules, int64_t *n_includes) {
    if (!r) return fail(TMB_E_INVALID, "rules_info: NULL");
    if (n_rules) *n_rules = r->R;
    if (n_includes) *n_includes = r->n_inc;
    return TMB_OK;
}

int tmb_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes, int64_t *pred,
              const int64_t *labels, uint64_t *correct, void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (!r || N < 0 || (N > 0 && !x) || (labels && !correct))
        return fail(TMB_E_INVALID, "infer: bad arguments");
    cudaStream_t st = as_stream(stream);
    return launch_infer(r, x, N, votes, pred, labels, (unsigned long long *)correct, st);
}

int tmb_infer_packed(const tmb_rules *r, const uint64_t *xb, int64_t N, int64_t W64,
                     int64_t *votes, int64_t *pred, const int64_t *labels, uint64_t *correct,
                     void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (!r || N < 0 || (N > 0 && !xb) || (labels && !correct) || W64 * 64 < r->F)
        return fail(TMB_E_INVALID, "infer_packed: bad arguments");
    if (N == 0) return TMB_OK;
    if (!r->heads_ok && !r->sheads_ok)
        return fail(TMB_E_UNSUPPORTED, "infer_packed: rule set needs the cluster or solo kernel");
    if (!g_bad_flag) {
        TMB_CUDA(cudaMalloc(&g_bad_flag, sizeof(unsigned)));
        TMB_CUDA(cudaMemset(g_bad_flag, 0, sizeof(unsigned)));
    }
    bool launched = false;
    rc = launch_infer_solo(r, nullptr, xb, W64, N, votes, pred, labels,
                           (unsigned long long *)correct, g_bad_flag, as_stream(stream), &launched);
    if (rc || launched) return rc;
    rc = launch_infer_cluster(r, nullptr, N, votes, pred, labels, (unsigned long long *)correct,
                              as_stream(stream), &launched, xb, W64);
    if (rc) return rc;
    if (!launched)
        return fail(TMB_E_UNSUPPORTED, "infer_packed: shape not supported by the cluster kernel");
    return TMB_OK;
}

int tmb_explain(const tmb_rules *r, const uint8_t *x, int64_t N, int for_class, int64_t *votes,
                int64_t *pred, int64_t *scores, void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (!r || N < 0 || (N > 0 && !x)) return fail(TMB_E_INVALID, "explain: bad arguments");
    if (for_class >= (int)r->K) return fail(TMB_E_INVALID, "explain: for_class out of range");
    if (N == 0) return TMB_OK;
    ExplainK k;
    k.x = x; k.N = N; k.F = r->F; k.inc = r->inc; k.ptr = r->ptr; k.w = r->weights;
    k.R = (int)r->R; k.K = (int)r->K; k.negations = r->negations;
    k.for_class = for_class < 0 ? -1 : for_class;
    k.votes = votes; k.pred = pred; k.scores = scores;
    const int threads = 256, nw = threads / 32;
    const size_t per = 8 * (size_t)k.K + 4 * (size_t)((k.R + 31) / 32) + (size_t)((r->F + 15) & ~15LL);
    const size_t smem = nw * ((per + 15) & ~(size_t)15);
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (smem > (size_t)max_smem)
        return fail(TMB_E_UNSUPPORTED, "explain: rule set / feature width too large");
    TMB_CUDA(cudaFuncSetAttribute((const void *)k_explain,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>((N + nw - 1) / nw, (int64_t)sm_count() * 8);
    k_explain<<<(unsigned)blocks, threads, smem, as_stream(stream)>>>(k);
    TMB_LAUNCHED();
    return TMB_OK;
}

int tmb_set_option(const char *name, int64_t value) {
    if (!name) return fail(TMB_E_INVALID, "set_option: NULL name");
    if (std::string(name) == "infer.force_generic") {
        g_force_generic_infer = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "train.key_chunk") {  // keyed trainer: steps per launch (0 = auto)
        g_train_key_chunk = value;
        return TMB_OK;
    }
    if (std::string(name) == "train.spec_window") {  // 0: k_train_fast; 1..16: k_train_spec
        if (value < 0 || value > 16) return fail(TMB_E_INVALID, "set_option: train.spec_window must be 0..16");
        g_train_spec = (int)value;                   // (applies to trainers created afterwards)
        return TMB_OK;
    }
    if (std::string(name) == "train.hbm_threads") {  // 512 | 1024 (applies at create)
        if (value != 512 && value != 1024) return fail(TMB_E_INVALID, "set_option: train.hbm_threads must be 512 or 1024");
        g_train_hbm_threads = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "train.tiny") {  // 1 (default): k_train_tiny for tiny banks, 0: k_train_warp
        g_train_tiny = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "train.gbal_weights") {  // packed bytes: Type II, Type I silent, Type I firing
        g_train_gbw = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "train.spec_entries") {  // 0 auto, else 64..256 (multiple of 32; default 64)
        g_train_spec_ent = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "train.debug_skip") {  // timing ablations only (not bit-exact)
        g_train_dbg = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "sparse.phase_buffer") {  // device uint64 [n_cta*16] or 0
        g_sparse_phase = reinterpret_cast<unsigned long long *>(value);
        return TMB_OK;
    }
    if (std::string(name) == "sparse.counters32") {  // 1: 32-bit counters in the counting kernel
        g_sparse_cnt32 = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "sparse.infer_key") {  // 1: key-literal sparse inference kernel
        g_sparse_infer_key = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "sparse.resident") {  // 0: keep clause lists in global memory
        g_sparse_resident = (int)value;            // (applies to banks created afterwards)
        return TMB_OK;
    }
    if (std::string(name) == "infer.solo") {  // 0: the 4-CTA cluster kernels instead
        g_infer_solo = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "infer.warp_specialized") {
        g_infer_ws = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "infer.eval_mode") {
        g_infer_eval = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "infer.debug_skip") {  // timing experiments only
        g_infer_dbg = (int)value;
        return TMB_OK;
    }
    if (std::string(name) == "infer.phase_buffer") {  // device uint64 [grid*8] or 0
        g_infer_phase = reinterpret_cast<unsigned long long *>(value);
        return TMB_OK;
    }
    return fail(TMB_E_INVALID, std::string("set_option: unknown option ") + name);
}

int tmb_infer_status(void *stream) {
    int rc = require_device();
    if (rc) return rc;
    return check_bad_input(as_stream(stream));
}

int tmbh_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes, int64_t *pred,
               int64_t chunk) {
    int rc = require_device();
    if (rc) return rc;
    if (!r || N < 0 || (N > 0 && !x)) return fail(TMB_E_INVALID, "infer: bad arguments");
    if (N == 0) return TMB_OK;
    const int64_t F = r->F, K = r->K;
    // ~48 MB of raw input per chunk: long enough copies for the PCIe / DMA
    // engine, enough chunks for a 3-deep copy / compute / drain pipeline
    if (chunk <= 0) chunk = std::max<int64_t>(128, ((48 << 20) / std::max<int64_t>(F, 1)) / 128 * 128);
    chunk = std::min(chunk, N);
    HostPipe *hp = r->pipe;
    if (!hp || hp->chunk < chunk || (votes && !hp->votes)) {
        if (hp) host_pipe_free(hp);
        hp = new HostPipe();
        const_cast<tmb_rules *>(r)->pipe = hp;
        hp->chunk = chunk;
        hp->votes = votes != nullptr;
        TMB_CUDA(cudaStreamCreateWithFlags(&hp->cs, cudaStreamNonBlocking));
        TMB_CUDA(cudaStreamCreateWithFlags(&hp->ks, cudaStreamNonBlocking));
        for (int b = 0; b < kPipe; ++b) {
            TMB_CUDA(cudaMalloc(&hp->dx[b], chunk * F));
            TMB_CUDA(cudaMalloc(&hp->dp[b], 8 * chunk));
            TMB_CUDA(cudaMallocHost(&hp->hp[b], 8 * chunk));
            if (hp->votes) {
                TMB_CUDA(cudaMalloc(&hp->dv[b], 8 * chunk * K));
                TMB_CUDA(cudaMallocHost(&hp->hv[b], 8 * chunk * K));
            }
            TMB_CUDA(cudaEventCreateWithFlags(&hp->kdone[b], cudaEventDisableTiming));
            TMB_CUDA(cudaEventCreateWithFlags(&hp->copied[b], cudaEventDisableTiming));
            TMB_CUDA(cudaEventCreateWithFlags(&hp->done[b], cudaEventDisableTiming));
        }
    }
    int64_t prev_off[kPipe], prev_n[kPipe];
    for (int b = 0; b < kPipe; ++b) prev_off[b] = -1, prev_n[b] = 0;
    auto drain = [&](int b) {
        if (prev_off[b] < 0) return;
        cudaEventSynchronize(hp->done[b]);
        if (votes) memcpy(votes + prev_off[b] * K, hp->hv[b], 8 * prev_n[b] * K);
        if (pred) memcpy(pred + prev_off[b], hp->hp[b], 8 * prev_n[b]);
        prev_off[b] = -1;
    };
    int64_t idx = 0;
    rc = TMB_OK;
    for (int64_t off = 0; off < N && !rc; off += chunk, ++idx) {
        const int b = (int)(idx % kPipe);
        const int64_t n = std::min(chunk, N - off);
        drain(b);  // chunk idx - kPipe's results are on the host; buffer b is free
        // the copy into dx[b] waits for the kernel that last read it
        if (idx >= kPipe) cudaStreamWaitEvent(hp->cs, hp->kdone[b], 0);
        rc = check_cuda(cudaMemcpyAsync(hp->dx[b], x + off * F, n * F, cudaMemcpyHostToDevice,
                                        hp->cs), "H2D");
        cudaEventRecord(hp->copied[b], hp->cs);
        cudaStreamWaitEvent(hp->ks, hp->copied[b], 0);
        if (!rc) rc = launch_infer(r, hp->dx[b], n, votes ? hp->dv[b] : nullptr, hp->dp[b],
                                   nullptr, nullptr, hp->ks);
        cudaEventRecord(hp->kdone[b], hp->ks);
        if (!rc && votes)
            rc = check_cuda(cudaMemcpyAsync(hp->hv[b], hp->dv[b], 8 * n * K, cudaMemcpyDeviceToHost,
                                            hp->ks), "D2H");
        if (!rc && pred)
            rc = check_cuda(cudaMemcpyAsync(hp->hp[b], hp->dp[b], 8 * n, cudaMemcpyDeviceToHost,
                                            hp->ks), "D2H");
        cudaEventRecord(hp->done[b], hp->ks);
        prev_off[b] = off;
        prev_n[b] = n;
    }
    for (int b = 0; b < kPipe; ++b) drain(b);
    if (!rc) rc = check_cuda(cudaStreamSynchronize(hp->ks), "sync");
    if (!rc) rc = check_bad_input(hp->ks);
    return rc;
}

}  // extern "C"
