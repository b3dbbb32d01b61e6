// tmb_infer.cuh -- the compiled rule set (tmb_rules) and the shared-memory /
// mbarrier / bulk-copy helpers of the inference kernels (tmb_infer.cu,
// tmb_infer_solo.cu).
#pragma once

#include <cstdint>
#include <vector>

#include "tmb_common.cuh"

// Host-buffer inference pipeline state (tmbh_infer), kept with the rule set
// between calls: kPipe device input / output buffers, pinned output staging,
// a copy stream and a compute stream.
constexpr int kPipe = 3;
struct HostPipe {
    int64_t chunk = 0;
    bool votes = false;
    uint8_t *dx[kPipe] = {};
    int64_t *dp[kPipe] = {}, *dv[kPipe] = {};
    int64_t *hp[kPipe] = {}, *hv[kPipe] = {};
    cudaEvent_t kdone[kPipe] = {}, copied[kPipe] = {}, done[kPipe] = {};
    cudaStream_t cs = nullptr, ks = nullptr;
};

struct tmb_rules {
    int64_t R = 0, K = 0, F = 0, n_inc = 0;
    int negations = 0;
    uint32_t *inc = nullptr;     // device [n_inc]: (feature << 1) | negated
    int64_t *ptr = nullptr;      // device [R+1]
    int32_t *weights = nullptr;  // device [R, K]
    // head/tail form for the cluster kernel (uint16 codes; F + 1 < 32768):
    // the first 16 include codes of every rule, padded with the always-true
    // code (F << 1) that addresses an all-ones X^T row; the rest in a CSR tail
    uint16_t *heads = nullptr;   // device [R, 16]
    int32_t *tail_ptr = nullptr; // device [R+1]
    uint16_t *tails = nullptr;   // device [n_tail]
    int heads_ok = 0;
    // per-CTA ("solo") kernel form (tmb_infer_solo.cu): 16 head slots per
    // rule as 8 (positive, negated) pairs of X^T row indices -- slot 2i reads
    // row f of a positive include (padding: the all-ones row F), slot 2i+1
    // row f of a negated include (padding: the all-zeros row F+1) -- so one
    // LOP3 tests two includes per word; the remaining includes in a CSR tail
    // of (feature << 1 | negated) codes.  Rules padded to a multiple of 64.
    uint16_t *sheads = nullptr;    // device [R_pad, 16]
    int32_t *stail_ptr = nullptr;  // device [R+1]
    uint16_t *stails = nullptr;    // device [n_stail]
    int64_t R_pad = 0;
    int sheads_ok = 0;
    HostPipe *pipe = nullptr;  // tmbh_infer buffers (lazily created)
};

namespace tmb {

__device__ __forceinline__ uint32_t pack8(unsigned long long q) {
    return (uint32_t)(((q & 0x0101010101010101ull) * 0x0102040810204080ull) >> 56);
}

// ---- mbarrier / bulk-copy helpers (shared::cta / shared::cluster, sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *mb, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t *mb, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)),
                 "r"(bytes) : "memory");
}
// try_wait suspend-time hint: a waiting warp is parked until the phase
// completes instead of re-polling (spin loops were ~16% of all issued
// instructions of the warp-specialised inference kernel)
constexpr uint32_t kSuspendNs = 0x989680;
__device__ __forceinline__ void mbar_wait(uint64_t *mb, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done) : "r"(smem_u32(mb)), "r"(parity), "r"(kSuspendNs) : "memory");
    } while (!done);
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void bulk_copy_to_peer(uint32_t dst_cluster, uint32_t src_cta,
                                                  uint32_t bytes, uint32_t mbar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(dst_cluster), "r"(src_cta), "r"(bytes), "r"(mbar_cluster) : "memory");
}

// shared-window atomic (a generic-pointer atomicAdd on a pointer derived from
// the mbarrier area compiles to a generic ATOM, not ATOMS)
__device__ __forceinline__ uint32_t atom_add_shared(void *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
    return old;
}
// predicated 16-byte shared load into v (v unchanged when !p)
__device__ __forceinline__ void lds128_if(uint4 &v, bool p, uint32_t addr) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %4, 0;\n"
                 " @q ld.shared.v4.u32 {%0, %1, %2, %3}, [%5];\n}"
                 : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w) : "r"((uint32_t)p), "r"(addr));
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

// 4 bytes of 0/1 -> 4 bits (bit t = byte t)
__device__ __forceinline__ uint32_t pack4(uint32_t w) {
    return ((w & 0x01010101u) * 0x01020408u) >> 24;
}

// 8x8 bit-matrix transpose: byte i = row i (bit t = column t) -> byte t =
// column t (bit i = row i)
__device__ __forceinline__ unsigned long long transpose8x8(unsigned long long x) {
    unsigned long long t;
    t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
    x = x ^ t ^ (t << 7);
    t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
    x = x ^ t ^ (t << 14);
    t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
    x = x ^ t ^ (t << 28);
    return x;
}

// up to 8 feature bytes starting at column f (bounds-checked against F)
__device__ __forceinline__ unsigned long long load8_tail(const uint8_t *src, int64_t f, int64_t F) {
    unsigned long long v = 0;
    for (int bb = 0; bb < 8; ++bb)
        if (f + bb < F) v |= (unsigned long long)src[bb] << (8 * bb);
    return v;
}

// 32x32 bit transpose across the warp: lane i holds row i (bit j = A[i][j]);
// afterwards lane j holds column j (bit i = A[i][j]).
__device__ __forceinline__ uint32_t warp_transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int j = 16; j >= 1; j >>= 1) {
        const uint32_t m0 = j == 16 ? 0x0000FFFFu : j == 8 ? 0x00FF00FFu : j == 4 ? 0x0F0F0F0Fu
                          : j == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, j);
        x = (lane & j) ? ((x & ~m0) | ((y >> j) & m0)) : ((x & m0) | ((y << j) & ~m0));
    }
    return x;
}

__device__ __forceinline__ void mbar_arrive_local(uint64_t *mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t mb_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(mb_cluster)
                 : "memory");
}
// arrival that publishes nothing (the barrier only orders reads before it)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t mb_cluster) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(mb_cluster)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *mb, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done) : "r"(smem_u32(mb)), "r"(parity) : "memory");
    } while (!done);
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}



// solo kernel (tmb_infer_solo.cu)
int build_solo_heads(const std::vector<int64_t> &ptr, const std::vector<uint32_t> &inc,
                     int64_t R, int64_t F, tmb_rules *r);
int launch_infer_solo(const tmb_rules *r, const uint8_t *x, const uint64_t *xb, int64_t W64,
                      int64_t N, int64_t *votes, int64_t *pred, const int64_t *labels,
                      unsigned long long *correct, unsigned int *bad_flag, cudaStream_t st,
                      bool *launched);
extern int g_infer_solo;  // tmb_set_option("infer.solo", 0|1)
extern int g_infer_dbg;   // tmb_set_option("infer.debug_skip", ...)

}  // namespace tmb
