// tmb_plugin.cu -- the fine-grained plugin surface: the sm_100a counterparts of
// kernels.clause_outputs / clause_outputs_batch / bank_feedback
// (kernels/_numba.py:53-125) plus the explicit-draws test hook, literal
// packing and include-mask construction shared with the fused trainer.
#include <algorithm>
#include <cstring>
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"

namespace tmb {

// ------------------------------------------------------------ packing --
// x uint8 [N, F] -> words [N, W]; bit p = literal position p (core.py:232-242).
__global__ void k_pack_literals(const uint8_t *__restrict__ x, int64_t N, int64_t F,
                                int negations, int64_t P, int64_t W,
                                uint32_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N * W) return;
    int64_t e = i / W, w = i % W;
    const uint8_t *row = x + e * F;
    uint32_t word = 0;
#pragma unroll 4
    for (int b = 0; b < 32; ++b) {
        int64_t p = w * 32 + b;
        uint32_t bit;
        if (p < F) bit = row[p] != 0;
        else if (p < P) bit = row[p - F] == 0;  // negated half
        else bit = 1;                            // padding never violates
        word |= bit << b;
    }
    out[i] = word;
}

// states int8 [C,P] -> include masks [C,W] (bit = state >= 0) and counts [C].
__global__ void k_build_masks(const int8_t *__restrict__ states, int64_t C, int64_t P,
                              int64_t W, uint32_t *__restrict__ masks,
                              int32_t *__restrict__ counts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= C * W) return;
    int64_t c = i / W, w = i % W;
    const int8_t *row = states + c * P;
    uint32_t word = 0;
    for (int b = 0; b < 32; ++b) {
        int64_t p = w * 32 + b;
        if (p < P && row[p] >= 0) word |= 1u << b;
    }
    masks[i] = word;
    if (word) atomicAdd(&counts[c], __popc(word));
}

// out[e, c] for masks / literal words (kernels/_numba.py:36-50).
__global__ void k_outputs_batch(const uint32_t *__restrict__ masks,
                                const int32_t *__restrict__ counts, int64_t C, int64_t W,
                                const uint32_t *__restrict__ lits, int64_t N, int training,
                                int64_t budget, uint8_t *__restrict__ out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N * C) return;
    int64_t e = i / C, c = i % C;
    const uint32_t *m = masks + c * W;
    const uint32_t *l = lits + e * W;
    uint32_t viol = 0;
    for (int64_t w = 0; w < W; ++w) viol |= m[w] & ~l[w];
    int cnt = counts[c];
    uint8_t o;
    if (viol) o = 0;
    else if (training) o = cnt > budget ? 0 : 1;
    else o = cnt == 0 ? 0 : 1;
    out[i] = o;
}

// ------------------------------------------------------------ feedback --
// Exclusive scan of (ut + un) over clauses -> window ordinal of each
// clause's first event; total -> *total.  Single CTA (C is at most ~10^6).
__global__ void k_event_scan(const uint8_t *__restrict__ ut, const uint8_t *__restrict__ un,
                             int64_t C, int64_t *__restrict__ prefix,
                             uint64_t *__restrict__ total) {
    __shared__ int64_t warp_sums[32];
    __shared__ int64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = 0; base < C; base += blockDim.x) {
        int64_t j = base + threadIdx.x;
        int v = (j < C) ? (int)(ut[j] != 0) + (int)(un[j] != 0) : 0;
        int x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int64_t s = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;  // inclusive
        }
        __syncthreads();
        int64_t before = carry + (wid > 0 ? warp_sums[wid - 1] : 0) + (x - v);
        if (j < C) prefix[j] = before;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = before + v;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = (uint64_t)carry;
}

// One CTA per clause with at least one applied event; threads over literal
// positions apply the target event then the negative event (SPEC order,
// kernels/_numba.py:101-125).  draws != NULL selects the explicit-draws hook.
__global__ void k_bank_feedback(int8_t *__restrict__ states, int32_t *__restrict__ weights,
                                int64_t C, int64_t P, int64_t K,
                                const uint32_t *__restrict__ litw, const uint8_t *__restrict__ outputs,
                                int64_t label, int64_t negative, const uint8_t *__restrict__ ut,
                                const uint8_t *__restrict__ un, const int64_t *__restrict__ prefix,
                                FbParams fp, uint64_t seed, uint64_t counter,
                                const double *__restrict__ draws, int64_t n_rows) {
    int64_t j = blockIdx.x;
    bool t_ev = ut[j] != 0, n_ev = un[j] != 0;
    if (!t_ev && !n_ev) return;
    int out = outputs[j];
    int32_t wl = weights[j * K + label], wn = weights[j * K + negative];
    bool t_type1 = wl >= 0, n_type1 = wn < 0;
    uint64_t ord_t = (uint64_t)prefix[j], ord_n = ord_t + (t_ev ? 1 : 0);
    uint64_t win_t = (counter + ord_t) << 32, win_n = (counter + ord_n) << 32;
    uint64_t sk_t = seed + kGolden * (win_t + 1), sk_n = seed + kGolden * (win_n + 1);
    int8_t *row = states + j * P;
    for (int64_t p = threadIdx.x; p < P; p += blockDim.x) {
        int st = row[p];
        int lit = (litw[p >> 5] >> (p & 31)) & 1;
        int st0 = st;
        uint64_t nd = 0;
        if (t_ev) {
            if (t_type1) {
                if (draws) st = type_i_explicit(st, lit, out, fp,
                                                ord_t < (uint64_t)n_rows ? draws[ord_t * P + p] : 0.0);
                else st = type_i_stream(st, lit, out, fp, sk_t, (uint32_t)p, nd);
            } else if (out && !lit && st < 0) {
                st += 1;
            }
        }
        if (n_ev) {
            if (n_type1) {
                if (draws) st = type_i_explicit(st, lit, out, fp,
                                                ord_n < (uint64_t)n_rows ? draws[ord_n * P + p] : 0.0);
                else st = type_i_stream(st, lit, out, fp, sk_n, (uint32_t)p, nd);
            } else if (out && !lit && st < 0) {
                st += 1;
            }
        }
        if (st != st0) row[p] = (int8_t)st;
    }
    if (threadIdx.x == 0 && out) {
        if (t_ev) weights[j * K + label] = wl + 1;
        if (n_ev) weights[j * K + negative] = wn - 1;
    }
}

}  // namespace tmb

using namespace tmb;

namespace {

int pack_lits_rows(const uint8_t *x, int64_t N, int64_t cols, int negations, int64_t P,
                   uint32_t *out, cudaStream_t st) {
    int64_t W = ceil_div(P, 32);
    int64_t n = N * W;
    if (n == 0) return TMB_OK;
    k_pack_literals<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(x, N, cols, negations, P, W, out);
    TMB_LAUNCHED();
    return TMB_OK;
}

int build_masks(const int8_t *states, int64_t C, int64_t P, uint32_t *masks, int32_t *counts,
                cudaStream_t st) {
    int64_t W = ceil_div(P, 32);
    TMB_CUDA(cudaMemsetAsync(counts, 0, sizeof(int32_t) * C, st));
    int64_t n = C * W;
    k_build_masks<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(states, C, P, W, masks, counts);
    TMB_LAUNCHED();
    return TMB_OK;
}

struct DevBuf {
    void *p = nullptr;
    cudaStream_t st = nullptr;
    int alloc(size_t n, cudaStream_t s) {
        st = s;
        return check_cuda(cudaMallocAsync(&p, n ? n : 1, s), "cudaMallocAsync");
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    template <class T> T *as() { return reinterpret_cast<T *>(p); }
};

int outputs_batch_dev(const int8_t *states, int64_t C, int64_t P, const uint8_t *x_lit,
                      int64_t N, int training, int64_t budget, uint8_t *out, cudaStream_t st) {
    int64_t W = ceil_div(P, 32);
    DevBuf masks, counts, lits;
    int rc;
    if ((rc = masks.alloc(sizeof(uint32_t) * C * W, st))) return rc;
    if ((rc = counts.alloc(sizeof(int32_t) * C, st))) return rc;
    if ((rc = lits.alloc(sizeof(uint32_t) * (N > 0 ? N : 1) * W, st))) return rc;
    if ((rc = build_masks(states, C, P, masks.as<uint32_t>(), counts.as<int32_t>(), st))) return rc;
    if ((rc = pack_lits_rows(x_lit, N, P, 0, P, lits.as<uint32_t>(), st))) return rc;
    int64_t n = N * C;
    if (n > 0) {
        k_outputs_batch<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
            masks.as<uint32_t>(), counts.as<int32_t>(), C, W, lits.as<uint32_t>(), N, training,
            budget, out);
        TMB_LAUNCHED();
    }
    return TMB_OK;
}

int feedback_dev(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                 const uint8_t *lits, const uint8_t *outputs, int64_t label, int64_t negative,
                 const uint8_t *ut, const uint8_t *un, double s, int boost, int smin, int smax,
                 uint64_t seed, uint64_t counter, const double *draws, int64_t n_rows,
                 uint64_t *counter_out, cudaStream_t st, uint64_t *total_pinned = nullptr) {
    if (C < 1 || P < 1 || K < 2 || label < 0 || label >= K || negative < 0 || negative >= K)
        return fail(TMB_E_INVALID, "bank_feedback: bad shape or class index");
    if (!(s > 1.0) && !draws) return fail(TMB_E_INVALID, "bank_feedback: s must exceed 1");
    int64_t W = ceil_div(P, 32);
    DevBuf prefix, total, litw;
    int rc;
    if ((rc = prefix.alloc(sizeof(int64_t) * C, st))) return rc;
    if ((rc = total.alloc(sizeof(uint64_t), st))) return rc;
    if ((rc = litw.alloc(sizeof(uint32_t) * W, st))) return rc;
    if ((rc = pack_lits_rows(lits, 1, P, 0, P, litw.as<uint32_t>(), st))) return rc;
    k_event_scan<<<1, 1024, 0, st>>>(ut, un, C, prefix.as<int64_t>(), total.as<uint64_t>());
    TMB_LAUNCHED();
    FbParams fp = make_fb_params(s, boost, smin, smax);
    k_bank_feedback<<<(unsigned)C, 256, 0, st>>>(states, weights, C, P, K, litw.as<uint32_t>(),
                                                 outputs, label, negative, ut, un,
                                                 prefix.as<int64_t>(), fp, seed, counter, draws,
                                                 n_rows);
    TMB_LAUNCHED();
    if (total_pinned) {  // the caller synchronises and adds the counter
        TMB_CUDA(cudaMemcpyAsync(total_pinned, total.as<uint64_t>(), sizeof(uint64_t),
                                 cudaMemcpyDeviceToHost, st));
        return TMB_OK;
    }
    uint64_t tot = 0;
    TMB_CUDA(cudaMemcpyAsync(&tot, total.as<uint64_t>(), sizeof(uint64_t),
                             cudaMemcpyDeviceToHost, st));
    TMB_CUDA(cudaStreamSynchronize(st));
    if (counter_out) *counter_out = counter + tot;
    return TMB_OK;
}

}  // namespace

extern "C" {

int tmb_pack_literals(const uint8_t *x, int64_t N, int64_t F, int negations, uint32_t *out,
                      void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (N < 0 || F < 1 || (N > 0 && (!x || !out)))
        return fail(TMB_E_INVALID, "pack_literals: bad arguments");
    int64_t P = negations ? 2 * F : F;
    return pack_lits_rows(x, N, F, negations, P, out, as_stream(stream));
}

int tmb_clause_outputs(const int8_t *states, int64_t C, int64_t P, const uint8_t *lits,
                       int training, int64_t budget, uint8_t *out, void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (C < 1 || P < 1 || !states || !lits || !out)
        return fail(TMB_E_INVALID, "clause_outputs: bad arguments");
    return outputs_batch_dev(states, C, P, lits, 1, training, budget, out, as_stream(stream));
}

int tmb_clause_outputs_batch(const int8_t *states, int64_t C, int64_t P, const uint8_t *x_lit,
                             int64_t N, int training, int64_t budget, uint8_t *out,
                             void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (C < 1 || P < 1 || N < 0 || !states || (N > 0 && (!x_lit || !out)))
        return fail(TMB_E_INVALID, "clause_outputs_batch: bad arguments");
    return outputs_batch_dev(states, C, P, x_lit, N, training, budget, out, as_stream(stream));
}

int tmb_bank_feedback(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                      const uint8_t *lits, const uint8_t *outputs, int64_t label,
                      int64_t negative, const uint8_t *ut, const uint8_t *un, double s,
                      int boost, int state_min, int state_max, uint64_t seed, uint64_t counter,
                      uint64_t *counter_out, void *stream) {
    int rc = require_device();
    if (rc) return rc;
    return feedback_dev(states, weights, C, P, K, lits, outputs, label, negative, ut, un, s,
                        boost, state_min, state_max, seed, counter, nullptr, 0, counter_out,
                        as_stream(stream));
}

int tmb_bank_feedback_draws(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                            const uint8_t *lits, const uint8_t *outputs, int64_t label,
                            int64_t negative, const uint8_t *ut, const uint8_t *un, double s,
                            int boost, int state_min, int state_max, uint64_t counter,
                            const double *draws, int64_t n_rows, uint64_t *counter_out,
                            void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (!draws || n_rows < 0) return fail(TMB_E_INVALID, "bank_feedback_draws: no draws");
    return feedback_dev(states, weights, C, P, K, lits, outputs, label, negative, ut, un, s,
                        boost, state_min, state_max, 0, counter, draws, n_rows, counter_out,
                        as_stream(stream));
}

// ------------------------------------------------------- host variants --
}  // extern "C"

namespace {
// Per host thread: one stream, a device arena and a pinned staging buffer,
// kept between calls (the reference calls the plugin once per example per
// block, so per-call stream / allocation setup would dominate).  Inputs are
// packed into the staging buffer and moved with ONE host->device copy.
struct PluginCtx {
    cudaStream_t st = nullptr;
    char *dev = nullptr, *pin = nullptr;
    size_t dev_cap = 0, pin_cap = 0;
    int ensure(size_t dbytes, size_t pbytes) {
        if (!st) TMB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        if (dbytes > dev_cap) {
            if (dev) cudaFree(dev);
            dev_cap = std::max(dbytes, 2 * dev_cap);
            TMB_CUDA(cudaMalloc(&dev, dev_cap));
        }
        if (pbytes > pin_cap) {
            if (pin) cudaFreeHost(pin);
            pin_cap = std::max(pbytes, 2 * pin_cap);
            TMB_CUDA(cudaMallocHost(&pin, pin_cap));
        }
        return TMB_OK;
    }
};
thread_local PluginCtx *t_pc = nullptr;  // never freed: outlives the CUDA runtime at exit
PluginCtx &plugin_ctx() {
    if (!t_pc) t_pc = new PluginCtx();
    return *t_pc;
}
inline size_t al16(size_t n) { return (n + 15) & ~(size_t)15; }
}  // namespace

extern "C" {

int tmbh_clause_outputs_batch(const int8_t *states, int64_t C, int64_t P, const uint8_t *x_lit,
                              int64_t N, int training, int64_t budget, uint8_t *out) {
    int rc = require_device();
    if (rc) return rc;
    if (C < 1 || P < 1 || N < 0 || !states || (N > 0 && (!x_lit || !out)))
        return fail(TMB_E_INVALID, "clause_outputs_batch: bad arguments");
    PluginCtx &pc = plugin_ctx();
    const size_t o_s = 0, o_x = al16(C * P), o_out = o_x + al16(N * P), tot_in = o_out;
    if ((rc = pc.ensure(o_out + al16(N * C), std::max(tot_in, (size_t)(N * C))))) return rc;
    memcpy(pc.pin + o_s, states, C * P);
    if (N > 0) memcpy(pc.pin + o_x, x_lit, N * P);
    TMB_CUDA(cudaMemcpyAsync(pc.dev, pc.pin, tot_in, cudaMemcpyHostToDevice, pc.st));
    rc = outputs_batch_dev(reinterpret_cast<int8_t *>(pc.dev + o_s), C, P,
                           reinterpret_cast<uint8_t *>(pc.dev + o_x), N, training, budget,
                           reinterpret_cast<uint8_t *>(pc.dev + o_out), pc.st);
    if (!rc && N > 0)
        rc = check_cuda(cudaMemcpyAsync(pc.pin, pc.dev + o_out, N * C, cudaMemcpyDeviceToHost,
                                        pc.st), "copy out");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(pc.st), "sync");
    if (!rc && N > 0) memcpy(out, pc.pin, N * C);
    return rc;
}

int tmbh_clause_outputs(const int8_t *states, int64_t C, int64_t P, const uint8_t *lits,
                        int training, int64_t budget, uint8_t *out) {
    return tmbh_clause_outputs_batch(states, C, P, lits, 1, training, budget, out);
}

int tmbh_bank_feedback(int8_t *states, int32_t *weights, int64_t C, int64_t P, int64_t K,
                       const uint8_t *lits, const uint8_t *outputs, int64_t label,
                       int64_t negative, const uint8_t *ut, const uint8_t *un, double s,
                       int boost, int state_min, int state_max, uint64_t seed, uint64_t counter,
                       uint64_t *counter_out) {
    int rc = require_device();
    if (rc) return rc;
    if (C < 1 || P < 1 || K < 2 || !states || !weights || !lits || !outputs || !ut || !un)
        return fail(TMB_E_INVALID, "bank_feedback: bad arguments");
    PluginCtx &pc = plugin_ctx();
    // staging layout: states | weights | lits | outputs | ut | un
    const size_t o_s = 0, o_w = al16(C * P), o_l = o_w + al16(4 * C * K), o_o = o_l + al16(P),
                 o_t = o_o + al16(C), o_n = o_t + al16(C), tot = o_n + al16(C);
    if ((rc = pc.ensure(tot, tot + 16))) return rc;
    uint64_t *ev_total = reinterpret_cast<uint64_t *>(pc.pin + tot);
    memcpy(pc.pin + o_s, states, C * P);
    memcpy(pc.pin + o_w, weights, 4 * C * K);
    memcpy(pc.pin + o_l, lits, P);
    memcpy(pc.pin + o_o, outputs, C);
    memcpy(pc.pin + o_t, ut, C);
    memcpy(pc.pin + o_n, un, C);
    TMB_CUDA(cudaMemcpyAsync(pc.dev, pc.pin, tot, cudaMemcpyHostToDevice, pc.st));
    char *d = pc.dev;
    rc = feedback_dev(reinterpret_cast<int8_t *>(d + o_s), reinterpret_cast<int32_t *>(d + o_w),
                      C, P, K, reinterpret_cast<uint8_t *>(d + o_l),
                      reinterpret_cast<uint8_t *>(d + o_o), label, negative,
                      reinterpret_cast<uint8_t *>(d + o_t), reinterpret_cast<uint8_t *>(d + o_n),
                      s, boost, state_min, state_max, seed, counter, nullptr, 0, counter_out,
                      pc.st, ev_total);
    if (!rc) rc = check_cuda(cudaMemcpyAsync(pc.pin, d, o_l, cudaMemcpyDeviceToHost, pc.st), "D2H");
    if (!rc) rc = check_cuda(cudaStreamSynchronize(pc.st), "sync");
    if (!rc) {
        if (counter_out) *counter_out = counter + *ev_total;
        memcpy(states, pc.pin + o_s, C * P);
        memcpy(weights, pc.pin + o_w, 4 * C * K);
    }
    return rc;
}

}  // extern "C"

// Exposed to the other translation units.
namespace tmb {
int dev_pack_literals(const uint8_t *x, int64_t N, int64_t cols, int negations, int64_t P,
                      uint32_t *out, cudaStream_t st) {
    return pack_lits_rows(x, N, cols, negations, P, out, st);
}
int dev_build_masks(const int8_t *states, int64_t C, int64_t P, uint32_t *masks,
                    int32_t *counts, cudaStream_t st) {
    return build_masks(states, C, P, masks, counts, st);
}
}  // namespace tmb
