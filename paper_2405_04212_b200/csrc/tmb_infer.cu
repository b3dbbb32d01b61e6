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
#include <vector>

#include "tmb_common.cuh"
#include "tmb_device.cuh"

struct tmb_rules {
    int64_t R = 0, K = 0, F = 0, n_inc = 0;
    int negations = 0;
    uint32_t *inc = nullptr;     // device [n_inc]: (feature << 1) | negated
    int64_t *ptr = nullptr;      // device [R+1]
    int32_t *weights = nullptr;  // device [R, K]
    int vote_bits = 32;
};

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

int launch_infer(const tmb_rules *r, const uint8_t *x, int64_t N, int64_t *votes, int64_t *pred,
                 const int64_t *labels, unsigned long long *correct, cudaStream_t st) {
    if (N == 0) return TMB_OK;
    int dev = 0;
    cudaGetDevice(&dev);
    int max_smem = 0;
    TMB_CUDA(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    if (!g_bad_flag) {
        TMB_CUDA(cudaMalloc(&g_bad_flag, sizeof(unsigned)));
        TMB_CUDA(cudaMemset(g_bad_flag, 0, sizeof(unsigned)));
    }
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
    if (chunk <= 0) chunk = 1 << 18;
    chunk = std::min(chunk, N);
    const int64_t F = r->F, K = r->K;
    cudaStream_t cs, ks;
    TMB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    TMB_CUDA(cudaStreamCreateWithFlags(&ks, cudaStreamNonBlocking));
    uint8_t *dx[2] = {nullptr, nullptr};
    int64_t *dv[2] = {nullptr, nullptr}, *dp[2] = {nullptr, nullptr};
    int64_t *hv[2] = {nullptr, nullptr}, *hp[2] = {nullptr, nullptr};
    cudaEvent_t copied[2], done[2];
    rc = TMB_OK;
    for (int b = 0; b < 2 && !rc; ++b) {
        rc = check_cuda(cudaMalloc(&dx[b], chunk * F), "cudaMalloc");
        if (!rc && votes) rc = check_cuda(cudaMalloc(&dv[b], 8 * chunk * K), "cudaMalloc");
        if (!rc && votes) rc = check_cuda(cudaMallocHost(&hv[b], 8 * chunk * K), "cudaMallocHost");
        if (!rc && pred) rc = check_cuda(cudaMalloc(&dp[b], 8 * chunk), "cudaMalloc");
        if (!rc && pred) rc = check_cuda(cudaMallocHost(&hp[b], 8 * chunk), "cudaMallocHost");
        cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming);
    }
    int64_t prev_off[2] = {-1, -1}, prev_n[2] = {0, 0};
    auto drain = [&](int b) {
        if (prev_off[b] < 0) return;
        cudaEventSynchronize(done[b]);
        if (votes) memcpy(votes + prev_off[b] * K, hv[b], 8 * prev_n[b] * K);
        if (pred) memcpy(pred + prev_off[b], hp[b], 8 * prev_n[b]);
        prev_off[b] = -1;
    };
    int64_t idx = 0;
    for (int64_t off = 0; off < N && !rc; off += chunk, ++idx) {
        const int b = (int)(idx & 1);
        const int64_t n = std::min(chunk, N - off);
        drain(b);  // buffer b's previous results are on the host and it is free
        rc = check_cuda(cudaMemcpyAsync(dx[b], x + off * F, n * F, cudaMemcpyHostToDevice, cs),
                        "H2D");
        cudaEventRecord(copied[b], cs);
        cudaStreamWaitEvent(ks, copied[b], 0);
        if (!rc) rc = launch_infer(r, dx[b], n, dv[b], dp[b], nullptr, nullptr, ks);
        if (!rc && votes)
            rc = check_cuda(cudaMemcpyAsync(hv[b], dv[b], 8 * n * K, cudaMemcpyDeviceToHost, ks), "D2H");
        if (!rc && pred)
            rc = check_cuda(cudaMemcpyAsync(hp[b], dp[b], 8 * n, cudaMemcpyDeviceToHost, ks), "D2H");
        cudaEventRecord(done[b], ks);
        prev_off[b] = off;
        prev_n[b] = n;
    }
    drain(0);
    drain(1);
    if (!rc) rc = check_cuda(cudaStreamSynchronize(ks), "sync");
    if (!rc) rc = check_bad_input(ks);
    for (int b = 0; b < 2; ++b) {
        cudaFree(dx[b]);
        if (dv[b]) cudaFree(dv[b]);
        if (dp[b]) cudaFree(dp[b]);
        if (hv[b]) cudaFreeHost(hv[b]);
        if (hp[b]) cudaFreeHost(hp[b]);
        cudaEventDestroy(copied[b]);
        cudaEventDestroy(done[b]);
    }
    cudaStreamDestroy(cs);
    cudaStreamDestroy(ks);
    return rc;
}

}  // extern "C"
