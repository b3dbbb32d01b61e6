// tmb_common.cuh -- shared device helpers: SplitMix64 counter streams, error
// plumbing, launch accounting.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <string>

#include "../../include/tsetlin_b200.h"

namespace tmb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kMixC1 = 0xBF58476D1CE4E5B9ULL;
constexpr uint64_t kMixC2 = 0x94D049BB133111EBULL;

// core.py:66-71.  Identical on host and device.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * kMixC1;
    z = (z ^ (z >> 27)) * kMixC2;
    return z ^ (z >> 31);
}

// core.py:74-85
__host__ __device__ __forceinline__ uint64_t derive_stream(uint64_t seed, uint64_t index) {
    uint64_t v = index + 1;
    return mix64(seed ^ ((v << 32) | (v >> 32)));
}

// Top 53 bits of draw k: u01 = m * 2^-53 exactly (core.py:93-95).
__host__ __device__ __forceinline__ uint64_t draw53(uint64_t seed, uint64_t k) {
    return mix64(seed + kGolden * (k + 1)) >> 11;
}

// u < p  <=>  m < ceil(p * 2^53) for m = u * 2^53 in [0, 2^53): exact,
// because p * 2^53 is an exact power-of-two scaling of a double.
__host__ __device__ __forceinline__ uint64_t prob_threshold(double p) {
    double x = p * 9007199254740992.0;  // 2^53
    if (x <= 0.0) return 0;
    if (x >= 9007199254740992.0) return (1ULL << 53);
    double c = ceil(x);
    return (uint64_t)c;
}

__host__ __device__ __forceinline__ double u01_from53(uint64_t m) {
    return (double)m * (1.0 / 9007199254740992.0);
}

// ------------------------------------------------------------ errors --
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int check_cuda(cudaError_t e, const char *what);
int require_device();
void note_launch(uint64_t n = 1);

#define TMB_CUDA(call)                                                  \
    do {                                                                \
        int _rc = ::tmb::check_cuda((call), #call);                     \
        if (_rc) return _rc;                                            \
    } while (0)

#define TMB_LAUNCHED()                                                  \
    do {                                                                \
        ::tmb::note_launch();                                           \
        int _rc = ::tmb::check_cuda(cudaGetLastError(), "kernel launch"); \
        if (_rc) return _rc;                                            \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

int sm_count();
extern int64_t g_train_key_chunk;
extern int g_train_dbg;  // trainer timing ablations (tmb_train.cu)
extern int g_train_spec;  // speculative window of the fast grid trainer (tmb_train.cu)
extern int g_train_spec_ent;  // staged flag entries per step head (0 = auto)
extern int g_train_hbm_threads;  // CTA size of the HBM-state grid trainer
extern int g_train_tiny;         // tiny banks: one warp per clause (k_train_tiny) instead of one warp
extern int g_train_gbw;          // balanced-feedback cost weights (packed bytes)
//  // keyed trainer: steps per launch override (tmb_train.cu)

}  // namespace tmb
