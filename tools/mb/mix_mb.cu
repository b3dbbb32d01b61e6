// Draw-throughput microbenchmark: SplitMix64 finalizer variants (shift-based
// vs shifts as IMAD.HI on the FMA pipe).  nvcc -arch=sm_100a -O3 mix_mb.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix_ref(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t mulhi(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
// z ^ (z >> k) for 0 < k < 32 with the shifts done by multiplies
template <int K>
__device__ __forceinline__ uint64_t xs_mul(uint64_t z, uint32_t c /* = 2^(32-K) */) {
    const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
    const uint32_t nlo = mulhi(lo, c) + hi * c;  // (lo >> K) | (hi << (32-K))
    const uint32_t nhi = mulhi(hi, c);           // hi >> K
    return z ^ (((uint64_t)nhi << 32) | nlo);
}
__device__ __forceinline__ uint64_t mix_mul(uint64_t z, uint32_t c30, uint32_t c27, uint32_t c31) {
    z = xs_mul<30>(z, c30) * 0xBF58476D1CE4E5B9ULL;
    z = xs_mul<27>(z, c27) * 0x94D049BB133111EBULL;
    return xs_mul<31>(z, c31);
}

__global__ void k_mix(int mode, int iters, uint64_t seed, unsigned long long *out, uint32_t c30,
                      uint32_t c27, uint32_t c31) {
    uint64_t z = seed + threadIdx.x + (uint64_t)blockIdx.x * blockDim.x;
    uint64_t acc = 0;
    const uint64_t G = 0x9E3779B97F4A7C15ULL;
    uint64_t k0 = z * G, k1 = k0 + G, k2 = k1 + G, k3 = k2 + G;
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {
            acc += (mix_ref(k0) >> 11) < 900719925474099ULL;
            acc += (mix_ref(k1) >> 11) < 900719925474099ULL;
            acc += (mix_ref(k2) >> 11) < 900719925474099ULL;
            acc += (mix_ref(k3) >> 11) < 900719925474099ULL;
        } else {
            acc += (mix_mul(k0, c30, c27, c31) >> 11) < 900719925474099ULL;
            acc += (mix_mul(k1, c30, c27, c31) >> 11) < 900719925474099ULL;
            acc += (mix_mul(k2, c30, c27, c31) >> 11) < 900719925474099ULL;
            acc += (mix_mul(k3, c30, c27, c31) >> 11) < 900719925474099ULL;
        }
        k0 += 4 * G; k1 += 4 * G; k2 += 4 * G; k3 += 4 * G;
    }
    if (acc == 0xFFFFFFFF) out[0] = acc;
}
__global__ void k_check(unsigned long long *bad, uint32_t c30, uint32_t c27, uint32_t c31) {
    uint64_t z = 0x123456789ULL + (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ULL;
    for (int i = 0; i < 1000; ++i) {
        if (mix_ref(z) != mix_mul(z, c30, c27, c31)) atomicAdd(bad, 1ull);
        z = z * 6364136223846793005ULL + 1442695040888963407ULL;
    }
}
int main() {
    unsigned long long *d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const uint32_t c30 = 1u << 2, c27 = 1u << 5, c31 = 1u << 1;
    k_check<<<148, 256>>>(d + 1, c30, c27, c31);
    unsigned long long bad = 0;
    cudaMemcpy(&bad, d + 1, 8, cudaMemcpyDeviceToHost);
    printf("mismatches %llu\n", bad);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            const int iters = 4096;
            cudaEventRecord(a);
            k_mix<<<148 * 4, 512>>>(mode, iters, 7, d, c30, c27, c31);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            double draws = 148.0 * 4 * 512 * iters * 4;
            if (rep) printf("mode %d: %.1f G draws/s (%.2f ms)\n", mode, draws / ms / 1e6, ms);
        }
    }
    return 0;
}
