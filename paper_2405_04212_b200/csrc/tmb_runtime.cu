// tmb_runtime.cu -- error plumbing, device facts, host RNG helpers, the host
// Fisher-Yates shuffle (executor.py:50-58) and launch accounting.
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "tmb_common.cuh"

namespace tmb {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int code, const std::string &msg) {
    g_last_error = msg;
    return code;
}

int check_cuda(cudaError_t e, const char *what) {
    if (e == cudaSuccess) return TMB_OK;
    g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return TMB_E_CUDA;
}

void note_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int g_dev_state = -1;  // -1 unknown, 0 ok, else error code
static std::string g_dev_msg;
static std::mutex g_dev_mu;
static int g_sm_count = 0;

int require_device() {
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (g_dev_state == -1) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0) {
            g_dev_state = TMB_E_NO_DEVICE;
            g_dev_msg = std::string("no CUDA device available (") +
                        (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                        "); libtmb200 has no CPU fallback";
            cudaGetLastError();
        } else {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceProp prop;
            cudaGetDeviceProperties(&prop, dev);
            if (prop.major != 10) {
                g_dev_state = TMB_E_NO_DEVICE;
                g_dev_msg = "libtmb200 is built for sm_100a (B200); device is sm_" +
                            std::to_string(prop.major) + std::to_string(prop.minor);
            } else {
                g_dev_state = TMB_OK;
                g_sm_count = prop.multiProcessorCount;
                // stream-ordered scratch (cudaMallocAsync) stays mapped between
                // calls: with the default release threshold of 0 every
                // synchronisation unmapped it and the next per-example plugin
                // call paid ~1 ms to map it again
                cudaMemPool_t pool;
                if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
                    uint64_t keep = UINT64_MAX;
                    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
                }
                cudaGetLastError();
            }
        }
    }
    if (g_dev_state != TMB_OK) g_last_error = g_dev_msg;
    return g_dev_state;
}

int sm_count() {
    if (g_sm_count == 0) require_device();
    return g_sm_count > 0 ? g_sm_count : 148;
}

}  // namespace tmb

using namespace tmb;

extern "C" {

int tmb_abi_version(void) { return TMB_ABI_VERSION; }

const char *tmb_last_error(void) { return g_last_error.c_str(); }

uint64_t tmb_launch_count(void) { return g_launches.load(); }

int tmb_device_info(int device, int *sm, int *cc_major, int *cc_minor, int64_t *l2_bytes,
                    int *max_smem_per_block) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device >= n) {
        cudaGetLastError();
        return fail(TMB_E_NO_DEVICE, "no such CUDA device");
    }
    cudaDeviceProp p;
    TMB_CUDA(cudaGetDeviceProperties(&p, device));
    if (sm) *sm = p.multiProcessorCount;
    if (cc_major) *cc_major = p.major;
    if (cc_minor) *cc_minor = p.minor;
    if (l2_bytes) *l2_bytes = p.l2CacheSize;
    if (max_smem_per_block) *max_smem_per_block = (int)p.sharedMemPerBlockOptin;
    return TMB_OK;
}

uint64_t tmb_derive_stream(uint64_t seed, uint64_t index) { return derive_stream(seed, index); }

int tmb_shuffle_permutation(int64_t n, uint64_t stream_seed, uint64_t counter, int64_t *perm,
                            uint64_t *counter_out) {
    if (n < 0 || (n > 0 && !perm)) return fail(TMB_E_INVALID, "shuffle: bad arguments");
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    if (n > 1) {
        uint64_t k = counter;
        for (int64_t i = n - 1; i > 0; --i, ++k) {
            double u = u01_from53(draw53(stream_seed, k));
            int64_t j = (int64_t)(u * (double)(i + 1));
            int64_t t = perm[i];
            perm[i] = perm[j];
            perm[j] = t;
        }
        counter += (uint64_t)(n - 1);
    }
    if (counter_out) *counter_out = counter;
    return TMB_OK;
}

}  // extern "C"
