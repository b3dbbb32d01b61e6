// tmb_rng.cu -- device fill of a counter-stream block (core.py:98-104); used
// by tests to pin the device SplitMix64 against the reference's values.
#include "tmb_common.cuh"

namespace tmb {
__global__ void k_stream_u64(uint64_t seed, uint64_t start, int64_t count, uint64_t *out) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < count) out[i] = mix64(seed + kGolden * (start + (uint64_t)i + 1));
}
}  // namespace tmb

using namespace tmb;

extern "C" int tmb_stream_u64_block(uint64_t seed, uint64_t start, int64_t count, uint64_t *out,
                                    void *stream) {
    int rc = require_device();
    if (rc) return rc;
    if (count < 0 || (count > 0 && !out)) return fail(TMB_E_INVALID, "stream_u64_block: bad args");
    if (count == 0) return TMB_OK;
    k_stream_u64<<<(unsigned)ceil_div(count, 256), 256, 0, as_stream(stream)>>>(seed, start, count,
                                                                                 out);
    TMB_LAUNCHED();
    return TMB_OK;
}
