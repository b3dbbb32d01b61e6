// tmb_sparse.cu -- SparseTM (sparse.py:78-256) on the device.  Placeholder
// until the sparse kernels land: every entry point reports TMB_E_UNSUPPORTED.
#include "tmb_common.cuh"

using namespace tmb;

struct tmb_sparse {
    int unused;
};

extern "C" {
int tmb_sparse_create(const tmb_sparse_cfg *, const int32_t *, int64_t, tmb_sparse **) {
    return fail(TMB_E_UNSUPPORTED, "sparse: not built yet");
}
int tmb_sparse_destroy(tmb_sparse *) { return TMB_OK; }
int tmb_sparse_train(tmb_sparse *, const int64_t *, const int32_t *, const int32_t *,
                     const int32_t *, int64_t, uint64_t, tmb_train_stats *, void *) {
    return fail(TMB_E_UNSUPPORTED, "sparse: not built yet");
}
int tmb_sparse_get(const tmb_sparse *, int32_t *, int32_t *, int8_t *, int32_t *, uint64_t *,
                   void *) {
    return fail(TMB_E_UNSUPPORTED, "sparse: not built yet");
}
int tmb_sparse_set(tmb_sparse *, const int32_t *, const int32_t *, const int8_t *,
                   const int32_t *, const uint64_t *, void *) {
    return fail(TMB_E_UNSUPPORTED, "sparse: not built yet");
}
int tmb_sparse_infer(const tmb_sparse *, const int64_t *, const int32_t *, int64_t, int64_t *,
                     int64_t *, void *) {
    return fail(TMB_E_UNSUPPORTED, "sparse: not built yet");
}
}
