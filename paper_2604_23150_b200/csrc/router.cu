// K1 placeholder: replaced by the tcgen05 router GEMM in the next commit.
#include "internal.cuh"

using namespace mpb;

extern "C" mpb_status mpb_router_topk(mpb_context *ctx, const void *X, const void *W, uint64_t T,
                                      uint32_t H, uint32_t E, uint32_t k, int score_fn, int renorm,
                                      int32_t *idx, float *weights, float *logits_out) {
    (void)ctx; (void)X; (void)W; (void)T; (void)H; (void)E; (void)k; (void)score_fn;
    (void)renorm; (void)idx; (void)weights; (void)logits_out;
    return fail(MPB_ERROR, "mpb_router_topk: not built yet");
}
