// score_tc.cu -- K1: tcgen05/TMEM tensor-core scorer (bf16 in, fp32 accum).
#include "epk_internal.cuh"

namespace epk {

int launch_score_tc(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int hq, int p,
                    int agg_max, int64_t n_max, float* scores) {
    (void)ctx; (void)c; (void)q; (void)kp; (void)hq; (void)p; (void)agg_max; (void)n_max; (void)scores;
    return fail(EPK_ERR_UNSUPPORTED, "tensor-core scorer not built yet");
}

}  // namespace epk
