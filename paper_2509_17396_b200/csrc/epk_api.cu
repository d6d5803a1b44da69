// epk_api.cu -- the C ABI (include/epk/epk.h): argument checking, context,
// workspace, and the host orchestration that must stay on the host (the
// k-means++ seeding and empty-cluster repair consume the reference RNG
// stream, clustering.hpp:158-191,213-232).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <vector>

#include "epk_internal.cuh"

namespace epk {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e);
    return EPK_ERR_CUDA;
}

int ws_require(epk_ctx* ctx, int64_t bytes) {
    if (bytes <= ctx->ws_bytes) return EPK_OK;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (ctx->stream) cudaStreamIsCapturing(ctx->stream, &st);
    if (st != cudaStreamCaptureStatusNone)
        return fail(EPK_ERR_ARG, "workspace must be reserved (epk_ctx_reserve) before graph capture");
    if (ctx->ws) {
        EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        EPK_CUDA_CHECK(cudaFree(ctx->ws));
        ctx->ws = nullptr;
        ctx->ws_bytes = 0;
    }
    const int64_t grow = align_up(bytes + bytes / 4, 1 << 20);
    EPK_CUDA_CHECK(cudaMalloc(&ctx->ws, size_t(grow)));
    ctx->ws_bytes = grow;
    return EPK_OK;
}

int ensure_aux_stream(epk_ctx* ctx) {
    if (ctx->aux) return EPK_OK;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (ctx->stream) cudaStreamIsCapturing(ctx->stream, &st);
    if (st != cudaStreamCaptureStatusNone) return fail(EPK_ERR_ARG, "run the call once before graph capture");
    int least = 0, greatest = 0;
    EPK_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    EPK_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, greatest));
    EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_aux_fork, cudaEventDisableTiming));
    EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_aux_join, cudaEventDisableTiming));
    return EPK_OK;
}

void prof_begin(epk_ctx* ctx, const char* name) {
    if (!ctx->profiling) return;
    epk_prof_rec r;
    std::snprintf(r.name, sizeof(r.name), "%s", name);
    cudaEventCreate(&r.start);
    cudaEventCreate(&r.stop);
    cudaEventRecord(r.start, ctx->stream);
    r.side = (ctx->side && ctx->stream == ctx->side) ? 1 : 0;
    ctx->prof.push_back(r);
}

void prof_end(epk_ctx* ctx) {
    static const bool trace_sync = std::getenv("EPK_DEBUG_SYNC") != nullptr;
    if (trace_sync) {  // diagnostics: name and completion of every launch
        std::fprintf(stderr, "[epk] launched %s\n", ctx->profiling && !ctx->prof.empty() ? ctx->prof.back().name : "?");
        std::fflush(stderr);
        cudaStreamSynchronize(ctx->stream);
        std::fprintf(stderr, "[epk] done\n");
        std::fflush(stderr);
    }
    if (!ctx->profiling || ctx->prof.empty()) return;
    cudaEventRecord(ctx->prof.back().stop, ctx->stream);
}

static void prof_clear(epk_ctx* ctx) {
    for (auto& r : ctx->prof) {
        cudaEventDestroy(r.start);
        cudaEventDestroy(r.stop);
    }
    ctx->prof.clear();
}

int ws2_require(epk_ctx* ctx, int64_t bytes) {
    if (bytes <= ctx->ws2_bytes) return EPK_OK;
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (ctx->stream) cudaStreamIsCapturing(ctx->stream, &st);
    if (st != cudaStreamCaptureStatusNone)
        return fail(EPK_ERR_ARG, "workspace must be reserved (run one step) before graph capture");
    if (ctx->ws2) {
        EPK_CUDA_CHECK(cudaDeviceSynchronize());
        EPK_CUDA_CHECK(cudaFree(ctx->ws2));
        ctx->ws2 = nullptr;
        ctx->ws2_bytes = 0;
    }
    const int64_t grow = align_up(bytes + bytes / 4, 1 << 20);
    EPK_CUDA_CHECK(cudaMalloc(&ctx->ws2, size_t(grow)));
    ctx->ws2_bytes = grow;
    return EPK_OK;
}

int make_layer_table(const epk_cache_desc* c, LayerTable* t) {
    if (!c) return fail(EPK_ERR_ARG, "null cache descriptor");
    if (c->layers < 1 || c->layers > kMaxLayers) return fail(EPK_ERR_UNSUPPORTED, "layers must be in [1, 128]");
    if (c->kv_heads < 1) return fail(EPK_ERR_ARG, "kv_heads must be >= 1");
    if (!c->layer_base) return fail(EPK_ERR_ARG, "layer_base is null");
    for (int l = 0; l <= c->layers; ++l) {
        t->base[l] = c->layer_base[l];
        if (l > 0 && t->base[l] < t->base[l - 1]) return fail(EPK_ERR_ARG, "layer_base must be non-decreasing");
    }
    for (int l = c->layers + 1; l <= kMaxLayers; ++l) t->base[l] = t->base[c->layers];
    return EPK_OK;
}

int launch_select(epk_ctx*, const epk_cache_desc*, const void*, int, const int64_t*, const int32_t*, int, uint8_t*,
                  int32_t*, int);
int launch_compact(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, const uint8_t*, int, const uint32_t*,
                   const uint64_t*, uint32_t*, uint32_t*);
int launch_select_threshold(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, int, const FusedSelect*,
                            const int64_t*, uint64_t*, int32_t*);
int launch_step_tc_grouped(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, const void*, const void*, int, int,
                           int, const int64_t*, int, cudaStream_t, cudaEvent_t, int, float*, uint8_t*,
                           const FusedSelect&, uint64_t*, int32_t*,
                           int (*)(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, int, const FusedSelect*,
                                   const int64_t*, uint64_t*, int32_t*),
                           int (*)(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, const uint8_t*, int,
                                   const uint32_t*, const uint64_t*, uint32_t*, uint32_t*),
                           epk_cache_desc (*)(const epk_cache_desc*, int, int));
int launch_append(epk_ctx*, const epk_cache_desc*, const void*, const void*, const int32_t*, int);
int launch_pool_scores(epk_ctx*, const epk_cache_desc*, const float*, float*, int);
int scan_epkv(const uint8_t*, int64_t, int64_t*, int64_t*, int64_t*);
int launch_load_epkv(epk_ctx*, const uint8_t*, int64_t, const int64_t*, const epk_cache_desc*);
int kmeans_shards(epk_ctx* const*, int, const double* const*, const int64_t*, int64_t, int64_t, uint64_t, int64_t,
                  int64_t*, double*, int64_t*, double*);
int launch_score_f32(epk_ctx*, const epk_cache_desc*, const float*, const float*, int, int, int, int64_t, float*);
int launch_score_tc(epk_ctx*, const epk_cache_desc*, const void*, const void*, int, int, int, int64_t, float*,
                    const FusedSelect*);
int launch_score_grids(epk_ctx*, int, int, int, const int64_t*, const double*, int, double*);
int launch_expf_probe(epk_ctx*, const float*, float*, int64_t);
int launch_km_dist(epk_ctx*, const double*, int64_t, int64_t, const double*, int64_t, double*);
int launch_km_assign(epk_ctx*, const double*, int64_t, int64_t, const double*, int64_t, int64_t*, double*);
int launch_km_sums(epk_ctx*, const double*, int64_t, int64_t, const int64_t*, int64_t, double*, int64_t*, int);
int launch_km_finalize(epk_ctx*, const double*, const int64_t*, int64_t, int64_t, double*);
int launch_km_sqdist(epk_ctx*, const double*, int64_t, int64_t, const double*, const int64_t*, double*);
int launch_key_cosine(epk_ctx*, const void*, const void*, int, int, int, int64_t, int, double*, int64_t*);
int launch_keydiff(epk_ctx*, const epk_cache_desc*, double*);
int launch_serialize_epkv(epk_ctx*, const epk_cache_desc*, uint64_t, const char*, uint64_t, const int64_t*, int32_t,
                          uint8_t*, int64_t, int64_t*, int64_t*);

bool pdl_enabled() {
    static const bool on = std::getenv("EPK_NO_PDL") == nullptr;
    return on;
}

static int check_ctx(epk_ctx* ctx) {
    if (!ctx) return fail(EPK_ERR_ARG, "null context");
    int dev = -1;
    EPK_CUDA_CHECK(cudaGetDevice(&dev));
    if (dev != ctx->device) EPK_CUDA_CHECK(cudaSetDevice(ctx->device));
    return EPK_OK;
}

static int check_cache(const epk_cache_desc* c) {
    if (!c) return fail(EPK_ERR_ARG, "null cache descriptor");
    if (c->dtype != EPK_F32 && c->dtype != EPK_BF16 && c->dtype != EPK_F64) return fail(EPK_ERR_ARG, "bad cache dtype");
    if (c->head_dim < 1) return fail(EPK_ERR_ARG, "head_dim must be >= 1");
    if (!c->head_off || !c->head_len || !c->pos) return fail(EPK_ERR_ARG, "cache head_off/head_len/pos null");
    if (c->layers < 1 || c->layers > kMaxLayers) return fail(EPK_ERR_UNSUPPORTED, "layers must be in [1, 128]");
    return EPK_OK;
}

}  // namespace epk

using namespace epk;

extern "C" {

const char* epk_last_error(void) { return g_last_error.c_str(); }

const char* epk_status_string(int s) {
    switch (s) {
        case EPK_OK: return "ok";
        case EPK_ERR_ARG: return "invalid argument";
        case EPK_ERR_PIN_OVERFLOW: return "pinned entries exceed layer budget";
        case EPK_ERR_DIM: return "dimension mismatch";
        case EPK_ERR_ZERO_NORM: return "zero-norm input";
        case EPK_ERR_EMPTY_PROMPT: return "empty prompt";
        case EPK_ERR_CUDA: return "CUDA error";
        case EPK_ERR_UNSUPPORTED: return "unsupported shape";
        case EPK_ERR_NAN: return "NaN score";
        default: return "unknown status";
    }
}

int epk_version(void) { return 10000; }

int epk_ctx_create(int device, void* stream, epk_ctx** out) {
    if (!out) return fail(EPK_ERR_ARG, "null out pointer");
    int n = 0;
    EPK_CUDA_CHECK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) return fail(EPK_ERR_ARG, "bad device ordinal");
    EPK_CUDA_CHECK(cudaSetDevice(device));
    cudaDeviceProp prop;
    EPK_CUDA_CHECK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(EPK_ERR_UNSUPPORTED, std::string("needs an sm_100 (B200) device, got ") + prop.name);
    epk_ctx* ctx = new epk_ctx();
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->num_sms = prop.multiProcessorCount;
    // experiments: SM split between the scorer and an overlapped gather
    if (const char* e = std::getenv("EPK_GATHER_SMS")) ctx->gather_sms = std::max(0, std::min(ctx->num_sms - 8, std::atoi(e)));
    if (const char* e = std::getenv("EPK_GATHER_CTAS")) ctx->gather_ctas = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("EPK_GATHER_THREADS")) ctx->gather_threads = std::max(32, std::min(512, std::atoi(e)));
    if (const char* e = std::getenv("EPK_GATHER_SMEM_KB")) ctx->gather_smem = std::max(0, std::atoi(e)) * 1024;
    cudaError_t e = cudaMalloc(&ctx->err_flag, sizeof(int));
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_fail(e, "cudaMalloc(err_flag)");
    }
    e = cudaMemset(ctx->err_flag, 0, sizeof(int));
    if (e != cudaSuccess) {
        cudaFree(ctx->err_flag);
        delete ctx;
        return cuda_fail(e, "cudaMemset(err_flag)");
    }
    *out = ctx;
    return EPK_OK;
}

int epk_ctx_destroy(epk_ctx* ctx) {
    if (!ctx) return EPK_OK;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    else cudaDeviceSynchronize();
    prof_clear(ctx);
    if (ctx->hi) {
        cudaStreamSynchronize(ctx->hi);
        cudaStreamDestroy(ctx->hi);
        cudaEventDestroy(ctx->ev_hi);
    }
    if (ctx->side) {
        cudaStreamSynchronize(ctx->side);
        cudaStreamDestroy(ctx->side);
    }
    if (ctx->aux) {
        cudaStreamSynchronize(ctx->aux);
        cudaStreamDestroy(ctx->aux);
        cudaEventDestroy(ctx->ev_aux_fork);
        cudaEventDestroy(ctx->ev_aux_join);
    }
    if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
    if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
    if (ctx->ws2) cudaFree(ctx->ws2);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->step_buf) cudaFree(ctx->step_buf);
    if (ctx->err_flag) cudaFree(ctx->err_flag);
    delete ctx;
    return EPK_OK;
}

int epk_ctx_set_stream(epk_ctx* ctx, void* stream) {
    if (!ctx) return fail(EPK_ERR_ARG, "null context");
    ctx->stream = static_cast<cudaStream_t>(stream);
    return EPK_OK;
}

int epk_ctx_reserve(epk_ctx* ctx, int64_t bytes) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return ws_require(ctx, bytes);
}

int epk_ctx_synchronize(epk_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return EPK_OK;
}

int epk_ctx_poll_error(epk_ctx* ctx) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    int v = 0;
    EPK_CUDA_CHECK(cudaMemcpyAsync(&v, ctx->err_flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    if (v != 0) {
        EPK_CUDA_CHECK(cudaMemsetAsync(ctx->err_flag, 0, sizeof(int), ctx->stream));
        EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (v == EPK_ERR_PIN_OVERFLOW) return fail(v, "evict_to_budget: pinned entries exceed layer budget");
        if (v == EPK_ERR_NAN) return fail(v, "evict_to_budget: NaN score (non-finite keys or prompt)");
        if (v == EPK_ERR_CUDA) return fail(v, "device-side wait timed out (a producer kernel never ran)");
        return fail(v, "device-side check failed: a head longer than n_max_per_head, or slack / output capacity "
                       "too small");
    }
    return EPK_OK;
}

int64_t epk_ctx_launch_count(epk_ctx* ctx) { return ctx ? ctx->launches : -1; }

#ifdef EPK_TIMELINE
extern "C++" {
namespace epk {
static std::vector<int (*)(int, unsigned long long*, int)>& tl_readers() {
    static std::vector<int (*)(int, unsigned long long*, int)> r;
    return r;
}
int tl_register(int (*reader)(int, unsigned long long*, int)) {
    tl_readers().push_back(reader);
    return 1;
}
}  // namespace epk
}
// experiment builds only: copies every translation unit's timeline records
// out (reset != 0 clears the rings after copying); returns the record count
extern "C" int epk_debug_timeline(int reset, unsigned long long* out, int max_records) {
    if (cudaDeviceSynchronize() != cudaSuccess) return -1;
    int n = 0;
    for (auto f : epk::tl_readers()) n += f(reset, out ? out + int64_t(n) * 4 : nullptr, max_records - n);
    return n;
}
#endif

int epk_ctx_profile(epk_ctx* ctx, int32_t enable) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    prof_clear(ctx);
    ctx->profiling = enable != 0;
    return EPK_OK;
}

int64_t epk_ctx_profile_read(epk_ctx* ctx, int64_t index, char* name_out, float* ms_out) {
    if (!ctx) return -1;
    if (index < 0) {
        if (cudaStreamSynchronize(ctx->stream) != cudaSuccess) return -1;
        return int64_t(ctx->prof.size());
    }
    if (index >= int64_t(ctx->prof.size())) return -1;
    const epk_prof_rec& r = ctx->prof[size_t(index)];
    std::snprintf(name_out, 32, "%s", r.name);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.start, r.stop);
    *ms_out = ms;
    return int64_t(ctx->prof.size());
}

int epk_ctx_profile_timeline(epk_ctx* ctx, int64_t index, char* name_out, float* start_ms, float* dur_ms,
                             int32_t* side) {
    if (!ctx || index < 0 || index >= int64_t(ctx->prof.size())) return EPK_ERR_ARG;
    const epk_prof_rec& r = ctx->prof[size_t(index)];
    std::snprintf(name_out, 32, "%s", r.name);
    float t0 = 0.f, d = 0.f;
    cudaEventElapsedTime(&t0, ctx->prof[0].start, r.start);
    cudaEventElapsedTime(&d, r.start, r.stop);
    *start_ms = t0;
    *dur_ms = d;
    *side = r.side;
    return EPK_OK;
}

int epk_score(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int32_t q_heads,
              int32_t prompt_len, int32_t aggregation, int32_t mode, int64_t n_max, float* scores) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(c))) return rc;
    if (prompt_len <= 0) return fail(EPK_ERR_EMPTY_PROMPT, "score_with_prompt: empty prompt");
    if (q_heads < c->kv_heads || q_heads % c->kv_heads != 0)
        return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
    if (!q || !kp || !scores) return fail(EPK_ERR_ARG, "score: null pointer");
    if (aggregation != EPK_AGG_MAX && aggregation != EPK_AGG_AVG) return fail(EPK_ERR_ARG, "bad aggregation");
    if (mode == EPK_SCORE_EXACT_F32)
        return launch_score_f32(ctx, c, static_cast<const float*>(q), static_cast<const float*>(kp), q_heads,
                                prompt_len, aggregation == EPK_AGG_MAX, n_max, scores);
    if (mode == EPK_SCORE_TC_BF16)
        return launch_score_tc(ctx, c, q, kp, q_heads, prompt_len, aggregation == EPK_AGG_MAX, n_max, scores, nullptr);
    return fail(EPK_ERR_ARG, "bad score mode");
}

int epk_score_grids(epk_ctx* ctx, int32_t q_heads, int32_t kv_heads, int32_t prompt_len, const int64_t* head_off,
                    const double* grids, int32_t aggregation, double* scores) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (!head_off) return fail(EPK_ERR_ARG, "null head_off");
    return launch_score_grids(ctx, q_heads, kv_heads, prompt_len, head_off, grids, aggregation == EPK_AGG_MAX,
                              scores);
}

int epk_select_pooled(epk_ctx* ctx, const epk_cache_desc* c, const void* scores, int32_t score_dtype,
                      const int64_t* budgets, const int32_t* pins, int32_t n_pins, uint8_t* keep, int32_t* kept,
                      int32_t synchronous) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(c))) return rc;
    if (!scores || !budgets || !keep) return fail(EPK_ERR_ARG, "select: null pointer");
    if (n_pins < 0) return fail(EPK_ERR_ARG, "select: negative pin count");
    rc = launch_select(ctx, c, scores, score_dtype, budgets, pins, n_pins, keep, kept, 0);
    if (rc) return rc;
    if (synchronous) return epk_ctx_poll_error(ctx);
    return EPK_OK;
}

int epk_pool_scores(epk_ctx* ctx, const epk_cache_desc* c, const float* scores, float* pooled, int32_t kernel) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(c))) return rc;
    if (!scores || !pooled) return fail(EPK_ERR_ARG, "pool_scores: null pointer");
    if (scores == pooled) return fail(EPK_ERR_ARG, "pool_scores: in-place pooling is not supported");
    return launch_pool_scores(ctx, c, scores, pooled, kernel);
}

int epk_select_per_head(epk_ctx* ctx, const epk_cache_desc* c, const void* scores, int32_t score_dtype,
                        const int64_t* k_per_layer, uint8_t* keep) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(c))) return rc;
    if (!scores || !k_per_layer || !keep) return fail(EPK_ERR_ARG, "select: null pointer");
    return launch_select(ctx, c, scores, score_dtype, k_per_layer, nullptr, 0, keep, nullptr, 1);
}

int epk_compact(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out, const uint8_t* keep,
                int32_t slack) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(in)) || (rc = check_cache(out))) return rc;
    if (!keep) return fail(EPK_ERR_ARG, "compact: null keep");
    return launch_compact(ctx, in, out, keep, slack, nullptr, nullptr, nullptr, nullptr);
}

int epk_append(epk_ctx* ctx, const epk_cache_desc* c, const void* k_new, const void* v_new, const int32_t* positions,
               int32_t len, int32_t slack) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(c))) return rc;
    if (!k_new || !v_new || !positions) return fail(EPK_ERR_ARG, "append: null pointer");
    if (slack < 0) return fail(EPK_ERR_ARG, "append: negative slack");
    // slack > 0: the gap the caller left after every head (epk_compact's
    // out_slack); a block longer than it can never fit.  The device checks
    // every head's actual gap either way (deferred EPK_ERR_ARG).
    if (slack > 0 && len > slack)
        return fail(EPK_ERR_ARG, "append: block of " + std::to_string(len) + " rows exceeds the slack of " +
                                     std::to_string(slack) + " rows per head");
    return launch_append(ctx, c, k_new, v_new, positions, len);
}

int epk_ctx_set_option(epk_ctx* ctx, int32_t option, int64_t value) {
    if (!ctx) return fail(EPK_ERR_ARG, "null context");
    switch (option) {
        case EPK_OPT_LAYER_GROUP:
            if (value < 0) return fail(EPK_ERR_ARG, "layer group must be >= 0");
            ctx->layer_group = int(value);
            return EPK_OK;
        case EPK_OPT_OVERLAP:
            ctx->overlap = value != 0;
            return EPK_OK;
        case EPK_OPT_POOL_KERNEL:
            if (value < 1 || value % 2 == 0 || value > 4095) return fail(EPK_ERR_ARG, "pool kernel must be odd, 1..4095");
            ctx->pool_kernel = int(value);
            return EPK_OK;
        default:
            return fail(EPK_ERR_ARG, "unknown option");
    }
}

static epk_cache_desc layer_view(const epk_cache_desc* c, int l0, int l1) {
    epk_cache_desc v = *c;
    v.layers = l1 - l0;
    v.head_off = c->head_off + int64_t(l0) * (c->kv_heads + 1);
    v.head_len = c->head_len + int64_t(l0) * c->kv_heads;
    v.layer_base = c->layer_base + l0;
    return v;
}

int epk_evict_step(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out, const void* q,
                   const void* kp, int32_t q_heads, int32_t prompt_len, const int64_t* budgets, const int32_t* pins,
                   int32_t n_pins, int32_t aggregation, int32_t mode, int64_t n_max, int32_t out_slack,
                   float* scores_ws, int32_t* kept) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(in)) || (rc = check_cache(out))) return rc;
    if (in->layers != out->layers) return fail(EPK_ERR_DIM, "evict_step: in/out layer counts differ");
    const int64_t rows = in->layer_base[in->layers];
    const int L = in->layers;
    // Tensor-core steps without pins take the fused selection: the scorer
    // writes keys + score histograms, select_threshold_kernel finds each
    // layer's threshold from them, the compaction derives keep[] itself.
    const bool pooled = ctx->pool_kernel > 1;  // opt-in smoothing: scores -> pool -> generic select
    const bool fused = mode == EPK_SCORE_TC_BF16 && n_pins == 0 && in->kv_heads <= 64 && !pooled;
    // Step buffers live in their own allocation so the kernels' workspace
    // growth never aliases them.  Layout: histograms at fixed offsets for
    // kMaxLayers layers (zeroed once here, re-zeroed by every step's P1
    // launch), thresholds, then the row-indexed scores / keep mask / keys.
    const int64_t o_hc = int64_t(kMaxLayers) * 65536 * 4;
    const int64_t o_thr = o_hc + int64_t(kMaxLayers) * 256 * 4;
    const int64_t o_cand = o_thr + int64_t(kMaxLayers) * 16;             // [kMaxLayers][1024] uint4
    const int64_t o_cnt = o_cand + int64_t(kMaxLayers) * 1024 * 16;     // cand_n, done: [kMaxLayers] each
    const int64_t o_scores = o_cnt + int64_t(kMaxLayers) * 8;
    const int64_t o_keep = o_scores + align_up(rows * 4, 256);
    const int64_t o_keys = o_keep + align_up(rows, 256);
    const int64_t o_pool = o_keys + align_up(rows * 4, 256);
    const int64_t need = o_pool + (pooled ? align_up(rows * 4, 256) : 0);
    const bool capturing = [&] {
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(ctx->stream, &st);
        return st != cudaStreamCaptureStatusNone;
    }();
    if (need > ctx->step_bytes) {
        if (capturing) return fail(EPK_ERR_ARG, "run one step before capturing a graph");
        if (ctx->step_buf) {
            EPK_CUDA_CHECK(cudaDeviceSynchronize());
            EPK_CUDA_CHECK(cudaFree(ctx->step_buf));
            ctx->step_buf = nullptr;
            ctx->step_bytes = 0;
        }
        EPK_CUDA_CHECK(cudaMalloc(&ctx->step_buf, size_t(need)));
        EPK_CUDA_CHECK(cudaMemsetAsync(ctx->step_buf, 0, size_t(need), ctx->stream));
        ctx->step_bytes = need;
    }
    char* sb = static_cast<char*>(ctx->step_buf);
    float* scores = scores_ws ? scores_ws : reinterpret_cast<float*>(sb + o_scores);
    uint8_t* keep = reinterpret_cast<uint8_t*>(sb + o_keep);
    uint32_t* keys = reinterpret_cast<uint32_t*>(sb + o_keys);
    uint32_t* hist_f = reinterpret_cast<uint32_t*>(sb);
    uint32_t* hist_c = reinterpret_cast<uint32_t*>(sb + o_hc);
    uint64_t* thr = reinterpret_cast<uint64_t*>(sb + o_thr);

    // Layer groups (EPK_OPT_LAYER_GROUP): 0 = auto = all layers in one group.
    // Smaller groups let a group's select+compact (side stream) overlap the
    // next group's scoring, at the cost of more, smaller launches.
    int G = ctx->layer_group;
    if (G <= 0) G = L;
    G = std::min(G, L);
    const bool overlap = ctx->overlap && G < L;
    if (overlap && !ctx->side) {
        if (capturing) return fail(EPK_ERR_ARG, "run one step before capturing a graph");
        // compaction at the lowest priority, the scoring / select chain at the
        // highest: when SM slots free up, the latency-critical select CTAs go first
        int least = 0, greatest = 0;
        EPK_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        EPK_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, least));
        EPK_CUDA_CHECK(cudaStreamCreateWithPriority(&ctx->hi, cudaStreamNonBlocking, greatest));
        EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
        EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
        EPK_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->ev_hi, cudaEventDisableTiming));
    }
    const int64_t qlayer = int64_t(q_heads) * prompt_len * in->head_dim * dtype_size(in->dtype);
    const int64_t klayer = int64_t(in->kv_heads) * prompt_len * in->head_dim * dtype_size(in->dtype);
    cudaStream_t main = ctx->stream;
    if (fused) {
        // P1 over all layers, then per group: P2 -> threshold select (main)
        // -> count/plan/gather (side stream when overlapping)
        if (prompt_len <= 0) return fail(EPK_ERR_EMPTY_PROMPT, "score_with_prompt: empty prompt");
        if (q_heads < in->kv_heads || q_heads % in->kv_heads != 0)
            return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
        if (aggregation != EPK_AGG_MAX && aggregation != EPK_AGG_AVG) return fail(EPK_ERR_ARG, "bad aggregation");
        unsigned* cnt = reinterpret_cast<unsigned*>(sb + o_cnt);
        const FusedSelect fs_all{keys, hist_f, hist_c, reinterpret_cast<uint4*>(sb + o_cand), cnt, cnt + kMaxLayers};
        static const bool no_hi = std::getenv("EPK_NO_HI_STREAM") != nullptr;  // A/B
        const bool use_hi = overlap && !no_hi;
        if (use_hi) {  // fork the user's stream onto the high-priority one
            EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_hi, main));
            EPK_CUDA_CHECK(cudaStreamWaitEvent(ctx->hi, ctx->ev_hi, 0));
            ctx->stream = ctx->hi;
        }
        // the fused selection works from the keys: the fp32 scores are written
        // only when the caller asked for them
        rc = launch_step_tc_grouped(ctx, in, out, q, kp, q_heads, prompt_len, aggregation == EPK_AGG_MAX, budgets, G,
                                    overlap ? ctx->side : nullptr, ctx->ev_fork, out_slack, scores_ws, keep, fs_all, thr,
                                    kept, launch_select_threshold, launch_compact, layer_view);
        ctx->stream = main;
        if (rc) return rc;
        if (overlap) {
            EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_join, ctx->side));
            EPK_CUDA_CHECK(cudaStreamWaitEvent(main, ctx->ev_join, 0));
        }
        if (use_hi) {
            EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_hi, ctx->hi));
            EPK_CUDA_CHECK(cudaStreamWaitEvent(main, ctx->ev_hi, 0));
        }
        return EPK_OK;
    }
    for (int l0 = 0; l0 < L; l0 += G) {
        const int l1 = std::min(L, l0 + G);
        const epk_cache_desc vin = layer_view(in, l0, l1);
        const epk_cache_desc vout = layer_view(out, l0, l1);
        const void* qg = static_cast<const char*>(q) + l0 * qlayer;
        const void* kpg = static_cast<const char*>(kp) + l0 * klayer;
        unsigned* cnt = reinterpret_cast<unsigned*>(sb + o_cnt);
        const FusedSelect fs{keys,
                             hist_f + int64_t(l0) * 65536,
                             hist_c + int64_t(l0) * 256,
                             reinterpret_cast<uint4*>(sb + o_cand) + int64_t(l0) * 1024,
                             cnt + l0,
                             cnt + kMaxLayers + l0};
        if (fused) {
            if (prompt_len <= 0) return fail(EPK_ERR_EMPTY_PROMPT, "score_with_prompt: empty prompt");
            if (q_heads < in->kv_heads || q_heads % in->kv_heads != 0)
                return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
            if (aggregation != EPK_AGG_MAX && aggregation != EPK_AGG_AVG) return fail(EPK_ERR_ARG, "bad aggregation");
            rc = launch_score_tc(ctx, &vin, qg, kpg, q_heads, prompt_len, aggregation == EPK_AGG_MAX, n_max, scores,
                                 &fs);
        } else {
            rc = epk_score(ctx, &vin, qg, kpg, q_heads, prompt_len, aggregation, mode, n_max, scores);
            if (rc == EPK_OK && pooled)
                rc = launch_pool_scores(ctx, &vin, scores, reinterpret_cast<float*>(sb + o_pool), ctx->pool_kernel);
        }
        if (rc) return rc;
        // select + compact of this group run on the side stream (when
        // overlapping) so the main stream goes straight on to the next
        // group's scoring; scores/keys/keep are row-indexed and the
        // histograms/thresholds layer-indexed, so groups never alias.
        if (overlap) {
            EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_fork, main));
            EPK_CUDA_CHECK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
            ctx->stream = ctx->side;
        }
        if (fused) {
            rc = launch_select_threshold(ctx, &vin, &vout, out_slack, &fs, budgets + l0, thr + 2 * l0,
                                         kept ? kept + l0 : nullptr);
            if (rc == EPK_OK)
                rc = launch_compact(ctx, &vin, &vout, keep, out_slack, keys, thr + 2 * l0, fs.hist_fine, fs.hist_coarse);
        } else {
            rc = launch_select(ctx, &vin, pooled ? reinterpret_cast<const float*>(sb + o_pool) : scores, EPK_F32,
                               budgets + l0, pins, n_pins, keep, kept ? kept + l0 : nullptr, 0);
            if (rc == EPK_OK) rc = launch_compact(ctx, &vin, &vout, keep, out_slack, nullptr, nullptr, nullptr, nullptr);
        }
        ctx->stream = main;
        if (rc) return rc;
    }
    if (overlap) {
        EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_join, ctx->side));
        EPK_CUDA_CHECK(cudaStreamWaitEvent(main, ctx->ev_join, 0));
    }
    return EPK_OK;
}

// ---- K4 ---------------------------------------------------------------------
int epk_kmeans_assign(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const double* cent, int64_t k,
                      int64_t* assign, double* best_d2) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (n < 1 || dim < 1 || k < 1) return fail(EPK_ERR_ARG, "kmeans_assign: empty input");
    return launch_km_assign(ctx, pts, n, dim, cent, k, assign, best_d2);
}

int epk_kmeans_partial_sums(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const int64_t* assign, int64_t k,
                            double* sums, int64_t* counts, int32_t accumulate) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return launch_km_sums(ctx, pts, n, dim, assign, k, sums, counts, accumulate);
}

int epk_kmeans_finalize(epk_ctx* ctx, const double* sums, const int64_t* counts, int64_t k, int64_t dim,
                        double* cent) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return launch_km_finalize(ctx, sums, counts, k, dim, cent);
}

int epk_kmeans_sq_dist(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const double* cent,
                       const int64_t* assign, double* d2) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return launch_km_sqdist(ctx, pts, n, dim, cent, assign, d2);
}

int epk_kmeans(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, int64_t k, uint64_t seed, int64_t max_iters,
               int64_t* assign_out, double* cent_out, int64_t* iters_out, double* sse_out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    // one shard of the multi-GPU orchestration (multigpu.cu): one code path
    epk_ctx* ctxs[1] = {ctx};
    const double* shards[1] = {pts};
    const int64_t ns[1] = {n};
    return kmeans_shards(ctxs, 1, shards, ns, dim, k, seed, max_iters, assign_out, cent_out, iters_out, sse_out);
}

// ---- K5 ---------------------------------------------------------------------
int epk_key_cosine_sigma(epk_ctx* ctx, const void* kf, const void* kb, int32_t dtype, int32_t layers, int32_t H,
                         int64_t ntok, int32_t dim, double* sigma, int64_t* skipped) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if (layers < 1 || H < 1 || ntok < 1 || dim < 1) return fail(EPK_ERR_ARG, "key_cosine: empty input");
    if (dtype != EPK_F32 && dtype != EPK_BF16 && dtype != EPK_F64) return fail(EPK_ERR_ARG, "key_cosine: bad dtype");
    return launch_key_cosine(ctx, kf, kb, dtype, layers, H, ntok, dim, sigma, skipped);
}

int epk_score_keydiff(epk_ctx* ctx, const epk_cache_desc* cache, double* scores) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(cache))) return rc;
    if (!scores) return fail(EPK_ERR_ARG, "keydiff: null scores");
    return launch_keydiff(ctx, cache, scores);
}

int epk_serialize_epkv(epk_ctx* ctx, const epk_cache_desc* cache, uint64_t episode_id, const char* scorer,
                       uint64_t budget_per_head, const int64_t* layer_budgets, int32_t n_layer_budgets,
                       uint8_t* out, int64_t capacity, int64_t* offset_out, int64_t* total_out) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(cache))) return rc;
    if (n_layer_budgets < 0) return fail(EPK_ERR_ARG, "persist: negative layer budget count");
    return launch_serialize_epkv(ctx, cache, episode_id, scorer, budget_per_head, layer_budgets, n_layer_budgets, out,
                                 capacity, offset_out, total_out);
}

int epk_epkv_scan(const uint8_t* bytes, int64_t nbytes, int64_t* info, int64_t* counts, int64_t* entry_off) {
    if (!info) return fail(EPK_ERR_ARG, "load: null info");
    return scan_epkv(bytes, nbytes, info, counts, entry_off);
}

int epk_load_epkv(epk_ctx* ctx, const uint8_t* dev_file, int64_t pad, const int64_t* entry_off,
                  const epk_cache_desc* cache) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    if ((rc = check_cache(cache))) return rc;
    if (!dev_file || !entry_off) return fail(EPK_ERR_ARG, "load: null pointer");
    return launch_load_epkv(ctx, dev_file, pad, entry_off, cache);
}

// ---- diagnostics ---------------------------------------------------------------
int epk_debug_expf(epk_ctx* ctx, const float* x, float* y, int64_t n) {
    int rc = check_ctx(ctx);
    if (rc) return rc;
    return launch_expf_probe(ctx, x, y, n);
}

}  // extern "C"
