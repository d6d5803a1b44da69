/*
 * epk.h -- C ABI of the B200-native EpiCache block-prefill eviction step.
 *
 * This is the drop-in boundary.  Everything below the
 * boundary is sm_100a CUDA (paper_2509_17396_b200/csrc/); everything above it
 * is host code that mirrors the reference epikv C++ API
 * (include/epikv/epikv_gpu.hpp for C++, paper_2509_17396_b200/ for Python).
 *
 * Signatures use plain pointers and sizes only.  Device pointers are marked
 * [dev], host pointers [host].  Every call is enqueued on the context's stream
 * and returns an EPK_* status; epk_last_error() holds the thread's last
 * message.  Functions documented "synchronous" block until the stream drains
 * because their result (an error the reference throws, a host count) is
 * data-dependent.  The library never allocates inside a call except the
 * context's grow-only workspace (reserve it with epk_ctx_reserve before CUDA
 * graph capture).
 *
 * Reference interfaces replaced (file:line under /root/reference/proj/include/epikv):
 *   epk_score            score_with_prompt (scoring.hpp:80) fused with the
 *                        attention-weight loop of forward (toymodel.hpp:327-391)
 *   epk_score_grids      score_with_prompt (scoring.hpp:80) on given grids
 *   epk_select_pooled    evict_to_budget selection (kvcache.hpp:142-190)
 *   epk_select_per_head  top_k_indices (numerics.hpp:111-125) per kv-head
 *   epk_compact          evict_to_budget output loop (kvcache.hpp:192-199)
 *   epk_append           append_to_cache (toymodel.hpp:428-443)
 *   epk_evict_step       one block step of block_prefill (blockprefill.hpp:157-226):
 *                        score -> per-layer evict, all layers
 *   epk_kmeans*          kmeans (clustering.hpp:148-260); epk_kmeans_sharded: the same
 *                        over embeddings sharded across GPUs (NCCL ordered chain)
 *   epk_key_cosine_sigma measure_sensitivity reduction (allocation.hpp:80-100)
 *   epk_score_keydiff    keydiff_scores (scoring.hpp:186-221), the KeyDiff baseline
 *   epk_serialize_epkv   persist (kvcache.hpp:281-317), the episodic cache store's writer
 *   epk_toy_forward      forward (toymodel.hpp:228-411), the model step before the path
 */
#ifndef EPK_EPK_H
#define EPK_EPK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (C++ shim maps them back to the reference exceptions) --- */
#define EPK_OK 0
#define EPK_ERR_ARG (-1)          /* bad argument (epikv::Error)                    */
#define EPK_ERR_PIN_OVERFLOW (-2) /* pinned entries exceed budget (epikv::Error,    */
                                  /*   kvcache.hpp:175-178)                          */
#define EPK_ERR_DIM (-3)          /* shape mismatch (epikv::DimensionError)         */
#define EPK_ERR_ZERO_NORM (-4)    /* epikv::ZeroNormError                           */
#define EPK_ERR_EMPTY_PROMPT (-6) /* score_with_prompt: empty prompt (scoring.hpp:82) */
#define EPK_ERR_CUDA (-7)         /* CUDA runtime / launch failure                  */
#define EPK_ERR_UNSUPPORTED (-8)  /* shape outside what the kernels support         */
#define EPK_ERR_NAN (-9)          /* a score is NaN (non-finite K/Q): no selection   */
                                  /*   order exists (kvcache.hpp:181-185); deferred  */

/* ---- enums ---------------------------------------------------------------- */
#define EPK_F32 0
#define EPK_BF16 1
#define EPK_F64 2

#define EPK_AGG_AVG 0 /* Aggregation::Avg (scoring.hpp:35) */
#define EPK_AGG_MAX 1 /* Aggregation::Max, the default      */

#define EPK_SCORE_EXACT_F32 0 /* CUDA-core fp32, EPK-F32 v1 op order (bit-exact vs oracle) */
#define EPK_SCORE_TC_BF16 1   /* tcgen05/TMEM tensor-core scorer, bf16 inputs, fp32 accum  */

typedef struct epk_ctx epk_ctx;

/*
 * A layered CSR cache ("episode cache"), all layers in one allocation.
 * Layer l owns rows [layer_base[l], layer_base[l+1]) of k/v/pos.  Inside the
 * layer, kv-head h owns the REGION [head_off[h], head_off[h+1]) (layer-relative
 * rows); its live entries are the first head_len[h] rows of the region,
 * position-sorted (the per-head KVEntry list of kvcache.hpp:38-53).  Rows
 * after head_len[h] are free slack that epk_append fills with the next block.
 *   k, v     [dev]  [rows][head_dim] of dtype, row-major, 16-byte aligned rows
 *   pos      [dev]  [rows] int32 token positions
 *   head_off [dev]  [layers][kv_heads+1] int32 (data dependent after eviction)
 *   head_len [dev]  [layers][kv_heads]   int32
 *   layer_base [host] [layers+1] int64 capacity layout (layer_base[layers] = rows)
 */
typedef struct epk_cache_desc {
    int32_t layers;
    int32_t kv_heads;
    int32_t head_dim;
    int32_t dtype;
    void* k;
    void* v;
    int32_t* pos;
    int32_t* head_off;
    int32_t* head_len;
    const int64_t* layer_base;
} epk_cache_desc;

/* ---- context ---------------------------------------------------------------- */
int epk_ctx_create(int device, void* cuda_stream, epk_ctx** out);
int epk_ctx_destroy(epk_ctx* ctx);
int epk_ctx_set_stream(epk_ctx* ctx, void* cuda_stream);
int epk_ctx_reserve(epk_ctx* ctx, int64_t workspace_bytes);
int epk_ctx_synchronize(epk_ctx* ctx);
/* Deferred device-side errors (pin overflow inside epk_evict_step): returns the
 * first EPK_* error raised since the last call and clears it.  Synchronous. */
int epk_ctx_poll_error(epk_ctx* ctx);
const char* epk_last_error(void);
const char* epk_status_string(int status);
int epk_version(void);
/* Options for epk_evict_step:
 *   EPK_OPT_LAYER_GROUP  layers scored/selected/compacted per group (0 = auto:
 *                        all layers in one group)
 *   EPK_OPT_OVERLAP      1 (default): with more than one group, each group's
 *                        select + compaction runs on a second stream,
 *                        overlapping the next group's scoring
 *   EPK_OPT_POOL_KERNEL  1 (default, the reference's semantics) or an odd
 *                        kernel w > 1: the step max-pools every head's scores
 *                        over a w-row window before selecting (opt-in; see
 *                        epk_pool_scores) */
#define EPK_OPT_LAYER_GROUP 1
#define EPK_OPT_OVERLAP 2
#define EPK_OPT_POOL_KERNEL 4
int epk_ctx_set_option(epk_ctx* ctx, int32_t option, int64_t value);
/* Number of kernels this library launched on the context since creation. */
int64_t epk_ctx_launch_count(epk_ctx* ctx);
/* Live per-kernel timing: while enabled, every kernel launch is bracketed by
 * CUDA events on the context stream.  Enabling clears the record.
 * epk_ctx_profile_read(ctx, -1, ...) synchronises and returns the record
 * count; index >= 0 returns the kernel name (<= 31 chars) and milliseconds. */
int epk_ctx_profile(epk_ctx* ctx, int32_t enable);
int64_t epk_ctx_profile_read(epk_ctx* ctx, int64_t index, char* name_out, float* ms_out);
/* Timeline of record `index` (after epk_ctx_profile_read(ctx, -1, ...)):
 * start relative to record 0's start, duration, and whether it was launched
 * on the context's side stream (overlapped select/compaction). */
int epk_ctx_profile_timeline(epk_ctx* ctx, int64_t index, char* name_out, float* start_ms, float* dur_ms,
                             int32_t* side);

/* ---- K1 / K1': fused patched-prompt scoring --------------------------------- *
 * scores[layer_base[l] + r] = score of live row r of layer l (fp32 [dev]).
 *   q_prompt [dev] [layers][q_heads][prompt_len][head_dim]  (dtype of cache)
 *   k_prompt [dev] [layers][kv_heads][prompt_len][head_dim]
 * mode EPK_SCORE_EXACT_F32 needs dtype F32; EPK_SCORE_TC_BF16 needs dtype BF16,
 * head_dim 128, prompt_len <= 256 and (q_heads/kv_heads)*prompt_len <= 2048
 * (longer prompts, e.g. KVzip's block repetition: epk_score_grids).
 * n_max_per_head [host] must bound every head's live count: the exact-f32
 * scorer sizes its logits scratch with it and refuses a longer head (deferred
 * EPK_ERR_ARG, epk_ctx_poll_error; that head's scores are not written); the
 * tensor-core scorer reads the live lengths on the device and needs no bound.
 * Asynchronous. */
int epk_score(epk_ctx* ctx, const epk_cache_desc* cache, const void* q_prompt,
              const void* k_prompt, int32_t q_heads, int32_t prompt_len, int32_t aggregation,
              int32_t mode, int64_t n_max_per_head, float* scores);

/* score_with_prompt on explicit fp64 attention grids for ONE layer.
 *   grids [dev] concatenated per query head qh: prompt_len x (n_h + prompt_len),
 *   n_h = head_off[h+1]-head_off[h] with h = qh / (q_heads/kv_heads)
 *   head_off [host] [kv_heads+1]; scores [dev] fp64 [head_off[kv_heads]].
 * Bit-exact with the reference (sequential window sum). Asynchronous. */
int epk_score_grids(epk_ctx* ctx, int32_t q_heads, int32_t kv_heads, int32_t prompt_len,
                    const int64_t* head_off, const double* grids, int32_t aggregation,
                    double* scores);

/* ---- opt-in score smoothing (north_star's "1-D max-pool smoothing") -------- *
 * NOT part of the reference (score_with_prompt has no pooling, scoring.hpp:
 * 80-128): SnapKV-style max_pool1d, odd kernel w, stride 1, "same" padding,
 * over every (layer, head)'s live rows in position order, never across heads:
 *   pooled[r] = max scores[i], i live in r's head, |i - r| <= w / 2.
 * scores, pooled [dev] fp32 [rows] (distinct buffers).  Asynchronous. */
int epk_pool_scores(epk_ctx* ctx, const epk_cache_desc* cache, const float* scores, float* pooled, int32_t kernel);

/* ---- K2: selection -------------------------------------------------------- *
 * Pooled selection of evict_to_budget for every layer of `cache`:
 * keep[layer_base[l]+r] = 1 iff row r is retained.  Per layer: under budget
 * (live <= kv_heads*budget[l]) keeps everything; else pins (sorted positions,
 * [dev]) are kept and the best kv_heads*budget[l]-pinned_live candidates by
 * (score desc, position asc, head asc) are kept.  scores are fp32 or fp64
 * (score_dtype) in cache row order.  kept_per_layer [dev, optional] int32 [layers].
 * Pin overflow raises EPK_ERR_PIN_OVERFLOW (synchronous check when
 * `synchronous` != 0, else deferred to epk_ctx_poll_error). */
int epk_select_pooled(epk_ctx* ctx, const epk_cache_desc* cache, const void* scores,
                      int32_t score_dtype, const int64_t* layer_budgets, const int32_t* pins,
                      int32_t n_pins, uint8_t* keep, int32_t* kept_per_layer, int32_t synchronous);

/* Per-head top-k (top_k_indices semantics, ties to the lower row). */
int epk_select_per_head(epk_ctx* ctx, const epk_cache_desc* cache, const void* scores,
                        int32_t score_dtype, const int64_t* k_per_layer, uint8_t* keep);

/* ---- K3: compaction ----------------------------------------------------- *
 * Stable gather of the kept rows (K, V, pos) of `in` into `out` (same layers,
 * heads, dim, dtype; out->layer_base is out's capacity layout).  Each head of
 * `out` is followed by `slack` free rows for the next block's append;
 * out->head_off is written on the device.  Asynchronous. */
int epk_compact(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out,
                const uint8_t* keep, int32_t slack);

/* ---- append_to_cache ------------------------------------------------------ *
 * Writes a block of new rows into the free rows after each head's live rows:
 *   k_new, v_new [dev] [layers][kv_heads][len][head_dim], positions [dev] [len]
 * and advances head_len (head_off is unchanged).  `slack` is the gap the
 * caller left after every head (the out_slack of the compaction that built
 * the cache): len > slack > 0 fails at once with EPK_ERR_ARG; slack = 0 skips
 * that host check.  On the device every head's actual gap is checked; a head
 * whose gap is too small is left unchanged and EPK_ERR_ARG is deferred to
 * epk_ctx_poll_error.  Asynchronous. */
int epk_append(epk_ctx* ctx, const epk_cache_desc* cache, const void* k_new, const void* v_new,
               const int32_t* positions, int32_t len, int32_t slack);

/* ---- fused block step ------------------------------------------------------ *
 * score (mode) -> pooled select -> compact, for all layers, in -> out.
 * scores_ws [dev, optional] fp32 [in rows] receives the scores.
 * kept_per_layer [dev, optional] int32 [layers].  Asynchronous; pin overflow
 * is deferred to epk_ctx_poll_error. */
int epk_evict_step(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out,
                   const void* q_prompt, const void* k_prompt, int32_t q_heads,
                   int32_t prompt_len, const int64_t* layer_budgets, const int32_t* pins,
                   int32_t n_pins, int32_t aggregation, int32_t mode, int64_t n_max_per_head,
                   int32_t out_slack, float* scores_ws, int32_t* kept_per_layer);

/* ---- K4: k-means (fp64, bit-exact vs clustering.hpp:148-260) -------------- *
 * points [dev] [n][dim] fp64.  Device kernels: */
int epk_kmeans_assign(epk_ctx* ctx, const double* points, int64_t n, int64_t dim,
                      const double* centroids, int64_t k, int64_t* assign, double* best_d2);
/* sums [dev] [k][dim] = sum over points i in index order with assign[i]==c
 * (accumulated ON TOP of the incoming sums when accumulate != 0, the ordered
 * chain used for sharded points), counts [dev] int64 [k] likewise. */
int epk_kmeans_partial_sums(epk_ctx* ctx, const double* points, int64_t n, int64_t dim,
                            const int64_t* assign, int64_t k, double* sums, int64_t* counts,
                            int32_t accumulate);
int epk_kmeans_finalize(epk_ctx* ctx, const double* sums, const int64_t* counts, int64_t k,
                        int64_t dim, double* centroids);
int epk_kmeans_sq_dist(epk_ctx* ctx, const double* points, int64_t n, int64_t dim,
                       const double* centroids, const int64_t* assign, double* d2);
/* Whole kmeans (k-means++ seeding with the reference RNG stream on the host,
 * Lloyd on the device).  Synchronous.  assign_out, centroids_out, sse_out [host];
 * sse_out has room for max_iters values. */
int epk_kmeans(epk_ctx* ctx, const double* points, int64_t n, int64_t dim, int64_t k,
               uint64_t seed, int64_t max_iters, int64_t* assign_out, double* centroids_out,
               int64_t* iterations_out, double* sse_out);

/* The same k-means with the points sharded in index order over `nshards`
 * contexts (one per GPU; a device may appear more than once): shard s holds
 * points [sum of n_per_shard[<s], + n_per_shard[s]) as points[s] [dev of
 * ctxs[s]] fp64 [n][dim].  The centroid sums run as an ordered chain (shard s
 * adds its points in index order on top of shard s-1's sums) and the last
 * shard broadcasts the centroids, so every result is bit-identical to
 * epk_kmeans on the concatenated points.  Transport: NCCL ncclSend/ncclRecv +
 * ncclBroadcast over ncclCommInitAll of the devices when they are distinct
 * (libnccl.so.2 loaded at first use; EPK_ERR_UNSUPPORTED if absent), device
 * copies when shards share a device.  Synchronous; replaces kmeans
 * (clustering.hpp:148-260) for embeddings sharded across GPUs. */
int epk_kmeans_sharded(epk_ctx* const* ctxs, int32_t nshards, const double* const* points,
                       const int64_t* n_per_shard, int64_t dim, int64_t k, uint64_t seed, int64_t max_iters,
                       int64_t* assign_out, double* centroids_out, int64_t* iterations_out, double* sse_out);

/* ---- K6: KeyDiff baseline scorer ------------------------------------------ *
 * scores[layer_base[l] + r] = -cosine(key_r, mean key of r's (layer, head)),
 * or 0 when either norm is zero (keydiff_scores, scoring.hpp:186-221), fp64
 * [dev] in cache row order; gap rows are not written.  Bit-exact with the
 * reference (fp64, sequential sums, no FMA).  Feed the scores to
 * epk_select_pooled (score_dtype EPK_F64) + epk_compact.  Cache dtype F32,
 * BF16 or F64 (keys only are read), head_dim <= 256.  Asynchronous. */
int epk_score_keydiff(epk_ctx* ctx, const epk_cache_desc* cache, double* scores);

/* ---- K7: episodic cache store (.epkv) --------------------------------------- *
 * Serialises `cache` into the byte stream persist (kvcache.hpp:281-317) writes:
 * header (magic "EPKV", version 1, episode_id, layer / head counts, provenance
 * scorer string, budget_per_head, layer_budgets [host, n_layer_budgets]), then
 * per layer its budget (layer_budgets[l], else budget_per_head) and heads, per
 * head its entry count, per entry position (u64), dim (u32) and key + value
 * widened to fp64 (bitwise the reference's reals).  out [dev, 16-byte aligned]
 * receives the file's bytes at out + *offset_out (0..15 leading pad bytes),
 * *total_out bytes long; out = NULL only computes the two sizes.  Capacity
 * must be >= offset + total.  Synchronous (reads the head lengths). */
int epk_serialize_epkv(epk_ctx* ctx, const epk_cache_desc* cache, uint64_t episode_id, const char* scorer,
                       uint64_t budget_per_head, const int64_t* layer_budgets, int32_t n_layer_budgets,
                       uint8_t* out, int64_t capacity, int64_t* offset_out, int64_t* total_out);

/* The reader (load_cache, kvcache.hpp:321-374; Phase B "KVs Retrieve").
 * epk_epkv_scan walks a file's structure on the host: info [4] = {layers,
 * kv_heads, dim, header bytes}; counts [layers*kv_heads] entry counts and
 * entry_off [layers*kv_heads] byte offsets of each head's first entry (either
 * may be NULL).  Fails closed on bad magic / version / truncation, like the
 * reference.  epk_load_epkv narrows every entry of the file (copied to the
 * device at dev_file + pad, pad chosen so that pad + entry_off[0] is a
 * multiple of 4) into `cache` (F32 / BF16 / F64; head_off / head_len already
 * laid out for the counts): positions, keys, values.  A value that does not
 * round-trip to the cache dtype, or a dim that differs, raises a deferred
 * EPK_ERR_ARG.  Asynchronous. */
int epk_epkv_scan(const uint8_t* bytes, int64_t nbytes, int64_t* info, int64_t* counts, int64_t* entry_off);
int epk_load_epkv(epk_ctx* ctx, const uint8_t* dev_file, int64_t pad, const int64_t* entry_off,
                  const epk_cache_desc* cache);

/* ---- K5: layer sensitivity ------------------------------------------------ *
 * sigma[l] = mean over (h, t) of cosine(k_full, k_block), zero-norm pairs
 * skipped (allocation.hpp:80-100).  k_full, k_block [dev] [layers][kv_heads][ntok][dim]
 * of dtype (F32, BF16 or F64); sigma [dev] fp64 [layers]; skipped [dev] int64 [1].
 * Asynchronous. */
int epk_key_cosine_sigma(epk_ctx* ctx, const void* k_full, const void* k_block, int32_t dtype,
                         int32_t layers, int32_t kv_heads, int64_t ntok, int32_t dim,
                         double* sigma, int64_t* skipped);

/* ---- the model step before the hot path -------------------- *
 * The reference's toy GQA transformer forward (toymodel.hpp:228-411) on the
 * GPU, fp64, the reference's operation order (no FMA).  Weights [dev], per
 * layer in this order: wq [D][D], wk [D][Hkv*dh], wv [D][Hkv*dh], wo [D][D],
 * mlp_in [D][2D], mlp_out [2D][D] (row-major, as the reference's Matrix). */
typedef struct epk_toy_model {
    int32_t layers;
    int32_t query_heads;
    int32_t kv_heads;
    int32_t head_dim;
    int32_t model_dim; /* = query_heads * head_dim */
    int64_t vocab;
    const double* token_embedding; /* [dev] [vocab][model_dim] */
    const double* weights;         /* [dev] all layers, layout above */
} epk_toy_model;

/* forward (toymodel.hpp:228) over n new tokens at `positions` attending to
 * the past cache (F64 layered CSR, may be NULL) and to earlier new tokens.
 *   tokens [dev] int32 [n]; pos_emb [dev] [n][D] = Model::position_embedding
 *   rows; positions [dev] int64 [n]; mask_kind 0 causal, 1 sink+recent
 *   (sink, recent as MaskSpec).
 *   k_out, v_out [dev] [layers][n][kv_heads*head_dim]: the new keys / values.
 *   attention [dev, optional]: query head qh of layer l writes its n x
 *   (cache_len(h) + n) weight grid at attention + attn_offsets[l*Hq + qh]
 *   (attn_offsets [host]); hidden_out [dev, optional] [n][D].
 * softmax_on_host != 0: each attention row's max / exp / denominator runs on
 * the host with std::exp (the reference's code): every output is bit-identical
 * to the reference forward.  0: on the device (CUDA exp, <= 1 ulp away).
 * Synchronous when softmax_on_host (or a past cache is given), else async. */
int epk_toy_forward(epk_ctx* ctx, const epk_toy_model* model, const int32_t* tokens, const double* pos_emb,
                    const int64_t* positions, int64_t n, int32_t mask_kind, int64_t sink, int64_t recent,
                    const epk_cache_desc* past, double* k_out, double* v_out, double* attention,
                    const int64_t* attn_offsets, double* hidden_out, int32_t softmax_on_host);

/* ---- diagnostics ---------------------------------------------------------- *
 * y[i] = epk_expf(x[i]) as the EPK-F32 v1 kernels compute it ([dev] fp32),
 * for the bitwise host/device parity test. */
int epk_debug_expf(epk_ctx* ctx, const float* x, float* y, int64_t n);

#ifdef __cplusplus
}
#endif
#endif /* EPK_EPK_H */
