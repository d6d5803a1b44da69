// compact.cu -- K3: stable gather-compaction of the kept rows, and append.
//
// Restates the output loop of evict_to_budget (kvcache.hpp:192-199): every
// head keeps its surviving entries in their original (position) order, heads
// stay in order.  The result is written out of place into a second cache
// (ping-pong buffers), each head followed by `slack` free rows so the next
// block's append_to_cache (toymodel.hpp:428-443) lands in place without
// moving the cache again.
//
// Launches, all free of shared memory (their small CTAs may share an SM with
// a scorer CTA of a next layer group):
//   count   one warp per 128-row chunk: kept rows in the chunk;
//   plan    one CTA per layer: exclusive scan of the chunk counts and the kept
//           count in front of every head region -> output head_off/head_len;
//   gather  one warp per 128-row chunk: ballot prefix per 32 rows, then
//           16-byte vector copies of K and V (8 in flight per lane) and the
//           positions.
// Given a keep[] mask (generic select) all three run; keep[] must be 0 on gap
// rows.  In threshold mode (the tensor-core step) select_threshold_kernel has
// already written the plan and the gather evaluates the keep rule itself from
// the scorer's keys, so the gather is the only launch here.
#include <algorithm>

#include "epk_internal.cuh"

namespace epk {

constexpr int kWarpsPerCta = 4;
#ifndef EPK_GATHER_U
#define EPK_GATHER_U 8  // measured cfg2: 4 -> 8 takes the gather from 0.307 to 0.298 ms (16 spills)
#endif
constexpr int kGatherU = EPK_GATHER_U;  // kept rows per half-warp in flight (K and V: 2 x 16 B per lane each)
static_assert(32 % (2 * kGatherU) == 0, "gather unroll");

struct CompactParams {
    LayerTable in_lt;
    LayerTable out_lt;
    int H;
    int max_chunks;
    int layers;
    int slack;
    int row_vec;  // row bytes / 16
    const int32_t* in_off;
    const int32_t* in_len;
    const uint8_t* keep;
    const uint4* in_k;
    const uint4* in_v;
    const int32_t* in_pos;
    uint4* out_k;
    uint4* out_v;
    int32_t* out_pos;
    int32_t* out_off;
    int32_t* out_len;
    int32_t* chunk_cnt;     // [layers][max_chunks]
    int32_t* chunk_prefix;  // [layers][max_chunks]
    int32_t* layer_bad;     // [layers] plan: kept rows + slack exceed the output layer (gather skips it)
    int* err_flag;
    // threshold mode (the tensor-core step): the gather derives keep from
    // the scorer's keys and the per-layer threshold, and select_threshold_kernel
    // (select.cu) wrote the plan (chunk prefixes, output heads, layer_bad)
    const uint32_t* keys;  // [rows] global, or null (keep[] given)
    const uint64_t* thr;   // [layers][2]
};

__device__ __forceinline__ int head_of_row(const int32_t* off, int H, int64_t r) {
    int lo = 0, hi = H - 1;
    while (lo < hi) {  // last h with off[h] <= r
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= r) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(32 * kWarpsPerCta) compact_count_kernel(const __grid_constant__ CompactParams P) {
    pdl_wait();
    const int layer = blockIdx.y;
    const int chunk = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (chunk >= P.max_chunks) return;
    const int64_t rows = P.in_off[layer * (P.H + 1) + P.H];
    const int64_t r0 = int64_t(chunk) * kChunkRows;
    int c = 0;
    if (r0 < rows) {
        const uint8_t* kp = P.keep + P.in_lt.base[layer];
#pragma unroll
        for (int i = 0; i < kChunkRows / 32; ++i) {
            const int64_t r = r0 + i * 32 + lane;
            c += (r < rows && kp[r]) ? 1 : 0;
        }
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) P.chunk_cnt[layer * P.max_chunks + chunk] = c;
}

// One CTA per layer: exclusive scan of the chunk counts, then the kept count
// in front of every head-region start -> output head offsets and lengths.
__global__ void __launch_bounds__(256) compact_plan_kernel(const __grid_constant__ CompactParams P) {
    pdl_wait();
    const int layer = blockIdx.x;
    const int H = P.H;
    __shared__ int32_t s_warp[8];
    __shared__ int64_t s_head_prefix[65];
    const int32_t* off = P.in_off + layer * (H + 1);
    const int64_t rows = off[H];
    const int nchunks = int((rows + kChunkRows - 1) / kChunkRows);
    const int32_t* cnt = P.chunk_cnt + layer * P.max_chunks;
    int32_t* pre = P.chunk_prefix + layer * P.max_chunks;
    // block-wide exclusive scan, each thread owns a contiguous run of chunks
    const int per = (nchunks + blockDim.x - 1) / blockDim.x;
    const int c0 = threadIdx.x * per, c1 = min(nchunks, c0 + per);
    int32_t mine = 0;
    for (int c = c0; c < c1; ++c) mine += cnt[c];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int32_t incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int32_t run = incl - mine;
    for (int w = 0; w < warp; ++w) run += s_warp[w];
    for (int c = c0; c < c1; ++c) {
        pre[c] = run;
        run += cnt[c];
    }
    __syncthreads();
    const uint8_t* kp = P.keep + P.in_lt.base[layer];
    // kept rows before every head start: the chunk prefix plus a warp-wide
    // count of the kept rows in [chunk start, head start)
    for (int h = warp; h <= H; h += blockDim.x / 32) {
        const int64_t x = off[h];
        const int64_t c = x / kChunkRows;
        int64_t v;
        if (c >= nchunks) {
            v = nchunks == 0 ? 0 : int64_t(pre[nchunks - 1]) + cnt[nchunks - 1];
        } else {
            int part = 0;
            for (int64_t r = c * kChunkRows + lane; r < x; r += 32) part += kp[r] ? 1 : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            v = int64_t(pre[c]) + part;
        }
        if (lane == 0) s_head_prefix[h] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int64_t cap = P.out_lt.base[layer + 1] - P.out_lt.base[layer];
        const int64_t need = s_head_prefix[H] + int64_t(P.slack) * H;
        P.layer_bad[layer] = need > cap;
        if (need > cap) {
            // the output layer cannot hold the kept rows: flag it, leave the
            // layer empty and let the gather skip it (no store past the layer)
            atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
            for (int h = 0; h <= H; ++h) P.out_off[layer * (H + 1) + h] = 0;
            for (int h = 0; h < H; ++h) P.out_len[layer * H + h] = 0;
            return;
        }
        for (int h = 0; h < H; ++h) {
            P.out_off[layer * (H + 1) + h] = int32_t(s_head_prefix[h] + int64_t(P.slack) * h);
            P.out_len[layer * H + h] = int32_t(s_head_prefix[h + 1] - s_head_prefix[h]);
        }
        P.out_off[layer * (H + 1) + H] = int32_t(s_head_prefix[H] + int64_t(P.slack) * H);
    }
}

// Warps walk the flattened (layer, chunk) items; the default launch gives
// every warp one item, a persistent launch (ctx->gather_ctas) strides.
__global__ void __launch_bounds__(512) compact_gather_kernel(const __grid_constant__ CompactParams P) {
    TL_BEGIN();
    pdl_wait();
    TL_GO();
    const int wpb = blockDim.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t items = int64_t(P.layers) * P.max_chunks;
    for (int64_t it = int64_t(blockIdx.x) * wpb + (threadIdx.x >> 5); it < items; it += int64_t(gridDim.x) * wpb) {
        const int layer = int(it / P.max_chunks);
        const int chunk = int(it % P.max_chunks);
        if (P.layer_bad[layer]) continue;
        const int32_t* off = P.in_off + layer * (P.H + 1);
        const int64_t rows = off[P.H];
        const int64_t r0 = int64_t(chunk) * kChunkRows;
        if (r0 >= rows) continue;
        const int64_t in_base = P.in_lt.base[layer];
        const int64_t out_base = P.out_lt.base[layer];
        const uint8_t* kp = P.keep + in_base;
        int32_t run = __ldcg(P.chunk_prefix + layer * P.max_chunks + chunk);
        const int rv = P.row_vec;
        const int hl = lane >> 4, cl = lane & 15;
        // threshold mode: keep = live && (key < T || key == T && (position << 8 | head) <= U)
        // (thr[2l] bit 32: keep every live row, bit 33: keep none)
        const bool thr_mode = P.keys != nullptr;
        uint64_t t0 = 0, U = 0;
        if (thr_mode) {
            t0 = __ldcg(P.thr + 2 * layer);
            U = __ldcg(P.thr + 2 * layer + 1);
        }
        // the chunk's first head and where the next one starts (a chunk rarely
        // crosses a head boundary: rows past it take the binary search)
        const bool need_h = P.slack || thr_mode;
        const int h0 = need_h ? head_of_row(off, P.H, r0) : 0;
        const int64_t h0_end = need_h ? int64_t(off[h0 + 1]) : 0;
        for (int sc = 0; sc < kChunkRows / 32; ++sc) {
            const int64_t rs = r0 + sc * 32;
            if (rs >= rows) break;
            const int64_t r = rs + lane;
            const int h = (need_h && r < rows) ? (r < h0_end ? h0 : head_of_row(off, P.H, r)) : 0;
            int32_t ps = 0;
            bool k;
            if (thr_mode) {
                k = false;
                if (r < rows && !((t0 >> 33) & 1) && r - off[h] < P.in_len[layer * P.H + h]) {
                    const uint32_t key = __ldcg(P.keys + in_base + r);
                    k = ((t0 >> 32) & 1) || key < uint32_t(t0);
                    if (!k && key == uint32_t(t0)) {  // inside the threshold tie: (position, head) decides
                        ps = P.in_pos[in_base + r];
                        k = ((uint64_t(uint32_t(ps)) << 8) | uint64_t(h)) <= U;
                    } else if (k) {
                        ps = P.in_pos[in_base + r];
                    }
                }
            } else {
                k = r < rows && kp[r];
                if (k) ps = P.in_pos[in_base + r];
            }
            const unsigned bal = __ballot_sync(0xffffffffu, k);
            if (bal == 0) continue;
            int64_t dst = 0;
            if (k) {
                dst = out_base + run + __popc(bal & ((1u << lane) - 1u));
                if (P.slack) dst += int64_t(P.slack) * h;
                P.out_pos[dst] = ps;
            }
            run += __popc(bal);
            // copy the kept rows: a half-warp per row, kGatherU rows per half-warp in flight
            for (int k0 = 0; k0 < 32; k0 += 2 * kGatherU) {
                uint4 kv[kGatherU], vv[kGatherU];
                int64_t dsts[kGatherU];
                bool ok[kGatherU];
#pragma unroll
                for (int u = 0; u < kGatherU; ++u) {
                    const int idx = k0 + 2 * u + hl;
                    ok[u] = (bal >> idx) & 1u;
                    dsts[u] = __shfl_sync(0xffffffffu, dst, idx);
                }
                for (int c = cl; c < rv; c += 16) {
#pragma unroll
                    for (int u = 0; u < kGatherU; ++u) {
                        if (ok[u]) {
                            const int64_t src = (in_base + rs + k0 + 2 * u + hl) * rv + c;
                            kv[u] = __ldg(P.in_k + src);
                            vv[u] = __ldg(P.in_v + src);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < kGatherU; ++u) {
                        if (ok[u]) {
                            P.out_k[dsts[u] * rv + c] = kv[u];
                            P.out_v[dsts[u] * rv + c] = vv[u];
                        }
                    }
                }
            }
        }
    }
    TL_END(6);
}

int compact_ws(epk_ctx* ctx, const epk_cache_desc* in, CompactWs* w) {
    int64_t max_rows = 0;
    for (int l = 0; l < in->layers; ++l)
        max_rows = std::max<int64_t>(max_rows, in->layer_base[l + 1] - in->layer_base[l]);
    w->max_chunks = int(std::max<int64_t>(1, (max_rows + kChunkRows - 1) / kChunkRows));
    const int64_t ws = 2 * int64_t(in->layers) * w->max_chunks * 4 + int64_t(in->layers) * 4 + 1024;
    int rc = ws2_require(ctx, ws);
    if (rc) return rc;
    WsCarver carve(ctx->ws2);
    w->chunk_cnt = carve.take<int32_t>(int64_t(in->layers) * w->max_chunks);
    w->chunk_prefix = carve.take<int32_t>(int64_t(in->layers) * w->max_chunks);
    w->layer_bad = carve.take<int32_t>(in->layers);
    return EPK_OK;
}

int launch_compact(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out, const uint8_t* keep,
                   int slack, const uint32_t* keys, const uint64_t* thr, uint32_t* hist_fine, uint32_t* hist_coarse) {
    if (in->layers != out->layers || in->kv_heads != out->kv_heads || in->head_dim != out->head_dim ||
        in->dtype != out->dtype)
        return fail(EPK_ERR_DIM, "compact: in/out cache shapes differ");
    if (in->kv_heads > 64) return fail(EPK_ERR_UNSUPPORTED, "compact: more than 64 kv heads");
    const int64_t row_bytes = int64_t(in->head_dim) * dtype_size(in->dtype);
    if (row_bytes % 16 != 0) return fail(EPK_ERR_UNSUPPORTED, "compact: row bytes must be a multiple of 16");
    if (slack < 0) return fail(EPK_ERR_ARG, "compact: negative slack");
    CompactParams P;
    int rc = make_layer_table(in, &P.in_lt);
    if (rc) return rc;
    rc = make_layer_table(out, &P.out_lt);
    if (rc) return rc;
    CompactWs w;
    if ((rc = compact_ws(ctx, in, &w))) return rc;
    P.H = in->kv_heads;
    P.max_chunks = w.max_chunks;
    P.layers = in->layers;
    P.slack = slack;
    P.row_vec = int(row_bytes / 16);
    P.in_off = in->head_off;
    P.in_len = in->head_len;
    P.keep = keep;
    P.in_k = static_cast<const uint4*>(in->k);
    P.in_v = static_cast<const uint4*>(in->v);
    P.in_pos = in->pos;
    P.out_k = static_cast<uint4*>(out->k);
    P.out_v = static_cast<uint4*>(out->v);
    P.out_pos = out->pos;
    P.out_off = out->head_off;
    P.out_len = out->head_len;
    P.err_flag = ctx->err_flag;
    P.keys = keys;
    P.thr = thr;
    (void)hist_fine;  // zeroed for the next step by the P1 launch (score_tc.cu)
    (void)hist_coarse;
    P.chunk_cnt = w.chunk_cnt;
    P.chunk_prefix = w.chunk_prefix;
    P.layer_bad = w.layer_bad;
    dim3 grid((P.max_chunks + kWarpsPerCta - 1) / kWarpsPerCta, in->layers);
#ifdef EPK_COMPACT_CARVEOUT
    // experiment: a shared-memory carveout matching the scorer's, so the
    // compaction CTAs may share an SM with a resident scorer CTA
    EPK_CUDA_CHECK(cudaFuncSetAttribute(compact_count_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        EPK_COMPACT_CARVEOUT));
    EPK_CUDA_CHECK(cudaFuncSetAttribute(compact_plan_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        EPK_COMPACT_CARVEOUT));
    EPK_CUDA_CHECK(cudaFuncSetAttribute(compact_gather_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                        EPK_COMPACT_CARVEOUT));
#endif
    if (!keys) {  // threshold mode: select_threshold_kernel planned the compaction already
        EPK_PROF(ctx, "compact_count");
        EPK_CUDA_CHECK(launch_pdl(compact_count_kernel, grid, dim3(32 * kWarpsPerCta), 0, ctx->stream, P));
        EPK_LAUNCH_CHECK(ctx);
        EPK_PROF(ctx, "compact_plan");
        EPK_CUDA_CHECK(launch_pdl(compact_plan_kernel, dim3(in->layers), dim3(256), 0, ctx->stream, P));
        EPK_LAUNCH_CHECK(ctx);
    }
    EPK_PROF(ctx, "compact_gather");
    if (ctx->gather_ctas > 0) {  // persistent (experiments: an SM-partitioned overlapped gather)
        if (ctx->gather_smem > 0)
            EPK_CUDA_CHECK(cudaFuncSetAttribute(compact_gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                ctx->gather_smem));
        EPK_CUDA_CHECK(launch_pdl(compact_gather_kernel, dim3(ctx->gather_ctas), dim3(ctx->gather_threads),
                                  size_t(ctx->gather_smem), ctx->stream, P));
    } else {
        const int64_t items = int64_t(in->layers) * P.max_chunks;
        EPK_CUDA_CHECK(launch_pdl(compact_gather_kernel, dim3(unsigned((items + kWarpsPerCta - 1) / kWarpsPerCta)),
                                  dim3(32 * kWarpsPerCta), 0, ctx->stream, P));
    }
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// ---------------------------------------------------------------------------
// append_to_cache: new rows land after each head's live rows.
// ---------------------------------------------------------------------------
struct AppendParams {
    LayerTable lt;
    int H;
    int len;
    int row_vec;
    const int32_t* off;
    int32_t* head_len;
    const uint4* k_new;  // [layers][H][len][row_vec]
    const uint4* v_new;
    const int32_t* positions;
    uint4* k;
    uint4* v;
    int32_t* pos;
    int* err_flag;
};

__global__ void append_copy_kernel(const __grid_constant__ AppendParams P) {
    const int lh = blockIdx.y;  // layer * H + h
    const int layer = lh / P.H, h = lh % P.H;
    const int32_t start = P.off[layer * (P.H + 1) + h];
    const int32_t region = P.off[layer * (P.H + 1) + h + 1] - start;
    const int32_t len0 = P.head_len[lh];
    if (len0 + P.len > region) {
        if (threadIdx.x == 0 && blockIdx.x == 0) atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
        return;
    }
    const int64_t dst_row0 = P.lt.base[layer] + start + len0;
    const int64_t src_row0 = int64_t(lh) * P.len;
    const int64_t nvec = int64_t(P.len) * P.row_vec;
    for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < nvec; v += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = v / P.row_vec, c = v % P.row_vec;
        P.k[(dst_row0 + row) * P.row_vec + c] = P.k_new[(src_row0 + row) * P.row_vec + c];
        P.v[(dst_row0 + row) * P.row_vec + c] = P.v_new[(src_row0 + row) * P.row_vec + c];
    }
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < P.len; i += int64_t(gridDim.x) * blockDim.x)
        P.pos[dst_row0 + i] = P.positions[i];
}

__global__ void append_len_kernel(int32_t* head_len, const int32_t* off, int H, int n, int len) {
    const int lh = blockIdx.x * blockDim.x + threadIdx.x;
    if (lh >= n) return;
    const int layer = lh / H, h = lh % H;
    const int32_t region = off[layer * (H + 1) + h + 1] - off[layer * (H + 1) + h];
    if (head_len[lh] + len <= region) head_len[lh] += len;
}

int launch_append(epk_ctx* ctx, const epk_cache_desc* c, const void* k_new, const void* v_new,
                  const int32_t* positions, int len) {
    if (len <= 0) return fail(EPK_ERR_ARG, "append: empty block");
    const int64_t row_bytes = int64_t(c->head_dim) * dtype_size(c->dtype);
    if (row_bytes % 16 != 0) return fail(EPK_ERR_UNSUPPORTED, "append: row bytes must be a multiple of 16");
    AppendParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.H = c->kv_heads;
    P.len = len;
    P.row_vec = int(row_bytes / 16);
    P.off = c->head_off;
    P.head_len = c->head_len;
    P.k_new = static_cast<const uint4*>(k_new);
    P.v_new = static_cast<const uint4*>(v_new);
    P.positions = positions;
    P.k = static_cast<uint4*>(c->k);
    P.v = static_cast<uint4*>(c->v);
    P.pos = c->pos;
    P.err_flag = ctx->err_flag;
    const int64_t nvec = int64_t(len) * P.row_vec;
    const int bx = int(std::min<int64_t>(64, (nvec + 255) / 256));
    dim3 grid(bx, c->layers * c->kv_heads);
    EPK_PROF(ctx, "append_copy");
    append_copy_kernel<<<grid, 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    const int n = c->layers * c->kv_heads;
    EPK_PROF(ctx, "append_len");
    append_len_kernel<<<(n + 255) / 256, 256, 0, ctx->stream>>>(c->head_len, c->head_off, c->kv_heads, n, len);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk

namespace epk {

// ---------------------------------------------------------------------------
// Opt-in 1-D max-pool smoothing of the scores (north_star's "1-D max-pool
// smoothing"; NOT in the reference, whose score_with_prompt has no pooling,
// scoring.hpp:80-128 -- SURVEY 0.4): SnapKV-style max_pool1d with an odd
// kernel w, stride 1 and "same" padding over each (layer, head)'s live rows in
// position order: pooled[j] = max of scores[i], |i - j| <= w / 2, i live in
// j's head.  One thread per cache row; the window never crosses a head.
// ---------------------------------------------------------------------------
struct PoolParams {
    LayerTable lt;
    int H;
    int half;
    int64_t max_region;
    const int32_t* off;
    const int32_t* len;
    const float* in;
    float* out;
};

__global__ void __launch_bounds__(256) pool_scores_kernel(const __grid_constant__ PoolParams P) {
    const int layer = blockIdx.y;
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int32_t* off = P.off + layer * (P.H + 1);
    if (r >= off[P.H]) return;
    const int h = head_of_row(off, P.H, r);
    const int64_t lo = off[h], n = P.len[layer * P.H + h];
    if (r - lo >= n) return;  // slack row
    const int64_t base = P.lt.base[layer];
    const int64_t a = max(lo, r - P.half), b = min(lo + n - 1, r + P.half);
    float m = __ldg(P.in + base + a);
    for (int64_t i = a + 1; i <= b; ++i) m = fmaxf(m, __ldg(P.in + base + i));
    P.out[base + r] = m;
}

int launch_pool_scores(epk_ctx* ctx, const epk_cache_desc* c, const float* in, float* out, int kernel) {
    if (kernel < 1 || kernel % 2 == 0) return fail(EPK_ERR_ARG, "pool_scores: kernel must be odd and >= 1");
    if (c->kv_heads > 64) return fail(EPK_ERR_UNSUPPORTED, "pool_scores: more than 64 kv heads");
    PoolParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.H = c->kv_heads;
    P.half = kernel / 2;
    P.max_region = 0;
    for (int l = 0; l < c->layers; ++l) P.max_region = std::max<int64_t>(P.max_region, P.lt.base[l + 1] - P.lt.base[l]);
    P.off = c->head_off;
    P.len = c->head_len;
    P.in = in;
    P.out = out;
    const dim3 grid(unsigned(std::max<int64_t>(1, (P.max_region + 255) / 256)), unsigned(c->layers));
    EPK_PROF(ctx, "pool_scores");
    EPK_CUDA_CHECK(launch_pdl(pool_scores_kernel, grid, dim3(256), 0, ctx->stream, P));
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
