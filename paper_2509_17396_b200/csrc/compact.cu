// compact.cu -- K3: stable gather-compaction of the kept rows, and append.
//
// Restates the output loop of evict_to_budget (kvcache.hpp:192-199): every
// head keeps its surviving entries in their original (position) order, heads
// stay in order.  The result is written out of place into a second cache
// (ping-pong buffers), each head followed by `slack` free rows so the next
// block's append_to_cache (toymodel.hpp:428-443) lands in place without
// moving the cache again.
//
// Three launches per call:
//   count   (layer, chunk) CTAs count kept rows per 2048-row chunk;
//   plan    one CTA per layer scans the chunk counts and derives the per-head
//           kept totals -> the output head_off / head_len;
//   gather  (layer, chunk) CTAs recompute their in-chunk exclusive prefix and
//           copy K, V (16-byte vectors, 4 in flight per thread) and positions.
#include <algorithm>

#include "epk_internal.cuh"

namespace epk {

constexpr int kChunkRows = 2048;
constexpr int kCompactThreads = 256;
constexpr int kMaxHeadsC = 64;

struct CompactParams {
    LayerTable in_lt;
    LayerTable out_lt;
    int H;
    int max_chunks;
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
    int* err_flag;
};

__device__ __forceinline__ int head_of_row(const int32_t* off, int H, int64_t r) {
    int lo = 0, hi = H - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    return lo;
}

template <int NT>
__device__ __forceinline__ int block_sum(int v, int* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    int t = 0;
    for (int w = 0; w < NT / 32; ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(kCompactThreads) compact_count_kernel(const __grid_constant__ CompactParams P) {
    const int layer = blockIdx.y;
    const int chunk = blockIdx.x;
    __shared__ int32_t s_off[kMaxHeadsC + 1];
    __shared__ int32_t s_len[kMaxHeadsC];
    __shared__ int s_red[kCompactThreads / 32];
    const int H = P.H;
    for (int i = threadIdx.x; i <= H; i += blockDim.x) s_off[i] = P.in_off[layer * (H + 1) + i];
    for (int i = threadIdx.x; i < H; i += blockDim.x) s_len[i] = P.in_len[layer * H + i];
    __syncthreads();
    const int64_t rows = s_off[H];
    const int64_t r0 = int64_t(chunk) * kChunkRows;
    if (r0 >= rows) {
        if (threadIdx.x == 0) P.chunk_cnt[layer * P.max_chunks + chunk] = 0;
        return;
    }
    const int64_t base = P.in_lt.base[layer];
    int c = 0;
    for (int i = threadIdx.x; i < kChunkRows; i += blockDim.x) {
        const int64_t r = r0 + i;
        if (r < rows) {
            const int h = head_of_row(s_off, H, r);
            if (r - s_off[h] < s_len[h] && P.keep[base + r]) ++c;
        }
    }
    c = block_sum<kCompactThreads>(c, s_red);
    if (threadIdx.x == 0) P.chunk_cnt[layer * P.max_chunks + chunk] = c;
}

// One CTA per layer: exclusive scan of the chunk counts, then the kept count
// in front of every head-region start -> output head offsets.
__global__ void __launch_bounds__(1024) compact_plan_kernel(const __grid_constant__ CompactParams P) {
    const int layer = blockIdx.x;
    const int H = P.H;
    __shared__ int32_t s_off[kMaxHeadsC + 1];
    __shared__ int32_t s_len[kMaxHeadsC];
    __shared__ int s_red[32];
    __shared__ int64_t s_head_prefix[kMaxHeadsC + 1];
    for (int i = threadIdx.x; i <= H; i += blockDim.x) s_off[i] = P.in_off[layer * (H + 1) + i];
    for (int i = threadIdx.x; i < H; i += blockDim.x) s_len[i] = P.in_len[layer * H + i];
    __syncthreads();
    const int64_t rows = s_off[H];
    const int nchunks = int((rows + kChunkRows - 1) / kChunkRows);
    const int32_t* cnt = P.chunk_cnt + layer * P.max_chunks;
    int32_t* pre = P.chunk_prefix + layer * P.max_chunks;
    if (threadIdx.x == 0) {
        int32_t run = 0;
        for (int c = 0; c < nchunks; ++c) {
            pre[c] = run;
            run += cnt[c];
        }
    }
    __syncthreads();
    const int64_t base = P.in_lt.base[layer];
    // kept rows before row x = pre[x / chunk] + kept in [chunk start, x)
    for (int h = 0; h <= H; ++h) {
        const int64_t x = s_off[h];
        const int64_t c = x / kChunkRows;
        int part = 0;
        for (int64_t r = c * kChunkRows + threadIdx.x; r < x; r += blockDim.x) {
            const int hh = head_of_row(s_off, H, r);
            if (r - s_off[hh] < s_len[hh] && P.keep[base + r]) ++part;
        }
        part = block_sum<1024>(part, s_red);
        if (threadIdx.x == 0) {
            const int64_t before = (c < nchunks ? int64_t(P.chunk_prefix[layer * P.max_chunks + c]) : 0) + part;
            // x == rows may sit past the last chunk start: count everything.
            int64_t v = before;
            if (c >= nchunks) {
                v = 0;
                for (int cc = 0; cc < nchunks; ++cc) v += cnt[cc];
            }
            s_head_prefix[h] = v;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t cap = P.out_lt.base[layer + 1] - P.out_lt.base[layer];
        const int64_t need = s_head_prefix[H] + int64_t(P.slack) * H;
        if (need > cap) atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
        for (int h = 0; h < H; ++h) {
            P.out_off[layer * (H + 1) + h] = int32_t(s_head_prefix[h] + int64_t(P.slack) * h);
            P.out_len[layer * H + h] = int32_t(s_head_prefix[h + 1] - s_head_prefix[h]);
        }
        P.out_off[layer * (H + 1) + H] = int32_t(s_head_prefix[H] + int64_t(P.slack) * H);
    }
}

__global__ void __launch_bounds__(kCompactThreads) compact_gather_kernel(const __grid_constant__ CompactParams P) {
    const int layer = blockIdx.y;
    const int chunk = blockIdx.x;
    const int H = P.H;
    __shared__ int32_t s_off[kMaxHeadsC + 1];
    __shared__ int32_t s_len[kMaxHeadsC];
    __shared__ int32_t s_src[kChunkRows];  // in-layer source row
    __shared__ int32_t s_dst[kChunkRows];  // out-layer destination row
    __shared__ int s_warp[kCompactThreads / 32];
    for (int i = threadIdx.x; i <= H; i += blockDim.x) s_off[i] = P.in_off[layer * (H + 1) + i];
    for (int i = threadIdx.x; i < H; i += blockDim.x) s_len[i] = P.in_len[layer * H + i];
    __syncthreads();
    const int64_t rows = s_off[H];
    const int64_t r0 = int64_t(chunk) * kChunkRows;
    if (r0 >= rows) return;
    const int64_t in_base = P.in_lt.base[layer];
    const int64_t out_base = P.out_lt.base[layer];
    const int32_t chunk_pre = P.chunk_prefix[layer * P.max_chunks + chunk];

    // Each thread owns 8 consecutive rows of the chunk.
    constexpr int kPer = kChunkRows / kCompactThreads;
    uint32_t bits = 0;
    int hs[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int64_t r = r0 + threadIdx.x * kPer + i;
        hs[i] = 0;
        if (r < rows) {
            const int h = head_of_row(s_off, H, r);
            hs[i] = h;
            if (r - s_off[h] < s_len[h] && P.keep[in_base + r]) bits |= 1u << i;
        }
    }
    const int mine = __popc(bits);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int warp_pre = 0;
    for (int w = 0; w < warp; ++w) warp_pre += s_warp[w];
    int total = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) total += s_warp[w];
    int slot = warp_pre + incl - mine;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        if (bits & (1u << i)) {
            const int64_t r = r0 + threadIdx.x * kPer + i;
            s_src[slot] = int32_t(r);
            s_dst[slot] = chunk_pre + slot + P.slack * hs[i];
            ++slot;
        }
    }
    __syncthreads();

    // Positions.
    for (int j = threadIdx.x; j < total; j += blockDim.x)
        P.out_pos[out_base + s_dst[j]] = P.in_pos[in_base + s_src[j]];

    // K and V rows: flattened (row, 16-byte column) loop, 4 vectors in flight.
    const int rv = P.row_vec;
    const int64_t nvec = int64_t(total) * rv;
    constexpr int U = 4;
    for (int64_t v0 = threadIdx.x; v0 < nvec; v0 += int64_t(blockDim.x) * U) {
        uint4 ka[U], va[U];
        int64_t dst[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + int64_t(u) * blockDim.x;
            if (v < nvec) {
                const int j = int(v / rv), c = int(v % rv);
                const int64_t src = (in_base + s_src[j]) * rv + c;
                dst[u] = (out_base + s_dst[j]) * rv + c;
                ka[u] = __ldcs(P.in_k + src);
                va[u] = __ldcs(P.in_v + src);
            } else {
                dst[u] = -1;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (dst[u] >= 0) {
                __stcs(P.out_k + dst[u], ka[u]);
                __stcs(P.out_v + dst[u], va[u]);
            }
        }
    }
}

int launch_compact(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out,
                   const uint8_t* keep, int slack) {
    if (in->layers != out->layers || in->kv_heads != out->kv_heads || in->head_dim != out->head_dim ||
        in->dtype != out->dtype)
        return fail(EPK_ERR_DIM, "compact: in/out cache shapes differ");
    if (in->kv_heads > kMaxHeadsC) return fail(EPK_ERR_UNSUPPORTED, "compact: more than 64 kv heads");
    const int64_t row_bytes = int64_t(in->head_dim) * dtype_size(in->dtype);
    if (row_bytes % 16 != 0) return fail(EPK_ERR_UNSUPPORTED, "compact: row bytes must be a multiple of 16");
    if (slack < 0) return fail(EPK_ERR_ARG, "compact: negative slack");
    CompactParams P;
    int rc = make_layer_table(in, &P.in_lt);
    if (rc) return rc;
    rc = make_layer_table(out, &P.out_lt);
    if (rc) return rc;
    int64_t max_rows = 0;
    for (int l = 0; l < in->layers; ++l) max_rows = std::max<int64_t>(max_rows, P.in_lt.base[l + 1] - P.in_lt.base[l]);
    P.H = in->kv_heads;
    P.max_chunks = int(std::max<int64_t>(1, (max_rows + kChunkRows - 1) / kChunkRows));
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
    const int64_t ws = 2 * int64_t(in->layers) * P.max_chunks * 4 + 1024;
    rc = ws_require(ctx, ws);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.chunk_cnt = carve.take<int32_t>(int64_t(in->layers) * P.max_chunks);
    P.chunk_prefix = carve.take<int32_t>(int64_t(in->layers) * P.max_chunks);
    dim3 grid(P.max_chunks, in->layers);
    EPK_PROF(ctx, "compact_count");
    compact_count_kernel<<<grid, kCompactThreads, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "compact_plan");
    compact_plan_kernel<<<in->layers, 1024, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "compact_gather");
    compact_gather_kernel<<<grid, kCompactThreads, 0, ctx->stream>>>(P);
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
