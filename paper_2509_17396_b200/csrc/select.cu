// select.cu -- K2: deterministic pooled (and per-head) top-k selection.
//
// Restates the selection of evict_to_budget (kvcache.hpp:142-190): per layer,
// if live <= H*M the layer is unchanged (:148-151); otherwise pinned rows are
// kept (:160-164) and the remaining H*M - pinned_live slots go to the smallest
// composite keys (score desc, position asc, head asc) (:181-190).  The
// per-head mode restates top_k_indices (numerics.hpp:111-125): ties to the
// lower index.
//
// Algorithm: MSB-first radix select.  One 8-CTA thread-block cluster per
// segment (layer, or (layer, head) in per-head mode); each CTA histograms the
// 8-bit digit of its slice of the segment into shared memory with
// warp-aggregated atomics (__match_any_sync), the cluster sums the 8
// histograms through distributed shared memory, and every CTA derives the
// same bucket.  After the score digits the exact threshold score key T is
// known; if T is shared by more rows than slots remain, a second radix select
// over the unique tiebreak (position << 8 | head) picks exactly the lowest
// ones.  Result: the same set std::sort would give, with no sort.
#include <cooperative_groups.h>

#include "epk_internal.cuh"

namespace cg = cooperative_groups;

namespace epk {

constexpr int kSelCluster = 8;
constexpr int kSelThreads = 1024;
constexpr int kMaxHeads = 64;

struct SelectParams {
    LayerTable lt;
    int64_t budget[kMaxLayers];
    const int32_t* head_off;
    const int32_t* head_len;
    const int32_t* pos;
    const void* scores;
    const int32_t* pins;
    int n_pins;
    int H;
    int per_head;
    uint8_t* keep;
    int32_t* kept_per_layer;
    int* err_flag;
    int key_cap;  // keys of this CTA's slice cached in dynamic shared memory
};

template <typename ScoreT>
struct KeyOf;
template <>
struct KeyOf<float> {
    using T = uint32_t;
};
template <>
struct KeyOf<double> {
    using T = uint64_t;
};

__device__ __forceinline__ bool is_pinned(const int32_t* pins, int n, int32_t p) {
    int lo = 0, hi = n - 1;
    while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const int32_t v = pins[mid];
        if (v == p) return true;
        if (v < p) lo = mid + 1; else hi = mid - 1;
    }
    return false;
}

// Finds the bucket holding the k-th smallest element (1-based) from 256
// totals; writes (bucket, count strictly before it, count in it).
__device__ void find_bucket(const uint32_t* tot, int64_t k, int* out_bucket, int64_t* out_before,
                            int64_t* out_eq) {
    const int lane = threadIdx.x & 31;
    int64_t local[8];
    int64_t lsum = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        local[i] = tot[lane * 8 + i];
        lsum += local[i];
    }
    int64_t incl = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const int64_t excl = incl - lsum;
    const bool mine = excl < k && k <= incl;
    const unsigned owner = __ballot_sync(0xffffffffu, mine);
    if (owner == 0) {  // cannot happen for a valid k; be defensive
        if (lane == 0) {
            *out_bucket = 255;
            *out_before = 0;
            *out_eq = 0;
        }
        return;
    }
    if (lane == __ffs(owner) - 1) {
        int64_t c = excl;
        for (int i = 0; i < 8; ++i) {
            if (c + local[i] >= k) {
                *out_bucket = lane * 8 + i;
                *out_before = c;
                *out_eq = local[i];
                break;
            }
            c += local[i];
        }
    }
}

template <typename ScoreT>
__global__ void __cluster_dims__(kSelCluster, 1, 1) __launch_bounds__(kSelThreads, 1)
    select_kernel(const __grid_constant__ SelectParams P) {
    using KeyT = typename KeyOf<ScoreT>::T;
    constexpr int kKeyBits = int(sizeof(KeyT) * 8);
    constexpr int kTieBits = 40;  // (position < 2^31) << 8 | head (< 256)

    cg::cluster_group cluster = cg::this_cluster();
    const int rank = int(cluster.block_rank());
    const int seg = blockIdx.x / kSelCluster;
    const int H = P.H;
    const int layer = P.per_head ? seg / H : seg;
    const int seg_head = P.per_head ? seg % H : -1;

    __shared__ int32_t s_off[kMaxHeads + 1];
    __shared__ int32_t s_len[kMaxHeads];
    __shared__ uint32_t s_hist[2][256];
    __shared__ uint32_t s_tot[256];
    __shared__ int64_t s_red[kSelThreads / 32];
    __shared__ int s_bucket;
    __shared__ int64_t s_before, s_eq;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    constexpr int nwarps = kSelThreads / 32;

    for (int i = tid; i <= H; i += blockDim.x) s_off[i] = P.head_off[layer * (H + 1) + i];
    for (int i = tid; i < H; i += blockDim.x) s_len[i] = P.head_len[layer * H + i];
    __syncthreads();

    // Segment row space (layer-relative rows, gaps included).
    int64_t seg_begin, seg_end, n_live = 0;
    if (P.per_head) {
        seg_begin = s_off[seg_head];
        seg_end = seg_begin + s_len[seg_head];
        n_live = s_len[seg_head];
    } else {
        seg_begin = 0;
        seg_end = s_off[H];
        for (int h = 0; h < H; ++h) n_live += s_len[h];
    }
    const int64_t span = seg_end - seg_begin;
    const int64_t my_begin = seg_begin + span * rank / kSelCluster;
    const int64_t my_end = seg_begin + span * (rank + 1) / kSelCluster;
    const int64_t base = P.lt.base[layer];
    const ScoreT* scores = static_cast<const ScoreT*>(P.scores) + base;
    const int32_t* pos = P.pos + base;
    uint8_t* keep = P.keep + base;
    const bool use_pins = !P.per_head && P.n_pins > 0;

    auto head_of = [&](int64_t r) -> int {
        if (P.per_head) return seg_head;
        int lo = 0, hi = H - 1;
        while (lo < hi) {  // last h with s_off[h] <= r
            const int mid = (lo + hi + 1) >> 1;
            if (s_off[mid] <= r) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    auto is_live = [&](int64_t r, int h) -> bool { return r - s_off[h] < s_len[h]; };

    // ---- pinned count (pooled mode with pins) -------------------------------
    int64_t pinned_live = 0;
    if (use_pins) {
        int64_t c = 0;
        for (int64_t r = my_begin + tid; r < my_end; r += blockDim.x) {
            const int h = head_of(r);
            if (is_live(r, h) && is_pinned(P.pins, P.n_pins, pos[r])) ++c;
        }
        for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        if (lane == 0) s_red[warp] = c;
        __syncthreads();
        if (tid == 0) {
            int64_t t = 0;
            for (int w = 0; w < nwarps; ++w) t += s_red[w];
            s_hist[0][0] = uint32_t(t);
        }
        cluster.sync();
        if (tid == 0) {
            int64_t t = 0;
            for (int q = 0; q < kSelCluster; ++q) t += *cluster.map_shared_rank(&s_hist[0][0], q);
            s_before = t;
        }
        cluster.sync();  // everyone has read s_hist[0][0] before it is reused
        __syncthreads();
        pinned_live = s_before;
    }

    if (P.per_head && rank == 0)  // gap rows after the head's live rows: never kept
        for (int64_t r = seg_end + tid; r < s_off[seg_head + 1]; r += blockDim.x) keep[r] = 0;
    const int64_t limit = P.per_head ? P.budget[layer] : int64_t(H) * P.budget[layer];
    if (n_live <= limit) {
        for (int64_t r = my_begin + tid; r < my_end; r += blockDim.x) keep[r] = is_live(r, head_of(r)) ? 1 : 0;
        if (rank == 0 && tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(n_live);
        return;
    }
    if (pinned_live > limit) {
        if (tid == 0 && rank == 0) atomicCAS(P.err_flag, 0, EPK_ERR_PIN_OVERFLOW);
        for (int64_t r = my_begin + tid; r < my_end; r += blockDim.x) keep[r] = 0;
        return;
    }
    int64_t k_rem = limit - pinned_live;
    if (k_rem == 0) {  // only the pins survive
        for (int64_t r = my_begin + tid; r < my_end; r += blockDim.x) {
            const int h = head_of(r);
            keep[r] = (is_live(r, h) && use_pins && is_pinned(P.pins, P.n_pins, pos[r])) ? 1 : 0;
        }
        if (rank == 0 && tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(limit);
        return;
    }

    // ---- this CTA's candidate keys -> shared memory (one global pass) ---------
    // Non-candidates (gap rows, pinned rows) hold the sentinel ~0, which no
    // finite or infinite score maps to.
    extern __shared__ __align__(16) unsigned char s_dyn[];
    KeyT* s_keys = reinterpret_cast<KeyT*>(s_dyn);
    const KeyT kNone = ~KeyT(0);
    const int64_t nmine = my_end - my_begin;
    const bool cached = nmine <= P.key_cap;
    auto fetch_key = [&](int64_t r) -> KeyT {
        const int h = head_of(r);
        if (!is_live(r, h) || (use_pins && is_pinned(P.pins, P.n_pins, pos[r]))) return kNone;
        return desc_key(scores[r]);
    };
    if (cached) {
#pragma unroll 4
        for (int64_t i = tid; i < nmine; i += blockDim.x) s_keys[i] = fetch_key(my_begin + i);
        __syncthreads();
    }
    auto key_of = [&](int64_t r) -> KeyT { return cached ? s_keys[r - my_begin] : fetch_key(r); };

    // ---- radix select on the score key --------------------------------------
    KeyT prefix = 0, mask = 0;
    int pass = 0;
    for (int shift = kKeyBits - 8; shift >= 0; shift -= 8, ++pass) {
        uint32_t* hist = s_hist[pass & 1];
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int64_t b0 = my_begin + int64_t(warp) * 32; b0 < my_end; b0 += int64_t(nwarps) * 32) {
            const int64_t r = b0 + lane;
            int digit = 256;
            if (r < my_end) {
                const KeyT key = key_of(r);
                if (key != kNone && ((key ^ prefix) & mask) == 0) digit = int((key >> shift) & 0xFF);
            }
            const unsigned grp = __match_any_sync(0xffffffffu, digit);
            if (digit != 256 && lane == __ffs(grp) - 1) atomicAdd(&hist[digit], uint32_t(__popc(grp)));
        }
        cluster.sync();
        if (tid < 256) {
            uint32_t t = 0;
            for (int q = 0; q < kSelCluster; ++q) t += cluster.map_shared_rank(hist, q)[tid];
            s_tot[tid] = t;
        }
        __syncthreads();
        if (warp == 0) find_bucket(s_tot, k_rem, &s_bucket, &s_before, &s_eq);
        __syncthreads();
        k_rem -= s_before;
        prefix |= KeyT(s_bucket) << shift;
        mask |= KeyT(0xFF) << shift;
    }
    const KeyT T = prefix;
    const int64_t eq_count = s_eq;

    // ---- tiebreak among rows whose score key equals T ----------------------
    uint64_t U = ~uint64_t(0);
    if (eq_count > k_rem) {
        uint64_t tprefix = 0, tmask = 0;
        for (int shift = kTieBits - 8; shift >= 0; shift -= 8, ++pass) {
            uint32_t* hist = s_hist[pass & 1];
            for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
            __syncthreads();
            for (int64_t b0 = my_begin + int64_t(warp) * 32; b0 < my_end; b0 += int64_t(nwarps) * 32) {
                const int64_t r = b0 + lane;
                int digit = 256;
                if (r < my_end && key_of(r) == T) {
                    const int h = head_of(r);
                    {
                        const uint64_t tb = P.per_head ? uint64_t(r) : ((uint64_t(uint32_t(pos[r])) << 8) | uint64_t(h));
                        if (((tb ^ tprefix) & tmask) == 0) digit = int((tb >> shift) & 0xFF);
                    }
                }
                const unsigned grp = __match_any_sync(0xffffffffu, digit);
                if (digit != 256 && lane == __ffs(grp) - 1) atomicAdd(&hist[digit], uint32_t(__popc(grp)));
            }
            cluster.sync();
            if (tid < 256) {
                uint32_t t = 0;
                for (int q = 0; q < kSelCluster; ++q) t += cluster.map_shared_rank(hist, q)[tid];
                s_tot[tid] = t;
            }
            __syncthreads();
            if (warp == 0) find_bucket(s_tot, k_rem, &s_bucket, &s_before, &s_eq);
            __syncthreads();
            k_rem -= s_before;
            tprefix |= uint64_t(s_bucket) << shift;
            tmask |= uint64_t(0xFF) << shift;
        }
        U = tprefix;
    }

    // ---- write the keep mask -------------------------------------------------
    for (int64_t r = my_begin + tid; r < my_end; r += blockDim.x) {
        const KeyT key = key_of(r);
        uint8_t kf = 0;
        if (key != kNone) {
            if (key < T) {
                kf = 1;
            } else if (key == T) {
                const int h = head_of(r);
                const uint64_t tb = P.per_head ? uint64_t(r) : ((uint64_t(uint32_t(pos[r])) << 8) | uint64_t(h));
                kf = tb <= U ? 1 : 0;
            }
        } else if (use_pins) {
            const int h = head_of(r);
            kf = (is_live(r, h) && is_pinned(P.pins, P.n_pins, pos[r])) ? 1 : 0;
        }
        keep[r] = kf;
    }
    if (rank == 0 && tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(limit);
    cluster.sync();  // no CTA exits while others may still read its histograms
}

int launch_select(epk_ctx* ctx, const epk_cache_desc* c, const void* scores, int score_dtype,
                  const int64_t* budgets, const int32_t* pins, int n_pins, uint8_t* keep,
                  int32_t* kept, int per_head) {
    if (c->kv_heads > kMaxHeads) return fail(EPK_ERR_UNSUPPORTED, "select: more than 64 kv heads");
    if (c->layers > kMaxLayers) return fail(EPK_ERR_UNSUPPORTED, "select: more than 128 layers");
    if (score_dtype != EPK_F32 && score_dtype != EPK_F64) return fail(EPK_ERR_ARG, "select: score dtype must be F32 or F64");
    SelectParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    for (int l = 0; l < c->layers; ++l) {
        if (budgets[l] < 0) return fail(EPK_ERR_ARG, "select: negative budget");
        P.budget[l] = budgets[l];
    }
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.pos = c->pos;
    P.scores = scores;
    P.pins = pins;
    P.n_pins = pins ? n_pins : 0;
    P.H = c->kv_heads;
    P.per_head = per_head;
    P.keep = keep;
    P.kept_per_layer = kept;
    P.err_flag = ctx->err_flag;
    const int segs = per_head ? c->layers * c->kv_heads : c->layers;
    dim3 grid(segs * kSelCluster), block(kSelThreads);
    constexpr int kKeySmem = 96 * 1024;
    static bool attr = false;
    if (!attr) {
        EPK_CUDA_CHECK(cudaFuncSetAttribute(select_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, kKeySmem));
        EPK_CUDA_CHECK(cudaFuncSetAttribute(select_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kKeySmem));
        attr = true;
    }
    P.key_cap = kKeySmem / (score_dtype == EPK_F32 ? 4 : 8);
    EPK_PROF(ctx, per_head ? "select_per_head" : "select");
    if (score_dtype == EPK_F32)
        select_kernel<float><<<grid, block, kKeySmem, ctx->stream>>>(P);
    else
        select_kernel<double><<<grid, block, kKeySmem, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
