// select.cu -- K2: deterministic pooled (and per-head) top-k selection.
//
// Restates the selection of evict_to_budget (kvcache.hpp:142-190): per layer,
// if live <= H*M the layer is unchanged (:148-151); otherwise pinned rows are
// kept (:160-164) and the remaining H*M - pinned_live slots go to the smallest
// composite keys (score desc, position asc, head asc) (:181-190).  The
// per-head mode restates top_k_indices (numerics.hpp:111-125): ties to the
// lower index.
//
// One lean CTA per segment (layer, or (layer, head) in per-head mode): 512
// threads, <= 32 registers, ~20 KB of shared memory, so a select CTA can
// co-reside with a scorer CTA and the side stream's selection overlaps the
// next layer group's scoring.  Passes over the segment (global memory, L2
// resident after the first):
//   keys     every row -> its order-preserving score key (desc_key; ~0 for
//            gap rows and pinned rows) in a key buffer; min/max of the
//            candidate keys (their common leading bits are skipped); pinned
//            count;
//   radix    11-bit digit histograms of the candidates below the known
//            prefix, until the bucket holding the k-th smallest key has at
//            most kCap candidates (one pass for softmax scores);
//   collect  that bucket's candidates (key, tiebreak = position << 8 | head)
//            -> shared memory; the rest of the key bits and the tiebreak are
//            resolved by 8-bit radix passes over the shared list;
//   final    keep[r] = key < T || (key == T && tiebreak <= U) || pinned.
// If the bucket never gets small (massive exact ties), the tiebreak radix runs
// over global memory instead.  Result: the set std::sort would give.
#include <algorithm>

#include "epk_internal.cuh"

namespace epk {

constexpr int kSelThreads = 512;
constexpr int kSelWarps = kSelThreads / 32;
constexpr int kMaxHeads = 64;
constexpr int kDigit = 11;  // global radix digit (2048 bins)
constexpr int kBins = 1 << kDigit;
constexpr int kCap = 1024;  // candidates resolved in shared memory

struct SelectParams {
    LayerTable lt;
    int64_t budget[kMaxLayers];
    const int32_t* head_off;
    const int32_t* head_len;
    const int32_t* pos;
    const void* scores;
    void* keys;  // [rows] key buffer (u32 for fp32 scores, u64 for fp64)
    const int32_t* pins;
    int n_pins;
    int H;
    int per_head;
    uint8_t* keep;
    int32_t* kept_per_layer;
    int* err_flag;
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

template <typename KeyT>
struct SelShared {
    int32_t off[kMaxHeads + 1];
    int32_t len[kMaxHeads];
    int64_t red[kSelWarps];
    KeyT mm[2 * kSelWarps];
    int bucket;
    int ncand;
    int64_t before, eq;
    union {
        uint32_t hist[2][kBins];  // global radix passes (two copies: odd/even warps)
        struct {
            KeyT key[kCap];
            uint64_t tb[kCap];
            uint32_t hist[256];
        } c;  // shared-list radix
    } u;
};

// Block-wide: the bucket of `tot[0..nbins)` holding the k-th smallest element
// (1-based) -> S.bucket, S.before (count strictly before), S.eq (in it).
template <typename KeyT>
__device__ void find_bucket(SelShared<KeyT>& S, const uint32_t* tot, int nbins, int64_t k) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nbins + kSelThreads - 1) / kSelThreads;
    const int b0 = tid * per;
    int64_t mine = 0;
    for (int i = 0; i < per; ++i)
        if (b0 + i < nbins) mine += tot[b0 + i];
    int64_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    __syncthreads();
    if (lane == 31) S.red[warp] = incl;
    __syncthreads();
    int64_t excl = incl - mine;
    for (int w = 0; w < warp; ++w) excl += S.red[w];
    if (mine > 0 && excl < k && k <= excl + mine) {  // exactly one thread
        int64_t c = excl;
        for (int i = 0; i < per; ++i) {
            const int64_t t = b0 + i < nbins ? tot[b0 + i] : 0;
            if (c + t >= k) {
                S.bucket = b0 + i;
                S.before = c;
                S.eq = t;
                break;
            }
            c += t;
        }
    }
    __syncthreads();
}

// The exact selection below a known key prefix: `eq` candidates match
// (prefix, mask) with `lo` key bits still open and `k_rem` slots left among
// them.  Global 11-bit radix passes narrow the bucket until it fits the
// shared list (kCap), the list is resolved by 8-bit passes, and ties on the
// threshold key T are cut by the tiebreak (position << 8 | head), giving U.
// load4(i, k) reads group i's keys (~0 for non-candidates); tiebreak(r) of a
// layer row; rows of group i are g0 + 4 i + u.
template <typename KeyT, typename Load4, typename TieOf>
__device__ __forceinline__ void radix_core(SelShared<KeyT>& S, int ngroups, Load4& load4, TieOf& tiebreak, int g0,
                                           KeyT& prefix, KeyT& mask, int& lo, int64_t& eq, int64_t& k_rem, KeyT& T,
                                           uint64_t& U) {
    constexpr int kTieBits = 40;  // (position < 2^31) << 8 | head (< 256)
    const KeyT kNone = ~KeyT(0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // ---- global radix passes until the bucket fits the shared list ----------
    uint32_t* hist = S.u.hist[warp & 1];
    while (lo > 0 && eq > kCap) {
        const int hi = lo;
        lo = hi > kDigit ? hi - kDigit : 0;
        const KeyT dmask = (KeyT(1) << (hi - lo)) - 1;
        for (int i = tid; i < 2 * kBins; i += blockDim.x) (&S.u.hist[0][0])[i] = 0;
        __syncthreads();
        for (int i = tid; i < ngroups; i += 2 * blockDim.x) {
            KeyT k[2][4];
            load4(i, k[0]);
            const bool two = i + int(blockDim.x) < ngroups;
            if (two) load4(i + blockDim.x, k[1]);
#pragma unroll
            for (int v = 0; v < 2; ++v)
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if ((v == 0 || two) && k[v][u] != kNone && ((k[v][u] ^ prefix) & mask) == 0)
                        atomicAdd(&hist[int((k[v][u] >> lo) & dmask)], 1u);
        }
        __syncthreads();
        for (int i = tid; i < kBins; i += blockDim.x) S.u.hist[0][i] += S.u.hist[1][i];
        __syncthreads();
        find_bucket(S, S.u.hist[0], int(dmask) + 1, k_rem);
        k_rem -= S.before;
        eq = S.eq;
        prefix |= KeyT(S.bucket) << lo;
        mask |= dmask << lo;
    }

    U = ~uint64_t(0);
    if (eq <= kCap) {
        // ---- collect the bucket's candidates into shared memory -------------
        if (tid == 0) S.ncand = 0;
        __syncthreads();
        for (int ib = warp * 32; ib < ngroups; ib += blockDim.x) {  // warp-uniform
            const int i = ib + lane;
            KeyT k[4] = {kNone, kNone, kNone, kNone};
            if (i < ngroups) load4(i, k);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool c = k[u] != kNone && ((k[u] ^ prefix) & mask) == 0;
                const unsigned bal = __ballot_sync(0xffffffffu, c);
                if (bal == 0) continue;
                const int leader = __ffs(bal) - 1;
                int at = 0;
                if (lane == leader) at = atomicAdd(&S.ncand, __popc(bal));
                at = __shfl_sync(0xffffffffu, at, leader) + __popc(bal & ((1u << lane) - 1u));
                if (c) {
                    S.u.c.key[at] = k[u];
                    S.u.c.tb[at] = tiebreak(g0 + 4 * i + u);
                }
            }
        }
        __syncthreads();
        const int n = S.ncand;  // == eq
        // ---- remaining key bits: 8-bit radix over the shared list -----------
        uint32_t* h2 = S.u.c.hist;
        while (lo > 0) {
            const int hi = lo;
            lo = hi > 8 ? hi - 8 : 0;
            const KeyT dmask = (KeyT(1) << (hi - lo)) - 1;
            for (int i = tid; i < 256; i += blockDim.x) h2[i] = 0;
            __syncthreads();
            for (int i = tid; i < n; i += blockDim.x) {
                const KeyT k = S.u.c.key[i];
                if (((k ^ prefix) & mask) == 0) atomicAdd(&h2[int((k >> lo) & dmask)], 1u);
            }
            __syncthreads();
            find_bucket(S, h2, int(dmask) + 1, k_rem);
            k_rem -= S.before;
            eq = S.eq;
            prefix |= KeyT(S.bucket) << lo;
            mask |= dmask << lo;
        }
        T = prefix;
        // ---- tiebreak among the list's rows with key T -----------------------
        if (eq > k_rem) {
            uint64_t tprefix = 0, tmask = 0;
            for (int shift = kTieBits - 8; shift >= 0; shift -= 8) {
                for (int i = tid; i < 256; i += blockDim.x) h2[i] = 0;
                __syncthreads();
                for (int i = tid; i < n; i += blockDim.x) {
                    const uint64_t tb = S.u.c.tb[i];
                    if (S.u.c.key[i] == T && ((tb ^ tprefix) & tmask) == 0)
                        atomicAdd(&h2[int((tb >> shift) & 0xFF)], 1u);
                }
                __syncthreads();
                find_bucket(S, h2, 256, k_rem);
                k_rem -= S.before;
                tprefix |= uint64_t(S.bucket) << shift;
                tmask |= uint64_t(0xFF) << shift;
            }
            U = tprefix;
        }
    } else {
        // every key bit resolved and still more than kCap rows share key T:
        // tiebreak radix over global memory
        T = prefix;
        if (eq > k_rem) {
            uint64_t tprefix = 0, tmask = 0;
            for (int shift = kTieBits - 8; shift >= 0; shift -= 8) {
                for (int i = tid; i < 2 * kBins; i += blockDim.x) (&S.u.hist[0][0])[i] = 0;
                __syncthreads();
                for (int i = tid; i < ngroups; i += blockDim.x) {
                    KeyT k[4];
                    load4(i, k);
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        if (k[u] != T) continue;
                        const uint64_t tb = tiebreak(g0 + 4 * i + u);
                        if (((tb ^ tprefix) & tmask) == 0) atomicAdd(&hist[int((tb >> shift) & 0xFF)], 1u);
                    }
                }
                __syncthreads();
                for (int i = tid; i < 256; i += blockDim.x) S.u.hist[0][i] += S.u.hist[1][i];
                __syncthreads();
                find_bucket(S, S.u.hist[0], 256, k_rem);
                k_rem -= S.before;
                tprefix |= uint64_t(S.bucket) << shift;
                tmask |= uint64_t(0xFF) << shift;
            }
            U = tprefix;
        }
    }

}

template <typename ScoreT>
__global__ void __launch_bounds__(kSelThreads, 4) select_kernel(const __grid_constant__ SelectParams P) {
    using KeyT = typename KeyOf<ScoreT>::T;
    constexpr int kKeyBits = int(sizeof(KeyT) * 8);
    const KeyT kNone = ~KeyT(0);  // no finite or infinite score maps to it
    __shared__ SelShared<KeyT> S;

    const int seg = blockIdx.x;
    const int H = P.H;
    const int layer = P.per_head ? seg / H : seg;
    const int seg_head = P.per_head ? seg % H : -1;
    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;

    for (int i = tid; i <= H; i += blockDim.x) S.off[i] = P.head_off[layer * (H + 1) + i];
    for (int i = tid; i < H; i += blockDim.x) S.len[i] = P.head_len[layer * H + i];
    __syncthreads();

    // Segment row space (layer-relative rows [sb, se), gaps included).
    int sb, se;
    int64_t n_live = 0;
    if (P.per_head) {
        sb = S.off[seg_head];
        se = sb + S.len[seg_head];
        n_live = S.len[seg_head];
    } else {
        sb = 0;
        se = S.off[H];
        for (int h = 0; h < H; ++h) n_live += S.len[h];
    }
    const int64_t base = P.lt.base[layer];
    // 4-row groups aligned in global row space: group i covers layer rows
    // [g0 + 4i, g0 + 4i + 4), g0 = (base + sb rounded down to 4) - base.
    const int g0 = int(((base + sb) & ~int64_t(3)) - base);
    const int ngroups = se > sb ? (se - g0 + 3) / 4 : 0;
    const ScoreT* scores = static_cast<const ScoreT*>(P.scores) + base;
    KeyT* keys = static_cast<KeyT*>(P.keys) + base;
    const int32_t* pos = P.pos + base;
    uint8_t* keep = P.keep + base;
    const bool use_pins = !P.per_head && P.n_pins > 0;

    auto head_of = [&](int r) -> int {
        if (P.per_head) return seg_head;
        int lo = 0, hi = H - 1;
        while (lo < hi) {  // last h with off[h] <= r
            const int mid = (lo + hi + 1) >> 1;
            if (S.off[mid] <= r) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    auto is_live = [&](int r, int h) -> bool { return r - S.off[h] < S.len[h]; };
    auto block_sum = [&](int64_t v) -> int64_t {
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) S.red[warp] = v;
        __syncthreads();
        int64_t t = 0;
        for (int w = 0; w < kSelWarps; ++w) t += S.red[w];
        __syncthreads();
        return t;
    };
    auto tiebreak = [&](int r) -> uint64_t {
        return P.per_head ? uint64_t(r) : ((uint64_t(uint32_t(pos[r])) << 8) | uint64_t(head_of(r)));
    };
    // Keys of group i (rows outside [sb, se) -> kNone).
    auto load4 = [&](int i, KeyT (&k)[4]) {
        const int r0 = g0 + 4 * i;
        if (r0 >= sb && r0 + 4 <= se) {
            if constexpr (sizeof(KeyT) == 4) {
                const uint4 v = __ldcg(reinterpret_cast<const uint4*>(keys + r0));
                k[0] = v.x;
                k[1] = v.y;
                k[2] = v.z;
                k[3] = v.w;
            } else {
                const ulonglong2 v0 = __ldcg(reinterpret_cast<const ulonglong2*>(keys + r0));
                const ulonglong2 v1 = __ldcg(reinterpret_cast<const ulonglong2*>(keys + r0 + 2));
                k[0] = v0.x;
                k[1] = v0.y;
                k[2] = v1.x;
                k[3] = v1.y;
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) k[u] = (r0 + u >= sb && r0 + u < se) ? keys[r0 + u] : kNone;
        }
    };

    if (P.per_head)  // gap rows after the head's live rows: never kept
        for (int r = se + tid; r < S.off[seg_head + 1]; r += blockDim.x) keep[r] = 0;

    // ---- keys (gap and pinned rows -> kNone), min/max, pinned count ---------
    int64_t pinned_mine = 0;
    KeyT kmin = kNone, kmax = 0;
    for (int i = tid; i < ngroups; i += blockDim.x) {
        const int r0 = g0 + 4 * i;
        KeyT k[4];
        int h = head_of(max(r0, sb));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = r0 + u;
            k[u] = kNone;
            if (r < sb || r >= se) continue;
            while (!P.per_head && h + 1 < H && S.off[h + 1] <= r) ++h;
            if (!is_live(r, h)) continue;
            if (use_pins && is_pinned(P.pins, P.n_pins, pos[r])) {
                ++pinned_mine;
                continue;
            }
            const ScoreT sv = __ldcg(scores + r);
            if (sv != sv) atomicCAS(P.err_flag, 0, EPK_ERR_NAN);  // no order for NaN (kvcache.hpp:181-185)
            k[u] = desc_key(sv);
            kmin = k[u] < kmin ? k[u] : kmin;
            kmax = k[u] > kmax ? k[u] : kmax;
        }
        if (r0 >= sb && r0 + 4 <= se) {
            if constexpr (sizeof(KeyT) == 4) {
                *reinterpret_cast<uint4*>(keys + r0) = make_uint4(k[0], k[1], k[2], k[3]);
            } else {
                *reinterpret_cast<ulonglong2*>(keys + r0) = make_ulonglong2(k[0], k[1]);
                *reinterpret_cast<ulonglong2*>(keys + r0 + 2) = make_ulonglong2(k[2], k[3]);
            }
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (r0 + u >= sb && r0 + u < se) keys[r0 + u] = k[u];
        }
    }
    const int64_t pinned_live = use_pins ? block_sum(pinned_mine) : 0;

    const int64_t limit = P.per_head ? P.budget[layer] : int64_t(H) * P.budget[layer];
    auto write_keep_all = [&](int mode) {  // 0: live rows, 1: nothing, 2: pinned live rows
        for (int r = sb + tid; r < se; r += blockDim.x) {
            uint8_t kf = 0;
            if (mode == 0) {
                kf = is_live(r, head_of(r)) ? 1 : 0;
            } else if (mode == 2) {
                kf = (is_live(r, head_of(r)) && use_pins && is_pinned(P.pins, P.n_pins, pos[r])) ? 1 : 0;
            }
            keep[r] = kf;
        }
    };
    if (n_live <= limit) {
        write_keep_all(0);
        if (tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(n_live);
        return;
    }
    if (pinned_live > limit) {
        if (tid == 0) atomicCAS(P.err_flag, 0, EPK_ERR_PIN_OVERFLOW);
        write_keep_all(1);
        return;
    }
    int64_t k_rem = limit - pinned_live;
    if (k_rem == 0) {  // only the pins survive
        write_keep_all(2);
        if (tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(limit);
        return;
    }
    const int64_t n_cand = n_live - pinned_live;  // > k_rem > 0

    // ---- common leading bits of the candidates ------------------------------
    for (int o = 16; o > 0; o >>= 1) {
        const KeyT a = __shfl_xor_sync(0xffffffffu, kmin, o), b = __shfl_xor_sync(0xffffffffu, kmax, o);
        kmin = a < kmin ? a : kmin;
        kmax = b > kmax ? b : kmax;
    }
    if (lane == 0) {
        S.mm[2 * warp] = kmin;
        S.mm[2 * warp + 1] = kmax;
    }
    __syncthreads();
    for (int w = 0; w < kSelWarps; ++w) {
        kmin = S.mm[2 * w] < kmin ? S.mm[2 * w] : kmin;
        kmax = S.mm[2 * w + 1] > kmax ? S.mm[2 * w + 1] : kmax;
    }
    const KeyT diff = kmin ^ kmax;
    int lo = diff == 0 ? 0 : kKeyBits - (sizeof(KeyT) == 4 ? __clz(uint32_t(diff)) : __clzll(uint64_t(diff)));
    KeyT mask = lo >= kKeyBits ? KeyT(0) : ~((KeyT(1) << lo) - 1);
    KeyT prefix = kmin & mask;
    int64_t eq = n_cand;  // candidates matching (prefix, mask)

    KeyT T;
    uint64_t U;
    radix_core<KeyT>(S, ngroups, load4, tiebreak, g0, prefix, mask, lo, eq, k_rem, T, U);

    // ---- write the keep mask -------------------------------------------------
    for (int i = tid; i < ngroups; i += blockDim.x) {
        const int r0 = g0 + 4 * i;
        KeyT k[4];
        load4(i, k);
        uint8_t kf[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int r = r0 + u;
            kf[u] = 0;
            if (r < sb || r >= se) continue;
            if (k[u] != kNone) {
                if (k[u] < T) kf[u] = 1;
                else if (k[u] == T) kf[u] = tiebreak(r) <= U ? 1 : 0;
            } else if (use_pins) {
                kf[u] = (is_live(r, head_of(r)) && is_pinned(P.pins, P.n_pins, pos[r])) ? 1 : 0;
            }
        }
        if (r0 >= sb && r0 + 4 <= se && (reinterpret_cast<uintptr_t>(keep + r0) & 3) == 0) {
            *reinterpret_cast<uint32_t*>(keep + r0) =
                uint32_t(kf[0]) | (uint32_t(kf[1]) << 8) | (uint32_t(kf[2]) << 16) | (uint32_t(kf[3]) << 24);
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (r0 + u >= sb && r0 + u < se) keep[r0 + u] = kf[u];
        }
    }
    if (tid == 0 && P.kept_per_layer && !P.per_head) P.kept_per_layer[layer] = int32_t(limit);
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
    // key buffer: the side-stream workspace (compaction reuses it afterwards,
    // in stream order)
    const int64_t rows = c->layer_base[c->layers];
    rc = ws2_require(ctx, rows * (score_dtype == EPK_F32 ? 4 : 8) + 4096);
    if (rc) return rc;
    P.keys = ctx->ws2;
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
    EPK_PROF(ctx, per_head ? "select_per_head" : "select");
    if (score_dtype == EPK_F32)
        select_kernel<float><<<segs, kSelThreads, 0, ctx->stream>>>(P);
    else
        select_kernel<double><<<segs, kSelThreads, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// ---------------------------------------------------------------------------
// Threshold select (the tensor-core step, no pins), with the compaction plan
// folded in.  The scorer (score_tc.cu, SCORE pass) already wrote each live
// row's key and counted float_bits(score) >> 14 into a 65536-bin per-layer
// histogram (+ a 256-bin coarse one).  Scores are softmax weights in [0, 1]
// (bin and key prefix agree for any score in [0, 2)), so bin b holds exactly
// the keys with key >> 14 == 0x1FFFF - b.  Grid: `parts` CTAs per layer (128
// threads), each owning a chunk-aligned slice of the layer's rows:
//   every CTA   finds the threshold bin kb and its rank from the coarse and
//               fine histograms (two 1 KB reads); over its slice it counts,
//               per 128-row compaction chunk, the live rows certainly kept
//               (key bin < kb) and appends the undecided ones (bin == kb) to
//               the layer's candidate list {key, row, position << 8 | head};
//   last CTA    (per-layer arrival counter) resolves the exact threshold key T
//               and tiebreak U among the candidates (8-bit radix on the
//               remaining 14 key bits, then on position << 8 | head), adds
//               the kept candidates to their chunks, scans the chunk counts
//               into the compaction plan (chunk prefixes, output head
//               offsets/lengths, the does-not-fit flag -- the former
//               count/plan launches), writes thr[l] = {T | flags << 32, U}
//               and resets the counters for the next step (the next P1
//               launch zeroes the histograms).
// The gather (compact.cu) then keeps live rows with key < T || (key == T &&
// tiebreak <= U).
// ---------------------------------------------------------------------------
constexpr int kTSThreads = 128;
constexpr int kTSCand = 1024;  // candidates resolved in shared memory
#ifndef EPK_TS_BLK
#define EPK_TS_BLK 16  // 32 spills at the 4-CTA/SM register budget
#endif
constexpr int kTSBlk = EPK_TS_BLK;  // 128-row chunks per slice iteration (keys loaded up front: one round trip)

struct ThreshParams {
    LayerTable lt;
    LayerTable out_lt;  // output cache capacity layout (the plan's fit check)
    int64_t budget[kMaxLayers];
    const int32_t* head_off;
    const int32_t* head_len;
    const int32_t* pos;
    const uint32_t* keys;    // [rows] global cache rows
    uint32_t* hist_fine;     // [layers][65536]
    uint32_t* hist_coarse;   // [layers][256]
    uint64_t* thr;           // [layers][2]
    uint4* cand;             // [layers][kTSCand] {key, layer row, tiebreak lo, tiebreak hi}
    unsigned* cand_n;        // [layers]
    unsigned* done;          // [layers]
    int32_t* kept_per_layer;
    // compaction plan (CompactWs) and the output head layout
    int32_t* chunk_cnt;
    int32_t* chunk_prefix;
    int32_t* layer_bad;
    int32_t* out_off;  // [layers][H + 1]
    int32_t* out_len;  // [layers][H]
    int max_chunks;
    int rpp;  // rows per CTA slice (a multiple of kChunkRows)
    int slack;
    int H;
    int parts;
    int* err_flag;
};

struct TSShared {
    int32_t off[kMaxHeads + 1];
    int32_t len[kMaxHeads];
    uint32_t tot[256];
    uint32_t hist[256];
    union {
        struct {  // last CTA: the layer's candidates
            uint32_t ck[kTSCand];
            int32_t cr[kTSCand];
            uint64_t ct[kTSCand];
        };
        uint4 lc[kTSCand];  // every CTA: its slice's candidates {key, row, head, 0} before they go global
    };
    unsigned nlc;
    int64_t red[kTSThreads / 32];
    int64_t head_prefix[kMaxHeads + 1];
    int32_t wc[kTSBlk][kTSThreads / 32];  // per (chunk of the iteration, warp): certainly kept rows
    int bucket;
    int64_t before, eq;
    int last;
};

// Bucket of tot[0..nbins) (nbins <= 256) holding the k-th smallest (1-based).
__device__ void ts_find_bucket(TSShared& S, const uint32_t* tot, int nbins, int64_t k) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int b0 = tid * 2;
    const int64_t mine = (b0 < nbins ? tot[b0] : 0) + (b0 + 1 < nbins ? tot[b0 + 1] : 0);
    int64_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    __syncthreads();
    if (lane == 31) S.red[w] = incl;
    __syncthreads();
    int64_t excl = incl - mine;
    for (int q = 0; q < w; ++q) excl += S.red[q];
    if (mine > 0 && excl < k && k <= excl + mine) {
        const int64_t t0 = b0 < nbins ? tot[b0] : 0;
        if (excl + t0 >= k) {
            S.bucket = b0;
            S.before = excl;
            S.eq = t0;
        } else {
            S.bucket = b0 + 1;
            S.before = excl + t0;
            S.eq = tot[b0 + 1];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kTSThreads, 4) select_threshold_kernel(const __grid_constant__ ThreshParams P) {
    TL_BEGIN();
    pdl_wait();
    TL_GO();
    __shared__ TSShared S;
    const int l = blockIdx.y, part = blockIdx.x;
    const int H = P.H;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // independent loads first, in flight together: the head layout, the
    // coarse histogram and the keys of this CTA's first slice block (rows of
    // the layer's capacity; the slice bound is applied once the layout is in)
    for (int i = tid; i <= H; i += kTSThreads) S.off[i] = P.head_off[l * (H + 1) + i];
    for (int i = tid; i < H; i += kTSThreads) S.len[i] = P.head_len[l * H + i];
    const int64_t base = P.lt.base[l];
    const uint32_t* keys = P.keys + base;
    const int cap_l = int(P.lt.base[l + 1] - base);
    const int r_beg = part * P.rpp;
    uint32_t kv[kTSBlk];
#pragma unroll
    for (int u = 0; u < kTSBlk; ++u) {
        const int rr = r_beg + u * kTSThreads + tid;
        kv[u] = rr < cap_l ? __ldcg(keys + rr) : 0u;
    }
    uint32_t hc[256 / kTSThreads];
#pragma unroll
    for (int j = 0; j < 256 / kTSThreads; ++j) hc[j] = __ldcg(P.hist_coarse + l * 256 + 255 - (tid + j * kTSThreads));
    __syncthreads();
    int64_t n_live = 0;
    for (int h = 0; h < H; ++h) n_live += S.len[h];
    const int region = S.off[H];
    const int32_t* pos = P.pos + base;
    int32_t* ccnt = P.chunk_cnt + int64_t(l) * P.max_chunks;
    const int64_t limit = int64_t(H) * P.budget[l];
    auto head_of = [&](int r) -> int {
        int lo = 0, hi = H - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (S.off[mid] <= r) lo = mid; else hi = mid - 1;
        }
        return lo;
    };
    uint32_t kb = 0;
    int64_t k_rem = limit, eq = 0;
    // budget 0 keeps nothing (evict_to_budget with no pins, kvcache.hpp:180-190):
    // no threshold bin exists, the resolve below emits the "none" flag
    const bool none = n_live > limit && limit == 0;
    const bool select = n_live > limit && !none;
    const bool all = n_live <= limit;  // every live row stays
    if (select) {
        // threshold bin: coarse then fine histogram, bins in key order
#pragma unroll
        for (int j = 0; j < 256 / kTSThreads; ++j) S.tot[tid + j * kTSThreads] = hc[j];
        __syncthreads();
        ts_find_bucket(S, S.tot, 256, k_rem);
        k_rem -= S.before;
        const int cb = 255 - S.bucket;
        for (int i = tid; i < 256; i += kTSThreads)
            S.tot[i] = __ldcg(P.hist_fine + int64_t(l) * 65536 + cb * 256 + 255 - i);
        __syncthreads();
        ts_find_bucket(S, S.tot, 256, k_rem);
        k_rem -= S.before;
        eq = S.eq;
        kb = uint32_t(0x1FFFF - (cb * 256 + 255 - S.bucket));
    }
    TL_END(7);
    // this CTA's chunk-aligned slice: per chunk the rows certainly kept, and
    // the threshold bin's candidates -> the layer's list (keys loaded 16 per
    // thread at a time, the first block's before the histograms)
    const int r_end = min(region, r_beg + P.rpp);
    if (tid == 0) S.nlc = 0;
    __syncthreads();
    for (int b0 = r_beg; b0 < r_end; b0 += kTSBlk * kTSThreads) {  // block-uniform
        if (select && b0 != r_beg) {
#pragma unroll
            for (int u = 0; u < kTSBlk; ++u) {
                const int rr = b0 + u * kTSThreads + tid;
                kv[u] = rr < r_end ? __ldcg(keys + rr) : 0u;
            }
        }
        int h = head_of(min(b0 + tid, max(r_end - 1, 0)));
        TL_END(8);
#pragma unroll
        for (int u = 0; u < kTSBlk; ++u) {
            const int rr = b0 + u * kTSThreads + tid;
            bool c = false, def = false;
            if (rr < r_end) {
                while (h + 1 < H && S.off[h + 1] <= rr) ++h;
                const bool live = rr - S.off[h] < S.len[h];
                if (select) {
                    c = live && (kv[u] >> 14) == kb;
                    def = live && (kv[u] >> 14) < kb;
                } else {
                    def = live && all;
                }
            }
            const unsigned dball = __ballot_sync(0xffffffffu, def);
            if (lane == 0) S.wc[u][warp] = __popc(dball);
            const unsigned bal = __ballot_sync(0xffffffffu, c);
            if (bal == 0) continue;
            const int leader = __ffs(bal) - 1;
            unsigned at = 0;
            if (lane == leader) at = atomicAdd(&S.nlc, unsigned(__popc(bal)));  // shared memory: no round trip
            at = __shfl_sync(0xffffffffu, at, leader) + __popc(bal & ((1u << lane) - 1u));
            if (c && at < unsigned(kTSCand)) S.lc[at] = make_uint4(kv[u], uint32_t(rr), uint32_t(h), 0u);
        }
        __syncthreads();
        if (tid < kTSBlk && b0 + tid * kTSThreads < r_end) {
            int32_t v = 0;
#pragma unroll
            for (int w = 0; w < kTSThreads / 32; ++w) v += S.wc[tid][w];
            ccnt[(b0 + tid * kTSThreads) / kChunkRows] = v;
        }
        __syncthreads();
    }
    // the slice's candidates -> the layer's list: one global reservation per
    // CTA, positions loaded for all of them at once.  A slice with more than
    // kTSCand candidates pushes the count past kTSCand, so the last CTA takes
    // the unlisted path (it rescans the layer's rows).
    if (select) {
        if (tid == 0) {
            const unsigned n = S.nlc;
            S.before = n ? int64_t(atomicAdd(P.cand_n + l, n <= unsigned(kTSCand) ? n : n + kTSCand + 1)) : 0;
        }
        __syncthreads();
        const unsigned n = min(S.nlc, unsigned(kTSCand)), at0 = unsigned(S.before);
        for (unsigned i = tid; i < n && at0 + i < unsigned(kTSCand); i += kTSThreads) {
            const uint4 e = S.lc[i];
            const uint64_t tb = (uint64_t(uint32_t(pos[e.y])) << 8) | uint64_t(e.z);
            P.cand[int64_t(l) * kTSCand + at0 + i] = make_uint4(e.x, e.y, uint32_t(tb), uint32_t(tb >> 32));
        }
    }
    TL_END(9);
    // the last CTA of the layer resolves and plans
    __threadfence();
    __syncthreads();
    if (tid == 0) S.last = atomicAdd(P.done + l, 1u) == unsigned(P.parts - 1);
    __syncthreads();
    if (!S.last) {
        TL_END(4);
        return;
    }
    __threadfence();
    // thr[2l] bit 32: keep every live row; bit 33: keep none; else the exact
    // threshold key T in the low word and the (position << 8 | head) tiebreak U
    uint64_t t0 = uint64_t(1) << 32, t1 = ~uint64_t(0);  // keep every live row
    if (none) t0 = uint64_t(2) << 32;
    if (select) {
        const unsigned n = __ldcg(P.cand_n + l);
        const bool listed = int64_t(n) == eq && n <= unsigned(kTSCand);
        if (listed) {
            for (int i = tid; i < int(n); i += kTSThreads) {
                const uint4 cv = __ldcg(P.cand + int64_t(l) * kTSCand + i);
                S.ck[i] = cv.x;
                S.cr[i] = int32_t(cv.y);
                S.ct[i] = (uint64_t(cv.w) << 32) | cv.z;
            }
            __syncthreads();
        }
        // for_each(f): f(key, tiebreak, layer row) over the bin's candidates
        auto each = [&](auto&& f) {
            if (listed) {
                for (int i = tid; i < int(n); i += kTSThreads) f(S.ck[i], S.ct[i], S.cr[i]);
            } else {  // list overflow: the layer's rows in global memory
                for (int rr = tid; rr < region; rr += kTSThreads) {
                    const int h = head_of(rr);
                    if (rr - S.off[h] >= S.len[h]) continue;
                    const uint32_t key = __ldcg(keys + rr);
                    if ((key >> 14) == kb) f(key, (uint64_t(uint32_t(pos[rr])) << 8) | uint64_t(h), rr);
                }
            }
        };
        uint32_t prefix = kb << 14, mask = 0xFFFFC000u;
        int lo = 14;
        while (lo > 0) {
            const int hi = lo;
            lo = hi > 8 ? hi - 8 : 0;
            const uint32_t dmask = (1u << (hi - lo)) - 1;
            for (int i = tid; i < 256; i += kTSThreads) S.hist[i] = 0;
            __syncthreads();
            each([&](uint32_t k, uint64_t, int) {
                if (((k ^ prefix) & mask) == 0) atomicAdd(&S.hist[(k >> lo) & dmask], 1u);
            });
            __syncthreads();
            ts_find_bucket(S, S.hist, int(dmask) + 1, k_rem);
            k_rem -= S.before;
            eq = S.eq;
            prefix |= uint32_t(S.bucket) << lo;
            mask |= dmask << lo;
        }
        const uint32_t T = prefix;
        uint64_t U = ~uint64_t(0);
        if (eq > k_rem) {
            uint64_t tp = 0, tm = 0;
            for (int shift = 32; shift >= 0; shift -= 8) {
                for (int i = tid; i < 256; i += kTSThreads) S.hist[i] = 0;
                __syncthreads();
                each([&](uint32_t k, uint64_t tb, int) {
                    if (k == T && ((tb ^ tp) & tm) == 0) atomicAdd(&S.hist[(tb >> shift) & 0xFF], 1u);
                });
                __syncthreads();
                ts_find_bucket(S, S.hist, 256, k_rem);
                k_rem -= S.before;
                tp |= uint64_t(S.bucket) << shift;
                tm |= uint64_t(0xFF) << shift;
            }
            U = tp;
        }
        t0 = T;
        t1 = U;
        TL_END(10);
        // the kept candidates join their chunks' counts
        each([&](uint32_t k, uint64_t tb, int rr) {
            if (k < T || (k == T && tb <= U)) atomicAdd(ccnt + rr / kChunkRows, 1);
        });
        __threadfence();
        __syncthreads();
    }
    // ---- compaction plan: chunk prefixes, output head offsets / lengths ----
    const uint32_t T = uint32_t(t0);
    auto keep_row = [&](int r) -> bool {  // the gather's keep rule
        const int h = head_of(r);
        if (none || r - S.off[h] >= S.len[h]) return false;
        if (all) return true;
        const uint32_t key = __ldcg(keys + r);
        return key < T || (key == T && ((uint64_t(uint32_t(pos[r])) << 8) | uint64_t(h)) <= t1);
    };
    TL_END(11);
    const int nchunks = (region + kChunkRows - 1) / kChunkRows;
    int32_t* cpre = P.chunk_prefix + int64_t(l) * P.max_chunks;
    {  // block-wide exclusive scan, each thread owns a contiguous run of chunks
       // (loaded kScanU at a time, so a run costs one L2 round trip per kScanU)
        constexpr int kScanU = 8;
        const int per = (nchunks + kTSThreads - 1) / kTSThreads;
        const int c0 = tid * per, c1 = min(nchunks, c0 + per);
        int64_t mine = 0;
        for (int cb = c0; cb < c1; cb += kScanU) {
            int32_t v[kScanU];
#pragma unroll
            for (int u = 0; u < kScanU; ++u) v[u] = cb + u < c1 ? __ldcg(ccnt + cb + u) : 0;
#pragma unroll
            for (int u = 0; u < kScanU; ++u) mine += v[u];
        }
        int64_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) S.red[warp] = incl;
        __syncthreads();
        int64_t run = incl - mine;
        for (int w = 0; w < warp; ++w) run += S.red[w];
        for (int cb = c0; cb < c1; cb += kScanU) {
            int32_t v[kScanU];
#pragma unroll
            for (int u = 0; u < kScanU; ++u) v[u] = cb + u < c1 ? __ldcg(ccnt + cb + u) : 0;
#pragma unroll
            for (int u = 0; u < kScanU; ++u) {
                if (cb + u < c1) cpre[cb + u] = int32_t(run);
                run += v[u];
            }
        }
    }
    __threadfence();
    __syncthreads();
    TL_END(12);
    // kept rows before every head start: the chunk prefix plus a warp-wide
    // count of the kept rows in [chunk start, head start)
    for (int h = warp; h <= H; h += kTSThreads / 32) {
        const int x = S.off[h];
        const int c = x / kChunkRows;
        int64_t v;
        if (c >= nchunks) {
            v = nchunks == 0 ? 0 : int64_t(__ldcg(cpre + nchunks - 1)) + __ldcg(ccnt + nchunks - 1);
        } else {
            int cnt = 0;
            for (int r = c * kChunkRows + lane; r < x; r += 32) cnt += keep_row(r) ? 1 : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            v = int64_t(__ldcg(cpre + c)) + cnt;
        }
        if (lane == 0) S.head_prefix[h] = v;
    }
    __syncthreads();
    if (tid == 0) {
        P.thr[2 * l] = t0;
        P.thr[2 * l + 1] = t1;
        if (P.kept_per_layer) P.kept_per_layer[l] = int32_t(min(n_live, limit));
        P.cand_n[l] = 0;
        P.done[l] = 0;
        const int64_t cap = P.out_lt.base[l + 1] - P.out_lt.base[l];
        const int64_t need = S.head_prefix[H] + int64_t(P.slack) * H;
        const bool bad = need > cap;
        P.layer_bad[l] = bad;
        if (bad) {
            // the output layer cannot hold the kept rows: flag it, leave the
            // layer empty and let the gather skip it (no store past the layer)
            atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
            for (int h = 0; h <= H; ++h) P.out_off[l * (H + 1) + h] = 0;
            for (int h = 0; h < H; ++h) P.out_len[l * H + h] = 0;
        } else {
            for (int h = 0; h < H; ++h) {
                P.out_off[l * (H + 1) + h] = int32_t(S.head_prefix[h] + int64_t(P.slack) * h);
                P.out_len[l * H + h] = int32_t(S.head_prefix[h + 1] - S.head_prefix[h]);
            }
            P.out_off[l * (H + 1) + H] = int32_t(S.head_prefix[H] + int64_t(P.slack) * H);
        }
    }
    TL_END(5);
}

int launch_select_threshold(epk_ctx* ctx, const epk_cache_desc* c, const epk_cache_desc* out, int out_slack,
                            const FusedSelect* fs, const int64_t* budgets, uint64_t* thr, int32_t* kept) {
    if (c->kv_heads > kMaxHeads) return fail(EPK_ERR_UNSUPPORTED, "select: more than 64 kv heads");
    if (out_slack < 0) return fail(EPK_ERR_ARG, "compact: negative slack");
    ThreshParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    if ((rc = make_layer_table(out, &P.out_lt))) return rc;
    int64_t max_region = 0;
    for (int l = 0; l < c->layers; ++l) {
        if (budgets[l] < 0) return fail(EPK_ERR_ARG, "select: negative budget");
        P.budget[l] = budgets[l];
        max_region = std::max<int64_t>(max_region, P.lt.base[l + 1] - P.lt.base[l]);
    }
    CompactWs w;
    if ((rc = compact_ws(ctx, c, &w))) return rc;
    P.chunk_cnt = w.chunk_cnt;
    P.chunk_prefix = w.chunk_prefix;
    P.layer_bad = w.layer_bad;
    P.max_chunks = w.max_chunks;
    P.out_off = out->head_off;
    P.out_len = out->head_len;
    P.slack = out_slack;
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.pos = c->pos;
    P.keys = fs->keys;
    P.hist_fine = fs->hist_fine;
    P.hist_coarse = fs->hist_coarse;
    P.thr = thr;
    P.cand = fs->cand;
    P.cand_n = fs->cand_n;
    P.done = fs->done;
    P.kept_per_layer = kept;
    P.H = c->kv_heads;
    // one CTA per 4096-row slice (measured: 8192 -> 4096 rows takes the cfg2
    // select from 35 to 27 us; smaller slices no longer help), slices aligned
    // to the compaction chunks, at most 64 per layer
    P.parts = int(std::max<int64_t>(1, std::min<int64_t>(64, (max_region + 4095) / 4096)));
    const int64_t per = (max_region + P.parts - 1) / P.parts;
    P.rpp = int(std::max<int64_t>(kChunkRows, (per + kChunkRows - 1) / kChunkRows * kChunkRows));
    P.err_flag = ctx->err_flag;
    EPK_PROF(ctx, "select");
    EPK_CUDA_CHECK(launch_pdl(select_threshold_kernel, dim3(P.parts, c->layers), dim3(kTSThreads), 0, ctx->stream, P));
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
