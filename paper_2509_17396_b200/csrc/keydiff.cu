// keydiff.cu -- K6: the KeyDiff baseline scorer on the
// shared selection/compaction path.
//
// Restates keydiff_scores (scoring.hpp:186-221) in fp64, bit-exact with the
// reference: per (layer, kv-head) the anchor is the mean key state -- a
// per-dimension sum over the head's live entries in cache (= position) order,
// then / n -- and every entry scores -clamp(dot(k, anchor) / (|k| |anchor|),
// -1, 1) with the sequential dot / norm loops of numerics.hpp:52-87, or 0
// when the anchor or the key has zero norm.  The reference build uses
// -ffp-contract=off, so every product and sum here is an explicitly rounded
// __dmul_rn / __dadd_rn (no FMA contraction).
//
// Two launches:
//   anchor  one CTA per (layer, head): the head's rows (contiguous in the
//           cache) stream through a 4-stage ring of 16 KB shared-memory chunks
//           filled by 1-D bulk copies (TMA engine, mbarrier completion), so
//           the HBM latency hides behind the sequential fp64 sums; thread i
//           keeps the running sums of dimensions i and i + 128 in row order,
//           / n, and thread 0 the anchor's norm (sequential over d).
//   score   grid (row block, head, layer): the head's anchor in shared
//           memory, one thread per live row (16-byte vector loads of the row):
//           |k| and dot(k, anchor) as two sequential chains.  fp64 throughput
//           is ample on sm_100; the pass reads K once.
// The scores (fp64, cache row order) feed epk_select_pooled / epk_compact,
// which already reproduce evict_to_budget bit for bit.
#include <cuda_bf16.h>

#include "epk_internal.cuh"
#include "sm100.cuh"

namespace epk {

using namespace sm100;

namespace {

template <typename T>
__device__ __forceinline__ double kd_load(const T* p);
template <>
__device__ __forceinline__ double kd_load<float>(const float* p) { return double(__ldg(p)); }
template <>
__device__ __forceinline__ double kd_load<double>(const double* p) { return __ldg(p); }
template <>
__device__ __forceinline__ double kd_load<__nv_bfloat16>(const __nv_bfloat16* p) {
    return double(__bfloat162float(__ldg(p)));
}

struct KeyDiffParams {
    LayerTable lt;
    int H, d;
    int rowbytes;             // d * sizeof(T)
    int chunk_rows;           // anchor: rows per bulk-copied chunk
    const int32_t* head_off;  // [L][H+1]
    const int32_t* head_len;  // [L][H]
    const void* k;
    double* anchor;  // [L][H][d]
    double* norm;    // [L][H]
    double* scores;  // [rows]
};

constexpr int kKdThreads = 128;
constexpr int kKdStages = 4;
constexpr int kKdChunkBytes = 16384;

template <typename T>
__device__ __forceinline__ double kd_elem(const uint8_t* row, int j) {
    return kd_load<T>(reinterpret_cast<const T*>(row) + j);
}
template <typename T>
__device__ __forceinline__ double kd_smem(const uint8_t* row, int j) {
    const T x = reinterpret_cast<const T*>(row)[j];
    if constexpr (sizeof(T) == 2) return double(__bfloat162float(x));
    else return double(x);
}

// anchor: one CTA per (layer, head); the head's rows stream through a ring of
// kKdStages shared-memory chunks (1-D bulk copies, TMA engine), thread i keeps
// the sequential sums of dimensions i and i + 128.
template <typename T>
__global__ void __launch_bounds__(kKdThreads) keydiff_anchor_kernel(const __grid_constant__ KeyDiffParams P) {
    extern __shared__ __align__(128) uint8_t kd_smem_raw[];
    __shared__ uint64_t full[kKdStages];
    __shared__ double s_a[256];
    const int h = blockIdx.x, l = blockIdx.y, i = threadIdx.x;
    const int64_t r0 = P.lt.base[l] + P.head_off[l * (P.H + 1) + h];
    const int n = P.head_len[l * P.H + h];
    const int R = P.chunk_rows;
    const int nchunks = (n + R - 1) / R;
    const uint8_t* src = static_cast<const uint8_t*>(P.k) + r0 * P.rowbytes;
    const int chunk_bytes = R * P.rowbytes;
    if (i == 0) {
        for (int s = 0; s < kKdStages; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int c) {
        const int s = c % kKdStages;
        const uint32_t bytes = uint32_t(min(R, n - c * R)) * uint32_t(P.rowbytes);
        mbar_expect_tx(&full[s], bytes);
        bulk_load_1d(kd_smem_raw + s * chunk_bytes, src + int64_t(c) * chunk_bytes, bytes, &full[s]);
    };
    if (i == 0)
        for (int c = 0; c < min(kKdStages, nchunks); ++c) issue(c);
    double acc0 = 0.0, acc1 = 0.0;
    const bool two = i + kKdThreads < P.d;
    for (int c = 0; c < nchunks; ++c) {
        const int s = c % kKdStages;
        mbar_wait(&full[s], (c / kKdStages) & 1);
        const int rows = min(R, n - c * R);
        const uint8_t* base = kd_smem_raw + s * chunk_bytes;
        if (i < P.d) {
            if (two) {
                for (int rr = 0; rr < rows; ++rr) {
                    acc0 = __dadd_rn(acc0, kd_smem<T>(base + rr * P.rowbytes, i));
                    acc1 = __dadd_rn(acc1, kd_smem<T>(base + rr * P.rowbytes, i + kKdThreads));
                }
            } else {
#pragma unroll 8
                for (int rr = 0; rr < rows; ++rr) acc0 = __dadd_rn(acc0, kd_smem<T>(base + rr * P.rowbytes, i));
            }
        }
        __syncthreads();  // stage s drained by every thread
        if (i == 0 && c + kKdStages < nchunks) issue(c + kKdStages);
    }
    double* a = P.anchor + (int64_t(l) * P.H + h) * P.d;
    if (i < P.d) {
        const double m = n > 0 ? __ddiv_rn(acc0, double(n)) : 0.0;
        a[i] = m;
        s_a[i] = m;
    }
    if (two) {
        const double m = n > 0 ? __ddiv_rn(acc1, double(n)) : 0.0;
        a[i + kKdThreads] = m;
        s_a[i + kKdThreads] = m;
    }
    __syncthreads();
    if (i == 0) {
        double nb = 0.0;
        for (int j = 0; j < P.d; ++j) nb = __dadd_rn(nb, __dmul_rn(s_a[j], s_a[j]));
        P.norm[int64_t(l) * P.H + h] = __dsqrt_rn(nb);
    }
}

// anchor, rows whose size is not a multiple of 16 bytes: plain loads.
template <typename T>
__global__ void __launch_bounds__(256) keydiff_anchor_small_kernel(const __grid_constant__ KeyDiffParams P) {
    const int h = blockIdx.x, l = blockIdx.y, i = threadIdx.x;
    const int64_t r0 = P.lt.base[l] + P.head_off[l * (P.H + 1) + h];
    const int n = P.head_len[l * P.H + h];
    __shared__ double s_a[256];
    if (i < P.d) {
        const T* k = static_cast<const T*>(P.k) + r0 * P.d + i;
        double acc = 0.0;
        for (int r = 0; r < n; ++r) acc = __dadd_rn(acc, kd_load<T>(k + int64_t(r) * P.d));
        const double m = n > 0 ? __ddiv_rn(acc, double(n)) : 0.0;
        P.anchor[(int64_t(l) * P.H + h) * P.d + i] = m;
        s_a[i] = m;
    }
    __syncthreads();
    if (i == 0) {
        double nb = 0.0;
        for (int j = 0; j < P.d; ++j) nb = __dadd_rn(nb, __dmul_rn(s_a[j], s_a[j]));
        P.norm[int64_t(l) * P.H + h] = __dsqrt_rn(nb);
    }
}

// score: grid (row blocks, head, layer); the head's anchor in shared memory,
// one thread per live row: |k| and dot(k, anchor) as two sequential chains.
template <typename T>
__global__ void __launch_bounds__(kKdThreads) keydiff_score_kernel(const __grid_constant__ KeyDiffParams P) {
    __shared__ double s_a[256];
    const int h = blockIdx.y, l = blockIdx.z;
    const int n = P.head_len[l * P.H + h];
    if (int(blockIdx.x) * kKdThreads >= n) return;
    const double* a = P.anchor + (int64_t(l) * P.H + h) * P.d;
    for (int j = threadIdx.x; j < P.d; j += kKdThreads) s_a[j] = a[j];
    __syncthreads();
    const int r = blockIdx.x * kKdThreads + threadIdx.x;
    if (r >= n) return;
    const int64_t g = P.lt.base[l] + P.head_off[l * (P.H + 1) + h] + r;
    const uint8_t* row = static_cast<const uint8_t*>(P.k) + g * P.rowbytes;
    double na = 0.0, dot = 0.0;
    if (P.rowbytes % 16 == 0) {
        constexpr int V = 16 / sizeof(T);
        for (int j0 = 0; j0 < P.d; j0 += V) {
            const uint4 w = __ldg(reinterpret_cast<const uint4*>(row) + j0 / V);
            const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
            for (int u = 0; u < V; ++u) {
                double x;
                if constexpr (sizeof(T) == 2) x = double(__bfloat162float(e[u]));
                else x = double(e[u]);
                na = __dadd_rn(na, __dmul_rn(x, x));
                dot = __dadd_rn(dot, __dmul_rn(x, s_a[j0 + u]));
            }
        }
    } else {
        for (int j = 0; j < P.d; ++j) {
            const double x = kd_elem<T>(row, j);
            na = __dadd_rn(na, __dmul_rn(x, x));
            dot = __dadd_rn(dot, __dmul_rn(x, s_a[j]));
        }
    }
    na = __dsqrt_rn(na);
    const double nb = P.norm[int64_t(l) * P.H + h];
    double s = 0.0;
    if (nb != 0.0 && na != 0.0) {
        double c = __ddiv_rn(dot, __dmul_rn(na, nb));
        c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);  // std::clamp
        s = -c;
    }
    P.scores[g] = s;
}

}  // namespace

int launch_keydiff(epk_ctx* ctx, const epk_cache_desc* c, double* scores) {
    if (c->head_dim < 1 || c->head_dim > 256) return fail(EPK_ERR_UNSUPPORTED, "keydiff: head_dim must be 1..256");
    if (c->dtype != EPK_BF16 && c->dtype != EPK_F32 && c->dtype != EPK_F64)
        return fail(EPK_ERR_UNSUPPORTED, "keydiff: cache dtype F32, BF16 or F64");
    KeyDiffParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.H = c->kv_heads;
    P.d = c->head_dim;
    P.rowbytes = int(c->head_dim * dtype_size(c->dtype));
    P.chunk_rows = std::max(1, kKdChunkBytes / P.rowbytes);
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.k = c->k;
    P.scores = scores;
    const int64_t na = int64_t(c->layers) * P.H * P.d, nn = int64_t(c->layers) * P.H;
    rc = ws_require(ctx, (na + nn) * 8 + 1024);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.anchor = carve.take<double>(na);
    P.norm = carve.take<double>(nn);
    int64_t max_len = 1;
    for (int l = 0; l < c->layers; ++l) max_len = std::max<int64_t>(max_len, P.lt.base[l + 1] - P.lt.base[l]);
    const dim3 ga(P.H, c->layers), gs(unsigned((max_len + kKdThreads - 1) / kKdThreads), P.H, c->layers);
    const bool bulk = P.rowbytes % 16 == 0 && (reinterpret_cast<uintptr_t>(c->k) & 15) == 0;
    const int smem = kKdStages * P.chunk_rows * P.rowbytes;
    EPK_PROF(ctx, "keydiff_anchor");
    auto anchor = [&](auto tag) {
        using T = decltype(tag);
        if (bulk) {
            EPK_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(keydiff_anchor_kernel<T>),
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
            keydiff_anchor_kernel<T><<<ga, kKdThreads, smem, ctx->stream>>>(P);
        } else {
            keydiff_anchor_small_kernel<T><<<ga, (P.d + 31) / 32 * 32, 0, ctx->stream>>>(P);
        }
        return EPK_OK;
    };
    if (c->dtype == EPK_BF16) rc = anchor(__nv_bfloat16());
    else if (c->dtype == EPK_F32) rc = anchor(float());
    else rc = anchor(double());
    if (rc) return rc;
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "keydiff_score");
    if (c->dtype == EPK_BF16)
        keydiff_score_kernel<__nv_bfloat16><<<gs, kKdThreads, 0, ctx->stream>>>(P);
    else if (c->dtype == EPK_F32)
        keydiff_score_kernel<float><<<gs, kKdThreads, 0, ctx->stream>>>(P);
    else
        keydiff_score_kernel<double><<<gs, kKdThreads, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
