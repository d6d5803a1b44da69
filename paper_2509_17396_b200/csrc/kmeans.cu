// kmeans.cu -- K4 (episode clustering) and K5 (layer sensitivity).
//
// K4 restates kmeans (clustering.hpp:148-260) in fp64, bit-exact: squared
// distances are sequential over dimensions with separate multiply and add
// (clustering.hpp:133-140), assignment ties go to the lower cluster (strict <,
// :200-205), centroid sums run over points in index order (:234-246).  Sums
// can be chained across shards (accumulate != 0) so a multi-GPU run that
// hands the running sums from rank r-1 to rank r reproduces the single-GPU
// bits.  The k-means++ seeding and the empty-cluster
// repair consume the reference RNG stream and stay on the host (epk_api.cu).
//
// K5 restates the reduction of measure_sensitivity (allocation.hpp:80-100), bit-exact:
// sigma_l = mean over (h, t) of clamp(cos(k_full, k_block)), zero-norm pairs
// skipped: per-pair cosines in the reference's operation order, then each
// layer's (h, t)-ordered running sum (see cosine_pair_kernel / cosine_mean_kernel).
#include <algorithm>

#include "epk_internal.cuh"

namespace epk {

// D[i][c] = sum_d (x_id - c_cd)^2, sequential d.
__global__ void km_dist_kernel(const double* __restrict__ pts, int64_t n, int64_t dim,
                               const double* __restrict__ cent, int64_t k, double* __restrict__ D) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= n * k) return;
    const int64_t i = idx / k, c = idx % k;
    const double* a = pts + i * dim;
    const double* b = cent + c * dim;
    double acc = 0.0;
    for (int64_t d = 0; d < dim; ++d) {
        const double t = __dsub_rn(a[d], b[d]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    D[idx] = acc;
}

__global__ void km_argmin_kernel(const double* __restrict__ D, int64_t n, int64_t k, int64_t* assign,
                                 double* best_d2) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int64_t best = 0;
    double bd = D[i * k];
    for (int64_t c = 1; c < k; ++c) {
        const double d = D[i * k + c];
        if (d < bd) {
            bd = d;
            best = c;
        }
    }
    assign[i] = best;
    if (best_d2) best_d2[i] = bd;
}

// One thread per (cluster, dim): points in index order.
__global__ void km_sums_kernel(const double* __restrict__ pts, int64_t n, int64_t dim,
                               const int64_t* __restrict__ assign, int64_t k, double* sums,
                               int accumulate) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * dim) return;
    const int64_t c = idx / dim, d = idx % dim;
    double acc = accumulate ? sums[idx] : 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (assign[i] == c) acc = __dadd_rn(acc, pts[i * dim + d]);
    sums[idx] = acc;
}

__global__ void km_counts_kernel(const int64_t* __restrict__ assign, int64_t n, int64_t k, int64_t* counts,
                                 int accumulate) {
    const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= k) return;
    int64_t cnt = accumulate ? counts[c] : 0;
    for (int64_t i = 0; i < n; ++i) cnt += assign[i] == c;
    counts[c] = cnt;
}

__global__ void km_finalize_kernel(const double* sums, const int64_t* counts, int64_t k, int64_t dim,
                                   double* cent) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= k * dim) return;
    cent[idx] = __ddiv_rn(sums[idx], double(counts[idx / dim]));
}

__global__ void km_sqdist_assigned_kernel(const double* __restrict__ pts, int64_t n, int64_t dim,
                                          const double* __restrict__ cent, const int64_t* __restrict__ assign,
                                          double* d2) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* a = pts + i * dim;
    const double* b = cent + assign[i] * dim;
    double acc = 0.0;
    for (int64_t d = 0; d < dim; ++d) {
        const double t = __dsub_rn(a[d], b[d]);
        acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
    d2[i] = acc;
}

int launch_km_dist(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const double* cent, int64_t k,
                   double* D) {
    const int64_t tot = n * k;
    EPK_PROF(ctx, "km_dist");
    km_dist_kernel<<<unsigned((tot + 127) / 128), 128, 0, ctx->stream>>>(pts, n, dim, cent, k, D);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

int launch_km_assign(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const double* cent, int64_t k,
                     int64_t* assign, double* best_d2) {
    int rc = ws_require(ctx, n * k * 8 + 256);
    if (rc) return rc;
    double* D = static_cast<double*>(ctx->ws);
    rc = launch_km_dist(ctx, pts, n, dim, cent, k, D);
    if (rc) return rc;
    EPK_PROF(ctx, "km_argmin");
    km_argmin_kernel<<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(D, n, k, assign, best_d2);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

int launch_km_sums(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const int64_t* assign, int64_t k,
                   double* sums, int64_t* counts, int accumulate) {
    EPK_PROF(ctx, "km_sums");
    km_sums_kernel<<<unsigned((k * dim + 127) / 128), 128, 0, ctx->stream>>>(pts, n, dim, assign, k, sums,
                                                                            accumulate);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "km_counts");
    km_counts_kernel<<<unsigned((k + 31) / 32), 32, 0, ctx->stream>>>(assign, n, k, counts, accumulate);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

int launch_km_finalize(epk_ctx* ctx, const double* sums, const int64_t* counts, int64_t k, int64_t dim,
                       double* cent) {
    EPK_PROF(ctx, "km_finalize");
    km_finalize_kernel<<<unsigned((k * dim + 255) / 256), 256, 0, ctx->stream>>>(sums, counts, k, dim, cent);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

int launch_km_sqdist(epk_ctx* ctx, const double* pts, int64_t n, int64_t dim, const double* cent,
                     const int64_t* assign, double* d2) {
    EPK_PROF(ctx, "km_sqdist");
    km_sqdist_assigned_kernel<<<unsigned((n + 127) / 128), 128, 0, ctx->stream>>>(pts, n, dim, cent, assign, d2);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// ---------------------------------------------------------------------------
// K5
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ double to_d(T x);
template <>
__device__ __forceinline__ double to_d<float>(float x) { return double(x); }
template <>
__device__ __forceinline__ double to_d<double>(double x) { return x; }
template <>
__device__ __forceinline__ double to_d<__nv_bfloat16>(__nv_bfloat16 x) { return double(__bfloat162float(x)); }

// K5, bit-exact with the reference's loop order (allocation.hpp:80-100 with
// cosine / l2_norm / dot of numerics.hpp:52-87, -ffp-contract=off):
//   pair  one thread per (layer, h, t): |a|^2, |b|^2 and a.b as sequential
//         chains over the dimensions (explicit __dmul_rn / __dadd_rn, no FMA),
//         correctly rounded sqrt and division, clamp to [-1, 1]; a zero-norm
//         pair is stored as NaN (skipped).
//   mean  one thread per layer: the (h, t)-ordered running sum of the pair
//         cosines -- the reference's sequential accumulation -- with a
//         64-deep rotating register prefetch so the dependent fp64 adds, not
//         the loads, set the pace; sigma = sum / counted (1 when none count).
template <typename T>
__device__ __forceinline__ void cos_vec(const T* p, int j, double (&x)[16 / sizeof(T)]) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + j);
    const T* e = reinterpret_cast<const T*>(&w);
#pragma unroll
    for (int u = 0; u < int(16 / sizeof(T)); ++u) x[u] = to_d(e[u]);
}

template <typename T>
__global__ void __launch_bounds__(256) cosine_pair_kernel(const T* __restrict__ kf, const T* __restrict__ kb,
                                                          int64_t rows_per_layer, int dim, double* cosv) {
    const int layer = blockIdx.y;
    const int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (row >= rows_per_layer) return;
    const int64_t g = int64_t(layer) * rows_per_layer + row;
    const T* a = kf + g * dim;
    const T* b = kb + g * dim;
    double na = 0.0, nb = 0.0, dot = 0.0;
    constexpr int V = 16 / sizeof(T);
    if ((dim * int(sizeof(T))) % 16 == 0) {
        for (int j = 0; j < dim / V; ++j) {
            double x[V], y[V];
            cos_vec<T>(a, j, x);
            cos_vec<T>(b, j, y);
#pragma unroll
            for (int u = 0; u < V; ++u) {
                na = __dadd_rn(na, __dmul_rn(x[u], x[u]));
                nb = __dadd_rn(nb, __dmul_rn(y[u], y[u]));
                dot = __dadd_rn(dot, __dmul_rn(x[u], y[u]));
            }
        }
    } else {
        for (int i = 0; i < dim; ++i) {
            const double x = to_d(a[i]), y = to_d(b[i]);
            na = __dadd_rn(na, __dmul_rn(x, x));
            nb = __dadd_rn(nb, __dmul_rn(y, y));
            dot = __dadd_rn(dot, __dmul_rn(x, y));
        }
    }
    na = __dsqrt_rn(na);
    nb = __dsqrt_rn(nb);
    double c;
    if (na == 0.0 || nb == 0.0) {
        c = __longlong_as_double(0x7ff8000000000000ll);  // skipped (zero norm)
    } else {
        c = __ddiv_rn(dot, __dmul_rn(na, nb));
        c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
    }
    cosv[g] = c;
}

__global__ void __launch_bounds__(32) cosine_mean_kernel(const double* __restrict__ cosv, int64_t rows,
                                                         double* sigma, int64_t* skipped_per_layer) {
    if (threadIdx.x != 0) return;
    const int l = blockIdx.x;
    const double* v = cosv + int64_t(l) * rows;
    constexpr int D = 64;
    double buf[D];
#pragma unroll
    for (int j = 0; j < D; ++j) buf[j] = j < rows ? __ldcg(v + j) : 0.0;
    double acc = 0.0;
    long long cnt = 0, sk = 0;
    for (int64_t b0 = 0; b0 < rows; b0 += D) {
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const int64_t i = b0 + j;
            if (i < rows) {
                const double x = buf[j];
                if (x == x) {
                    acc = __dadd_rn(acc, x);
                    ++cnt;
                } else {
                    ++sk;
                }
            }
            buf[j] = i + D < rows ? __ldcg(v + i + D) : 0.0;
        }
    }
    sigma[l] = cnt > 0 ? __ddiv_rn(acc, double(cnt)) : 1.0;
    skipped_per_layer[l] = sk;
}

__global__ void cosine_skip_total_kernel(const int64_t* per_layer, int layers, int64_t* skipped) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t t = 0;
        for (int l = 0; l < layers; ++l) t += per_layer[l];
        if (skipped) *skipped = t;
    }
}

int launch_key_cosine(epk_ctx* ctx, const void* kf, const void* kb, int dtype, int layers, int H, int64_t ntok,
                      int dim, double* sigma, int64_t* skipped) {
    const int64_t rows = int64_t(H) * ntok;
    int rc = ws_require(ctx, int64_t(layers) * rows * 8 + int64_t(layers) * 8 + 1024);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    double* cosv = carve.take<double>(int64_t(layers) * rows);
    int64_t* skl = carve.take<int64_t>(layers);
    const dim3 g(unsigned((rows + 255) / 256), layers);
    EPK_PROF(ctx, "cosine_pair");
    if (dtype == EPK_F64)
        cosine_pair_kernel<double><<<g, 256, 0, ctx->stream>>>(static_cast<const double*>(kf),
                                                               static_cast<const double*>(kb), rows, dim, cosv);
    else if (dtype == EPK_F32)
        cosine_pair_kernel<float><<<g, 256, 0, ctx->stream>>>(static_cast<const float*>(kf),
                                                              static_cast<const float*>(kb), rows, dim, cosv);
    else
        cosine_pair_kernel<__nv_bfloat16><<<g, 256, 0, ctx->stream>>>(
            static_cast<const __nv_bfloat16*>(kf), static_cast<const __nv_bfloat16*>(kb), rows, dim, cosv);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "cosine_mean");
    cosine_mean_kernel<<<layers, 32, 0, ctx->stream>>>(cosv, rows, sigma, skl);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "cosine_total");
    cosine_skip_total_kernel<<<1, 32, 0, ctx->stream>>>(skl, layers, skipped);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
