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
// K5 restates the reduction of measure_sensitivity (allocation.hpp:80-100):
// sigma_l = mean over (h, t) of clamp(cos(k_full, k_block)), zero-norm pairs
// skipped.  HBM-bound; one warp per key row, fixed-order block partials then
// a fixed-order per-layer reduction (deterministic, fp64).
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

constexpr int kCosThreads = 256;
constexpr int kCosRowsPerBlock = 64;

// partial[layer][blk] = (sum of cosines, counted, skipped) over a block of rows.
template <typename T>
__global__ void __launch_bounds__(kCosThreads) cosine_partial_kernel(const T* __restrict__ kf, const T* __restrict__ kb,
                                                                     int64_t rows_per_layer, int dim,
                                                                     int blocks_per_layer, double* psum,
                                                                     int64_t* pcnt, int64_t* pskip) {
    const int layer = blockIdx.y;
    const int blk = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ double s_cos[kCosRowsPerBlock];
    __shared__ int s_ok[kCosRowsPerBlock];
    const int64_t row0 = int64_t(blk) * kCosRowsPerBlock;
    for (int rr = warp; rr < kCosRowsPerBlock; rr += kCosThreads / 32) {
        const int64_t row = row0 + rr;
        double na = 0.0, nb = 0.0, dot = 0.0;
        if (row < rows_per_layer) {
            const T* a = kf + (int64_t(layer) * rows_per_layer + row) * dim;
            const T* b = kb + (int64_t(layer) * rows_per_layer + row) * dim;
            for (int i = lane; i < dim; i += 32) {
                const double x = to_d(a[i]), y = to_d(b[i]);
                na += x * x;
                nb += y * y;
                dot += x * y;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            na += __shfl_xor_sync(0xffffffffu, na, o);
            nb += __shfl_xor_sync(0xffffffffu, nb, o);
            dot += __shfl_xor_sync(0xffffffffu, dot, o);
        }
        if (lane == 0) {
            if (row >= rows_per_layer) {
                s_ok[rr] = -1;
                s_cos[rr] = 0.0;
            } else {
                const double sa = sqrt(na), sb = sqrt(nb);
                if (sa == 0.0 || sb == 0.0) {
                    s_ok[rr] = 0;
                    s_cos[rr] = 0.0;
                } else {
                    s_ok[rr] = 1;
                    s_cos[rr] = fmin(1.0, fmax(-1.0, dot / (sa * sb)));
                }
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        int64_t c = 0, sk = 0;
        for (int i = 0; i < kCosRowsPerBlock; ++i) {
            if (s_ok[i] == 1) {
                s += s_cos[i];
                ++c;
            } else if (s_ok[i] == 0) {
                ++sk;
            }
        }
        const int64_t o = int64_t(layer) * blocks_per_layer + blk;
        psum[o] = s;
        pcnt[o] = c;
        pskip[o] = sk;
    }
}

// One CTA per layer: fixed-order strided partial sums, then a fixed smem tree
// (deterministic run to run).  Skipped counts land in skipped_per_layer.
__global__ void __launch_bounds__(256) cosine_final_kernel(const double* psum, const int64_t* pcnt,
                                                           const int64_t* pskip, int blocks_per_layer,
                                                           double* sigma, int64_t* skipped_per_layer) {
    const int l = blockIdx.x;
    __shared__ double s_s[256];
    __shared__ long long s_c[256], s_k[256];
    double s = 0.0;
    long long c = 0, sk = 0;
    for (int b = threadIdx.x; b < blocks_per_layer; b += 256) {
        s += psum[int64_t(l) * blocks_per_layer + b];
        c += pcnt[int64_t(l) * blocks_per_layer + b];
        sk += pskip[int64_t(l) * blocks_per_layer + b];
    }
    s_s[threadIdx.x] = s;
    s_c[threadIdx.x] = c;
    s_k[threadIdx.x] = sk;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            s_s[threadIdx.x] += s_s[threadIdx.x + w];
            s_c[threadIdx.x] += s_c[threadIdx.x + w];
            s_k[threadIdx.x] += s_k[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        sigma[l] = s_c[0] > 0 ? s_s[0] / double(s_c[0]) : 1.0;
        skipped_per_layer[l] = s_k[0];
    }
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
    const int bpl = int((rows + kCosRowsPerBlock - 1) / kCosRowsPerBlock);
    const int64_t np = int64_t(layers) * bpl;
    int rc = ws_require(ctx, np * 24 + int64_t(layers) * 8 + 2048);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    double* psum = carve.take<double>(np);
    int64_t* pcnt = carve.take<int64_t>(np);
    int64_t* pskip = carve.take<int64_t>(np);
    int64_t* skl = carve.take<int64_t>(layers);
    dim3 g(bpl, layers);
    EPK_PROF(ctx, "cosine_partial");
    if (dtype == EPK_F64)
        cosine_partial_kernel<double><<<g, kCosThreads, 0, ctx->stream>>>(
            static_cast<const double*>(kf), static_cast<const double*>(kb), rows, dim, bpl, psum, pcnt, pskip);
    else if (dtype == EPK_F32)
        cosine_partial_kernel<float><<<g, kCosThreads, 0, ctx->stream>>>(
            static_cast<const float*>(kf), static_cast<const float*>(kb), rows, dim, bpl, psum, pcnt, pskip);
    else
        cosine_partial_kernel<__nv_bfloat16><<<g, kCosThreads, 0, ctx->stream>>>(
            static_cast<const __nv_bfloat16*>(kf), static_cast<const __nv_bfloat16*>(kb), rows, dim, bpl, psum,
            pcnt, pskip);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "cosine_final");
    cosine_final_kernel<<<layers, 256, 0, ctx->stream>>>(psum, pcnt, pskip, bpl, sigma, skl);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "cosine_total");
    cosine_skip_total_kernel<<<1, 32, 0, ctx->stream>>>(skl, layers, skipped);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
