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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "epk_internal.cuh"
#include "sm100.cuh"

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
// cosine / l2_norm / dot of numerics.hpp:52-87, -ffp-contract=off), as two
// kernels that run CONCURRENTLY (the chain kernel on the context's aux stream):
//   pair   a CTA of TR threads per tile of TR (h, t) pairs of one layer; the
//          tile's K_full / K_block rows are staged in shared memory with
//          coalesced cp.async copies (rows padded by 16 bytes, so the
//          per-thread 16-byte row reads are bank-conflict free), then each
//          thread runs |a|^2, |b|^2 and a.b as sequential chains over the
//          dimensions (explicit __dmul_rn / __dadd_rn, no FMA), correctly
//          rounded sqrt and division, clamp to [-1, 1]; a zero-norm pair is
//          stored as NaN (skipped).  Tiles go chunk-major over the layers and
//          each publishes a ready flag.
//   chain  one CTA per layer: warp 1 follows the ready flags, loads the
//          cosines in (h, t) order and compacts away the NaNs into a
//          shared-memory ring; lane 0 of warp 0 runs the reference's
//          sequential fp64 running sum from the ring (nothing but the
//          dependent adds on its critical path).  sigma = sum / counted
//          (1 when none count).
// pairs per tile (= threads per pair CTA): ~64 KB of staged rows at d = 128
template <typename T>
struct K5Shape;
template <>
struct K5Shape<double> {
    static constexpr int TR = 32;
};
template <>
struct K5Shape<float> {
    static constexpr int TR = 64;
};
template <>
struct K5Shape<__nv_bfloat16> {
    static constexpr int TR = 128;
};

struct K5Params {
    const void* kf;
    const void* kb;
    int64_t rows;        // (h, t) pairs per layer
    int64_t cos_stride;  // cosv layer stride (16-byte aligned)
    int dim, layers;
    int64_t tiles;       // tiles per layer
    double* cosv;
    unsigned* ready;     // [layers][tiles]
    double* sigma;
    int64_t* skipped_per_layer;
    int* err_flag;
};

template <typename T>
__device__ __forceinline__ void cos_accum(const uint4 w1, const uint4 w2, double& na, double& nb, double& dot) {
    const T* e1 = reinterpret_cast<const T*>(&w1);
    const T* e2 = reinterpret_cast<const T*>(&w2);
#pragma unroll
    for (int u = 0; u < int(16 / sizeof(T)); ++u) {
        const double x = to_d(e1[u]), y = to_d(e2[u]);
        na = __dadd_rn(na, __dmul_rn(x, x));
        nb = __dadd_rn(nb, __dmul_rn(y, y));
        dot = __dadd_rn(dot, __dmul_rn(x, y));
    }
}

__device__ __forceinline__ double finish_cosine(double na, double nb, double dot) {
    na = __dsqrt_rn(na);
    nb = __dsqrt_rn(nb);
    if (na == 0.0 || nb == 0.0) return __longlong_as_double(0x7ff8000000000000ll);  // skipped (zero norm)
    const double c = __ddiv_rn(dot, __dmul_rn(na, nb));
    return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}

// STAGED: rows staged through shared memory (row bytes a multiple of 16);
// else each thread reads its own row directly (any dim).
template <typename T, bool STAGED>
__global__ void __launch_bounds__(K5Shape<T>::TR) cosine_pair_kernel(const __grid_constant__ K5Params P) {
    constexpr int TR = K5Shape<T>::TR;
    extern __shared__ __align__(16) uint8_t k5_smem[];
    const int layer = int(blockIdx.x % P.layers);
    const int64_t tile = blockIdx.x / P.layers;  // chunk-major: every layer advances together
    const int64_t r0 = tile * TR;
    const int nrows = int(min(int64_t(TR), P.rows - r0));
    const int64_t g0 = int64_t(layer) * P.rows + r0;
    const T* kf = static_cast<const T*>(P.kf);
    const T* kb = static_cast<const T*>(P.kb);
    double na = 0.0, nb = 0.0, dot = 0.0;
    if (STAGED) {
        const int rowb = P.dim * int(sizeof(T));
        const int stride = rowb + 16;
        const int cpr = rowb / 16;
        uint8_t* sa = k5_smem;
        uint8_t* sb = k5_smem + TR * stride;
        const uint8_t* ga = reinterpret_cast<const uint8_t*>(kf + g0 * P.dim);
        const uint8_t* gb = reinterpret_cast<const uint8_t*>(kb + g0 * P.dim);
        const int nchunk = nrows * cpr;
        for (int q = threadIdx.x; q < nchunk; q += TR) {
            const int r = q / cpr, c = q % cpr;
            const uint32_t da = sm100::smem_u32(sa + r * stride + c * 16);
            const uint32_t db = sm100::smem_u32(sb + r * stride + c * 16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(da), "l"(ga + int64_t(q) * 16) : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(db), "l"(gb + int64_t(q) * 16) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        if (int(threadIdx.x) < nrows) {
            const uint4* ra = reinterpret_cast<const uint4*>(sa + threadIdx.x * stride);
            const uint4* rb = reinterpret_cast<const uint4*>(sb + threadIdx.x * stride);
            for (int j = 0; j < cpr; ++j) cos_accum<T>(ra[j], rb[j], na, nb, dot);
        }
    } else if (int(threadIdx.x) < nrows) {
        const T* a = kf + (g0 + threadIdx.x) * P.dim;
        const T* b = kb + (g0 + threadIdx.x) * P.dim;
        for (int i = 0; i < P.dim; ++i) {
            const double x = to_d(a[i]), y = to_d(b[i]);
            na = __dadd_rn(na, __dmul_rn(x, x));
            nb = __dadd_rn(nb, __dmul_rn(y, y));
            dot = __dadd_rn(dot, __dmul_rn(x, y));
        }
    }
    if (int(threadIdx.x) < nrows) P.cosv[int64_t(layer) * P.cos_stride + r0 + threadIdx.x] = finish_cosine(na, nb, dot);
    __threadfence();  // every writer's cosine is visible device-wide before the tile's flag
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(P.ready + int64_t(layer) * P.tiles + tile), "r"(1u)
                     : "memory");
    }
}

constexpr int kChainChunk = 1024;  // cosines per ring stage (8 KB)
constexpr int kChainStages = 4;

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// An L2 load the compiler may not hoist above the flag wait (__ldcg is not
// volatile and can move across it).
__device__ __forceinline__ double ld_cg_ordered(const double* p) {
    double v;
    asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
    return v;
}

__global__ void __launch_bounds__(64) cosine_chain_kernel(const __grid_constant__ K5Params P, int tr) {
    __shared__ __align__(128) double ring[kChainStages][kChainChunk];
    __shared__ int nvalid[kChainStages], nskip[kChainStages];
    __shared__ __align__(8) uint64_t full[kChainStages], empty[kChainStages];
    const int l = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const double* v = P.cosv + int64_t(l) * P.cos_stride;
    const unsigned* ready = P.ready + int64_t(l) * P.tiles;
    const int64_t nchunks = (P.rows + kChainChunk - 1) / kChainChunk;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kChainStages; ++s) {
            sm100::mbar_init(&full[s], 32);  // every loader lane releases its own ring stores
            sm100::mbar_init(&empty[s], 1);
        }
        sm100::fence_barrier_init();
    }
    __syncthreads();
    if (warp == 1) {  // loader: flags -> cosines -> NaN-free ring slot
        bool timed_out = false;
        for (int64_t c = 0; c < nchunks; ++c) {
            const int s = int(c % kChainStages);
            sm100::mbar_wait(&empty[s], (uint32_t(c / kChainStages) & 1u) ^ 1u);
            const int64_t i0 = c * kChainChunk;
            const int n = int(min(int64_t(kChainChunk), P.rows - i0));
            if (!timed_out) {  // every tile of this chunk published? lane j watches tile t0 + j (bounded wait)
                const int64_t t0 = i0 / tr, nt = (i0 + n - 1) / tr - t0 + 1;
                for (int64_t tb = 0; tb < nt; tb += 32) {
                    const bool mine = tb + lane < nt;
                    unsigned long long t_start = 0, t_now = 0;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
                    while (!__all_sync(0xffffffffu, !mine || ld_acquire_u32(ready + t0 + tb + lane) != 0u)) {
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_now));
                        if (t_now - t_start > 4000000000ull) {  // 4 s without progress: give up, flag the error
                            if (lane == 0) atomicCAS(P.err_flag, 0, EPK_ERR_CUDA);
                            timed_out = true;
                            break;
                        }
                        __nanosleep(32);
                    }
                    if (timed_out) break;
                }
            }
            __syncwarp();
            __threadfence();  // every lane ordered after the flags its neighbours acquired
            // all of the chunk's loads in flight at once (32 per lane), then
            // the order-preserving NaN compaction
            double xs[kChainChunk / 32];
#pragma unroll
            for (int u = 0; u < kChainChunk / 32; ++u) {
                const int i = u * 32 + lane;
                xs[u] = i < n ? ld_cg_ordered(v + i0 + i) : 0.0;
            }
            int base = 0, sk = 0;
#pragma unroll
            for (int u = 0; u < kChainChunk / 32; ++u) {
                const int i = u * 32 + lane;
                const bool ok = i < n && xs[u] == xs[u];
                const unsigned bal = __ballot_sync(0xffffffffu, ok);
                if (ok) ring[s][base + __popc(bal & ((1u << lane) - 1u))] = xs[u];
                base += __popc(bal);
                sk += __popc(__ballot_sync(0xffffffffu, i < n && !ok));
            }
            if (lane == 0) {
                nvalid[s] = base;
                nskip[s] = sk;
            }
            sm100::mbar_arrive(&full[s]);  // release: this lane's ring stores (and lane 0's counts) precede it
        }
        return;
    }
    if (lane != 0) return;
    double acc = 0.0;
    long long cnt = 0, sk = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const int s = int(c % kChainStages);
        sm100::mbar_wait(&full[s], uint32_t(c / kChainStages) & 1u);
        const int n = nvalid[s];
        const double* x = ring[s];
        int i = 0;
        if (n >= 8) {  // software-pipelined: the next 8 values load while the current 8 are added
            double2 b[4], nb[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) b[u] = reinterpret_cast<const double2*>(x)[u];
            for (; i + 16 <= n; i += 8) {
#pragma unroll
                for (int u = 0; u < 4; ++u) nb[u] = reinterpret_cast<const double2*>(x + i + 8)[u];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    acc = __dadd_rn(acc, b[u].x);
                    acc = __dadd_rn(acc, b[u].y);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) b[u] = nb[u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc = __dadd_rn(acc, b[u].x);
                acc = __dadd_rn(acc, b[u].y);
            }
            i += 8;
        }
        for (; i < n; ++i) acc = __dadd_rn(acc, x[i]);
        cnt += n;
        sk += nskip[s];
        sm100::mbar_arrive(&empty[s]);
    }
    P.sigma[l] = cnt > 0 ? __ddiv_rn(acc, double(cnt)) : 1.0;
    P.skipped_per_layer[l] = sk;
}

__global__ void cosine_skip_total_kernel(const int64_t* per_layer, int layers, int64_t* skipped) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        int64_t t = 0;
        for (int l = 0; l < layers; ++l) t += per_layer[l];
        if (skipped) *skipped = t;
    }
}

// With lazy module loading, the first launch of a kernel may wait for the
// kernels already running; the pair kernels must therefore be loaded before
// the chain kernel that spins on their flags starts.
static int k5_preload() {
    cudaFuncAttributes fa;
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<double, true>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<double, false>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<float, true>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<float, false>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<__nv_bfloat16, true>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_pair_kernel<__nv_bfloat16, false>));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_chain_kernel));
    EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, cosine_skip_total_kernel));
    return EPK_OK;
}

template <typename T>
static int k5_launch_pair(epk_ctx* ctx, const K5Params& P) {
    constexpr int TR = K5Shape<T>::TR;
    const int rowb = P.dim * int(sizeof(T));
    const size_t smem = size_t(2) * TR * (rowb + 16);
    const bool staged = rowb % 16 == 0 && smem <= 200 * 1024 && (reinterpret_cast<uintptr_t>(P.kf) & 15) == 0 &&
                        (reinterpret_cast<uintptr_t>(P.kb) & 15) == 0;
    const dim3 grid(unsigned(P.tiles * P.layers));
    EPK_PROF(ctx, "cosine_pair");
    if (staged) {
        EPK_CUDA_CHECK(cudaFuncSetAttribute(cosine_pair_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            int(smem)));
        cosine_pair_kernel<T, true><<<grid, TR, smem, ctx->stream>>>(P);
    } else {
        cosine_pair_kernel<T, false><<<grid, TR, 0, ctx->stream>>>(P);
    }
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

int launch_key_cosine(epk_ctx* ctx, const void* kf, const void* kb, int dtype, int layers, int H, int64_t ntok,
                      int dim, double* sigma, int64_t* skipped) {
    const int64_t rows = int64_t(H) * ntok;
    const int tr = dtype == EPK_F64 ? K5Shape<double>::TR : dtype == EPK_F32 ? K5Shape<float>::TR
                                                                             : K5Shape<__nv_bfloat16>::TR;
    const int64_t tiles = (rows + tr - 1) / tr;
    if (tiles * layers > int64_t(0x7fffffff)) return fail(EPK_ERR_UNSUPPORTED, "key_cosine: too many pairs");
    const int64_t stride = (rows + 1) & ~int64_t(1);  // 16-byte aligned layer rows
    int rc = ws_require(ctx, int64_t(layers) * stride * 8 + 16 + int64_t(layers) * 8 + tiles * layers * 4 + 2048);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    K5Params P;
    P.kf = kf;
    P.kb = kb;
    P.rows = rows;
    P.cos_stride = stride;
    P.dim = dim;
    P.layers = layers;
    P.tiles = tiles;
    P.cosv = carve.take<double>(int64_t(layers) * stride + 2);
    P.skipped_per_layer = carve.take<int64_t>(layers);
    P.ready = carve.take<unsigned>(tiles * layers);
    P.sigma = sigma;
    P.err_flag = ctx->err_flag;
    if ((rc = ensure_aux_stream(ctx)) || (rc = k5_preload())) return rc;
    cudaStream_t main = ctx->stream;
    EPK_CUDA_CHECK(cudaMemsetAsync(P.ready, 0, size_t(tiles * layers) * 4, main));
    // EPK_K5_SERIAL=1 (profilers that serialise kernels, e.g. ncu): pairs first,
    // then the chain on the same stream -- same results, no overlap
    static const bool serial = std::getenv("EPK_K5_SERIAL") != nullptr;
    if (serial) {
        if (dtype == EPK_F64) rc = k5_launch_pair<double>(ctx, P);
        else if (dtype == EPK_F32) rc = k5_launch_pair<float>(ctx, P);
        else rc = k5_launch_pair<__nv_bfloat16>(ctx, P);
        if (rc) return rc;
        EPK_PROF(ctx, "cosine_chain");
        cosine_chain_kernel<<<layers, 64, 0, main>>>(P, tr);
        EPK_LAUNCH_CHECK(ctx);
        EPK_PROF(ctx, "cosine_total");
        cosine_skip_total_kernel<<<1, 32, 0, main>>>(P.skipped_per_layer, layers, skipped);
        EPK_LAUNCH_CHECK(ctx);
        return EPK_OK;
    }
    // the chain CTAs follow the pair tiles' ready flags from the aux stream
    EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_aux_fork, main));
    EPK_CUDA_CHECK(cudaStreamWaitEvent(ctx->aux, ctx->ev_aux_fork, 0));
    ctx->stream = ctx->aux;
    EPK_PROF(ctx, "cosine_chain");
    cosine_chain_kernel<<<layers, 64, 0, ctx->aux>>>(P, tr);
    ctx->stream = main;
    {
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "cosine_chain launch");
        ctx->launches++;
        if (ctx->profiling && !ctx->prof.empty()) cudaEventRecord(ctx->prof.back().stop, ctx->aux);
    }
    if (dtype == EPK_F64) rc = k5_launch_pair<double>(ctx, P);
    else if (dtype == EPK_F32) rc = k5_launch_pair<float>(ctx, P);
    else rc = k5_launch_pair<__nv_bfloat16>(ctx, P);
    if (rc) return rc;
    EPK_CUDA_CHECK(cudaEventRecord(ctx->ev_aux_join, ctx->aux));
    EPK_CUDA_CHECK(cudaStreamWaitEvent(main, ctx->ev_aux_join, 0));
    EPK_PROF(ctx, "cosine_total");
    cosine_skip_total_kernel<<<1, 32, 0, ctx->stream>>>(P.skipped_per_layer, layers, skipped);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
