// score_f32.cu -- K1': the fp32 PARITY scorer (CUDA cores, EPK-F32 v1).
//
// Computes, for every live cache row of every (layer, kv-head), the patched
// prompt score of score_with_prompt (scoring.hpp:80-128) over the attention
// weights of forward (toymodel.hpp:327-391), in fp32 with a fixed operation
// order that oracle/epk_oracle.cpp (score_layer_f32) mirrors bit for bit:
//   logit  = (sum_d q_d*k_d, sequential d, separate mul/add) * d^-1/2
//   m      = max over the visible columns (n_h cache rows + prompt rows 0..t)
//   e      = epk_expf(logit - m)           (Cody-Waite + degree-7 Horner)
//   Z      = pairwise tree over 64-column sequential chunk sums
//   w      = e / Z
//   score  = max_g max_t w   (Aggregation::Max)   or max_g (sum_t w) / p (Avg)
// Every arithmetic op is an explicit round-to-nearest intrinsic, so nvcc
// cannot contract them into FMAs.  This is the correctness path; the
// throughput path is score_tc.cu (tcgen05/TMEM).
//
// Launches per layer: logits (64x64 tiles) -> row stats (one CTA per prompt
// row) -> column scores.  Scratch: (Hq*p) x (n_max+p) floats per layer.
#include <algorithm>

#include "epk_internal.cuh"

namespace epk {

__device__ __forceinline__ float epk_expf_dev(float x) {
    if (x > 88.72283935546875f) return __int_as_float(0x7f800000);
    if (x < -103.97207641601562f) return 0.0f;
    const float t = __fmul_rn(x, 1.44269502162933349609375f);
    const float kf = rintf(t);
    float r = __fsub_rn(x, __fmul_rn(kf, 0.693145751953125f));
    r = __fsub_rn(r, __fmul_rn(kf, 1.428606765330187045037746429443359375e-06f));
    float pz = 1.98412701138295233249664306640625e-04f;
    pz = __fadd_rn(__fmul_rn(pz, r), 1.3888889225199818611145019531250e-03f);
    pz = __fadd_rn(__fmul_rn(pz, r), 8.3333337679505348205566406250000e-03f);
    pz = __fadd_rn(__fmul_rn(pz, r), 4.1666667908430099487304687500000e-02f);
    pz = __fadd_rn(__fmul_rn(pz, r), 1.6666667163372039794921875000000e-01f);
    pz = __fadd_rn(__fmul_rn(pz, r), 0.5f);
    pz = __fadd_rn(__fmul_rn(pz, r), 1.0f);
    pz = __fadd_rn(__fmul_rn(pz, r), 1.0f);
    const int ki = int(kf);
    if (ki > 127) return __fmul_rn(__fmul_rn(pz, __int_as_float((127 + 127) << 23)), 2.0f);
    if (ki >= -126) return __fmul_rn(pz, __int_as_float((ki + 127) << 23));
    return __fmul_rn(__fmul_rn(pz, __int_as_float((ki + 127 + 64) << 23)), __int_as_float((127 - 64) << 23));
}

__global__ void expf_probe_kernel(const float* x, float* y, int64_t n) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) y[i] = epk_expf_dev(x[i]);
}

struct F32Params {
    int H, G, p, d;
    int64_t n_max;       // scratch column stride = n_max + p
    int64_t layer_base;  // global row base of the layer
    const int32_t* off;  // layer head_off [H+1]
    const int32_t* len;  // layer head_len [H]
    const float* k;      // global cache K
    const float* q;      // layer q [Hq][p][d]
    const float* kp;     // layer kp [H][p][d]
    float* logits;       // [Hq*p][n_max+p]
    float* rz;           // [Hq*p] denominators
    float* scores;       // global
    int agg_max;
    float scale;
    int* err_flag;  // a head longer than n_max: EPK_ERR_ARG, the head is not scored
};

constexpr int kT = 64;    // tile rows/cols
constexpr int kDc = 32;   // d staged per smem pass

// logits[(qh*p + t)][j] for j < n_h + p (cache rows then prompt rows).
__global__ void __launch_bounds__(256) f32_logits_kernel(const __grid_constant__ F32Params P) {
    const int qh = blockIdx.z;
    const int h = qh / P.G;
    const int t0 = blockIdx.y * kT;
    const int64_t j0 = int64_t(blockIdx.x) * kT;
    const int n_h = P.len[h];
    if (n_h > P.n_max) {  // the scratch stride is n_max + p: refuse rather than overrun
        if (threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0) atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
        return;
    }
    const int64_t cols = int64_t(n_h) + P.p;
    if (j0 >= cols || t0 >= P.p) return;
    __shared__ float sq[kT][kDc + 1];
    __shared__ float sk[kT][kDc + 1];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.0f;
    const int64_t krow0 = P.layer_base + P.off[h];
    for (int dc = 0; dc < P.d; dc += kDc) {
        for (int i = threadIdx.x; i < kT * kDc; i += blockDim.x) {
            const int r = i / kDc, c = i % kDc;
            const int t = t0 + r;
            sq[r][c] = (t < P.p && dc + c < P.d) ? P.q[(int64_t(qh) * P.p + t) * P.d + dc + c] : 0.0f;
            const int64_t j = j0 + r;
            float kv = 0.0f;
            if (dc + c < P.d) {
                if (j < n_h) kv = P.k[(krow0 + j) * P.d + dc + c];
                else if (j < cols) kv = P.kp[(int64_t(h) * P.p + (j - n_h)) * P.d + dc + c];
            }
            sk[r][c] = kv;
        }
        __syncthreads();
        const int dmax = min(kDc, P.d - dc);
        for (int c = 0; c < dmax; ++c) {
            float qa[4], kb[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) qa[a] = sq[ty * 4 + a][c];
#pragma unroll
            for (int b = 0; b < 4; ++b) kb[b] = sk[tx * 4 + b][c];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) acc[a][b] = __fadd_rn(acc[a][b], __fmul_rn(qa[a], kb[b]));
        }
        __syncthreads();
    }
    const int64_t stride = P.n_max + P.p;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const int t = t0 + ty * 4 + a;
        if (t >= P.p) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int64_t j = j0 + tx * 4 + b;
            if (j < cols) P.logits[(int64_t(qh) * P.p + t) * stride + j] = __fmul_rn(acc[a][b], P.scale);
        }
    }
}

// One CTA per (qh, t) row: m, e (in place), Z by the chunked pairwise tree.
__global__ void __launch_bounds__(256) f32_rowstat_kernel(const __grid_constant__ F32Params P) {
    extern __shared__ float s_chunks[];  // 2 * nchunks
    const int row = blockIdx.x;
    const int qh = row / P.p, t = row % P.p;
    const int h = qh / P.G;
    if (P.len[h] > P.n_max) return;  // flagged by the logits kernel
    const int64_t visible = int64_t(P.len[h]) + t + 1;
    const int64_t stride = P.n_max + P.p;
    float* lg = P.logits + int64_t(row) * stride;
    __shared__ float s_red[8];
    float m = -__int_as_float(0x7f800000);
    for (int64_t j = threadIdx.x; j < visible; j += blockDim.x) m = fmaxf(m, lg[j]);
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = m;
    __syncthreads();
    m = s_red[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, s_red[w]);
    const int64_t nchunks = (visible + 63) / 64;
    float* a = s_chunks;
    float* b = s_chunks + nchunks;
    for (int64_t c = threadIdx.x; c < nchunks; c += blockDim.x) {
        float s = 0.0f;
        const int64_t end = min(visible, (c + 1) * 64);
        for (int64_t j = c * 64; j < end; ++j) {
            const float e = epk_expf_dev(__fsub_rn(lg[j], m));
            lg[j] = e;
            s = __fadd_rn(s, e);
        }
        a[c] = s;
    }
    __syncthreads();
    int64_t len = nchunks;
    while (len > 1) {
        const int64_t half = len / 2;
        for (int64_t i = threadIdx.x; i < half; i += blockDim.x) b[i] = __fadd_rn(a[2 * i], a[2 * i + 1]);
        if ((len & 1) && threadIdx.x == 0) b[half] = a[len - 1];
        __syncthreads();
        float* tmp = a;
        a = b;
        b = tmp;
        len = (len + 1) / 2;
        __syncthreads();
    }
    if (threadIdx.x == 0) P.rz[row] = a[0];
}

// One thread per cache column j of kv-head h (blockIdx.y).
__global__ void __launch_bounds__(256) f32_colscore_kernel(const __grid_constant__ F32Params P) {
    const int h = blockIdx.y;
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int n_h = P.len[h];
    if (j >= n_h || n_h > P.n_max) return;
    const int64_t stride = P.n_max + P.p;
    float best = -__int_as_float(0x7f800000);
    for (int g = 0; g < P.G; ++g) {
        const int qh = h * P.G + g;
        float acc = P.agg_max ? -__int_as_float(0x7f800000) : 0.0f;
        for (int t = 0; t < P.p; ++t) {
            const int row = qh * P.p + t;
            const float w = __fdiv_rn(P.logits[int64_t(row) * stride + j], P.rz[row]);
            if (P.agg_max) acc = fmaxf(acc, w);
            else acc = __fadd_rn(acc, w);
        }
        if (!P.agg_max) acc = __fdiv_rn(acc, float(P.p));
        best = fmaxf(best, acc);
    }
    if (best != best) atomicCAS(P.err_flag, 0, EPK_ERR_NAN);
    P.scores[P.layer_base + P.off[h] + j] = best;
}

int launch_score_f32(epk_ctx* ctx, const epk_cache_desc* c, const float* q, const float* kp, int hq,
                     int p, int agg_max, int64_t n_max, float* scores) {
    if (c->dtype != EPK_F32) return fail(EPK_ERR_ARG, "score(exact f32): cache dtype must be F32");
    const int H = c->kv_heads, d = c->head_dim;
    if (hq % H != 0) return fail(EPK_ERR_ARG, "score: q_heads must be divisible by kv_heads");
    if (n_max < 0) return fail(EPK_ERR_ARG, "score: n_max_per_head must be >= 0");
    const int64_t stride = n_max + p;
    const int64_t rows = int64_t(hq) * p;
    int rc = ws_require(ctx, rows * stride * 4 + rows * 4 + 4096);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    F32Params P;
    P.logits = carve.take<float>(rows * stride);
    P.rz = carve.take<float>(rows);
    P.H = H;
    P.G = hq / H;
    P.p = p;
    P.d = d;
    P.n_max = n_max;
    P.k = static_cast<const float*>(c->k);
    P.scores = scores;
    P.agg_max = agg_max;
    P.scale = float(1.0 / std::sqrt(double(d)));
    P.err_flag = ctx->err_flag;
    const int64_t nchunks = (stride + 63) / 64;
    const size_t rs_smem = size_t(2 * nchunks) * 4;
    if (rs_smem > 200 * 1024) return fail(EPK_ERR_UNSUPPORTED, "score(exact f32): context too long for one CTA row");
    if (rs_smem > 48 * 1024)
        EPK_CUDA_CHECK(cudaFuncSetAttribute(f32_rowstat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(rs_smem)));
    for (int l = 0; l < c->layers; ++l) {
        P.layer_base = c->layer_base[l];
        P.off = c->head_off + l * (H + 1);
        P.len = c->head_len + l * H;
        P.q = q + int64_t(l) * hq * p * d;
        P.kp = kp + int64_t(l) * H * p * d;
        dim3 g1(unsigned((stride + kT - 1) / kT), unsigned((p + kT - 1) / kT), unsigned(hq));
        EPK_PROF(ctx, "f32_logits");
        f32_logits_kernel<<<g1, 256, 0, ctx->stream>>>(P);
        EPK_LAUNCH_CHECK(ctx);
        EPK_PROF(ctx, "f32_rowstat");
        f32_rowstat_kernel<<<unsigned(rows), 256, rs_smem, ctx->stream>>>(P);
        EPK_LAUNCH_CHECK(ctx);
        dim3 g3(unsigned((std::max<int64_t>(n_max, 1) + 255) / 256), unsigned(H));
        EPK_PROF(ctx, "f32_colscore");
        f32_colscore_kernel<<<g3, 256, 0, ctx->stream>>>(P);
        EPK_LAUNCH_CHECK(ctx);
    }
    return EPK_OK;
}

int launch_expf_probe(epk_ctx* ctx, const float* x, float* y, int64_t n) {
    EPK_PROF(ctx, "expf_probe");
    expf_probe_kernel<<<unsigned((n + 255) / 256), 256, 0, ctx->stream>>>(x, y, n);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// ---------------------------------------------------------------------------
// score_with_prompt on explicit fp64 grids (one layer): thread per (h, j).
// Window Max/Avg in row order (scoring.hpp:104-116), then max over the
// group's query heads with first-emplace semantics (:117-123).
// ---------------------------------------------------------------------------
struct GridParams {
    int hq, H, p;
    int64_t off[65];
    int64_t grid_off[257];  // element offset of query head qh's grid
    const double* grids;
    double* scores;
    int agg_max;
};

__global__ void grid_score_kernel(const __grid_constant__ GridParams P) {
    const int h = blockIdx.y;
    const int64_t n_h = P.off[h + 1] - P.off[h];
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n_h) return;
    const int G = P.hq / P.H;
    const int64_t cols = n_h + P.p;
    double slot = 0.0;
    for (int g = 0; g < G; ++g) {
        const double* grid = P.grids + P.grid_off[h * G + g];
        double acc = P.agg_max ? -__longlong_as_double(0x7ff0000000000000ll) : 0.0;
        for (int t = 0; t < P.p; ++t) {
            const double w = grid[int64_t(t) * cols + j];
            if (P.agg_max) acc = (acc < w) ? w : acc;  // std::max(acc, w)
            else acc = __dadd_rn(acc, w);
        }
        if (!P.agg_max) acc = __ddiv_rn(acc, double(P.p));
        if (g == 0 || acc > slot) slot = acc;
    }
    P.scores[P.off[h] + j] = slot;
}

int launch_score_grids(epk_ctx* ctx, int hq, int H, int p, const int64_t* head_off,
                       const double* grids, int agg_max, double* scores) {
    if (H < 1 || H > 64 || hq < 1 || hq > 256 || hq % H != 0)
        return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
    if (p <= 0) return fail(EPK_ERR_EMPTY_PROMPT, "score_with_prompt: empty prompt");
    GridParams P;
    P.hq = hq;
    P.H = H;
    P.p = p;
    int64_t n_max = 0;
    for (int h = 0; h <= H; ++h) P.off[h] = head_off[h];
    const int G = hq / H;
    int64_t acc = 0;
    for (int qh = 0; qh < hq; ++qh) {
        const int h = qh / G;
        const int64_t n_h = head_off[h + 1] - head_off[h];
        n_max = std::max(n_max, n_h);
        P.grid_off[qh] = acc;
        acc += int64_t(p) * (n_h + p);
    }
    P.grids = grids;
    P.scores = scores;
    P.agg_max = agg_max;
    dim3 g(unsigned((std::max<int64_t>(n_max, 1) + 255) / 256), unsigned(H));
    EPK_PROF(ctx, "grid_score");
    grid_score_kernel<<<g, 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
