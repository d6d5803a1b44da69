// toy_forward.cu -- the model step BEFORE the hot path: the
// reference's seeded GQA transformer forward (toymodel.hpp:228-411) on the
// GPU in fp64, so a block_prefill caller no longer runs the prompt pass's
// attention loop (toymodel.hpp:327-391) -- the bulk of the reference's block
// loop time -- on the host.
//
// Every value follows the reference's operation order, without FMA:
//   embed      hidden[t] = token_embedding[tok] + position_embedding(pos)
//              (the position rows come from the caller: Model::position_embedding);
//   layernorm  sequential mean, sequential variance, 1/sqrt(var + 1e-5)   (:196-214)
//   matmul     C[i][j] = sum_k A[i][k] B[k][j], k in order from 0.0      (:173-190)
//   attention  per (query head, row t): logits over the head's cache rows
//              then the new rows 0..t (sequential-d dot, * d^-1/2, masked
//              -inf), running max, e = exp(l - max), sequential denominator,
//              w = e / den; out[d] += w v[j][d] over j in order, skipping
//              w == 0                                                    (:327-391)
//   residual / ReLU MLP                                                  (:393-408)
// The softmax row (max, exp, denominator, weights) runs either on the host
// with std::exp -- the reference's own code, so every output is bit-identical
// -- or on the device (CUDA exp, <= 1 ulp from std::exp; the outputs then
// agree to ~1e-15 relative, not bitwise).  Everything else is on the device.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "epk_internal.cuh"

namespace epk {

// ---- kernels -------------------------------------------------------------------
__global__ void tf_embed_kernel(const double* __restrict__ emb, const int32_t* __restrict__ tok,
                                const double* __restrict__ pos_emb, int64_t n, int D, double* hidden) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n * D) return;
    const int64_t t = i / D, d = i % D;
    hidden[i] = __dadd_rn(emb[int64_t(tok[t]) * D + d], pos_emb[i]);
}

// one thread per row (toymodel.hpp:196-214)
__global__ void tf_layernorm_kernel(const double* __restrict__ in, double* __restrict__ out, int64_t n, int D) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double* x = in + t * D;
    double mean = 0.0;
    for (int i = 0; i < D; ++i) mean = __dadd_rn(mean, x[i]);
    mean = __ddiv_rn(mean, double(D));
    double var = 0.0;
    for (int i = 0; i < D; ++i) {
        const double dd = __dsub_rn(x[i], mean);
        var = __dadd_rn(var, __dmul_rn(dd, dd));
    }
    var = __ddiv_rn(var, double(D));
    const double inv = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, 1e-5)));
    for (int i = 0; i < D; ++i) out[t * D + i] = __dmul_rn(__dsub_rn(x[i], mean), inv);
}

// C (n x m) = A (n x k) B (k x m), each element a sequential k chain from 0.0
// (matmul_add into a zero matrix, toymodel.hpp:173-190).  relu: clamp x < 0 to 0.
__global__ void tf_matmul_kernel(const double* __restrict__ A, const double* __restrict__ B, double* __restrict__ C,
                                 int64_t n, int k, int m, int relu) {
    const int64_t i = int64_t(blockIdx.y);
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || j >= m) return;
    const double* a = A + i * k;
    double acc = 0.0;
    for (int q = 0; q < k; ++q) acc = __dadd_rn(acc, __dmul_rn(a[q], B[int64_t(q) * m + j]));
    if (relu && acc < 0.0) acc = 0.0;
    C[i * m + j] = acc;
}

__global__ void tf_add_kernel(double* __restrict__ x, const double* __restrict__ y, int64_t count) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) x[i] = __dadd_rn(x[i], y[i]);
}

struct TfAttn {
    int n, dh, Hkv, qh, h, group;
    int64_t cache_len;       // rows of this head in the past cache
    const double* q;         // [n][Hq*dh]
    int q_stride;
    const double* past_k;    // [cache_len][dh] (head-contiguous rows) or null
    const double* past_v;
    const int32_t* past_pos; // [cache_len]
    const double* new_k;     // [n][Hkv*dh]
    const double* new_v;
    const int64_t* pos;      // [n] new positions
    int mask_sinkrecent;
    int64_t sink, recent;
    double scale;
    double* logits;          // [n][ctx] (ctx = cache_len + n)
    double* out;             // attn_out [n][Hq*dh]
};

__device__ __forceinline__ bool tf_allows(const TfAttn& P, int64_t qpos, int64_t kpos) {
    if (kpos > qpos) return false;
    if (!P.mask_sinkrecent) return true;
    return kpos < P.sink || kpos + P.recent > qpos;
}

// logits[t][j] for j < visible_t = cache_len + t + 1: thread per (t, j)
__global__ void tf_logits_kernel(const __grid_constant__ TfAttn P) {
    const int t = blockIdx.y;
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t ctx = P.cache_len + P.n;
    if (t >= P.n || j >= ctx) return;
    if (j >= P.cache_len + t + 1) {  // a future new row: weight 0 in the grid (Matrix zero-init)
        P.logits[int64_t(t) * ctx + j] = 0.0;
        return;
    }
    const double* kv;
    int64_t kpos;
    if (j < P.cache_len) {
        kv = P.past_k + j * P.dh;
        kpos = P.past_pos[j];
    } else {
        kv = P.new_k + (j - P.cache_len) * int64_t(P.Hkv * P.dh) + P.h * P.dh;
        kpos = P.pos[j - P.cache_len];
    }
    double s = -__longlong_as_double(0x7ff0000000000000ll);
    if (tf_allows(P, P.pos[t], kpos)) {
        const double* qv = P.q + int64_t(t) * P.q_stride + P.qh * P.dh;
        double acc = 0.0;
        for (int d = 0; d < P.dh; ++d) acc = __dadd_rn(acc, __dmul_rn(qv[d], kv[d]));
        s = __dmul_rn(acc, P.scale);
    }
    P.logits[int64_t(t) * ctx + j] = s;
}

// device softmax row (one thread per row t; the sums are sequential)
__global__ void tf_softmax_kernel(const __grid_constant__ TfAttn P) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= P.n) return;
    const int64_t ctx = P.cache_len + P.n;
    const int64_t vis = P.cache_len + t + 1;
    double* l = P.logits + int64_t(t) * ctx;
    const double masked = -__longlong_as_double(0x7ff0000000000000ll);
    double m = masked;
    for (int64_t j = 0; j < vis; ++j)
        if (l[j] > m) m = l[j];
    double den = 0.0;
    for (int64_t j = 0; j < vis; ++j) {
        const double e = l[j] == masked ? 0.0 : exp(__dsub_rn(l[j], m));
        l[j] = e;
        den = __dadd_rn(den, e);
    }
    for (int64_t j = 0; j < vis; ++j) l[j] = __ddiv_rn(l[j], den);
}

// out[t][qh*dh + d] += w[t][j] v[j][d], j in order, w == 0 skipped: thread per (t, d)
__global__ void tf_attn_out_kernel(const __grid_constant__ TfAttn P) {
    const int t = blockIdx.x;
    const int d = threadIdx.x;
    if (t >= P.n || d >= P.dh) return;
    const int64_t ctx = P.cache_len + P.n;
    const int64_t vis = P.cache_len + t + 1;
    const double* w = P.logits + int64_t(t) * ctx;
    double acc = P.out[int64_t(t) * P.q_stride + P.qh * P.dh + d];
    for (int64_t j = 0; j < vis; ++j) {
        const double wgt = w[j];
        if (wgt != 0.0) {
            const double vv = j < P.cache_len ? P.past_v[j * P.dh + d]
                                              : P.new_v[(j - P.cache_len) * int64_t(P.Hkv * P.dh) + P.h * P.dh + d];
            acc = __dadd_rn(acc, __dmul_rn(wgt, vv));
        }
    }
    P.out[int64_t(t) * P.q_stride + P.qh * P.dh + d] = acc;
}

// ---- host --------------------------------------------------------------------------
static int tf_matmul(epk_ctx* ctx, const double* A, const double* B, double* C, int64_t n, int k, int m, int relu) {
    const dim3 grid(unsigned((m + 127) / 128), unsigned(n));
    EPK_PROF(ctx, "toy_matmul");
    tf_matmul_kernel<<<grid, 128, 0, ctx->stream>>>(A, B, C, n, k, m, relu);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

static int tf_layernorm(epk_ctx* ctx, const double* in, double* out, int64_t n, int D) {
    EPK_PROF(ctx, "toy_layernorm");
    tf_layernorm_kernel<<<unsigned((n + 127) / 128), 128, 0, ctx->stream>>>(in, out, n, D);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

static int tf_add(epk_ctx* ctx, double* x, const double* y, int64_t count) {
    EPK_PROF(ctx, "toy_add");
    tf_add_kernel<<<unsigned((count + 255) / 256), 256, 0, ctx->stream>>>(x, y, count);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// The reference's softmax row on the host (toymodel.hpp:348-385), rows split
// over host threads (each row is independent; its own order is the reference's).
static void host_softmax_rows(double* logits, int n, int64_t cache_len) {
    const int64_t ctx = cache_len + n;
    const double masked = -std::numeric_limits<double>::infinity();
    auto rows = [&](int a, int b) {
        for (int t = a; t < b; ++t) {
            double* l = logits + int64_t(t) * ctx;
            const int64_t vis = cache_len + t + 1;
            double m = masked;
            for (int64_t j = 0; j < vis; ++j)
                if (l[j] > m) m = l[j];
            double den = 0.0;
            for (int64_t j = 0; j < vis; ++j) {
                const double e = l[j] == masked ? 0.0 : std::exp(l[j] - m);
                l[j] = e;
                den += e;
            }
            for (int64_t j = 0; j < vis; ++j) l[j] = l[j] / den;
        }
    };
    const int nt = std::max(1, std::min<int>(n / 8, int(std::thread::hardware_concurrency())));
    if (nt <= 1) {
        rows(0, n);
        return;
    }
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i) th.emplace_back(rows, n * i / nt, n * (i + 1) / nt);
    for (auto& x : th) x.join();
}

}  // namespace epk

using namespace epk;

extern "C" int epk_toy_forward(epk_ctx* ctx, const epk_toy_model* m, const int32_t* tokens, const double* pos_emb,
                               const int64_t* positions, int64_t n, int32_t mask_kind, int64_t sink, int64_t recent,
                               const epk_cache_desc* past, double* k_out, double* v_out, double* attention,
                               const int64_t* attn_offsets, double* hidden_out, int32_t softmax_on_host) {
    if (!ctx || !m) return fail(EPK_ERR_ARG, "forward: null argument");
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(EPK_ERR_CUDA, "forward: cudaSetDevice");
    if (n < 1) return fail(EPK_ERR_ARG, "forward: empty token sequence");
    if (!tokens || !pos_emb || !positions || !k_out || !v_out || !m->token_embedding || !m->weights)
        return fail(EPK_ERR_ARG, "forward: null pointer");
    const int L = m->layers, Hq = m->query_heads, Hkv = m->kv_heads, dh = m->head_dim, D = m->model_dim;
    if (L < 1 || Hq < 1 || Hkv < 1 || dh < 1 || Hq % Hkv != 0 || D != Hq * dh)
        return fail(EPK_ERR_ARG, "forward: bad model shape");
    if (mask_kind != 0 && mask_kind != 1) return fail(EPK_ERR_ARG, "forward: bad mask kind");
    if (past && (past->dtype != EPK_F64 || past->layers != L || past->kv_heads != Hkv || past->head_dim != dh))
        return fail(EPK_ERR_DIM, "forward: cache layer count mismatch");
    const int KV = Hkv * dh, F = 2 * D;
    const int group = Hq / Hkv;
    // weights layout per layer: wq[D][D], wk[D][KV], wv[D][KV], wo[D][D], mlp_in[D][F], mlp_out[F][D]
    const int64_t per_layer = int64_t(D) * D * 2 + int64_t(D) * KV * 2 + int64_t(D) * F * 2;
    // past cache layout on the host (head offsets, lengths) for the attention launches
    std::vector<int32_t> p_off, p_len;
    if (past) {
        p_off.resize(size_t(L) * (Hkv + 1));
        p_len.resize(size_t(L) * Hkv);
        EPK_CUDA_CHECK(cudaMemcpyAsync(p_off.data(), past->head_off, p_off.size() * 4, cudaMemcpyDeviceToHost,
                                       ctx->stream));
        EPK_CUDA_CHECK(cudaMemcpyAsync(p_len.data(), past->head_len, p_len.size() * 4, cudaMemcpyDeviceToHost,
                                       ctx->stream));
        EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    }
    int64_t max_cache = 0;
    for (int32_t x : p_len) max_cache = std::max<int64_t>(max_cache, x);
    // scratch: hidden, normed, q, attn_out, proj, act, logits of one query head
    const int64_t logit_elems = n * (max_cache + n);
    const int64_t need = 8 * (n * D * 5 + n * F + logit_elems) + 8 * 256;
    int rc = ws_require(ctx, need);
    if (rc) return rc;
    WsCarver wc(ctx->ws);
    double* hidden = wc.take<double>(n * D);
    double* normed = wc.take<double>(n * D);
    double* q = wc.take<double>(n * D);
    double* attn = wc.take<double>(n * D);
    double* proj = wc.take<double>(n * D);
    double* act = wc.take<double>(n * F);
    double* logits = wc.take<double>(logit_elems);
    std::vector<double> host_logits(softmax_on_host ? size_t(logit_elems) : 0);
    EPK_PROF(ctx, "toy_embed");
    tf_embed_kernel<<<unsigned((n * D + 255) / 256), 256, 0, ctx->stream>>>(m->token_embedding, tokens, pos_emb, n, D,
                                                                           hidden);
    EPK_LAUNCH_CHECK(ctx);
    for (int l = 0; l < L; ++l) {
        const double* w = m->weights + l * per_layer;
        const double *wq = w, *wk = wq + int64_t(D) * D, *wv = wk + int64_t(D) * KV, *wo = wv + int64_t(D) * KV;
        const double *w_in = wo + int64_t(D) * D, *w_out = w_in + int64_t(D) * F;
        double* kl = k_out + int64_t(l) * n * KV;  // [n][Hkv*dh] of this layer
        double* vl = v_out + int64_t(l) * n * KV;
        if ((rc = tf_layernorm(ctx, hidden, normed, n, D)) || (rc = tf_matmul(ctx, normed, wq, q, n, D, D, 0)) ||
            (rc = tf_matmul(ctx, normed, wk, kl, n, D, KV, 0)) || (rc = tf_matmul(ctx, normed, wv, vl, n, D, KV, 0)))
            return rc;
        EPK_CUDA_CHECK(cudaMemsetAsync(attn, 0, size_t(n * D) * 8, ctx->stream));
        for (int qh = 0; qh < Hq; ++qh) {
            const int h = qh / group;
            TfAttn A;
            A.n = int(n);
            A.dh = dh;
            A.Hkv = Hkv;
            A.qh = qh;
            A.h = h;
            A.group = group;
            A.cache_len = past ? p_len[size_t(l) * Hkv + h] : 0;
            A.q = q;
            A.q_stride = D;
            const int64_t prow = past ? past->layer_base[l] + p_off[size_t(l) * (Hkv + 1) + h] : 0;
            A.past_k = past ? static_cast<const double*>(past->k) + prow * dh : nullptr;
            A.past_v = past ? static_cast<const double*>(past->v) + prow * dh : nullptr;
            A.past_pos = past ? past->pos + prow : nullptr;
            A.new_k = kl;
            A.new_v = vl;
            A.pos = positions;
            A.mask_sinkrecent = mask_kind;
            A.sink = sink;
            A.recent = recent;
            A.scale = 1.0 / std::sqrt(double(dh));
            A.logits = logits;
            A.out = attn;
            const int64_t ctx_total = A.cache_len + n;
            EPK_PROF(ctx, "toy_logits");
            tf_logits_kernel<<<dim3(unsigned((ctx_total + 127) / 128), unsigned(n)), 128, 0, ctx->stream>>>(A);
            EPK_LAUNCH_CHECK(ctx);
            if (softmax_on_host) {
                const size_t bytes = size_t(n * ctx_total) * 8;
                EPK_CUDA_CHECK(cudaMemcpyAsync(host_logits.data(), logits, bytes, cudaMemcpyDeviceToHost, ctx->stream));
                EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
                host_softmax_rows(host_logits.data(), int(n), A.cache_len);
                EPK_CUDA_CHECK(cudaMemcpyAsync(logits, host_logits.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
            } else {
                EPK_PROF(ctx, "toy_softmax");
                tf_softmax_kernel<<<unsigned((n + 63) / 64), 64, 0, ctx->stream>>>(A);
                EPK_LAUNCH_CHECK(ctx);
            }
            if (attention && attn_offsets) {  // the weight grid: visible columns, masked / future ones 0
                double* g = attention + attn_offsets[size_t(l) * Hq + qh];
                EPK_CUDA_CHECK(cudaMemcpyAsync(g, logits, size_t(n * ctx_total) * 8, cudaMemcpyDeviceToDevice,
                                               ctx->stream));
            }
            EPK_PROF(ctx, "toy_attn_out");
            tf_attn_out_kernel<<<unsigned(n), unsigned(std::max(32, (dh + 31) / 32 * 32)), 0, ctx->stream>>>(A);
            EPK_LAUNCH_CHECK(ctx);
        }
        if ((rc = tf_matmul(ctx, attn, wo, proj, n, D, D, 0)) || (rc = tf_add(ctx, hidden, proj, n * D)) ||
            (rc = tf_layernorm(ctx, hidden, normed, n, D)) || (rc = tf_matmul(ctx, normed, w_in, act, n, D, F, 1)) ||
            (rc = tf_matmul(ctx, act, w_out, proj, n, F, D, 0)) || (rc = tf_add(ctx, hidden, proj, n * D)))
            return rc;
    }
    if (hidden_out)
        EPK_CUDA_CHECK(cudaMemcpyAsync(hidden_out, hidden, size_t(n * D) * 8, cudaMemcpyDeviceToDevice, ctx->stream));
    return EPK_OK;
}
