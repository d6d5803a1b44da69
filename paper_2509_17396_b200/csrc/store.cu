// store.cu -- K7: the episodic cache store's writer:
// a device cache serialised into the reference's .epkv byte stream
// (persist, kvcache.hpp:281-317) on the GPU, so the D2H copy moves the
// finished file and the host only writes it out.
//
// Layout (little endian, no padding):
//   header  "EPKV" u16 version=1, u64 episode_id, u32 layers, u32 heads of
//           layer 0, u32 scorer length + bytes, u64 budget_per_head, u32 n +
//           n x u64 layer budgets                       (built on the host)
//   layer   u64 budget, u32 heads
//   head    u64 entry count
//   entry   u64 position, u32 dim, dim x f64 key, dim x f64 value
// Every field after the header sits at a multiple of 4 bytes from the header's
// end (12, 8, 12 + 16 dim), so the body is written with coalesced 32-bit
// stores into a buffer whose header ends 16-byte aligned (`pad` leading bytes
// that are not part of the file).  Keys and values are widened to fp64
// exactly (bf16 / fp32 -> fp64 is exact), i.e. bitwise the reference's reals.
#include <cuda_bf16.h>

#include <cstring>
#include <string>
#include <vector>

#include "epk_internal.cuh"

namespace epk {

namespace {

constexpr int kStoreEntriesPerCta = 64;

struct StoreParams {
    LayerTable lt;
    int H, d;
    const int32_t* head_off;   // [L][H+1]
    const int32_t* head_len;   // [L][H]
    const int32_t* pos;
    const void* k;
    const void* v;
    const int64_t* layer_word;  // [L] word offset of the layer record (from the body start)
    const int64_t* head_word;   // [L][H] word offset of the head's count field
    const uint64_t* budget;     // [L] per-layer budget field
    uint32_t* body;             // 16-byte aligned body start
};

template <typename T>
__device__ __forceinline__ double st_load(const T* p);
template <>
__device__ __forceinline__ double st_load<float>(const float* p) { return double(__ldg(p)); }
template <>
__device__ __forceinline__ double st_load<double>(const double* p) { return __ldg(p); }
template <>
__device__ __forceinline__ double st_load<__nv_bfloat16>(const __nv_bfloat16* p) {
    return double(__bfloat162float(__ldg(p)));
}

// grid (entry chunks, head, layer); each warp writes whole entries, lanes
// striding over the entry's 3 + 4 d words.
template <typename T>
__global__ void __launch_bounds__(256) epkv_write_kernel(const __grid_constant__ StoreParams P) {
    const int h = blockIdx.y, l = blockIdx.z;
    const int n = P.head_len[l * P.H + h];
    const int e0 = blockIdx.x * kStoreEntriesPerCta;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int64_t hw = P.head_word[l * P.H + h];
        P.body[hw] = uint32_t(uint64_t(n));
        P.body[hw + 1] = uint32_t(uint64_t(n) >> 32);
        if (h == 0) {
            const int64_t lw = P.layer_word[l];
            P.body[lw] = uint32_t(P.budget[l]);
            P.body[lw + 1] = uint32_t(P.budget[l] >> 32);
            P.body[lw + 2] = uint32_t(P.H);
        }
    }
    if (e0 >= n) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int words = 3 + 4 * P.d;
    const int64_t row0 = P.lt.base[l] + P.head_off[l * (P.H + 1) + h];
    const int64_t w_head = P.head_word[l * P.H + h] + 2;
    for (int e = e0 + warp; e < min(n, e0 + kStoreEntriesPerCta); e += 8) {
        const int64_t row = row0 + e;
        uint32_t* out = P.body + w_head + int64_t(e) * words;
        const uint64_t ps = uint64_t(uint32_t(P.pos[row]));
        const T* kr = static_cast<const T*>(P.k) + row * P.d;
        const T* vr = static_cast<const T*>(P.v) + row * P.d;
        for (int w = lane; w < words; w += 32) {
            uint32_t x;
            if (w < 2) {
                x = uint32_t(ps >> (32 * w));
            } else if (w == 2) {
                x = uint32_t(P.d);
            } else {
                const int q = w - 3;
                const int j = q >> 1;
                const double val = j < P.d ? st_load<T>(kr + j) : st_load<T>(vr + (j - P.d));
                const uint64_t b = uint64_t(__double_as_longlong(val));
                x = uint32_t(b >> (32 * (q & 1)));
            }
            out[w] = x;
        }
    }
}

void put_le(std::vector<uint8_t>& b, uint64_t v, int n) {
    for (int i = 0; i < n; ++i) b.push_back(uint8_t((v >> (8 * i)) & 0xFF));
}

}  // namespace

int launch_serialize_epkv(epk_ctx* ctx, const epk_cache_desc* c, uint64_t episode_id, const char* scorer,
                          uint64_t budget_per_head, const int64_t* layer_budgets, int32_t n_layer_budgets,
                          uint8_t* out, int64_t capacity, int64_t* offset_out, int64_t* total_out) {
    if (c->dtype != EPK_BF16 && c->dtype != EPK_F32 && c->dtype != EPK_F64)
        return fail(EPK_ERR_UNSUPPORTED, "persist: cache dtype F32, BF16 or F64");
    if (!layer_budgets && n_layer_budgets > 0) return fail(EPK_ERR_ARG, "persist: null layer budgets");
    if (!offset_out || !total_out) return fail(EPK_ERR_ARG, "persist: null size outputs");
    const int L = c->layers, H = c->kv_heads, d = c->head_dim;
    // header (kvcache.hpp:287-299)
    std::vector<uint8_t> hdr = {'E', 'P', 'K', 'V'};
    put_le(hdr, 1, 2);
    put_le(hdr, episode_id, 8);
    put_le(hdr, uint64_t(L), 4);
    put_le(hdr, uint64_t(H), 4);
    const size_t slen = scorer ? std::strlen(scorer) : 0;
    put_le(hdr, uint64_t(slen), 4);
    for (size_t i = 0; i < slen; ++i) hdr.push_back(uint8_t(scorer[i]));
    put_le(hdr, budget_per_head, 8);
    put_le(hdr, uint64_t(n_layer_budgets), 4);
    for (int i = 0; i < n_layer_budgets; ++i) put_le(hdr, uint64_t(layer_budgets[i]), 8);
    // entry counts -> word offsets of every layer / head record
    std::vector<int32_t> len(size_t(L) * H);
    EPK_CUDA_CHECK(cudaMemcpyAsync(len.data(), c->head_len, len.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    std::vector<int64_t> tab(size_t(L) + size_t(L) * H);
    std::vector<uint64_t> bud(static_cast<size_t>(L));
    const int64_t words = 3 + 4 * int64_t(d);
    int64_t w = 0;
    for (int l = 0; l < L; ++l) {
        tab[size_t(l)] = w;
        w += 3;
        for (int h = 0; h < H; ++h) {
            if (len[size_t(l) * H + h] < 0) return fail(EPK_ERR_ARG, "persist: negative head length");
            tab[size_t(L) + size_t(l) * H + h] = w;
            w += 2 + int64_t(len[size_t(l) * H + h]) * words;
        }
        bud[size_t(l)] = l < n_layer_budgets ? uint64_t(layer_budgets[l]) : budget_per_head;
    }
    const int64_t hb = int64_t(hdr.size());
    const int64_t pad = (16 - hb % 16) % 16;
    *offset_out = pad;
    *total_out = hb + 4 * w;
    if (!out) return EPK_OK;  // size query
    if (capacity < pad + *total_out) return fail(EPK_ERR_ARG, "persist: output buffer too small");
    if (reinterpret_cast<uintptr_t>(out) % 16) return fail(EPK_ERR_ARG, "persist: output buffer must be 16-byte aligned");
    StoreParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.H = H;
    P.d = d;
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.pos = c->pos;
    P.k = c->k;
    P.v = c->v;
    const int64_t tab_bytes = int64_t(tab.size()) * 8, bud_bytes = int64_t(bud.size()) * 8;
    rc = ws_require(ctx, tab_bytes + bud_bytes + 256);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    int64_t* d_tab = carve.take<int64_t>(int64_t(tab.size()));
    uint64_t* d_bud = carve.take<uint64_t>(int64_t(bud.size()));
    EPK_CUDA_CHECK(cudaMemcpyAsync(d_tab, tab.data(), tab_bytes, cudaMemcpyHostToDevice, ctx->stream));
    EPK_CUDA_CHECK(cudaMemcpyAsync(d_bud, bud.data(), bud_bytes, cudaMemcpyHostToDevice, ctx->stream));
    EPK_CUDA_CHECK(cudaMemcpyAsync(out + pad, hdr.data(), size_t(hb), cudaMemcpyHostToDevice, ctx->stream));
    P.layer_word = d_tab;
    P.head_word = d_tab + L;
    P.budget = d_bud;
    P.body = reinterpret_cast<uint32_t*>(out + pad + hb);
    int max_len = 1;
    for (int32_t x : len) max_len = std::max(max_len, x);
    const dim3 grid(unsigned((max_len + kStoreEntriesPerCta - 1) / kStoreEntriesPerCta), unsigned(H), unsigned(L));
    EPK_PROF(ctx, "epkv_write");
    if (c->dtype == EPK_BF16)
        epkv_write_kernel<__nv_bfloat16><<<grid, 256, 0, ctx->stream>>>(P);
    else if (c->dtype == EPK_F32)
        epkv_write_kernel<float><<<grid, 256, 0, ctx->stream>>>(P);
    else
        epkv_write_kernel<double><<<grid, 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    // the host vectors above must outlive the async copies
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    return EPK_OK;
}

}  // namespace epk
