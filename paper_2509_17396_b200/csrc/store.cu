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

// ---------------------------------------------------------------------------
// K7': the store's reader (load_cache, kvcache.hpp:321-374, Phase B "KVs
// Retrieve") on the GPU: the host walks the header and the per-head counts
// (epk_epkv_scan), the file bytes go to the device in one copy, and a kernel
// narrows every entry into a device cache, checking that each value
// round-trips (fails closed like the reference's loader).
// ---------------------------------------------------------------------------
namespace {

struct LoadParams {
    LayerTable lt;
    int H, d;
    const int32_t* head_off;     // [L][H+1] of the output cache
    const int32_t* head_len;     // [L][H]
    const int64_t* head_word;    // [L][H] word offset of the head's first entry (from the file start + pad)
    const uint32_t* words;       // the file, 4-byte aligned body
    void* k;
    void* v;
    int32_t* pos;
    int* err_flag;
};

template <typename T>
__device__ __forceinline__ T ld_narrow(double x, bool& exact);
template <>
__device__ __forceinline__ float ld_narrow<float>(double x, bool& exact) {
    const float f = __double2float_rn(x);
    exact = double(f) == x || (x != x);
    return f;
}
template <>
__device__ __forceinline__ double ld_narrow<double>(double x, bool& exact) {
    exact = true;
    return x;
}
template <>
__device__ __forceinline__ __nv_bfloat16 ld_narrow<__nv_bfloat16>(double x, bool& exact) {
    const __nv_bfloat16 b = __double2bfloat16(x);
    exact = double(__bfloat162float(b)) == x || (x != x);
    return b;
}

template <typename T>
__global__ void __launch_bounds__(256) epkv_read_kernel(const __grid_constant__ LoadParams P) {
    const int h = blockIdx.y, l = blockIdx.z;
    const int n = P.head_len[l * P.H + h];
    const int e0 = blockIdx.x * kStoreEntriesPerCta;
    if (e0 >= n) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t words = 3 + 4 * int64_t(P.d);
    const int64_t row0 = P.lt.base[l] + P.head_off[l * (P.H + 1) + h];
    const uint32_t* first = P.words + P.head_word[l * P.H + h];
    bool ok = true;
    for (int e = e0 + warp; e < min(n, e0 + kStoreEntriesPerCta); e += 8) {
        const uint32_t* in = first + int64_t(e) * words;
        const int64_t row = row0 + e;
        if (lane == 0) {
            const uint64_t ps = uint64_t(in[0]) | (uint64_t(in[1]) << 32);
            if (in[2] != uint32_t(P.d) || ps > 0x7fffffffull) ok = false;
            P.pos[row] = int32_t(ps);
        }
        for (int j = lane; j < 2 * P.d; j += 32) {
            const uint64_t b = uint64_t(in[3 + 2 * j]) | (uint64_t(in[4 + 2 * j]) << 32);
            bool ex;
            const T x = ld_narrow<T>(__longlong_as_double(static_cast<long long>(b)), ex);
            ok = ok && ex;
            if (j < P.d) static_cast<T*>(P.k)[row * P.d + j] = x;
            else static_cast<T*>(P.v)[row * P.d + (j - P.d)] = x;
        }
    }
    if (!ok) atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
}

int64_t rd_le(const uint8_t* b, int64_t at, int n) {
    uint64_t v = 0;
    for (int i = 0; i < n; ++i) v |= uint64_t(b[at + i]) << (8 * i);
    return int64_t(v);
}

}  // namespace

// Host walk of the file structure: info = {layers, heads, dim, header bytes};
// counts [L*H] and entry_off [L*H] (byte offset of each head's first entry).
int scan_epkv(const uint8_t* b, int64_t n, int64_t* info, int64_t* counts, int64_t* entry_off) {
    auto need = [&](int64_t at, int64_t len) { return at + len <= n; };
    if (!b || n < 34 || std::memcmp(b, "EPKV", 4) != 0) return fail(EPK_ERR_ARG, "load: bad magic");
    if (rd_le(b, 4, 2) != 1) return fail(EPK_ERR_ARG, "load: version mismatch");
    int64_t at = 14;
    const int64_t L = rd_le(b, at, 4);
    at += 8;  // layers, heads of layer 0
    if (!need(at, 4)) return fail(EPK_ERR_ARG, "load: cache file truncated");
    const int64_t slen = rd_le(b, at, 4);
    at += 4 + slen + 8;
    if (!need(at, 4)) return fail(EPK_ERR_ARG, "load: cache file truncated");
    const int64_t nb = rd_le(b, at, 4);
    at += 4 + 8 * nb;
    const int64_t header = at;
    int64_t H = -1, dim = -1;
    std::vector<int64_t> cnt, off;
    for (int64_t l = 0; l < L; ++l) {
        if (!need(at, 12)) return fail(EPK_ERR_ARG, "load: cache file truncated");
        const int64_t heads = rd_le(b, at + 8, 4);
        at += 12;
        if (H < 0) H = heads;
        if (heads != H) return fail(EPK_ERR_UNSUPPORTED, "load: layers with different head counts");
        for (int64_t h = 0; h < heads; ++h) {
            if (!need(at, 8)) return fail(EPK_ERR_ARG, "load: cache file truncated");
            const int64_t c = rd_le(b, at, 8);
            at += 8;
            if (c > 0) {
                if (!need(at, 12)) return fail(EPK_ERR_ARG, "load: cache file truncated");
                const int64_t dd = rd_le(b, at + 8, 4);
                if (dim < 0) dim = dd;
                if (dd != dim) return fail(EPK_ERR_UNSUPPORTED, "load: ragged key dimensions");
            }
            cnt.push_back(c);
            off.push_back(at);
            const int64_t ebytes = 12 + 16 * std::max<int64_t>(dim, 0);
            if (c < 0 || !need(at, c * ebytes)) return fail(EPK_ERR_ARG, "load: cache file truncated");
            at += c * ebytes;
        }
    }
    info[0] = L;
    info[1] = std::max<int64_t>(H, 0);
    info[2] = std::max<int64_t>(dim, 1);
    info[3] = header;
    if (counts) std::copy(cnt.begin(), cnt.end(), counts);
    if (entry_off) std::copy(off.begin(), off.end(), entry_off);
    return EPK_OK;
}

int launch_load_epkv(epk_ctx* ctx, const uint8_t* dev_file, int64_t pad, const int64_t* entry_off,
                     const epk_cache_desc* c) {
    const int L = c->layers, H = c->kv_heads, d = c->head_dim;
    if ((reinterpret_cast<uintptr_t>(dev_file) + pad + entry_off[0]) % 4 != 0)
        return fail(EPK_ERR_ARG, "load: the device copy of the file must put its body on a 4-byte boundary");
    std::vector<int64_t> word(size_t(L) * H);
    for (size_t i = 0; i < word.size(); ++i) word[i] = (pad + entry_off[i]) / 4;
    std::vector<int32_t> len(size_t(L) * H);
    EPK_CUDA_CHECK(cudaMemcpyAsync(len.data(), c->head_len, len.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    int rc = ws_require(ctx, int64_t(word.size()) * 8 + 256);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    int64_t* d_word = carve.take<int64_t>(int64_t(word.size()));
    EPK_CUDA_CHECK(cudaMemcpyAsync(d_word, word.data(), word.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
    LoadParams P;
    if ((rc = make_layer_table(c, &P.lt))) return rc;
    P.H = H;
    P.d = d;
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.head_word = d_word;
    P.words = reinterpret_cast<const uint32_t*>(dev_file);
    P.k = c->k;
    P.v = c->v;
    P.pos = c->pos;
    P.err_flag = ctx->err_flag;
    int max_len = 1;
    for (int32_t x : len) max_len = std::max(max_len, x);
    const dim3 grid(unsigned((max_len + kStoreEntriesPerCta - 1) / kStoreEntriesPerCta), unsigned(H), unsigned(L));
    EPK_PROF(ctx, "epkv_read");
    if (c->dtype == EPK_BF16)
        epkv_read_kernel<__nv_bfloat16><<<grid, 256, 0, ctx->stream>>>(P);
    else if (c->dtype == EPK_F32)
        epkv_read_kernel<float><<<grid, 256, 0, ctx->stream>>>(P);
    else
        epkv_read_kernel<double><<<grid, 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
