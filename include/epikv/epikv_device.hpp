// epikv_device.hpp -- the C++ host API of the THROUGHPUT path: one episode's
// cache resident in HBM (bf16 K/V, layered CSR, two ping-pong buffers) driven
// block by block through the C ABI (include/epk/epk.h):
//
//   append(k, v, positions, len)      append_to_cache        toymodel.hpp:428-443
//   evict(q_prompt, k_prompt, ...)    score_with_prompt ->    scoring.hpp:80-128
//                                     evict_to_budget         kvcache.hpp:142-201
//                                     (one fused step for all layers: the tcgen05
//                                     scorer K1, threshold select K2, gather K3)
//
// i.e. the per-block body of block_prefill (blockprefill.hpp:170-221) for a
// caller whose model forward already produced the block's K/V and the patched
// prompt's Q/K on the device.  Every call is asynchronous on the episode's
// stream; host views (retained_positions, entries_per_layer) synchronise and
// surface deferred device errors as epikv::gpu::DeviceError.
//
// Header-only, C++17, no dependency on the reference headers (epikv_gpu.hpp
// adds the conversion to the reference's EpisodicCache).  Link -lepk -lcudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "epk/epk.h"

namespace epikv {
namespace gpu {

/// A failed C-ABI call or a deferred device-side error (pin / capacity / NaN).
class DeviceError : public std::runtime_error {
  public:
    DeviceError(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
    int status() const { return status_; }

  private:
    int status_;
};

namespace device_detail {
inline void check(int rc, const char* call) {
    if (rc != EPK_OK) {
        const char* m = epk_last_error();
        throw DeviceError(rc, std::string(call) + ": " + (m && *m ? m : epk_status_string(rc)));
    }
}
inline void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(EPK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
}  // namespace device_detail

/// One episode cache on the device.  Layer l holds at most kv_heads *
/// budget[l] live entries after a step (pooled selection: per-head counts are
/// ragged), and every head keeps `block` free rows for the next append, so a
/// layer's capacity is kv_heads * (budget[l] + block) rows in each buffer.
class DeviceEpisode {
  public:
    DeviceEpisode(std::size_t layers, std::size_t kv_heads, std::vector<std::int64_t> budgets, std::size_t block,
                  int device = 0, cudaStream_t stream = nullptr, std::size_t head_dim = 128)
        : L_(layers), H_(kv_heads), d_(head_dim), block_(block), budgets_(std::move(budgets)), device_(device) {
        if (L_ == 0 || H_ == 0 || block_ == 0) throw DeviceError(EPK_ERR_ARG, "DeviceEpisode: empty shape");
        if (budgets_.size() == 1) budgets_.resize(L_, budgets_[0]);
        if (budgets_.size() != L_) throw DeviceError(EPK_ERR_DIM, "DeviceEpisode: one budget per layer");
        base_.resize(L_ + 1, 0);
        for (std::size_t l = 0; l < L_; ++l) {
            if (budgets_[l] < 0) throw DeviceError(EPK_ERR_ARG, "DeviceEpisode: negative budget");
            base_[l + 1] = base_[l] + std::int64_t(H_) * (budgets_[l] + std::int64_t(block_));
        }
        device_detail::cuda(cudaSetDevice(device_), "cudaSetDevice");
        device_detail::check(epk_ctx_create(device_, stream, &ctx_), "epk_ctx_create");
        stream_ = stream;
        try {
            allocate();
        } catch (...) {
            release();  // a constructor that throws runs no destructor
            throw;
        }
    }

    DeviceEpisode(const DeviceEpisode&) = delete;
    DeviceEpisode& operator=(const DeviceEpisode&) = delete;

    ~DeviceEpisode() { release(); }

  private:
    void allocate() {
        const std::size_t rows = std::size_t(base_[L_]);
        for (Buf& b : buf_) {
            device_detail::cuda(cudaMalloc(&b.k, rows * d_ * 2), "cudaMalloc(k)");
            device_detail::cuda(cudaMalloc(&b.v, rows * d_ * 2), "cudaMalloc(v)");
            device_detail::cuda(cudaMalloc(&b.pos, rows * 4), "cudaMalloc(pos)");
            device_detail::cuda(cudaMalloc(&b.off, L_ * (H_ + 1) * 4), "cudaMalloc(head_off)");
            device_detail::cuda(cudaMalloc(&b.len, L_ * H_ * 4), "cudaMalloc(head_len)");
        }
        device_detail::cuda(cudaMalloc(&kept_, L_ * 4), "cudaMalloc(kept)");
        // empty episode: head h of layer l owns rows [h (M_l + block), (h + 1) (M_l + block))
        std::vector<std::int32_t> off(L_ * (H_ + 1)), len(L_ * H_, 0);
        for (std::size_t l = 0; l < L_; ++l)
            for (std::size_t h = 0; h <= H_; ++h) off[l * (H_ + 1) + h] = std::int32_t(h * (budgets_[l] + block_));
        device_detail::cuda(cudaMemcpy(buf_[0].off, off.data(), off.size() * 4, cudaMemcpyHostToDevice), "H2D");
        device_detail::cuda(cudaMemcpy(buf_[0].len, len.data(), len.size() * 4, cudaMemcpyHostToDevice), "H2D");
    }

    void release() noexcept {
        if (!ctx_) return;
        cudaSetDevice(device_);
        epk_ctx_synchronize(ctx_);
        for (Buf& b : buf_) {
            cudaFree(b.k);  // cudaFree(nullptr) is a no-op
            cudaFree(b.v);
            cudaFree(b.pos);
            cudaFree(b.off);
            cudaFree(b.len);
            b = Buf{};
        }
        cudaFree(kept_);
        kept_ = nullptr;
        epk_ctx_destroy(ctx_);
        ctx_ = nullptr;
    }

  public:

    /// append_to_cache: k, v [dev] bf16 [layers][kv_heads][len][head_dim],
    /// positions [dev] int32 [len] (the block's token positions; the caller
    /// keeps them ascending and after every live position, as the reference's
    /// block loop does -- not re-checked on the device).  len <= block.
    void append(const void* k, const void* v, const std::int32_t* positions, std::size_t len) {
        const epk_cache_desc c = desc();
        device_detail::check(epk_append(ctx_, &c, k, v, positions, std::int32_t(len), std::int32_t(block_)),
                             "epk_append");
    }

    /// One block step (score -> pooled select -> compact) into the other
    /// buffer, which becomes the live cache.  q_prompt [dev] bf16
    /// [layers][q_heads][prompt_len][head_dim], k_prompt [dev] bf16
    /// [layers][kv_heads][prompt_len][head_dim].  scores_ws [dev, optional]
    /// fp32 [capacity rows] receives the step's scores of the INPUT cache's
    /// live rows.
    void evict(const void* q_prompt, const void* k_prompt, std::size_t q_heads, std::size_t prompt_len,
               bool aggregation_max = true, float* scores_ws = nullptr) {
        const epk_cache_desc in = desc(), out = desc_of(cur_ ^ 1);
        std::int64_t nmax = 0;
        for (std::int64_t b : budgets_) nmax = std::max<std::int64_t>(nmax, std::int64_t(H_) * b + std::int64_t(block_));
        device_detail::check(epk_evict_step(ctx_, &in, &out, q_prompt, k_prompt, std::int32_t(q_heads),
                                            std::int32_t(prompt_len), budgets_.data(), nullptr, 0,
                                            aggregation_max ? EPK_AGG_MAX : EPK_AGG_AVG, EPK_SCORE_TC_BF16, nmax,
                                            std::int32_t(block_), scores_ws, kept_),
                             "epk_evict_step");
        cur_ ^= 1;
        ++steps_;
    }

    /// Waits for the stream and raises any deferred device-side error.
    void synchronize() const {
        device_detail::check(epk_ctx_synchronize(ctx_), "epk_ctx_synchronize");
        device_detail::check(epk_ctx_poll_error(ctx_), "device-side check");
    }

    /// retained_positions (kvcache.hpp:220-236): [layer][head] -> positions.
    std::vector<std::vector<std::vector<std::int64_t>>> retained_positions() const {
        synchronize();
        const Buf& b = buf_[cur_];
        std::vector<std::int32_t> off(L_ * (H_ + 1)), len(L_ * H_), pos(std::size_t(base_[L_]));
        device_detail::cuda(cudaMemcpy(off.data(), b.off, off.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        device_detail::cuda(cudaMemcpy(len.data(), b.len, len.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        device_detail::cuda(cudaMemcpy(pos.data(), b.pos, pos.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        std::vector<std::vector<std::vector<std::int64_t>>> out(L_, std::vector<std::vector<std::int64_t>>(H_));
        for (std::size_t l = 0; l < L_; ++l)
            for (std::size_t h = 0; h < H_; ++h) {
                const std::int64_t r0 = base_[l] + off[l * (H_ + 1) + h];
                out[l][h].assign(pos.begin() + r0, pos.begin() + r0 + len[l * H_ + h]);
            }
        return out;
    }

    /// Live entries per layer (entry_count of every LayerCache).
    std::vector<std::size_t> entries_per_layer() const {
        synchronize();
        std::vector<std::int32_t> len(L_ * H_);
        device_detail::cuda(cudaMemcpy(len.data(), buf_[cur_].len, len.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        std::vector<std::size_t> out(L_, 0);
        for (std::size_t l = 0; l < L_; ++l)
            for (std::size_t h = 0; h < H_; ++h) out[l] += std::size_t(len[l * H_ + h]);
        return out;
    }

    /// The live cache (device pointers; valid until the next evict).
    epk_cache_desc desc() const { return desc_of(cur_); }
    epk_ctx* context() const { return ctx_; }
    cudaStream_t stream() const { return stream_; }
    std::size_t layers() const { return L_; }
    std::size_t kv_heads() const { return H_; }
    std::size_t head_dim() const { return d_; }
    std::size_t block() const { return block_; }
    std::size_t steps() const { return steps_; }
    const std::vector<std::int64_t>& budgets() const { return budgets_; }
    const std::vector<std::int64_t>& layer_base() const { return base_; }

  private:
    struct Buf {
        void* k = nullptr;
        void* v = nullptr;
        std::int32_t* pos = nullptr;
        std::int32_t* off = nullptr;
        std::int32_t* len = nullptr;
    };

    epk_cache_desc desc_of(int i) const {
        const Buf& b = buf_[i];
        return epk_cache_desc{std::int32_t(L_), std::int32_t(H_), std::int32_t(d_), EPK_BF16, b.k, b.v,
                              b.pos,           b.off,           b.len,            base_.data()};
    }

    std::size_t L_, H_, d_, block_;
    std::vector<std::int64_t> budgets_, base_;
    int device_;
    cudaStream_t stream_ = nullptr;
    epk_ctx* ctx_ = nullptr;
    Buf buf_[2];
    std::int32_t* kept_ = nullptr;
    int cur_ = 0;
    std::size_t steps_ = 0;
};

}  // namespace gpu
}  // namespace epikv
