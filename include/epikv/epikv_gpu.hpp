// epikv_gpu.hpp -- the drop-in C++ boundary: the reference epikv hot-path API
// (/root/reference/proj/include/epikv) with the same signatures, argument
// meaning, results and exceptions, computed by the sm_100a kernels behind the
// C ABI (include/epk/epk.h, libepk.so).
//
// The reference is a header-only library of inline functions in namespace
// epikv, so the GPU versions live in namespace epikv::gpu over the reference's
// OWN types (LayerCache, LayerScores, ForwardTrace, TokenScoreMap, Model,
// BlockPrefillConfig, PrefillReport, KMeansResult, SensitivityProfile).  A call
// site switches by qualification:
//
//   epikv::evict_to_budget(c, s, pins)      ->  epikv::gpu::evict_to_budget(c, s, pins)
//   epikv::score_with_prompt(trace, agg)    ->  epikv::gpu::score_with_prompt(trace, agg)
//   epikv::kmeans(points, k, seed, iters)   ->  epikv::gpu::kmeans(points, k, seed, iters)
//   epikv::measure_sensitivity(m, t, b, s)  ->  epikv::gpu::measure_sensitivity(m, t, b, s)
//   epikv::block_prefill(m, ctx, cfg, e, p) ->  epikv::gpu::block_prefill(m, ctx, cfg, e, p)
//
// Replaced reference interfaces (file:line under proj/include/epikv):
//   evict_to_budget      kvcache.hpp:142      (K2 pooled select on fp64 keys; the kept
//                                              KVEntry objects keep their stable order)
//   score_with_prompt    scoring.hpp:80       (grid reduction kernel, fp64, bit-exact)
//   kmeans               clustering.hpp:148   (K4, fp64, bit-exact)
//   measure_sensitivity  allocation.hpp:55    (K5 reduction; the two model forwards
//                                              stay the reference's, on the host)
//   block_prefill        blockprefill.hpp:92  (the block loop: the toy-model
//                                              forward stays on the host, scoring
//                                              and eviction run on the GPU)
//   build                episodic.hpp:108     (Phase A over several GPUs: one host
//                                              thread + one epk_ctx per GPU, episodes
//                                              round-robin; k-means optionally over
//                                              embeddings sharded across the GPUs,
//                                              NCCL ordered chain -- epk_kmeans_sharded)
// allocate (allocation.hpp:120) is L host scalars and stays the reference's.
//
// Link: -L<repo>/paper_2509_17396_b200 -lepk -lcudart.  Needs the reference
// headers (and nlohmann/json) on the include path, as epikv itself does.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "epikv/allocation.hpp"
#include "epikv/blockprefill.hpp"
#include "epikv/clustering.hpp"
#include "epikv/episodic.hpp"
#include "epikv/kvcache.hpp"
#include "epikv/scoring.hpp"
#include "epikv/toymodel.hpp"
#include "epk/epk.h"
#include "epikv/epikv_device.hpp"

namespace epikv {
namespace gpu {

namespace detail {

// Maps a C-ABI status to the reference's exception types.
inline void check(int rc) {
    if (rc == EPK_OK) return;
    const std::string msg = epk_last_error();
    switch (rc) {
        case EPK_ERR_DIM: throw DimensionError(msg);
        case EPK_ERR_ZERO_NORM: throw ZeroNormError(msg);
        default: throw Error(msg);
    }
}

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// One context per thread (the C ABI is reentrant; contexts are not shared).
inline epk_ctx* ctx() {
    thread_local struct Holder {
        epk_ctx* c = nullptr;
        ~Holder() {
            if (c) epk_ctx_destroy(c);
        }
    } h;
    if (!h.c) {
        int dev = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        check(epk_ctx_create(dev, nullptr, &h.c));
    }
    return h.c;
}

// Device buffer (RAII).
template <typename T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DBuf(size_t count) : n(count) {
        cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
    }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void upload(const T* h, size_t count) {
        cuda_check(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    void download(T* h, size_t count) const {
        cuda_check(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
};

}  // namespace detail

/// evict_to_budget (kvcache.hpp:142) on the GPU: pooled selection over the
/// layer's heads by (score desc, position asc, head asc) with pins; the kept
/// entries keep their per-head order.  Same result and exceptions as the
/// reference.  (The host KVEntry payload never moves to the device; the
/// device-resident cache path is epk_evict_step / epk_compact.)
inline LayerCache evict_to_budget(const LayerCache& cache, const LayerScores& scores,
                                  const std::unordered_set<std::size_t>& pinned = {}) {
    const std::size_t H = cache.heads.size();
    if (scores.size() != H) throw DimensionError("evict_to_budget: score head count mismatch");
    const std::size_t limit = H * cache.budget;
    if (cache.entry_count() <= limit) return cache;
    // marshal: CSR rows, fp64 scores (pinned rows carry a dummy score)
    std::vector<int32_t> pos, off(H + 1, 0), len(H, 0);
    std::vector<double> sc;
    std::size_t dim = 0;
    for (std::size_t h = 0; h < H; ++h) {
        for (const KVEntry& e : cache.heads[h]) {
            if (e.position > 0x7fffffffu) throw Error("evict_to_budget: position exceeds the device int32 range");
            pos.push_back(int32_t(e.position));
            if (pinned.count(e.position)) {
                sc.push_back(0.0);
            } else {
                auto it = scores[h].find(e.position);
                if (it == scores[h].end())
                    throw DimensionError("evict_to_budget: missing score for head " + std::to_string(h) +
                                         " position " + std::to_string(e.position));
                sc.push_back(it->second);
            }
            dim = std::max(dim, e.key.size());
        }
        len[h] = int32_t(cache.heads[h].size());
        off[h + 1] = off[h] + len[h];
    }
    const std::size_t n = pos.size();
    // the selection only needs positions and scores; the compaction order is
    // the stable per-head order, so the kept entries are copied on the host
    // from the device's keep mask (the K/V payload never has to move).
    epk_ctx* c = detail::ctx();
    detail::DBuf<int32_t> d_pos(n), d_off(H + 1), d_len(H);
    detail::DBuf<double> d_sc(n), d_kv(2 * std::max<std::size_t>(n, 1));
    detail::DBuf<uint8_t> d_keep(n);
    d_pos.upload(pos.data(), n);
    d_off.upload(off.data(), H + 1);
    d_len.upload(len.data(), H);
    d_sc.upload(sc.data(), n);
    std::vector<int32_t> pins_sorted;
    for (std::size_t p : pinned)
        if (p <= 0x7fffffffu) pins_sorted.push_back(int32_t(p));
    std::sort(pins_sorted.begin(), pins_sorted.end());
    detail::DBuf<int32_t> d_pins(pins_sorted.size());
    if (!pins_sorted.empty()) d_pins.upload(pins_sorted.data(), pins_sorted.size());
    const int64_t base[2] = {0, int64_t(n)};
    epk_cache_desc desc{1, int32_t(H), 2, EPK_F64, d_kv.p, d_kv.p, d_pos.p, d_off.p, d_len.p, base};
    const int64_t budget = int64_t(cache.budget);
    detail::check(epk_select_pooled(c, &desc, d_sc.p, EPK_F64, &budget, pins_sorted.empty() ? nullptr : d_pins.p,
                                    int32_t(pins_sorted.size()), d_keep.p, nullptr, 1));
    std::vector<uint8_t> keep(n);
    d_keep.download(keep.data(), n);
    LayerCache out(H, cache.budget);
    std::size_t r = 0;
    for (std::size_t h = 0; h < H; ++h)
        for (const KVEntry& e : cache.heads[h])
            if (keep[r++]) out.heads[h].push_back(e);
    return out;
}

/// score_with_prompt (scoring.hpp:80) on the GPU: window Max/Avg over the
/// prompt rows, max over a kv-head's query heads, cache columns only.
inline TokenScoreMap score_with_prompt(const ForwardTrace& prompt_trace, Aggregation agg) {
    const std::size_t p = prompt_trace.positions.size();
    if (p == 0) throw Error("score_with_prompt: empty prompt");
    TokenScoreMap map;
    map.layers.resize(prompt_trace.layers.size());
    epk_ctx* c = detail::ctx();
    for (std::size_t l = 0; l < prompt_trace.layers.size(); ++l) {
        const LayerTrace& lt = prompt_trace.layers[l];
        const std::size_t H = lt.context_positions.size();
        if (H == 0 || lt.attention.empty() || lt.attention.size() % H != 0)
            throw DimensionError("score_with_prompt: attention grid shape mismatch");
        const std::size_t group = lt.attention.size() / H;
        std::vector<int64_t> off(H + 1, 0);
        for (std::size_t h = 0; h < H; ++h) {
            if (lt.context_positions[h].size() < p) throw DimensionError("score_with_prompt: attention grid shape mismatch");
            off[h + 1] = off[h] + int64_t(lt.context_positions[h].size() - p);
        }
        std::vector<double> grids;
        for (std::size_t qh = 0; qh < lt.attention.size(); ++qh) {
            const Matrix& g = lt.attention[qh];
            const std::size_t h = qh / group;
            if (g.rows != p || g.cols != lt.context_positions[h].size())
                throw DimensionError("score_with_prompt: attention grid shape mismatch");
            grids.insert(grids.end(), g.values.begin(), g.values.end());
        }
        const std::size_t nout = static_cast<std::size_t>(off[H]);
        detail::DBuf<double> d_grids(grids.size()), d_out(nout);
        d_grids.upload(grids.data(), grids.size());
        detail::check(epk_score_grids(c, int32_t(lt.attention.size()), int32_t(H), int32_t(p), off.data(), d_grids.p,
                                      agg == Aggregation::Max ? EPK_AGG_MAX : EPK_AGG_AVG, d_out.p));
        std::vector<double> out(nout);
        d_out.download(out.data(), out.size());
        map.layers[l].resize(H);
        for (std::size_t h = 0; h < H; ++h)
            for (int64_t j = 0; j < off[h + 1] - off[h]; ++j)
                map.layers[l][h].emplace(lt.context_positions[h][std::size_t(j)], out[std::size_t(off[h] + j)]);
    }
    return map;
}

/// keydiff_scores (scoring.hpp:186) on the GPU, bit-exact (fp64 keys,
/// sequential sums, no FMA): the KeyDiff baseline's scores for every layer.
inline TokenScoreMap keydiff_scores(const EpisodicCache& cache) {
    TokenScoreMap map;
    map.layers.resize(cache.layers.size());
    epk_ctx* c = detail::ctx();
    for (std::size_t l = 0; l < cache.layers.size(); ++l) {
        const LayerCache& layer = cache.layers[l];
        const std::size_t H = layer.heads.size();
        map.layers[l].resize(H);
        std::vector<int32_t> pos, off(H + 1, 0), len(H, 0);
        std::vector<double> keys;
        std::size_t dim = 0;
        for (const auto& head : layer.heads)
            for (const KVEntry& e : head) dim = std::max(dim, e.key.size());
        if (dim == 0) {
            for (std::size_t h = 0; h < H; ++h)
                for (const KVEntry& e : layer.heads[h]) map.layers[l][h].emplace(e.position, 0.0);
            continue;
        }
        for (std::size_t h = 0; h < H; ++h) {
            for (const KVEntry& e : layer.heads[h]) {
                if (e.key.size() != dim) throw DimensionError("keydiff_scores: key dimension mismatch");
                pos.push_back(int32_t(e.position & 0x7fffffff));
                keys.insert(keys.end(), e.key.begin(), e.key.end());
            }
            len[h] = int32_t(layer.heads[h].size());
            off[h + 1] = off[h] + len[h];
        }
        const std::size_t n = pos.size();
        if (n == 0) continue;
        detail::DBuf<int32_t> d_pos(n), d_off(H + 1), d_len(H);
        detail::DBuf<double> d_k(n * dim), d_out(n);
        d_pos.upload(pos.data(), n);
        d_off.upload(off.data(), H + 1);
        d_len.upload(len.data(), H);
        d_k.upload(keys.data(), keys.size());
        const int64_t base[2] = {0, int64_t(n)};
        epk_cache_desc desc{1, int32_t(H), int32_t(dim), EPK_F64, d_k.p, d_k.p, d_pos.p, d_off.p, d_len.p, base};
        detail::check(epk_score_keydiff(c, &desc, d_out.p));
        std::vector<double> out(n);
        d_out.download(out.data(), n);
        std::size_t r = 0;
        for (std::size_t h = 0; h < H; ++h)
            for (const KVEntry& e : layer.heads[h]) map.layers[l][h].emplace(e.position, out[r++]);
    }
    return map;
}

/// kmeans (clustering.hpp:148) on the GPU, bit-exact (fp64, same RNG stream).
inline KMeansResult kmeans(const std::vector<Vec>& points, std::size_t k, std::uint64_t seed,
                           std::size_t max_iters = 64) {
    if (k < 1) throw Error("kmeans: cluster count must be >= 1");
    if (points.size() < k)
        throw Error("kmeans: fewer points (" + std::to_string(points.size()) + ") than clusters (" +
                    std::to_string(k) + ")");
    const std::size_t n = points.size(), dim = points[0].size();
    std::vector<double> flat;
    flat.reserve(n * dim);
    for (const Vec& p : points) {
        if (p.size() != dim) throw DimensionError("kmeans: points differ in dimension");
        flat.insert(flat.end(), p.begin(), p.end());
    }
    detail::DBuf<double> d_pts(flat.size());
    d_pts.upload(flat.data(), flat.size());
    std::vector<int64_t> assign(n);
    std::vector<double> cent(k * dim), sse(std::max<std::size_t>(max_iters, 1));
    int64_t iters = 0;
    detail::check(epk_kmeans(detail::ctx(), d_pts.p, int64_t(n), int64_t(dim), int64_t(k), seed, int64_t(max_iters),
                             assign.data(), cent.data(), &iters, sse.data()));
    KMeansResult r;
    r.assignments.assign(assign.begin(), assign.end());
    r.centroids.resize(k);
    for (std::size_t c = 0; c < k; ++c) r.centroids[c].assign(cent.begin() + c * dim, cent.begin() + (c + 1) * dim);
    r.iterations = std::size_t(iters);
    r.sse_per_iteration.assign(sse.begin(), sse.begin() + iters);
    return r;
}

namespace detail {
// The GPU key-cosine reduction of measure_sensitivity (allocation.hpp:80-100)
// over the two calibration traces.
inline SensitivityProfile sensitivity_from_traces(const Model& model, const ForwardTrace& full,
                                                  const ForwardTrace& block, std::size_t n,
                                                  std::size_t calibration_budget, std::size_t sink,
                                                  std::string input_id) {
    const std::size_t L = model.config.layers, H = model.config.kv_heads, d = model.config.head_dim;
    std::vector<double> kf(L * H * n * d), kb(L * H * n * d);
    for (std::size_t l = 0; l < L; ++l)
        for (std::size_t h = 0; h < H; ++h) {
            std::memcpy(kf.data() + (l * H + h) * n * d, full.layers[l].keys[h].values.data(), n * d * sizeof(double));
            std::memcpy(kb.data() + (l * H + h) * n * d, block.layers[l].keys[h].values.data(), n * d * sizeof(double));
        }
    detail::DBuf<double> d_kf(kf.size()), d_kb(kb.size()), d_sigma(L);
    detail::DBuf<int64_t> d_skip(1);
    d_kf.upload(kf.data(), kf.size());
    d_kb.upload(kb.data(), kb.size());
    detail::check(epk_key_cosine_sigma(detail::ctx(), d_kf.p, d_kb.p, EPK_F64, int32_t(L), int32_t(H), int64_t(n),
                                       int32_t(d), d_sigma.p, d_skip.p));
    SensitivityProfile profile;
    profile.sigma.resize(L);
    d_sigma.download(profile.sigma.data(), L);
    int64_t skipped = 0;
    d_skip.download(&skipped, 1);
    for (double s : profile.sigma) profile.sensitivity.push_back(1.0 - s);
    profile.mask_sink = sink;
    profile.mask_recent = calibration_budget - sink;
    profile.input_id = std::move(input_id);
    profile.model_seed = model.config.seed;
    profile.skipped_zero_norm = std::size_t(skipped);
    return profile;
}
}  // namespace detail

/// measure_sensitivity (allocation.hpp:55): the two forwards (causal and
/// sink+recent) are the reference's model substrate on the host; the key
/// cosine reduction sigma_l runs on the GPU (fp64, deterministic order).
inline SensitivityProfile measure_sensitivity(const Model& model, std::span<const TokenId> calibration_tokens,
                                              std::size_t calibration_budget, std::size_t sink,
                                              std::string input_id = "") {
    const std::size_t n = calibration_tokens.size();
    if (n < 2) throw Error("measure_sensitivity: need at least 2 calibration tokens");
    if (calibration_budget < sink + 1) throw Error("measure_sensitivity: budget must be >= sink + 1");
    TraceOptions opts;
    opts.store_attention = false;
    const ForwardTrace full = epikv::forward(model, calibration_tokens, MaskSpec::causal(), nullptr, opts);
    const ForwardTrace block =
        epikv::forward(model, calibration_tokens, MaskSpec::sink_recent(sink, calibration_budget - sink), nullptr, opts);
    return detail::sensitivity_from_traces(model, full, block, n, calibration_budget, sink, std::move(input_id));
}

// ---- the model forward on the GPU ----------------------------
/// Where the attention rows' softmax (max, exp, denominator) runs in
/// gpu::forward: on the host with std::exp -- the reference's own code, every
/// output bit-identical -- or on the device (CUDA exp, <= 1 ulp from std::exp,
/// outputs within ~1e-15 relative).
enum class Softmax { host, device };

namespace detail {

/// A reference Model's weights in HBM (epk_toy_model layout), cached per
/// thread by object identity and config (init_model is deterministic in the
/// config; a model whose weights are edited in place needs a fresh object).
struct DeviceModel {
    const Model* src = nullptr;
    ModelConfig cfg;
    std::unique_ptr<DBuf<double>> emb, weights;
    epk_toy_model desc{};
};

inline const DeviceModel& device_model(const Model& m) {
    thread_local std::vector<std::unique_ptr<DeviceModel>> cache;
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    for (auto& d : cache)
        if (d->src == &m && d->cfg == m.config) return *d;
    const ModelConfig& c = m.config;
    auto d = std::make_unique<DeviceModel>();
    d->src = &m;
    d->cfg = c;
    d->emb = std::make_unique<DBuf<double>>(m.token_embedding.values.size());
    d->emb->upload(m.token_embedding.values.data(), m.token_embedding.values.size());
    std::vector<double> w;
    for (const LayerWeights& lw : m.layers)
        for (const Matrix* x : {&lw.wq, &lw.wk, &lw.wv, &lw.wo, &lw.mlp_in, &lw.mlp_out})
            w.insert(w.end(), x->values.begin(), x->values.end());
    d->weights = std::make_unique<DBuf<double>>(w.size());
    d->weights->upload(w.data(), w.size());
    d->desc = epk_toy_model{int32_t(c.layers), int32_t(c.query_heads), int32_t(c.kv_heads), int32_t(c.head_dim),
                            int32_t(c.model_dim), int64_t(c.vocab), d->emb->p, d->weights->p};
    if (cache.size() >= 4) cache.erase(cache.begin());
    cache.push_back(std::move(d));
    return *cache.back();
}

/// An EpisodicCache as an fp64 layered CSR in HBM (the past cache of forward).
struct DeviceCache {
    std::unique_ptr<DBuf<double>> k, v;
    std::unique_ptr<DBuf<int32_t>> pos, off, len;
    std::vector<int64_t> base;
    epk_cache_desc desc{};
};

inline std::unique_ptr<DeviceCache> upload_cache(const EpisodicCache& c, std::size_t kv_heads, std::size_t dh) {
    auto d = std::make_unique<DeviceCache>();
    const std::size_t L = c.layers.size();
    std::vector<double> k, v;
    std::vector<int32_t> pos, off, len;
    d->base.push_back(0);
    for (const LayerCache& layer : c.layers) {
        int32_t o = 0;
        for (std::size_t h = 0; h < kv_heads; ++h) {
            off.push_back(o);
            const auto& head = layer.heads[h];
            len.push_back(int32_t(head.size()));
            for (const KVEntry& e : head) {
                if (e.key.size() != dh || e.value.size() != dh) throw DimensionError("forward: cache entry dimension mismatch");
                if (e.position > 0x7fffffffu) throw Error("forward: position exceeds the device int32 range");
                k.insert(k.end(), e.key.begin(), e.key.end());
                v.insert(v.end(), e.value.begin(), e.value.end());
                pos.push_back(int32_t(e.position));
            }
            o += int32_t(head.size());
        }
        off.push_back(o);
        d->base.push_back(d->base.back() + o);
    }
    d->k = std::make_unique<DBuf<double>>(std::max<std::size_t>(k.size(), 1));
    d->v = std::make_unique<DBuf<double>>(std::max<std::size_t>(v.size(), 1));
    d->pos = std::make_unique<DBuf<int32_t>>(std::max<std::size_t>(pos.size(), 1));
    d->off = std::make_unique<DBuf<int32_t>>(off.size());
    d->len = std::make_unique<DBuf<int32_t>>(len.size());
    if (!k.empty()) {
        d->k->upload(k.data(), k.size());
        d->v->upload(v.data(), v.size());
        d->pos->upload(pos.data(), pos.size());
    }
    d->off->upload(off.data(), off.size());
    d->len->upload(len.data(), len.size());
    d->desc = epk_cache_desc{int32_t(L), int32_t(kv_heads), int32_t(dh), EPK_F64, d->k->p, d->v->p,
                             d->pos->p, d->off->p, d->len->p, d->base.data()};
    return d;
}

}  // namespace detail

/// forward (toymodel.hpp:228-411) with the layers on the GPU (epk_toy_forward):
/// same signature and trace (keys, values, context positions, attention
/// grids, hidden), same validation and exceptions.  Softmax::host (default)
/// keeps every output bit-identical to the reference.
inline ForwardTrace forward(const Model& model, std::span<const TokenId> tokens, std::span<const std::size_t> positions,
                            const MaskSpec& mask, const EpisodicCache* past = nullptr, TraceOptions opts = {},
                            Softmax softmax = Softmax::host) {
    const ModelConfig& cfg = model.config;
    const std::size_t n = tokens.size();
    if (n == 0) throw Error("forward: empty token sequence");
    if (positions.size() != n) throw DimensionError("forward: positions size mismatch");
    for (std::size_t i = 0; i < n; ++i) {
        if (tokens[i] >= cfg.vocab) throw Error("forward: token id " + std::to_string(tokens[i]) + " out of vocab");
        if (i > 0 && positions[i] <= positions[i - 1]) throw Error("forward: positions must be strictly increasing");
    }
    if (past != nullptr) {
        if (past->layer_count() != cfg.layers) throw DimensionError("forward: cache layer count mismatch");
        if (!past->empty() && past->max_position() >= positions[0])
            throw Error("forward: position overlap between cache and new tokens");
    }
    const std::size_t L = cfg.layers, Hq = cfg.query_heads, Hkv = cfg.kv_heads, dh = cfg.head_dim, D = cfg.model_dim;
    const detail::DeviceModel& dm = detail::device_model(model);
    std::vector<int32_t> tok(tokens.begin(), tokens.end());
    std::vector<int64_t> pos(positions.begin(), positions.end());
    std::vector<double> pe;
    pe.reserve(n * D);
    for (std::size_t t = 0; t < n; ++t) {
        const Vec p = model.position_embedding(positions[t]);
        pe.insert(pe.end(), p.begin(), p.end());
    }
    detail::DBuf<int32_t> d_tok(n);
    detail::DBuf<int64_t> d_pos(n);
    detail::DBuf<double> d_pe(n * D), d_k(L * n * Hkv * dh), d_v(L * n * Hkv * dh), d_h(n * D);
    d_tok.upload(tok.data(), n);
    d_pos.upload(pos.data(), n);
    d_pe.upload(pe.data(), pe.size());
    std::unique_ptr<detail::DeviceCache> dc;
    std::vector<std::size_t> cache_len(L * Hkv, 0);
    if (past != nullptr) {
        dc = detail::upload_cache(*past, Hkv, dh);
        for (std::size_t l = 0; l < L; ++l)
            for (std::size_t h = 0; h < Hkv; ++h) cache_len[l * Hkv + h] = past->layers[l].heads[h].size();
    }
    std::vector<int64_t> attn_off;
    std::size_t attn_total = 0;
    if (opts.store_attention) {
        for (std::size_t l = 0; l < L; ++l)
            for (std::size_t qh = 0; qh < Hq; ++qh) {
                attn_off.push_back(int64_t(attn_total));
                attn_total += n * (cache_len[l * Hkv + cfg.kv_head_of(qh)] + n);
            }
    }
    std::unique_ptr<detail::DBuf<double>> d_attn;
    if (opts.store_attention) d_attn = std::make_unique<detail::DBuf<double>>(std::max<std::size_t>(attn_total, 1));
    const MaskSpec::Kind kind = mask.kind;
    detail::check(epk_toy_forward(detail::ctx(), &dm.desc, d_tok.p, d_pe.p, d_pos.p, int64_t(n),
                                  kind == MaskSpec::Kind::Causal ? 0 : 1, int64_t(mask.sink_count),
                                  int64_t(mask.recent_count), dc ? &dc->desc : nullptr, d_k.p, d_v.p,
                                  d_attn ? d_attn->p : nullptr, attn_off.empty() ? nullptr : attn_off.data(), d_h.p,
                                  softmax == Softmax::host ? 1 : 0));
    std::vector<double> hk(L * n * Hkv * dh), hv(hk.size()), hh(n * D), ha(attn_total);
    d_k.download(hk.data(), hk.size());
    d_v.download(hv.data(), hv.size());
    d_h.download(hh.data(), hh.size());
    if (d_attn && attn_total) d_attn->download(ha.data(), attn_total);
    ForwardTrace trace;
    trace.positions.assign(positions.begin(), positions.end());
    trace.layers.resize(L);
    for (std::size_t l = 0; l < L; ++l) {
        LayerTrace& lt = trace.layers[l];
        lt.keys.resize(Hkv);
        lt.values.resize(Hkv);
        lt.context_positions.resize(Hkv);
        for (std::size_t h = 0; h < Hkv; ++h) {
            lt.keys[h] = Matrix(n, dh);
            lt.values[h] = Matrix(n, dh);
            for (std::size_t t = 0; t < n; ++t)
                for (std::size_t d = 0; d < dh; ++d) {
                    const std::size_t src = (l * n + t) * Hkv * dh + h * dh + d;
                    lt.keys[h].values[t * dh + d] = hk[src];
                    lt.values[h].values[t * dh + d] = hv[src];
                }
            if (past != nullptr)
                for (const KVEntry& e : past->layers[l].heads[h]) lt.context_positions[h].push_back(e.position);
            lt.context_positions[h].insert(lt.context_positions[h].end(), positions.begin(), positions.end());
        }
        if (opts.store_attention) {
            lt.attention.resize(Hq);
            for (std::size_t qh = 0; qh < Hq; ++qh) {
                const std::size_t cols = cache_len[l * Hkv + cfg.kv_head_of(qh)] + n;
                lt.attention[qh] = Matrix(n, cols);
                std::copy(ha.begin() + attn_off[l * Hq + qh], ha.begin() + attn_off[l * Hq + qh] + n * cols,
                          lt.attention[qh].values.begin());
            }
        }
    }
    trace.hidden = Matrix(n, D);
    trace.hidden.values = std::move(hh);
    return trace;
}

/// measure_sensitivity (allocation.hpp:55) with its two calibration forwards
/// (causal and sink+recent, allocation.hpp:70-72) on the GPU as well.
inline SensitivityProfile measure_sensitivity(const Model& model, std::span<const TokenId> calibration_tokens,
                                              std::size_t calibration_budget, std::size_t sink, std::string input_id,
                                              Softmax softmax) {
    const std::size_t n = calibration_tokens.size();
    if (n < 2) throw Error("measure_sensitivity: need at least 2 calibration tokens");
    if (calibration_budget < sink + 1) throw Error("measure_sensitivity: budget must be >= sink + 1");
    TraceOptions opts;
    opts.store_attention = false;
    std::vector<std::size_t> pos(n);
    for (std::size_t i = 0; i < n; ++i) pos[i] = i;
    const ForwardTrace full = gpu::forward(model, calibration_tokens, pos, MaskSpec::causal(), nullptr, opts, softmax);
    const ForwardTrace block = gpu::forward(model, calibration_tokens, pos,
                                            MaskSpec::sink_recent(sink, calibration_budget - sink), nullptr, opts,
                                            softmax);
    return detail::sensitivity_from_traces(model, full, block, n, calibration_budget, sink, std::move(input_id));
}

/// Which forwards of gpu::block_prefill run on the GPU (default: none -- the
/// reference's host forward, as in the reference-signature overload).
struct PrefillForward {
    bool block_on_device = false;   // the block's own forward (appended K/V)
    bool prompt_on_device = false;  // the patched prompt's forward (attention grids for scoring)
    Softmax softmax = Softmax::host;
};

/// block_prefill (blockprefill.hpp:92) with scoring and eviction on the GPU.
/// The toy-model forwards (block and prompt) are the reference's own, on the
/// host; every block's prompt grids are scored by the GPU reduction and every
/// layer is evicted by the GPU selection, so the result is bit-identical to
/// the reference.  Supports every scorer: patched, snapkv, kvzip, infinipot
/// (GPU prompt scoring), keydiff (GPU KeyDiff scores) and streaming.
inline PrefillReport block_prefill(const Model& model, std::span<const TokenId> context,
                                   const BlockPrefillConfig& config, std::size_t episode_id,
                                   std::span<const std::size_t> positions, const PrefillForward& fwd) {
    const ModelConfig& cfg = model.config;
    if (context.empty()) throw Error("block_prefill: empty context");
    if (config.budget_per_head < 1 || config.block_size < 1)
        throw Error("block_prefill: budget and block size must be >= 1");
    if (config.scorer == ScorerKind::patched && !config.prompt_provider)
        throw Error("block_prefill: patched scorer needs a prompt provider");
    std::vector<std::size_t> default_positions;
    if (positions.empty()) {
        default_positions.resize(context.size());
        for (std::size_t i = 0; i < context.size(); ++i) default_positions[i] = i;
        positions = default_positions;
    } else if (positions.size() != context.size()) {
        throw DimensionError("block_prefill: positions size mismatch");
    }
    std::vector<std::size_t> layer_budgets(cfg.layers, config.budget_per_head);
    if (config.allocation) {
        if (config.allocation->layer_count() != cfg.layers)
            throw Error("block_prefill: allocation layer count != model layers");
        if (config.allocation->total() != cfg.layers * config.budget_per_head)
            throw Error("block_prefill: allocation does not target layers * budget");
        layer_budgets = config.allocation->layer_budgets;
    }
    PrefillReport report;
    report.layer_budgets = layer_budgets;
    report.cache.episode_id = episode_id;
    report.cache.provenance.scorer = std::string(scorer_name(config.scorer));
    report.cache.provenance.budget_per_head = config.budget_per_head;
    report.cache.provenance.layer_budgets = layer_budgets;
    for (std::size_t l = 0; l < cfg.layers; ++l) report.cache.layers.emplace_back(cfg.kv_heads, layer_budgets[l]);
    const std::size_t prompt_base = positions.back() + 1;
    const std::vector<std::size_t> zeros(cfg.layers, 0);
    std::unordered_set<std::size_t> pins;
    if (config.scorer == ScorerKind::streaming) {
        if (config.streaming_sink > config.budget_per_head) throw Error("block_prefill: streaming sink exceeds budget");
        if (config.allocation)
            for (std::size_t b : layer_budgets)
                if (config.streaming_sink > b) throw Error("block_prefill: streaming sink exceeds an allocated layer budget");
    }
    auto entries = [&](const EpisodicCache& c) {
        std::vector<std::size_t> out;
        for (const auto& layer : c.layers) out.push_back(layer.entry_count());
        return out;
    };
    TraceOptions block_opts;
    block_opts.store_attention = false;
    const std::size_t n = context.size();
    for (std::size_t start = 0; start < n; start += config.block_size) {
        const std::size_t len = std::min(config.block_size, n - start);
        const std::span<const TokenId> block = context.subspan(start, len);
        const std::span<const std::size_t> block_positions = positions.subspan(start, len);
        const std::size_t block_index = report.blocks_processed;
        ForwardTrace trace =
            fwd.block_on_device
                ? gpu::forward(model, block, block_positions, MaskSpec::causal(), &report.cache, block_opts, fwd.softmax)
                : epikv::forward(model, block, block_positions, MaskSpec::causal(), &report.cache, block_opts);
        append_to_cache(report.cache, trace);
        report.occupancy.record(OccupancyKind::Append, entries(report.cache), zeros);
        TokenScoreMap scores;
        if (scorer_uses_prompt(config.scorer)) {
            PatchedPrompt prompt;
            switch (config.scorer) {
                case ScorerKind::patched: prompt = config.prompt_provider(episode_id, block_index); break;
                case ScorerKind::snapkv: prompt = snapkv_prompt(block); break;
                case ScorerKind::kvzip: prompt = kvzip_prompt(block, cfg.vocab); break;
                case ScorerKind::infinipot: prompt = infinipot_prompt(cfg.vocab); break;
                default: break;
            }
            if (prompt.tokens.empty()) throw Error("block_prefill: empty patched prompt");
            std::vector<std::size_t> prompt_positions(prompt.tokens.size());
            for (std::size_t i = 0; i < prompt.tokens.size(); ++i) prompt_positions[i] = prompt_base + i;
            report.prompt_ranges.push_back({prompt_base, prompt.tokens.size()});
            const ForwardTrace prompt_trace =
                fwd.prompt_on_device
                    ? gpu::forward(model, prompt.tokens, prompt_positions, MaskSpec::causal(), &report.cache, {},
                                   fwd.softmax)
                    : epikv::forward(model, prompt.tokens, prompt_positions, MaskSpec::causal(), &report.cache);
            report.occupancy.record(OccupancyKind::PromptResident, entries(report.cache),
                                    std::vector<std::size_t>(cfg.layers, cfg.kv_heads * prompt.tokens.size()));
            scores = gpu::score_with_prompt(prompt_trace, config.aggregation);
        } else if (config.scorer == ScorerKind::keydiff) {
            scores = gpu::keydiff_scores(report.cache);
        } else {
            scores.layers.resize(report.cache.layers.size());
            for (std::size_t l = 0; l < report.cache.layers.size(); ++l) {
                scores.layers[l].resize(report.cache.layers[l].heads.size());
                for (std::size_t h = 0; h < report.cache.layers[l].heads.size(); ++h)
                    for (const KVEntry& e : report.cache.layers[l].heads[h])
                        scores.layers[l][h].emplace(e.position, double(e.position));
            }
            pins.clear();
            for (std::size_t p = 0; p < config.streaming_sink; ++p) pins.insert(p);
        }
        std::size_t evicted = 0;
        for (std::size_t l = 0; l < cfg.layers; ++l) {
            const std::size_t before = report.cache.layers[l].entry_count();
            report.cache.layers[l] = gpu::evict_to_budget(report.cache.layers[l], scores.layers[l], pins);
            evicted += before - report.cache.layers[l].entry_count();
        }
        report.evictions_per_block.push_back(evicted);
        report.occupancy.record(OccupancyKind::Evict, entries(report.cache), zeros);
        ++report.blocks_processed;
    }
    return report;
}

/// block_prefill with the reference's signature: host forwards (the
/// reference's), GPU scoring and eviction.
inline PrefillReport block_prefill(const Model& model, std::span<const TokenId> context,
                                   const BlockPrefillConfig& config, std::size_t episode_id = 0,
                                   std::span<const std::size_t> positions = {}) {
    return gpu::block_prefill(model, context, config, episode_id, positions, PrefillForward{});
}

/// kmeans (clustering.hpp:148) with the points split in index order over
/// `devices` (one shard per entry; a device may repeat): the centroid sums run
/// as an ordered chain over NCCL (epk_kmeans_sharded), so the result is
/// bit-identical to the reference's single-threaded kmeans.
inline KMeansResult kmeans_sharded(const std::vector<Vec>& points, std::size_t k, std::uint64_t seed,
                                   const std::vector<int>& devices, std::size_t max_iters = 64) {
    if (k < 1) throw Error("kmeans: cluster count must be >= 1");
    if (points.size() < k)
        throw Error("kmeans: fewer points (" + std::to_string(points.size()) + ") than clusters (" +
                    std::to_string(k) + ")");
    if (devices.empty()) throw Error("kmeans_sharded: no devices");
    const std::size_t n = points.size(), dim = points[0].size(), S = devices.size();
    struct Ctx {
        epk_ctx* c = nullptr;
        ~Ctx() {
            if (c) epk_ctx_destroy(c);
        }
    };
    std::vector<Ctx> ctxs(S);
    std::vector<std::unique_ptr<detail::DBuf<double>>> bufs;
    std::vector<epk_ctx*> handles(S);
    std::vector<const double*> shard_ptrs(S);
    std::vector<int64_t> ns(S);
    int cur = 0;
    detail::cuda_check(cudaGetDevice(&cur), "cudaGetDevice");
    for (std::size_t s = 0; s < S; ++s) {
        const std::size_t a = n * s / S, b = n * (s + 1) / S;
        std::vector<double> flat;
        flat.reserve((b - a) * dim);
        for (std::size_t i = a; i < b; ++i) {
            if (points[i].size() != dim) throw DimensionError("kmeans: points differ in dimension");
            flat.insert(flat.end(), points[i].begin(), points[i].end());
        }
        detail::cuda_check(cudaSetDevice(devices[s]), "cudaSetDevice");
        detail::check(epk_ctx_create(devices[s], nullptr, &ctxs[s].c));
        bufs.push_back(std::make_unique<detail::DBuf<double>>(std::max<std::size_t>(flat.size(), 1)));
        if (!flat.empty()) bufs.back()->upload(flat.data(), flat.size());
        handles[s] = ctxs[s].c;
        shard_ptrs[s] = bufs.back()->p;
        ns[s] = int64_t(b - a);
    }
    detail::cuda_check(cudaSetDevice(cur), "cudaSetDevice");
    std::vector<int64_t> assign(n);
    std::vector<double> cent(k * dim), sse(std::max<std::size_t>(max_iters, 1));
    int64_t iters = 0;
    detail::check(epk_kmeans_sharded(handles.data(), int32_t(S), shard_ptrs.data(), ns.data(), int64_t(dim),
                                     int64_t(k), seed, int64_t(max_iters), assign.data(), cent.data(), &iters,
                                     sse.data()));
    KMeansResult r;
    r.assignments.assign(assign.begin(), assign.end());
    r.centroids.resize(k);
    for (std::size_t c = 0; c < k; ++c) r.centroids[c].assign(cent.begin() + c * dim, cent.begin() + (c + 1) * dim);
    r.iterations = std::size_t(iters);
    r.sse_per_iteration.assign(sse.begin(), sse.begin() + iters);
    return r;
}

/// Where gpu::build runs: the GPUs the episodes are sharded over (one host
/// thread and one epk_ctx each; a device listed twice gets two threads), and
/// whether the A1 k-means also shards the segment embeddings over them.
struct BuildDevices {
    std::vector<int> devices;        // empty: every visible device
    bool shard_embeddings = false;   // k-means via epk_kmeans_sharded (NCCL ordered chain)
};

/// build (episodic.hpp:108-199), Phase A on several GPUs.  A1 clusters the
/// segment embeddings (gpu::kmeans or gpu::kmeans_sharded), A2 measures the
/// sensitivity (gpu::measure_sensitivity) and allocates (the reference's
/// allocate), A3 runs gpu::block_prefill once per episode with episodes
/// assigned round-robin to the devices (episodes are independent,
/// episodic.hpp:159-171; zero inter-GPU traffic) and persists each cache as it
/// finishes, then writes the manifest.  Every file is byte-identical to the
/// reference build's, whatever the device count (the multi-GPU analogue of
/// test_episodic.cpp:289-302); config.parallel_episodes is implied by
/// more than one device.
inline BuildResult build(const Model& model, const ConversationHistory& history, std::size_t episode_count,
                         std::size_t budget_per_head, double alpha, const Embedder& embedder,
                         const std::string& store_dir, const EpisodicBuildConfig& config = {},
                         const BuildDevices& where = {}) {
    std::vector<int> devices = where.devices;
    if (devices.empty()) {
        int nd = 0;
        detail::cuda_check(cudaGetDeviceCount(&nd), "cudaGetDeviceCount");
        for (int d = 0; d < nd; ++d) devices.push_back(d);
    }
    if (devices.empty()) throw Error("build: no CUDA device");
    const std::vector<Segment> segments = segment_history(history, config.w_embed);
    if (episode_count > segments.size()) {
        throw Error("build: more episodes (" + std::to_string(episode_count) + ") than segments (" +
                    std::to_string(segments.size()) + ")");
    }
    // A1: segment, embed, cluster, pick medoids and prompts.
    std::vector<Vec> embeddings;
    embeddings.reserve(segments.size());
    for (const Segment& s : segments) embeddings.push_back(embedder.embed(s.text));
    const KMeansResult clusters =
        where.shard_embeddings
            ? gpu::kmeans_sharded(embeddings, episode_count, config.cluster_seed, devices, config.kmeans_max_iters)
            : gpu::kmeans(embeddings, episode_count, config.cluster_seed, config.kmeans_max_iters);
    EpisodeModel episodes = finalize_episodes(history, segments, embeddings, clusters.assignments,
                                              config.prompt_window, model.config.vocab);
    // A2: sensitivity and per-layer budgets.
    BudgetAllocation allocation;
    SensitivityProfile profile;
    if (config.use_allocation) {
        const std::size_t cal_budget = config.calibration_budget > 0 ? config.calibration_budget : budget_per_head;
        const std::size_t cal_sink =
            config.calibration_sink > 0 ? config.calibration_sink : std::min<std::size_t>(128, cal_budget / 2);
        const std::size_t cal_len =
            config.calibration_tokens > 0 ? config.calibration_tokens : std::max<std::size_t>(4 * cal_budget, 256);
        const std::vector<TokenId> cal_tokens =
            synthetic_calibration_tokens(cal_len, config.calibration_seed, model.config.vocab);
        profile = gpu::measure_sensitivity(model, cal_tokens, cal_budget, cal_sink,
                                           "synthetic:seed=" + std::to_string(config.calibration_seed) +
                                               ",len=" + std::to_string(cal_len));
        allocation = allocate(profile, budget_per_head, alpha);
    } else {
        allocation = uniform_allocation(model.config.layers, budget_per_head);
        profile.sigma.assign(model.config.layers, 1.0);
        profile.sensitivity.assign(model.config.layers, 0.0);
        profile.input_id = "uniform";
        profile.model_seed = model.config.seed;
    }
    // A3: episodes round-robin over the devices, one host thread (and, through
    // detail::ctx(), one epk_ctx) per device entry.
    const RenderedHistory rendered = render_history_tokens(history, model.config.vocab);
    CacheStore store(store_dir);
    BuildResult result;
    result.reports.resize(episode_count);
    const std::size_t G = std::min(devices.size(), std::max<std::size_t>(episode_count, 1));
    std::vector<std::exception_ptr> errors(G);
    auto worker = [&](std::size_t g) {
        try {
            detail::cuda_check(cudaSetDevice(devices[g]), "cudaSetDevice");
            for (std::size_t e = g; e < episode_count; e += G) {
                BlockPrefillConfig prefill;
                prefill.budget_per_head = budget_per_head;
                prefill.block_size = config.block_size;
                prefill.scorer = ScorerKind::patched;
                prefill.aggregation = config.aggregation;
                prefill.allocation = allocation;
                const PatchedPrompt prompt = episodes.prompts[e];
                prefill.prompt_provider = [prompt](std::size_t, std::size_t) { return prompt; };
                result.reports[e] = gpu::block_prefill(model, rendered.tokens, prefill, e);
                store.save(result.reports[e].cache);
            }
        } catch (...) {
            errors[g] = std::current_exception();
        }
    };
    if (G == 1) {
        worker(0);
    } else {
        std::vector<std::thread> threads;
        for (std::size_t g = 0; g < G; ++g) threads.emplace_back(worker, g);
        for (std::thread& t : threads) t.join();
    }
    for (const std::exception_ptr& e : errors)
        if (e) std::rethrow_exception(e);
    store.write_manifest(
        epikv::detail::manifest_json(episodes, allocation, store, ScorerKind::patched, budget_per_head, embedder.dim()));
    result.set.episodes = std::move(episodes);
    result.set.allocation = std::move(allocation);
    result.set.profile = std::move(profile);
    result.set.store_dir = store_dir;
    result.set.budget_per_head = budget_per_head;
    return result;
}

// The live cache of a DeviceEpisode (the throughput path, epikv_device.hpp)
// as the reference's EpisodicCache: bf16 keys / values widened to double,
// every head's entries in position order, budgets as the layer budgets.  For
// persisting with the reference's CacheStore or decoding on the host.
inline EpisodicCache to_episodic_cache(const DeviceEpisode& e, std::size_t episode_id = 0,
                                       const std::string& scorer = "patched") {
    e.synchronize();
    const epk_cache_desc c = e.desc();
    const std::size_t L = e.layers(), H = e.kv_heads(), d = e.head_dim();
    const std::size_t rows = std::size_t(e.layer_base()[L]);
    std::vector<std::int32_t> off(L * (H + 1)), len(L * H), pos(rows);
    std::vector<std::uint16_t> k(rows * d), v(rows * d);
    detail::cuda_check(cudaMemcpy(off.data(), c.head_off, off.size() * 4, cudaMemcpyDeviceToHost), "D2H head_off");
    detail::cuda_check(cudaMemcpy(len.data(), c.head_len, len.size() * 4, cudaMemcpyDeviceToHost), "D2H head_len");
    detail::cuda_check(cudaMemcpy(pos.data(), c.pos, rows * 4, cudaMemcpyDeviceToHost), "D2H pos");
    detail::cuda_check(cudaMemcpy(k.data(), c.k, rows * d * 2, cudaMemcpyDeviceToHost), "D2H k");
    detail::cuda_check(cudaMemcpy(v.data(), c.v, rows * d * 2, cudaMemcpyDeviceToHost), "D2H v");
    auto widen = [](std::uint16_t b) {
        const std::uint32_t u = std::uint32_t(b) << 16;
        float f;
        std::memcpy(&f, &u, 4);
        return double(f);
    };
    EpisodicCache out;
    out.episode_id = episode_id;
    out.provenance.scorer = scorer;
    std::size_t mx = 0;
    for (std::size_t l = 0; l < L; ++l) {
        const std::size_t m = std::size_t(e.budgets()[l]);
        mx = std::max(mx, m);
        out.provenance.layer_budgets.push_back(m);
        LayerCache lc(H, m);
        for (std::size_t h = 0; h < H; ++h) {
            const std::size_t r0 = std::size_t(e.layer_base()[l]) + std::size_t(off[l * (H + 1) + h]);
            for (std::size_t i = 0; i < std::size_t(len[l * H + h]); ++i) {
                KVEntry en;
                en.position = std::size_t(pos[r0 + i]);
                en.key.resize(d);
                en.value.resize(d);
                for (std::size_t j = 0; j < d; ++j) {
                    en.key[j] = widen(k[(r0 + i) * d + j]);
                    en.value[j] = widen(v[(r0 + i) * d + j]);
                }
                lc.heads[h].push_back(std::move(en));
            }
        }
        out.layers.push_back(std::move(lc));
    }
    out.provenance.budget_per_head = mx;
    return out;
}

}  // namespace gpu
}  // namespace epikv
