// ref_shim.cpp -- extern "C" entry points into the UNMODIFIED reference
// headers (/root/reference/proj/include/epikv), compiled in place by
// oracle/Makefile into oracle/_ref/libepkref.so.
//
// TEST INFRASTRUCTURE ONLY (see oracle/epk_oracle.cpp header).  No reference
// source is copied: this file only #includes the reference headers from
// where they lie and marshals flat arrays into the reference types.
//
// Uses: pinning oracle/epk_oracle.cpp (tests/test_oracle_vs_ref.py),
// generating tests/golden/ fixtures, and bench.py --impl reference (the
// reference CPU path timed on the host cores).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <set>
#include <string>
#include <unordered_set>
#include <vector>

#include "epikv/allocation.hpp"
#include "epikv/blockprefill.hpp"
#include "epikv/clustering.hpp"
#include "epikv/kvcache.hpp"
#include "epikv/numerics.hpp"
#include "epikv/scoring.hpp"
#include "epikv/toymodel.hpp"

using i64 = std::int64_t;

namespace {

thread_local std::string g_err;

int map_exception(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const epikv::DimensionError*>(&e)) return -3;
    if (dynamic_cast<const epikv::ZeroNormError*>(&e)) return -4;
    if (dynamic_cast<const epikv::IoError*>(&e)) return -5;
    if (dynamic_cast<const epikv::Error*>(&e)) return -2;
    return -9;
}

// The synthetic-Q restatement of toymodel.hpp:327-391 (forward() never
// exposes Q), producing the LayerTrace the reference scorer consumes.
epikv::LayerTrace build_prompt_trace(int hq, int hkv, int d, int p, const i64* head_off,
                                     const i64* pos, i64 prompt_base, const double* q,
                                     const double* k, const double* kp) {
    epikv::LayerTrace lt;
    lt.context_positions.resize(size_t(hkv));
    for (int h = 0; h < hkv; ++h) {
        for (i64 r = head_off[h]; r < head_off[h + 1]; ++r)
            lt.context_positions[size_t(h)].push_back(size_t(pos[r]));
        for (int t = 0; t < p; ++t) lt.context_positions[size_t(h)].push_back(size_t(prompt_base + t));
    }
    const int group = hq / hkv;
    const double scale = 1.0 / std::sqrt(double(d));
    constexpr double kMasked = -std::numeric_limits<double>::infinity();
    std::vector<double> scratch;
    for (int qh = 0; qh < hq; ++qh) {
        const int h = qh / group;
        const i64 n = head_off[h + 1] - head_off[h];
        const i64 ctx_total = n + p;
        epikv::Matrix grid{static_cast<size_t>(p), static_cast<size_t>(ctx_total)};
        scratch.resize(size_t(ctx_total));
        for (int t = 0; t < p; ++t) {
            const double* qv = q + (i64(qh) * p + t) * d;
            const i64 visible = n + t + 1;
            double max_logit = kMasked;
            for (i64 j = 0; j < visible; ++j) {
                const double* kv = j < n ? k + (head_off[h] + j) * d : kp + (i64(h) * p + (j - n)) * d;
                double acc = 0.0;
                for (int dd = 0; dd < d; ++dd) acc += qv[dd] * kv[dd];
                const double s = acc * scale;
                if (s > max_logit) max_logit = s;
                scratch[size_t(j)] = s;
            }
            double denom = 0.0;
            for (i64 j = 0; j < visible; ++j) {
                const double e = std::exp(scratch[size_t(j)] - max_logit);
                scratch[size_t(j)] = e;
                denom += e;
            }
            for (i64 j = 0; j < visible; ++j) grid.at(size_t(t), size_t(j)) = scratch[size_t(j)] / denom;
        }
        lt.attention.push_back(std::move(grid));
    }
    return lt;
}

epikv::LayerCache build_layer(int hkv, i64 budget, int d, const i64* head_off, const i64* pos,
                              const double* k, const double* v) {
    epikv::LayerCache cache{static_cast<size_t>(hkv), static_cast<size_t>(budget)};
    for (int h = 0; h < hkv; ++h) {
        for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) {
            epikv::KVEntry e;
            e.position = size_t(pos[r]);
            if (d > 0) {
                e.key.assign(k + r * d, k + (r + 1) * d);
                e.value.assign(v + r * d, v + (r + 1) * d);
            }
            cache.heads[size_t(h)].push_back(std::move(e));
        }
    }
    return cache;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// score_with_prompt (scoring.hpp:80) over the restated prompt trace.
int ref_score_layer_f64(int hq, int hkv, int d, int p, const i64* head_off, const i64* pos,
                        const double* q, const double* k, const double* kp, int agg_max,
                        double* out) {
    try {
        i64 prompt_base = 0;
        for (i64 r = 0; r < head_off[hkv]; ++r) prompt_base = std::max(prompt_base, pos[r] + 1);
        epikv::ForwardTrace trace;
        for (int t = 0; t < p; ++t) trace.positions.push_back(size_t(prompt_base + t));
        trace.layers.push_back(build_prompt_trace(hq, hkv, d, p, head_off, pos, prompt_base, q, k, kp));
        const epikv::TokenScoreMap map = epikv::score_with_prompt(
            trace, agg_max ? epikv::Aggregation::Max : epikv::Aggregation::Avg);
        for (int h = 0; h < hkv; ++h)
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) out[r] = map.at(0, size_t(h), size_t(pos[r]));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// score_with_prompt on caller-supplied grids: grids[qh] is p x (n_h + p).
int ref_score_grids(int hq, int hkv, int p, const i64* head_off, const i64* pos,
                    const double* grids, int agg_max, double* out) {
    try {
        epikv::ForwardTrace trace;
        for (int t = 0; t < p; ++t) trace.positions.push_back(size_t(1u << 30) + size_t(t));
        epikv::LayerTrace lt;
        lt.context_positions.resize(size_t(hkv));
        for (int h = 0; h < hkv; ++h) {
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r)
                lt.context_positions[size_t(h)].push_back(size_t(pos[r]));
            for (int t = 0; t < p; ++t) lt.context_positions[size_t(h)].push_back(size_t(1u << 30) + size_t(t));
        }
        const int group = hq / hkv;
        const double* g = grids;
        for (int qh = 0; qh < hq; ++qh) {
            const int h = qh / group;
            const i64 cols = head_off[h + 1] - head_off[h] + p;
            epikv::Matrix m{static_cast<size_t>(p), static_cast<size_t>(cols)};
            std::memcpy(m.values.data(), g, sizeof(double) * size_t(p * cols));
            g += p * cols;
            lt.attention.push_back(std::move(m));
        }
        trace.layers.push_back(std::move(lt));
        const epikv::TokenScoreMap map = epikv::score_with_prompt(
            trace, agg_max ? epikv::Aggregation::Max : epikv::Aggregation::Avg);
        for (int h = 0; h < hkv; ++h)
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) out[r] = map.at(0, size_t(h), size_t(pos[r]));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// evict_to_budget (kvcache.hpp:142).  keep[r] = 1 for retained rows; the
// compacted K/V rows and positions are written in output order when k_out is
// non-null.  Returns the number of retained rows, or a negative error code.
i64 ref_evict_layer(int hkv, i64 budget, int d, const i64* head_off, const i64* pos,
                    const double* k, const double* v, const double* scores, const i64* pins,
                    i64 npins, std::uint8_t* keep, i64* out_head_counts, double* k_out,
                    double* v_out, i64* pos_out) {
    try {
        const epikv::LayerCache cache = build_layer(hkv, budget, d, head_off, pos, k, v);
        epikv::LayerScores scores_map(static_cast<size_t>(hkv));
        for (int h = 0; h < hkv; ++h)
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) scores_map[size_t(h)][size_t(pos[r])] = scores[r];
        std::unordered_set<std::size_t> pinned;
        for (i64 i = 0; i < npins; ++i) pinned.insert(size_t(pins[i]));
        const epikv::LayerCache out = epikv::evict_to_budget(cache, scores_map, pinned);
        i64 total = 0;
        for (int h = 0; h < hkv; ++h) {
            std::set<std::size_t> kept;
            for (const auto& e : out.heads[size_t(h)]) {
                kept.insert(e.position);
                if (pos_out) pos_out[total] = i64(e.position);
                if (k_out && d > 0) {
                    std::memcpy(k_out + total * d, e.key.data(), sizeof(double) * size_t(d));
                    std::memcpy(v_out + total * d, e.value.data(), sizeof(double) * size_t(d));
                }
                ++total;
            }
            if (out_head_counts) out_head_counts[h] = i64(out.heads[size_t(h)].size());
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) keep[r] = kept.count(size_t(pos[r])) ? 1 : 0;
        }
        return total;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// One reference CPU step for one layer: restated attention grids ->
// score_with_prompt -> evict_to_budget (the bench --impl reference unit).
i64 ref_step_layer_f64(int hq, int hkv, int d, int p, i64 budget, const i64* head_off,
                       const i64* pos, const double* q, const double* k, const double* v,
                       const double* kp, int agg_max, std::uint8_t* keep) {
    std::vector<double> scores(size_t(head_off[hkv]));
    const int rc = ref_score_layer_f64(hq, hkv, d, p, head_off, pos, q, k, kp, agg_max, scores.data());
    if (rc != 0) return rc;
    return ref_evict_layer(hkv, budget, d, head_off, pos, k, v, scores.data(), nullptr, 0, keep,
                           nullptr, nullptr, nullptr, nullptr);
}

// top_k_indices (numerics.hpp:111) -> ascending indices; returns count.
i64 ref_top_k_indices(const double* scores, i64 n, i64 k, i64* out) {
    const auto idx = epikv::top_k_indices(std::span<const double>(scores, size_t(n)), size_t(k));
    for (size_t i = 0; i < idx.size(); ++i) out[i] = i64(idx[i]);
    return i64(idx.size());
}

// keydiff_scores (scoring.hpp:186) over a one-layer EpisodicCache.
int ref_keydiff_layer(int hkv, int d, const i64* head_off, const i64* pos, const double* k, double* out) {
    try {
        std::vector<double> v(size_t(head_off[hkv]) * size_t(d), 0.0);
        epikv::EpisodicCache cache;
        cache.layers.push_back(build_layer(hkv, 0, d, head_off, pos, k, v.data()));
        const epikv::TokenScoreMap map = epikv::keydiff_scores(cache);
        for (int h = 0; h < hkv; ++h)
            for (i64 r = head_off[h]; r < head_off[h + 1]; ++r) out[r] = map.at(0, size_t(h), size_t(pos[r]));
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// persist (kvcache.hpp:281) of an EpisodicCache built from flat arrays:
// layer l's heads are rows [head_off[l*(H+1)+h], head_off[l*(H+1)+h+1]) of
// pos / k / v ([rows][d] fp64).  Returns the byte count or a negative code.
i64 ref_persist(const char* path, std::uint64_t episode_id, const char* scorer, std::uint64_t budget_per_head,
                const i64* layer_budgets, int n_layer_budgets, int layers, int hkv, int d, const i64* head_off,
                const i64* pos, const double* k, const double* v, const i64* layer_budget_fields) {
    try {
        epikv::EpisodicCache cache;
        cache.episode_id = episode_id;
        cache.provenance.scorer = scorer;
        cache.provenance.budget_per_head = budget_per_head;
        for (int i = 0; i < n_layer_budgets; ++i) cache.provenance.layer_budgets.push_back(size_t(layer_budgets[i]));
        for (int l = 0; l < layers; ++l)
            cache.layers.push_back(build_layer(hkv, layer_budget_fields[l], d, head_off + i64(l) * (hkv + 1), pos, k, v));
        return i64(epikv::persist(cache, path));
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// load_cache (kvcache.hpp:321) of `in`, persisted again to `out`: the
// reference reads our files (round trip).  Returns the bytes written.
i64 ref_load_repersist(const char* in, const char* out) {
    try {
        return i64(epikv::persist(epikv::load_cache(in), out));
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

double ref_cosine(const double* a, const double* b, i64 d) {
    try {
        return epikv::cosine(std::span<const double>(a, size_t(d)), std::span<const double>(b, size_t(d)));
    } catch (const std::exception& e) {
        map_exception(e);
        return std::numeric_limits<double>::quiet_NaN();
    }
}

// kmeans (clustering.hpp:148).
int ref_kmeans(const double* pts, i64 n, i64 dim, i64 k, std::uint64_t seed, i64 max_iters,
               i64* assign_out, double* centroids_out, i64* iters_out, double* sse_out) {
    try {
        std::vector<epikv::Vec> points(static_cast<size_t>(n));
        for (i64 i = 0; i < n; ++i) points[size_t(i)].assign(pts + i * dim, pts + (i + 1) * dim);
        const epikv::KMeansResult r = epikv::kmeans(points, size_t(k), seed, size_t(max_iters));
        for (i64 i = 0; i < n; ++i) assign_out[i] = i64(r.assignments[size_t(i)]);
        for (i64 c = 0; c < k; ++c)
            std::memcpy(centroids_out + c * dim, r.centroids[size_t(c)].data(), sizeof(double) * size_t(dim));
        *iters_out = i64(r.iterations);
        for (size_t i = 0; i < r.sse_per_iteration.size(); ++i) sse_out[i] = r.sse_per_iteration[i];
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// allocate (allocation.hpp:120).
int ref_allocate(const double* sens, int layers, i64 per_head_budget, double alpha,
                 i64* budgets_out, double* weights_out) {
    try {
        epikv::SensitivityProfile prof;
        for (int l = 0; l < layers; ++l) {
            prof.sensitivity.push_back(sens[l]);
            prof.sigma.push_back(1.0 - sens[l]);
        }
        const epikv::BudgetAllocation a = epikv::allocate(prof, size_t(per_head_budget), alpha);
        for (int l = 0; l < layers; ++l) {
            budgets_out[l] = i64(a.layer_budgets[size_t(l)]);
            if (weights_out) weights_out[l] = a.weights[size_t(l)];
        }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// measure_sensitivity (allocation.hpp:55) on a seeded toy model, plus the two
// key tensors it reduces ([L][Hkv][N][d] each), so the oracle and the GPU
// reduction can be checked on exactly the keys the reference used.
int ref_measure_sensitivity(int layers, int hq, int hkv, int d, std::uint64_t model_seed,
                            i64 ntok, std::uint64_t tok_seed, i64 budget, i64 sink,
                            double* sigma_out, i64* skipped_out, double* kf_out, double* kb_out) {
    try {
        epikv::ModelConfig cfg;
        cfg.layers = size_t(layers);
        cfg.query_heads = size_t(hq);
        cfg.kv_heads = size_t(hkv);
        cfg.head_dim = size_t(d);
        cfg.model_dim = size_t(hq * d);
        cfg.vocab = 128;
        cfg.seed = model_seed;
        const epikv::Model model = epikv::init_model(cfg);
        const auto tokens = epikv::synthetic_calibration_tokens(size_t(ntok), tok_seed, cfg.vocab);
        const epikv::SensitivityProfile prof =
            epikv::measure_sensitivity(model, tokens, size_t(budget), size_t(sink));
        for (int l = 0; l < layers; ++l) sigma_out[l] = prof.sigma[size_t(l)];
        *skipped_out = i64(prof.skipped_zero_norm);
        epikv::TraceOptions opts;
        opts.store_attention = false;
        const auto full = epikv::forward(model, tokens, epikv::MaskSpec::causal(), nullptr, opts);
        const auto blk = epikv::forward(model, tokens,
                                        epikv::MaskSpec::sink_recent(size_t(sink), size_t(budget - sink)),
                                        nullptr, opts);
        for (int l = 0; l < layers; ++l)
            for (int h = 0; h < hkv; ++h) {
                const i64 off = ((i64(l) * hkv + h) * ntok) * d;
                std::memcpy(kf_out + off, full.layers[size_t(l)].keys[size_t(h)].values.data(),
                            sizeof(double) * size_t(ntok * d));
                std::memcpy(kb_out + off, blk.layers[size_t(l)].keys[size_t(h)].values.data(),
                            sizeof(double) * size_t(ntok * d));
            }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

// block_prefill (blockprefill.hpp:92) on a seeded toy model with a fixed
// patched prompt.  Writes the append/evict occupancy series of layer 0
// (PromptResident samples skipped, as test_blockprefill.cpp:49-58 does), the
// evictions per block and the retained positions of every (layer, head).
int ref_block_prefill(int layers, int hq, int hkv, int d, std::uint64_t model_seed, i64 ntok,
                      std::uint64_t tok_seed, i64 budget, i64 block, const i64* prompt_tokens,
                      i64 prompt_len, const i64* layer_budgets, i64* series_out, i64* n_series,
                      i64* evictions_out, i64* n_blocks, i64* retained_out, i64* retained_counts) {
    try {
        epikv::ModelConfig cfg;
        cfg.layers = size_t(layers);
        cfg.query_heads = size_t(hq);
        cfg.kv_heads = size_t(hkv);
        cfg.head_dim = size_t(d);
        cfg.model_dim = size_t(hq * d);
        cfg.vocab = 128;
        cfg.seed = model_seed;
        const epikv::Model model = epikv::init_model(cfg);
        const auto context = epikv::synthetic_calibration_tokens(size_t(ntok), tok_seed, cfg.vocab);
        epikv::BlockPrefillConfig config;
        config.budget_per_head = size_t(budget);
        config.block_size = size_t(block);
        config.scorer = epikv::ScorerKind::patched;
        std::vector<epikv::TokenId> ptoks;
        for (i64 i = 0; i < prompt_len; ++i) ptoks.push_back(epikv::TokenId(prompt_tokens[i]));
        config.prompt_provider = [ptoks](std::size_t, std::size_t) {
            epikv::PatchedPrompt pp;
            pp.tokens = ptoks;
            return pp;
        };
        if (layer_budgets) {
            epikv::BudgetAllocation alloc;
            alloc.alpha = 1.0;
            alloc.per_head_budget = size_t(budget);
            for (int l = 0; l < layers; ++l) {
                alloc.layer_budgets.push_back(size_t(layer_budgets[l]));
                alloc.weights.push_back(1.0 / layers);
            }
            config.allocation = alloc;
        }
        const epikv::PrefillReport rep = epikv::block_prefill(model, context, config);
        i64 ns = 0;
        for (const auto& s : rep.occupancy.samples)
            if (s.kind != epikv::OccupancyKind::PromptResident) series_out[ns++] = i64(s.entries_per_layer[0]);
        *n_series = ns;
        for (size_t b = 0; b < rep.evictions_per_block.size(); ++b) evictions_out[b] = i64(rep.evictions_per_block[b]);
        *n_blocks = i64(rep.blocks_processed);
        i64 w = 0;
        const auto ret = epikv::retained_positions(rep.cache);
        for (int l = 0; l < layers; ++l)
            for (int h = 0; h < hkv; ++h) {
                retained_counts[l * hkv + h] = i64(ret[size_t(l)][size_t(h)].size());
                for (auto p : ret[size_t(l)][size_t(h)]) retained_out[w++] = i64(p);
            }
        return 0;
    } catch (const std::exception& e) {
        return map_exception(e);
    }
}

}  // extern "C"
