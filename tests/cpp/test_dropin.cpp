// test_dropin.cpp -- the C++ drop-in boundary (include/epikv/epikv_gpu.hpp)
// against the reference library itself, call for call, on the reference's own
// test scenarios (test_kvcache.cpp, acceptance_test.cpp C2/C3,
// test_scoring.cpp, test_clustering.cpp, test_allocation.cpp,
// test_blockprefill.cpp).  Built by tests/cpp/Makefile against the reference
// headers in place; run on a B200 by tests/test_gpu_cpp_dropin.py.
#include <cstdio>
#include <functional>
#include <set>

#include "epikv/epikv_gpu.hpp"

using namespace epikv;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, what)                                              \
    do {                                                               \
        if (cond) {                                                    \
            ++g_pass;                                                  \
        } else {                                                       \
            ++g_fail;                                                  \
            std::fprintf(stderr, "FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                              \
    } while (0)

template <typename F>
static std::string thrown(F f) {
    try {
        f();
    } catch (const DimensionError&) {
        return "DimensionError";
    } catch (const ZeroNormError&) {
        return "ZeroNormError";
    } catch (const Error&) {
        return "Error";
    }
    return "none";
}

static KVEntry entry(std::size_t p, Rng& rng, std::size_t dim = 4) {
    KVEntry e;
    e.position = p;
    for (std::size_t i = 0; i < dim; ++i) e.key.push_back(rng.gaussian());
    for (std::size_t i = 0; i < dim; ++i) e.value.push_back(rng.gaussian());
    return e;
}

static void test_evict() {
    Rng rng(2);
    {  // direct top-k (5,1,9,2), M=2 -> {0,2}   (test_kvcache.cpp:85-96)
        LayerCache cache(1, 2);
        LayerScores scores(1);
        const double s[] = {5, 1, 9, 2};
        for (std::size_t p = 0; p < 4; ++p) {
            cache.heads[0].push_back(entry(p, rng));
            scores[0][p] = s[p];
        }
        const LayerCache a = gpu::evict_to_budget(cache, scores);
        CHECK(a == evict_to_budget(cache, scores), "evict direct top-k");
        CHECK(a.heads[0].size() == 2 && a.heads[0][0].position == 0 && a.heads[0][1].position == 2, "evict {0,2}");
    }
    Rng r5(5);
    for (int trial = 0; trial < 200; ++trial) {  // test_kvcache.cpp:117-142
        const std::size_t heads = 1 + r5.uniform_index(2), budget = 1 + r5.uniform_index(4);
        LayerCache cache(heads, budget);
        LayerScores scores(heads);
        for (std::size_t h = 0; h < heads; ++h)
            for (std::size_t p = 0; p < 6; ++p) {
                cache.heads[h].push_back(entry(p, r5));
                scores[h][p] = double(r5.uniform_index(4));
            }
        std::unordered_set<std::size_t> pins;
        if (trial % 3 == 0 && heads * budget > heads) pins.insert(0);
        CHECK(gpu::evict_to_budget(cache, scores, pins) == evict_to_budget(cache, scores, pins), "evict 200 trials");
    }
    Rng r24(2024);
    for (int trial = 0; trial < 500; ++trial) {  // acceptance C3
        const std::size_t heads = 1 + r24.uniform_index(4), budget = 1 + r24.uniform_index(6),
                          block = 1 + r24.uniform_index(8), n = 1 + r24.uniform_index(budget + block);
        LayerCache cache(heads, budget);
        LayerScores scores(heads);
        for (std::size_t h = 0; h < heads; ++h)
            for (std::size_t p = 0; p < n; ++p) {
                KVEntry e;
                e.position = p;
                e.key = {r24.gaussian()};
                e.value = {r24.gaussian()};
                cache.heads[h].push_back(e);
                scores[h][p] = double(r24.uniform_index(5));
            }
        std::unordered_set<std::size_t> pins;
        if (trial % 4 == 0) pins.insert(0);
        CHECK(gpu::evict_to_budget(cache, scores, pins) == evict_to_budget(cache, scores, pins), "evict C3");
    }
    {  // errors: pin overflow -> Error, missing score -> DimensionError
        LayerCache cache(1, 1);
        LayerScores scores(1);
        std::unordered_set<std::size_t> pinned;
        for (std::size_t p = 0; p < 3; ++p) {
            cache.heads[0].push_back(entry(p, rng));
            scores[0][p] = 0.0;
            pinned.insert(p);
        }
        CHECK(thrown([&] { gpu::evict_to_budget(cache, scores, pinned); }) == "Error", "pin overflow throws Error");
        LayerScores missing(1);
        missing[0][0] = 1.0;
        CHECK(thrown([&] { gpu::evict_to_budget(cache, missing); }) == "DimensionError", "missing score");
        CHECK(thrown([&] { gpu::evict_to_budget(cache, LayerScores(2)); }) == "DimensionError", "head count");
    }
}

static ForwardTrace prompt_trace(std::size_t p, std::size_t cols, std::size_t H, std::size_t G, Rng* rng) {
    ForwardTrace trace;
    for (std::size_t i = 0; i < p; ++i) trace.positions.push_back(1000 + i);
    LayerTrace lt;
    lt.context_positions.resize(H);
    for (std::size_t h = 0; h < H; ++h) {
        for (std::size_t j = 0; j < cols; ++j) lt.context_positions[h].push_back(j);
        for (std::size_t i = 0; i < p; ++i) lt.context_positions[h].push_back(1000 + i);
    }
    for (std::size_t qh = 0; qh < H * G; ++qh) {
        Matrix grid(p, cols + p);
        if (rng)
            for (double& x : grid.values) x = rng->uniform();
        lt.attention.push_back(std::move(grid));
    }
    trace.layers.push_back(std::move(lt));
    return trace;
}

static bool same_map(const TokenScoreMap& a, const TokenScoreMap& b) {
    if (a.layers.size() != b.layers.size()) return false;
    for (std::size_t l = 0; l < a.layers.size(); ++l) {
        if (a.layers[l].size() != b.layers[l].size()) return false;
        for (std::size_t h = 0; h < a.layers[l].size(); ++h)
            if (a.layers[l][h] != b.layers[l][h]) return false;
    }
    return true;
}

static void test_scoring() {
    Rng rng(7);
    for (int trial = 0; trial < 100; ++trial) {  // test_scoring.cpp:97-111 shapes, bitwise
        const std::size_t p = 1 + rng.uniform_index(6), cols = 1 + rng.uniform_index(10);
        ForwardTrace t = prompt_trace(p, cols, 2, 2, &rng);
        for (Aggregation agg : {Aggregation::Avg, Aggregation::Max})
            CHECK(same_map(gpu::score_with_prompt(t, agg), score_with_prompt(t, agg)), "score random grids");
    }
    ForwardTrace t = prompt_trace(2, 3, 1, 2, nullptr);  // head 1 wins (test_scoring.cpp:136-149)
    for (std::size_t qh = 0; qh < 2; ++qh)
        for (std::size_t r = 0; r < 2; ++r)
            for (std::size_t j = 0; j < 3; ++j) t.layers[0].attention[qh].at(r, j) = 0.1 * double(j + 1) + 0.5 * double(qh);
    const TokenScoreMap m = gpu::score_with_prompt(t, Aggregation::Max);
    for (std::size_t j = 0; j < 3; ++j) CHECK(m.at(0, 0, j) == 0.1 * double(j + 1) + 0.5, "head 1 wins");
    ForwardTrace empty;
    empty.layers.resize(1);
    CHECK(thrown([&] { gpu::score_with_prompt(empty, Aggregation::Max); }) == "Error", "empty prompt throws");
    ForwardTrace bad = prompt_trace(2, 3, 1, 1, nullptr);
    bad.layers[0].attention.clear();
    CHECK(thrown([&] { gpu::score_with_prompt(bad, Aggregation::Max); }) == "DimensionError", "missing attention");
}

static void test_kmeans() {
    for (std::uint64_t seed : {1ull, 7ull, 11ull}) {
        Rng rng(seed);
        std::vector<Vec> pts(300, Vec(16));
        for (auto& p : pts)
            for (double& x : p) x = rng.gaussian();
        for (std::size_t k : {1u, 4u, 8u}) {
            const KMeansResult a = gpu::kmeans(pts, k, seed), b = kmeans(pts, k, seed);
            CHECK(a.assignments == b.assignments && a.centroids == b.centroids && a.iterations == b.iterations &&
                      a.sse_per_iteration == b.sse_per_iteration,
                  "kmeans bitwise");
        }
    }
    std::vector<Vec> few(2, Vec(3, 1.0));
    CHECK(thrown([&] { gpu::kmeans(few, 3, 1); }) == "Error", "kmeans fewer points");
}

static ModelConfig small(std::size_t layers, std::size_t q, std::size_t kv) {
    ModelConfig cfg;
    cfg.layers = layers;
    cfg.query_heads = q;
    cfg.kv_heads = kv;
    cfg.head_dim = 8;
    cfg.model_dim = q * 8;
    cfg.vocab = 128;
    cfg.seed = 3;
    return cfg;
}

static void test_sensitivity() {
    const Model model = init_model(small(3, 4, 2));
    const auto tokens = synthetic_calibration_tokens(64, 5, model.config.vocab);
    const SensitivityProfile a = gpu::measure_sensitivity(model, tokens, 16, 4);
    const SensitivityProfile b = measure_sensitivity(model, tokens, 16, 4);
    CHECK(a.sigma == b.sigma && a.sensitivity == b.sensitivity && a.skipped_zero_norm == b.skipped_zero_norm,
          "sensitivity bitwise");
    CHECK(allocate(a, 8, 1.1).layer_budgets == allocate(b, 8, 1.1).layer_budgets, "allocation from GPU sigma");
}

static PatchedPrompt fixed_prompt() {
    PatchedPrompt p;
    p.tokens = {7, 21, 42};
    return p;
}

static void test_block_prefill() {
    struct Case {
        std::size_t layers, q, kv, n, budget, block;
        ScorerKind scorer;
    };
    const Case cases[] = {{1, 1, 1, 9, 1, 3, ScorerKind::patched},   {2, 2, 2, 120, 8, 16, ScorerKind::patched},
                          {2, 4, 2, 100, 5, 12, ScorerKind::snapkv}, {2, 2, 1, 90, 6, 10, ScorerKind::kvzip},
                          {2, 2, 2, 70, 6, 16, ScorerKind::infinipot}, {2, 2, 2, 80, 8, 16, ScorerKind::streaming},
                          {2, 2, 2, 90, 7, 16, ScorerKind::keydiff},
                          {3, 6, 3, 200, 10, 24, ScorerKind::patched}};
    for (const Case& c : cases) {
        const Model model = init_model(small(c.layers, c.q, c.kv));
        const auto ctx = synthetic_calibration_tokens(c.n, 2, model.config.vocab);
        for (Aggregation agg : {Aggregation::Max, Aggregation::Avg}) {
            BlockPrefillConfig cfg;
            cfg.budget_per_head = c.budget;
            cfg.block_size = c.block;
            cfg.scorer = c.scorer;
            cfg.aggregation = agg;
            cfg.streaming_sink = 4;
            cfg.prompt_provider = [](std::size_t, std::size_t) { return fixed_prompt(); };
            const PrefillReport a = gpu::block_prefill(model, ctx, cfg), b = block_prefill(model, ctx, cfg);
            CHECK(retained_positions(a.cache) == retained_positions(b.cache), "block_prefill retained positions");
            CHECK(a.cache == b.cache, "block_prefill caches bitwise");
            CHECK(a.evictions_per_block == b.evictions_per_block, "block_prefill evictions");
            std::vector<std::size_t> sa, sb;
            for (const auto& s : a.occupancy.samples) sa.push_back(s.entries_per_layer[0]);
            for (const auto& s : b.occupancy.samples) sb.push_back(s.entries_per_layer[0]);
            CHECK(sa == sb, "block_prefill occupancy");
        }
    }
    {  // allocated budgets {4, 12} (test_blockprefill.cpp:176-189)
        const Model model = init_model(small(2, 2, 1));
        const auto ctx = synthetic_calibration_tokens(64, 17, model.config.vocab);
        BlockPrefillConfig cfg;
        cfg.budget_per_head = 8;
        cfg.block_size = 16;
        cfg.prompt_provider = [](std::size_t, std::size_t) { return fixed_prompt(); };
        BudgetAllocation alloc;
        alloc.alpha = 1.0;
        alloc.per_head_budget = 8;
        alloc.weights = {0.25, 0.75};
        alloc.layer_budgets = {4, 12};
        cfg.allocation = alloc;
        const PrefillReport a = gpu::block_prefill(model, ctx, cfg);
        CHECK(a.cache.layers[0].entry_count() == 4 && a.cache.layers[1].entry_count() == 12, "allocation {4,12}");
    }
}

int main() {
    test_evict();
    test_scoring();
    test_kmeans();
    test_sensitivity();
    test_block_prefill();
    std::printf("drop-in checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
