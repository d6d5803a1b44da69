// test_forward.cpp -- the model step before the hot path on the GPU
// (epikv::gpu::forward over epk_toy_forward) against the
// reference forward (toymodel.hpp:228-411) itself:
//   * Softmax::host: keys, values, context positions, attention grids and the
//     hidden state bit-identical, causal and sink+recent masks, with and
//     without a past cache (the reference's prefix-consistency setup,
//     test_toymodel.cpp:212-240);
//   * Softmax::device: within 1e-13 relative (CUDA exp vs std::exp);
//   * gpu::block_prefill with both forwards on the GPU == the reference
//     block_prefill bit for bit (reports, caches), and gpu::measure_sensitivity
//     with device forwards == the reference's;
//   * a timing line: reference block_prefill vs gpu::block_prefill with host
//     forwards vs with device forwards.
#include <chrono>
#include <cmath>
#include <cstdio>

#include "epikv/epikv_gpu.hpp"

using namespace epikv;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, what)                                                        \
    do {                                                                         \
        if (cond) {                                                              \
            ++g_pass;                                                            \
        } else {                                                                 \
            ++g_fail;                                                            \
            std::fprintf(stderr, "FAIL %s (%s:%d)\n", what, __FILE__, __LINE__); \
        }                                                                        \
    } while (0)

static ModelConfig config(std::size_t layers, std::size_t q, std::size_t kv, std::size_t dh, std::size_t vocab,
                          std::uint64_t seed) {
    ModelConfig c;
    c.layers = layers;
    c.query_heads = q;
    c.kv_heads = kv;
    c.head_dim = dh;
    c.model_dim = q * dh;
    c.vocab = vocab;
    c.seed = seed;
    return c;
}

// normwise: max |a - b| over max |a| of the array (attention weights span
// hundreds of orders of magnitude; elementwise ratios of the tiniest are noise)
static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return 1e300;
    double m = 0.0, s = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        m = std::max(m, std::fabs(a[i] - b[i]));
        s = std::max(s, std::fabs(a[i]));
    }
    return s > 0 ? m / s : m;
}

static double trace_rel(const ForwardTrace& a, const ForwardTrace& b) {
    double m = max_rel(a.hidden.values, b.hidden.values);
    for (std::size_t l = 0; l < a.layers.size(); ++l) {
        for (std::size_t h = 0; h < a.layers[l].keys.size(); ++h) {
            m = std::max(m, max_rel(a.layers[l].keys[h].values, b.layers[l].keys[h].values));
            m = std::max(m, max_rel(a.layers[l].values[h].values, b.layers[l].values[h].values));
        }
        for (std::size_t q = 0; q < a.layers[l].attention.size(); ++q)
            m = std::max(m, max_rel(a.layers[l].attention[q].values, b.layers[l].attention[q].values));
    }
    return m;
}

static bool trace_equal(const ForwardTrace& a, const ForwardTrace& b) {
    if (a.positions != b.positions || a.layers.size() != b.layers.size() || a.hidden.values != b.hidden.values)
        return false;
    for (std::size_t l = 0; l < a.layers.size(); ++l) {
        const LayerTrace &x = a.layers[l], &y = b.layers[l];
        if (x.context_positions != y.context_positions || x.keys.size() != y.keys.size() ||
            x.attention.size() != y.attention.size())
            return false;
        for (std::size_t h = 0; h < x.keys.size(); ++h)
            if (x.keys[h].values != y.keys[h].values || x.values[h].values != y.values[h].values) return false;
        for (std::size_t q = 0; q < x.attention.size(); ++q)
            if (x.attention[q].values != y.attention[q].values || x.attention[q].cols != y.attention[q].cols)
                return false;
    }
    return true;
}

static std::vector<TokenId> tokens(std::size_t n, std::size_t vocab, std::uint64_t seed) {
    Rng rng(seed);
    std::vector<TokenId> t(n);
    for (auto& x : t) x = TokenId(rng.uniform_index(vocab));
    return t;
}

static double worst_device_rel = 0.0;

static void test_forward() {
    for (const ModelConfig& cfg : {config(2, 4, 2, 8, 128, 3), config(3, 6, 2, 16, 300, 7), config(1, 8, 8, 32, 64, 9)}) {
        const Model model = init_model(cfg);
        const auto ctx_tok = tokens(40, cfg.vocab, 1);
        const auto new_tok = tokens(9, cfg.vocab, 2);
        std::vector<std::size_t> pos0(40), pos1(9);
        for (std::size_t i = 0; i < 40; ++i) pos0[i] = 3 * i;
        for (std::size_t i = 0; i < 9; ++i) pos1[i] = 200 + 2 * i;
        for (const MaskSpec& mask : {MaskSpec::causal(), MaskSpec::sink_recent(4, 11)}) {
            const ForwardTrace a = forward(model, ctx_tok, pos0, mask);
            const ForwardTrace b = gpu::forward(model, ctx_tok, pos0, mask);
            CHECK(trace_equal(a, b), "forward no cache bitwise");
            const ForwardTrace c = gpu::forward(model, ctx_tok, pos0, mask, nullptr, {}, gpu::Softmax::device);
            const double rel = trace_rel(a, c);
            worst_device_rel = std::max(worst_device_rel, rel);
            CHECK(rel < 1e-13, "forward device softmax 1e-13 (normwise)");
            // a past cache (appended + evicted, so heads are ragged)
            EpisodicCache cache = make_empty_cache(cfg, 12);
            append_to_cache(cache, a);
            Rng rng(5);
            for (auto& layer : cache.layers) {
                LayerScores sc(layer.heads.size());
                for (std::size_t h = 0; h < layer.heads.size(); ++h)
                    for (const KVEntry& e : layer.heads[h]) sc[h][e.position] = rng.uniform();
                layer = evict_to_budget(layer, sc);
            }
            const ForwardTrace d = forward(model, new_tok, pos1, mask, &cache);
            const ForwardTrace e = gpu::forward(model, new_tok, pos1, mask, &cache);
            CHECK(trace_equal(d, e), "forward with past cache bitwise");
            TraceOptions no;
            no.store_attention = false;
            CHECK(trace_equal(forward(model, new_tok, pos1, mask, &cache, no),
                              gpu::forward(model, new_tok, pos1, mask, &cache, no)),
                  "forward without attention bitwise");
        }
        // error paths as the reference
        std::vector<TokenId> bad = {TokenId(cfg.vocab)};
        std::vector<std::size_t> p1 = {0};
        bool threw = false;
        try {
            gpu::forward(model, bad, p1, MaskSpec::causal());
        } catch (const Error&) {
            threw = true;
        }
        CHECK(threw, "forward out-of-vocab throws");
    }
}

static PatchedPrompt fixed_prompt(std::size_t vocab) {
    PatchedPrompt p;
    p.tokens = {TokenId(7 % vocab), TokenId(21 % vocab), TokenId(42 % vocab), TokenId(5 % vocab)};
    return p;
}

static bool same_report(const PrefillReport& a, const PrefillReport& b) {
    if (a.evictions_per_block != b.evictions_per_block || a.blocks_processed != b.blocks_processed) return false;
    if (a.occupancy.samples.size() != b.occupancy.samples.size()) return false;
    if (retained_positions(a.cache) != retained_positions(b.cache)) return false;
    for (std::size_t l = 0; l < a.cache.layers.size(); ++l)
        if (!(a.cache.layers[l] == b.cache.layers[l])) return false;
    return true;
}

static void test_block_prefill_device_forward() {
    const ModelConfig cfg = config(2, 4, 2, 16, 256, 11);
    const Model model = init_model(cfg);
    const auto ctx = tokens(150, cfg.vocab, 3);
    BlockPrefillConfig bp;
    bp.budget_per_head = 16;
    bp.block_size = 24;
    const PatchedPrompt prompt = fixed_prompt(cfg.vocab);
    bp.prompt_provider = [prompt](std::size_t, std::size_t) { return prompt; };
    const PrefillReport ref = block_prefill(model, ctx, bp);
    gpu::PrefillForward fwd;
    fwd.block_on_device = fwd.prompt_on_device = true;
    const PrefillReport got = gpu::block_prefill(model, ctx, bp, 0, {}, fwd);
    CHECK(same_report(ref, got), "block_prefill with device forwards == reference");
    for (ScorerKind sk : {ScorerKind::snapkv, ScorerKind::keydiff}) {
        BlockPrefillConfig b2 = bp;
        b2.scorer = sk;
        CHECK(same_report(block_prefill(model, ctx, b2), gpu::block_prefill(model, ctx, b2, 0, {}, fwd)),
              "block_prefill device forwards, baseline scorers");
    }
    const auto cal = synthetic_calibration_tokens(64, 5, cfg.vocab);
    const SensitivityProfile a = measure_sensitivity(model, cal, 16, 4);
    const SensitivityProfile b = gpu::measure_sensitivity(model, cal, 16, 4, "", gpu::Softmax::host);
    CHECK(a.sigma == b.sigma && a.skipped_zero_norm == b.skipped_zero_norm, "measure_sensitivity device forwards");
}

static void timing() {
    // a toy model where the prompt pass's attention over the cache matters:
    // 2 layers, 8 query / 4 kv heads of 64 (model dim 512), 4,096-token
    // context, blocks of 256, budget 512 per head, a 32-token patched prompt
    const ModelConfig cfg = config(2, 8, 4, 64, 512, 13);
    const Model model = init_model(cfg);
    const auto ctx = tokens(4096, cfg.vocab, 9);
    BlockPrefillConfig bp;
    bp.budget_per_head = 512;
    bp.block_size = 256;
    PatchedPrompt prompt;
    prompt.tokens = tokens(32, cfg.vocab, 10);
    bp.prompt_provider = [prompt](std::size_t, std::size_t) { return prompt; };
    using clk = std::chrono::steady_clock;
    auto t0 = clk::now();
    const PrefillReport ref = block_prefill(model, ctx, bp);
    auto t1 = clk::now();
    const PrefillReport host_fwd = gpu::block_prefill(model, ctx, bp);
    auto t2 = clk::now();
    gpu::PrefillForward fwd;
    fwd.block_on_device = fwd.prompt_on_device = true;
    const PrefillReport dev_fwd = gpu::block_prefill(model, ctx, bp, 0, {}, fwd);
    auto t3 = clk::now();
    const double a = std::chrono::duration<double>(t1 - t0).count(), b = std::chrono::duration<double>(t2 - t1).count(),
                 c = std::chrono::duration<double>(t3 - t2).count();
    CHECK(same_report(ref, host_fwd) && same_report(ref, dev_fwd), "timing runs agree with the reference");
    std::printf("block_prefill 2x(8q/4kv x 64), 4096 tokens, block 256, M 512, p 32: reference %.2f s, "
                "gpu (host forwards) %.2f s, gpu (device forwards) %.2f s\n", a, b, c);
}

int main(int argc, char** argv) {
    try {
        test_forward();
        test_block_prefill_device_forward();
        if (argc > 1 && std::string(argv[1]) == "--timing") timing();
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("device-softmax forward: max normwise relative difference %.3g\n", worst_device_rel);
    std::printf("forward checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
