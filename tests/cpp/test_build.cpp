// test_build.cpp -- Phase A over several GPUs (epikv::gpu::build,
// include/epikv/epikv_gpu.hpp) against the reference build (episodic.hpp:108-199)
// itself: every persisted .epkv file and the manifest must be byte-identical
// to the reference's, for one device, for several host threads / contexts
// (one GPU listed twice or three times -- the multi-GPU code path on a
// one-GPU box) and with the k-means embeddings sharded over the devices (the
// ordered chain of epk_kmeans_sharded).  The analogue of
// test_episodic.cpp:274-302 (rebuild / parallel == sequential, bitwise).
// Also gpu::kmeans_sharded vs the reference kmeans on 1..4 shards.
// Built by tests/cpp/Makefile against the reference headers in place; run on
// a B200 by tests/test_gpu_cpp_dropin.py (also with EPK_FORCE_NCCL=1, which
// routes the one-device chain through NCCL).
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <sstream>

#include "epikv/epikv_gpu.hpp"

using namespace epikv;
namespace fs = std::filesystem;

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

// A topic-blocked synthetic conversation in the reference's JSONL format
// (parse_conversation, dialogue.hpp:96-154): each topic draws its words from
// its own pool, so k-means finds the topics as episodes.
static ConversationHistory conversation(std::size_t topics, std::size_t turns, std::uint64_t seed) {
    Rng rng(seed);
    std::ostringstream out;
    for (std::size_t t = 0; t < topics; ++t) {
        if (t > 0) out << "{\"kind\":\"session_break\"}\n";
        for (std::size_t j = 0; j < turns; ++j) {
            out << "{\"kind\":\"turn\",\"role\":\"" << (j % 2 ? "speaker_2" : "speaker_1") << "\",\"text\":\"";
            const std::size_t words = 6 + rng.uniform_index(5);
            for (std::size_t w = 0; w < words; ++w)
                out << (w ? " " : "") << "t" << t << "w" << rng.uniform_index(24);
            out << "\"}\n";
        }
    }
    out << "{\"kind\":\"query\",\"text\":\"t0w1 t0w2?\"}\n";
    std::istringstream in(out.str());
    return parse_conversation(in).first;
}

static std::vector<char> bytes(const fs::path& p) {
    std::ifstream in(p, std::ios::binary);
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

static void same_store(const fs::path& a, const fs::path& b, std::size_t E, const char* what) {
    bool ok = true;
    for (std::size_t e = 0; e < E; ++e) {
        const std::string name = "episode_" + std::to_string(e) + ".epkv";
        const auto x = bytes(a / name), y = bytes(b / name);
        ok = ok && !x.empty() && x == y;
    }
    ok = ok && bytes(a / "manifest.json") == bytes(b / "manifest.json");
    CHECK(ok, what);
}

static void test_build(const fs::path& root) {
    struct Case {
        ModelConfig cfg;
        std::size_t topics, turns, E, budget, block;
        bool alloc;
    };
    ModelConfig small;
    small.layers = 2;
    small.query_heads = 2;
    small.kv_heads = 1;
    small.head_dim = 8;
    small.model_dim = 16;
    small.seed = 9;
    ModelConfig gqa;
    gqa.layers = 3;
    gqa.query_heads = 4;
    gqa.kv_heads = 2;
    gqa.head_dim = 16;
    gqa.model_dim = 64;
    gqa.seed = 5;
    const Case cases[] = {{small, 3, 8, 3, 8, 16, true}, {gqa, 4, 10, 4, 12, 32, true}, {gqa, 5, 6, 5, 6, 8, false}};
    int ci = 0;
    for (const Case& c : cases) {
        const ConversationHistory history = conversation(c.topics, c.turns, 100 + ci);
        const Model model = init_model(c.cfg);
        const HashEmbedder embedder;
        EpisodicBuildConfig config;
        config.block_size = c.block;
        config.use_allocation = c.alloc;
        const fs::path dir = root / ("case" + std::to_string(ci++));
        const BuildResult ref = build(model, history, c.E, c.budget, 1.1, embedder, (dir / "ref").string(), config);
        const std::vector<std::pair<std::string, gpu::BuildDevices>> variants = {
            {"gpu1", {{0}, false}}, {"gpu2", {{0, 0}, false}}, {"gpu3_sharded_kmeans", {{0, 0, 0}, true}}};
        for (const auto& [name, where] : variants) {
            const BuildResult got =
                gpu::build(model, history, c.E, c.budget, 1.1, embedder, (dir / name).string(), config, where);
            same_store(dir / "ref", dir / name, c.E, ("build store bytes: " + name).c_str());
            bool reports = got.reports.size() == ref.reports.size();
            for (std::size_t e = 0; reports && e < c.E; ++e)
                reports = got.reports[e].evictions_per_block == ref.reports[e].evictions_per_block &&
                          retained_positions(got.reports[e].cache) == retained_positions(ref.reports[e].cache);
            CHECK(reports, ("build reports: " + name).c_str());
            CHECK(got.set.allocation.layer_budgets == ref.set.allocation.layer_budgets, "build allocation");
            CHECK(got.set.episodes.centroids == ref.set.episodes.centroids, "build centroids");
        }
    }
}

static void test_kmeans_sharded() {
    Rng rng(31);
    for (std::size_t trial = 0; trial < 4; ++trial) {
        const std::size_t n = 97 + 211 * trial, dim = 16 + 40 * trial, k = 2 + trial;
        std::vector<Vec> pts(n, Vec(dim));
        for (auto& p : pts)
            for (double& x : p) x = rng.gaussian() + double(rng.uniform_index(3));
        const KMeansResult ref = kmeans(pts, k, 7 + trial);
        for (std::size_t shards = 1; shards <= 4; ++shards) {
            const KMeansResult got = gpu::kmeans_sharded(pts, k, 7 + trial, std::vector<int>(shards, 0));
            CHECK(got.assignments == ref.assignments && got.centroids == ref.centroids &&
                      got.iterations == ref.iterations && got.sse_per_iteration == ref.sse_per_iteration,
                  "kmeans_sharded == reference kmeans");
        }
    }
    // an empty cluster forces the repair path: duplicated points
    std::vector<Vec> dup(40, Vec(4, 1.0));
    for (std::size_t i = 0; i < 5; ++i) dup[i] = Vec{double(i), 0.0, 2.0, -1.0};
    const KMeansResult ref = kmeans(dup, 6, 3);
    const KMeansResult got = gpu::kmeans_sharded(dup, 6, 3, {0, 0, 0});
    CHECK(got.assignments == ref.assignments && got.centroids == ref.centroids, "kmeans_sharded repair");
}

int main() {
    const fs::path root = fs::temp_directory_path() / "epk_test_build";
    fs::remove_all(root);
    fs::create_directories(root);
    try {
        test_kmeans_sharded();
        test_build(root);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        ++g_fail;
    }
    fs::remove_all(root);
    std::printf("build checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
