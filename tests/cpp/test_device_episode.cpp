// test_device_episode.cpp -- the C++ host API of the throughput path
// (include/epikv/epikv_device.hpp: epikv::gpu::DeviceEpisode) against the
// reference library itself.
//
// Parity: a 2-layer, 4-KV-head episode (G = 2, p = 32, block 256, ragged layer
// budgets 512 / 384) runs 8 blocks of append -> fused tensor-core step.  Before
// every step the live device cache is read back as the reference's
// EpisodicCache (to_episodic_cache); after it, the reference's own
// evict_to_budget (kvcache.hpp:142-201) runs on that cache with the step's own
// scores, and the device result must equal it exactly: every head's entries in
// order, positions, and the bf16 keys / values widened to double.
//
// --timing: the cfg2 workload (Llama-3.2-3B shape: 28 layers, 24 Q / 8 KV
// heads, budget 8,192, block 2,048, p = 128) driven from C++: the episode is
// filled to its steady state, then K blocks of append + evict are timed with
// CUDA events on the episode's stream (inputs resident in HBM).
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

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

static void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        std::fprintf(stderr, "CUDA %s: %s\n", what, cudaGetErrorString(e));
        std::exit(2);
    }
}

// bf16 bits of a standard normal sample (round to nearest even)
static std::uint16_t bf16_normal(std::mt19937_64& g, std::normal_distribution<float>& n) {
    const float f = n(g);
    std::uint32_t u;
    std::memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return std::uint16_t(u >> 16);
}

static void* upload_normal(std::size_t count, std::mt19937_64& g) {
    std::normal_distribution<float> n(0.f, 1.f);
    std::vector<std::uint16_t> h(count);
    for (auto& x : h) x = bf16_normal(g, n);
    void* d = nullptr;
    cuda(cudaMalloc(&d, count * 2), "cudaMalloc");
    cuda(cudaMemcpy(d, h.data(), count * 2, cudaMemcpyHostToDevice), "H2D");
    return d;
}

static void parity() {
    const std::size_t L = 2, H = 4, G = 2, d = 128, p = 32, block = 256, blocks = 8;
    gpu::DeviceEpisode ep(L, H, {512, 384}, block);
    std::mt19937_64 g(7);
    const std::size_t rows = std::size_t(ep.layer_base()[L]);
    float* scores = nullptr;
    std::int32_t* positions = nullptr;
    cuda(cudaMalloc(&scores, rows * 4), "cudaMalloc");
    cuda(cudaMalloc(&positions, block * 4), "cudaMalloc");
    for (std::size_t b = 0; b < blocks; ++b) {
        void* k = upload_normal(L * H * block * d, g);
        void* v = upload_normal(L * H * block * d, g);
        void* q = upload_normal(L * H * G * p * d, g);
        void* kp = upload_normal(L * H * p * d, g);
        std::vector<std::int32_t> pos(block);
        for (std::size_t i = 0; i < block; ++i) pos[i] = std::int32_t(b * block + i);
        cuda(cudaMemcpy(positions, pos.data(), block * 4, cudaMemcpyHostToDevice), "H2D");
        ep.append(k, v, positions, block);
        const EpisodicCache before = gpu::to_episodic_cache(ep);
        // the input cache's row layout, to read the step's scores per (head, position)
        const epk_cache_desc in = ep.desc();
        std::vector<std::int32_t> off(L * (H + 1)), len(L * H);
        cuda(cudaMemcpy(off.data(), in.head_off, off.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        cuda(cudaMemcpy(len.data(), in.head_len, len.size() * 4, cudaMemcpyDeviceToHost), "D2H");
        ep.evict(q, kp, H * G, p, /*aggregation_max*/ b % 3 != 2, scores);
        const EpisodicCache after = gpu::to_episodic_cache(ep);
        std::vector<float> s(rows);
        cuda(cudaMemcpy(s.data(), scores, rows * 4, cudaMemcpyDeviceToHost), "D2H");
        const auto counts = ep.entries_per_layer();
        for (std::size_t l = 0; l < L; ++l) {
            LayerScores ls(H);
            for (std::size_t h = 0; h < H; ++h) {
                const std::size_t r0 = std::size_t(ep.layer_base()[l]) + std::size_t(off[l * (H + 1) + h]);
                for (std::size_t i = 0; i < std::size_t(len[l * H + h]); ++i)
                    ls[h][before.layers[l].heads[h][i].position] = double(s[r0 + i]);
            }
            const LayerCache ref = evict_to_budget(before.layers[l], ls);
            CHECK(after.layers[l].heads == ref.heads, ("step " + std::to_string(b) + " layer " + std::to_string(l) +
                                                       ": device cache == reference evict_to_budget")
                                                          .c_str());
            const std::size_t live = before.layers[l].entry_count();
            CHECK(counts[l] == std::min(live, H * std::size_t(ep.budgets()[l])), "kept count");
        }
        cudaFree(k);
        cudaFree(v);
        cudaFree(q);
        cudaFree(kp);
    }
    const auto rp = ep.retained_positions();
    const EpisodicCache fin = gpu::to_episodic_cache(ep);
    bool same = true;
    for (std::size_t l = 0; l < L; ++l)
        for (std::size_t h = 0; h < H; ++h) {
            same = same && rp[l][h].size() == fin.layers[l].heads[h].size();
            for (std::size_t i = 0; same && i < rp[l][h].size(); ++i)
                same = std::size_t(rp[l][h][i]) == fin.layers[l].heads[h][i].position;
        }
    CHECK(same, "retained_positions == to_episodic_cache positions");
    CHECK(ep.steps() == blocks, "step count");
    cudaFree(scores);
    cudaFree(positions);
}

static void timing(int steps) {
    const std::size_t L = 28, H = 8, G = 3, d = 128, p = 128, block = 2048, M = 8192;
    gpu::DeviceEpisode ep(L, H, {std::int64_t(M)}, block);
    std::mt19937_64 g(11);
    void* k = upload_normal(L * H * block * d, g);
    void* v = upload_normal(L * H * block * d, g);
    void* q = upload_normal(L * H * G * p * d, g);
    void* kp = upload_normal(L * H * p * d, g);
    std::int32_t* positions = nullptr;
    cuda(cudaMalloc(&positions, block * 4), "cudaMalloc");
    std::vector<std::int32_t> pos(block);
    std::size_t t = 0;
    auto next_block = [&]() {
        for (std::size_t i = 0; i < block; ++i) pos[i] = std::int32_t(t + i);
        t += block;
        cuda(cudaMemcpy(positions, pos.data(), block * 4, cudaMemcpyHostToDevice), "H2D");
    };
    // fill to the steady state: M / block + 1 blocks (the cache then holds H*M per layer before each append)
    for (std::size_t b = 0; b < M / block + 2; ++b) {
        next_block();
        ep.append(k, v, positions, block);
        ep.evict(q, kp, H * G, p);
    }
    ep.synchronize();
    // every timed step appends the same block K/V at fresh positions (positions
    // uploaded beforehand: 32 KB per step, outside the timed region)
    std::vector<std::int32_t*> pos_d(static_cast<std::size_t>(steps));
    for (auto& pd : pos_d) {
        cuda(cudaMalloc(&pd, block * 4), "cudaMalloc");
        for (std::size_t i = 0; i < block; ++i) pos[i] = std::int32_t(t + i);
        t += block;
        cuda(cudaMemcpy(pd, pos.data(), block * 4, cudaMemcpyHostToDevice), "H2D");
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, ep.stream());
    for (int s = 0; s < steps; ++s) {
        ep.append(k, v, pos_d[std::size_t(s)], block);
        ep.evict(q, kp, H * G, p);
    }
    cudaEventRecord(e1, ep.stream());
    ep.synchronize();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per = double(ms) / steps;
    const double live = double(L * H * (M + block));
    std::printf("cfg2 via epikv::gpu::DeviceEpisode (C++ host, append + fused step per block): %.4f ms/step, "
                "%.3e entries/s (%d steps)\n",
                per, live / (per / 1e3), steps);
    const auto counts = ep.entries_per_layer();
    bool ok = true;
    for (auto c : counts) ok = ok && c == H * M;
    CHECK(ok, "steady state keeps H*M per layer");
    for (auto pd : pos_d) cudaFree(pd);
    cudaFree(k);
    cudaFree(v);
    cudaFree(q);
    cudaFree(kp);
    cudaFree(positions);
}

int main(int argc, char** argv) {
    try {
        parity();
        if (argc > 1 && std::string(argv[1]) == "--timing") timing(argc > 2 ? std::atoi(argv[2]) : 50);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 2;
    }
    std::printf("device-episode checks: %d passed, %d failed\n", g_pass, g_fail);
    return g_fail ? 1 : 0;
}
