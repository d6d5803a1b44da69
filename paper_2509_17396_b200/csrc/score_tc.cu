// score_tc.cu -- K1: the tensor-core patched-prompt scorer (bf16 in, fp32
// accumulate), tcgen05 MMAs with TMEM accumulators fed by TMA.
//
// Computes the same quantity as score_f32.cu / score_with_prompt
// (scoring.hpp:80-128 over the attention weights of toymodel.hpp:327-391):
//   score(j) = max_{g,t} exp(l_{g,t,j} - lse_{g,t})     (Aggregation::Max)
//   score(j) = max_g (1/p) sum_t exp(l_{g,t,j} - lse_{g,t})   (Avg)
// with l = q.k * d^-1/2 and lse_{g,t} the log-sum-exp of row (g,t) over the
// n_h cache columns plus the causal prompt columns 0..t.  The attention grid
// never exists in memory: two passes over K (the second mostly from L2):
//
//   P1 (row stats)  per (layer, kv-head, 128-query-row block, column split):
//       A = Q block [128 x 128] (smem, TMA), B = K tile [128 cols x 128]
//       (4-stage TMA ring), D = 128x128 fp32 in TMEM (2 slots).  Epilogue
//       warps own one query row each (TMEM lane) and keep an online
//       (max, sum of exp2) over the columns -> partial (m, Z) per split.
//   merge           lse2 = log2-sum-exp2 over splits (+inf for pad rows).
//   P2 (col scores) per (layer, kv-head, 128-row cache tile): A = K tile,
//       B = Q chunk [128 query rows] (resident per head when it fits),
//       D = 128x128 in TMEM (4 slots).  Epilogue lanes own one cache row and
//       reduce max_r (x*c2 - lse2[r]) over every query row -> one exp2 per
//       (cache row): score.
//
// Warp roles per CTA (192 threads): warp 0 TMA producer, warp 1 TMEM
// allocator + MMA issuer (one elected lane), warps 2-5 epilogue.
// Persistent grid (one CTA per SM), contiguous item ranges so Q stays in
// shared memory across consecutive items of the same head.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>

#include "epk_internal.cuh"
#include "sm100.cuh"

namespace epk {

using namespace sm100;

constexpr int kD = 128;
constexpr int kTile = 128;
constexpr int kTileBytes = kTile * kD * 2;  // 32 KB: two 16 KB swizzled d-halves
constexpr int kHalfBytes = kTileBytes / 2;
constexpr int kSplitTiles = 16;  // P1 column split: 2048 cache columns
constexpr int kP1Stages = 4;
constexpr int kP2Stages = 2;
constexpr int kP2QSlots = 4;
constexpr int kThreads = 192;
constexpr uint32_t kIdesc = idesc_bf16_f32(128, 128);

struct TcParams {
    LayerTable lt;
    int L, H, Hq, G, p, Gp, NQ;
    int tiles_max;     // ceil(n_max / 128)
    int splits;        // P1 splits per (layer, head, row block)
    int prompt_tiles;  // ceil(p / 128)
    const int32_t* head_off;
    const int32_t* head_len;
    float c2;  // d^-1/2 * log2(e)
    float* part_m;
    float* part_z;
    float* lse2;
    float* scores;
    int agg_max;
    int64_t items;
};

// MMA of one 128x128x128 tile: 8 K-steps of 16 (32 bytes) across the two
// 64-element swizzled halves of each operand.
__device__ __forceinline__ void mma_tile(uint32_t d_tmem, const uint8_t* a, const uint8_t* b) {
    const uint32_t a0 = smem_u32(a), b0 = smem_u32(b);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = uint32_t((kk >> 2) * kHalfBytes + (kk & 3) * 32);
        mma_bf16_ss(d_tmem, sdesc_k_sw128(a0 + off), sdesc_k_sw128(b0 + off), kIdesc, kk > 0 ? 1u : 0u);
    }
}

__device__ __forceinline__ void load_tile(uint8_t* dst, const CUtensorMap* map, uint64_t* bar, int row) {
    tma_load_2d(dst, map, bar, 0, row);
    tma_load_2d(dst + kHalfBytes, map, bar, 64, row);
}

struct P1Item {
    int l, h, rb, s;
    int n_h;
    int64_t krow0;   // first K row of the head (global)
    int cache_t0, cache_t1;
    int prompt_tiles;
    __device__ int ntiles() const { return (cache_t1 > cache_t0 ? cache_t1 - cache_t0 : 0) + prompt_tiles; }
};

__device__ __forceinline__ P1Item p1_item(const TcParams& P, int64_t it) {
    P1Item x;
    x.s = int(it % P.splits);
    int64_t r = it / P.splits;
    x.rb = int(r % P.NQ);
    r /= P.NQ;
    x.h = int(r % P.H);
    x.l = int(r / P.H);
    x.n_h = P.head_len[x.l * P.H + x.h];
    x.krow0 = P.lt.base[x.l] + P.head_off[x.l * (P.H + 1) + x.h];
    const int tiles = (x.n_h + kTile - 1) / kTile;
    x.cache_t0 = x.s * kSplitTiles;
    x.cache_t1 = min(tiles, x.cache_t0 + kSplitTiles);
    x.prompt_tiles = (x.s == P.splits - 1) ? P.prompt_tiles : 0;
    return x;
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_rowstats_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + kTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sK + kP1Stages * kTileBytes);
    uint64_t* k_full = bars;
    uint64_t* k_empty = bars + kP1Stages;
    uint64_t* q_full = bars + 2 * kP1Stages;
    uint64_t* q_empty = q_full + 1;
    uint64_t* t_full = q_empty + 1;
    uint64_t* t_empty = t_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = (P.items + gridDim.x - 1) / gridDim.x;
    const int64_t it_beg = int64_t(blockIdx.x) * per;
    const int64_t it_end = min(P.items, it_beg + per);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_kp);
        for (int s = 0; s < kP1Stages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&t_full[s], 1);
            mbar_init(&t_empty[s], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer ----------------
            int ks = 0;
            uint32_t kph = 0, qloads = 0;
            int64_t qkey = -1;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const P1Item x = p1_item(P, it);
                if (x.ntiles() == 0) continue;
                const int64_t key = it / P.splits;
                if (key != qkey) {
                    mbar_wait(q_empty, (qloads & 1) ^ 1);
                    mbar_expect_tx(q_full, kTileBytes);
                    const int qrow = (x.l * P.Hq + x.h * P.G) * P.p + x.rb * kTile;
                    load_tile(sQ, &tm_q, q_full, qrow);
                    ++qloads;
                    qkey = key;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    mbar_wait(&k_empty[ks], kph ^ 1);
                    mbar_expect_tx(&k_full[ks], kTileBytes);
                    const int nc = x.cache_t1 > x.cache_t0 ? x.cache_t1 - x.cache_t0 : 0;
                    if (t < nc)
                        load_tile(sK + ks * kTileBytes, &tm_k, &k_full[ks], int(x.krow0 + int64_t(x.cache_t0 + t) * kTile));
                    else
                        load_tile(sK + ks * kTileBytes, &tm_kp, &k_full[ks],
                                  (x.l * P.H + x.h) * P.p + (t - nc) * kTile);
                    if (++ks == kP1Stages) {
                        ks = 0;
                        kph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            int ks = 0, ts = 0;
            uint32_t kph = 0, tph = 0, qloads = 0;
            int64_t qkey = -1;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const P1Item x = p1_item(P, it);
                if (x.ntiles() == 0) continue;
                const int64_t key = it / P.splits;
                if (key != qkey) {
                    if (qloads > 0) mma_commit(q_empty);  // previous Q free once its MMAs retire
                    mbar_wait(q_full, qloads & 1);
                    ++qloads;
                    qkey = key;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    mbar_wait(&t_empty[ts], tph ^ 1);
                    mbar_wait(&k_full[ks], kph);
                    tc_fence_after();
                    mma_tile(tmem + uint32_t(ts * kTile), sQ, sK + ks * kTileBytes);
                    mma_commit(&k_empty[ks]);
                    mma_commit(&t_full[ts]);
                    if (++ks == kP1Stages) {
                        ks = 0;
                        kph ^= 1;
                    }
                    if (++ts == 2) {
                        ts = 0;
                        tph ^= 1;
                    }
                }
            }
        }
    } else {  // ---------------- epilogue: one query row per thread ----------------
        const int quarter = warp & 3;
        const int r_local = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        int ts = 0;
        uint32_t tph = 0;
        for (int64_t it = it_beg; it < it_end; ++it) {
            const P1Item x = p1_item(P, it);
            const int rq = x.rb * kTile + r_local;  // query row within the head (g*p + t)
            const int t_pos = rq % P.p;
            float m = -INFINITY, z = 0.0f;
            const int nc = x.cache_t1 > x.cache_t0 ? x.cache_t1 - x.cache_t0 : 0;
            for (int t = 0; t < x.ntiles(); ++t) {
                int lim;
                if (t < nc) {
                    lim = x.n_h - (x.cache_t0 + t) * kTile;
                } else {
                    const int c0 = (t - nc) * kTile;
                    lim = min(P.p, t_pos + 1) - c0;
                }
                mbar_wait(&t_full[ts], tph);
                tc_fence_after();
#pragma unroll 1
                for (int sub = 0; sub < 4; ++sub) {
                    float v[32];
                    tmem_ld32(tmem + lane_addr + uint32_t(ts * kTile + sub * 32), v);
                    const int base = sub * 32;
                    float mx = -INFINITY;
                    if (lim >= base + 32) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            v[i] *= P.c2;
                            mx = fmaxf(mx, v[i]);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            v[i] = (base + i < lim) ? v[i] * P.c2 : -INFINITY;
                            mx = fmaxf(mx, v[i]);
                        }
                    }
                    if (mx > m) {
                        z *= ex2(m - mx);
                        m = mx;
                    }
                    if (m != -INFINITY) {
                        float s0 = 0.f, s1 = 0.f;
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            s0 += ex2(v[i] - m);
                            s1 += ex2(v[i + 1] - m);
                        }
                        z += s0 + s1;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&t_empty[ts]);
                if (++ts == 2) {
                    ts = 0;
                    tph ^= 1;
                }
            }
            const int64_t o = ((int64_t(x.l) * P.H + x.h) * (P.NQ * kTile) + rq) * P.splits + x.s;
            P.part_m[o] = m;
            P.part_z[o] = z;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 256);
}

// lse2 per query row = log2 sum_s Z_s 2^(m_s - M) + M over the splits.
__global__ void tc_merge_kernel(const __grid_constant__ TcParams P) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t rows = int64_t(P.L) * P.H * P.NQ * kTile;
    if (idx >= rows) return;
    const int rq = int(idx % (P.NQ * kTile));
    if (rq >= P.Gp) {
        P.lse2[idx] = INFINITY;
        return;
    }
    float M = -INFINITY;
    for (int s = 0; s < P.splits; ++s) M = fmaxf(M, P.part_m[idx * P.splits + s]);
    float Z = 0.f;
    if (M != -INFINITY)
        for (int s = 0; s < P.splits; ++s) {
            const float ms = P.part_m[idx * P.splits + s];
            if (ms != -INFINITY) Z += P.part_z[idx * P.splits + s] * ex2(ms - M);
        }
    P.lse2[idx] = M + log2f(Z);
}

struct P2Item {
    int l, h, tile, n_h;
    int64_t krow0;
    __device__ bool live() const { return tile * kTile < n_h; }
};

__device__ __forceinline__ P2Item p2_item(const TcParams& P, int64_t it) {
    P2Item x;
    x.tile = int(it % P.tiles_max);
    const int64_t r = it / P.tiles_max;
    x.h = int(r % P.H);
    x.l = int(r / P.H);
    x.n_h = P.head_len[x.l * P.H + x.h];
    x.krow0 = P.lt.base[x.l] + P.head_off[x.l * (P.H + 1) + x.h];
    return x;
}

__global__ void __launch_bounds__(kThreads, 1)
    tc_colscore_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_q) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;                            // kP2QSlots x 32 KB
    uint8_t* sK = smem + kP2QSlots * kTileBytes;   // kP2Stages x 32 KB
    float* s_lse = reinterpret_cast<float*>(sK + kP2Stages * kTileBytes);  // NQ*128
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lse + P.NQ * kTile);
    uint64_t* k_full = bars;
    uint64_t* k_empty = k_full + kP2Stages;
    uint64_t* q_full = k_empty + kP2Stages;
    uint64_t* q_empty = q_full + kP2QSlots;
    uint64_t* t_full = q_empty + kP2QSlots;
    uint64_t* t_empty = t_full + 4;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = (P.items + gridDim.x - 1) / gridDim.x;
    const int64_t it_beg = int64_t(blockIdx.x) * per;
    const int64_t it_end = min(P.items, it_beg + per);
    const bool resident = P.NQ <= kP2QSlots;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_q);
        for (int s = 0; s < kP2Stages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < kP2QSlots; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < 4; ++s) {
            mbar_init(&t_full[s], 1);
            mbar_init(&t_empty[s], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer ----------------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kP2QSlots] = {0, 0, 0, 0};
            int64_t head_key = -1;
            int64_t job = 0;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const P2Item x = p2_item(P, it);
                if (!x.live()) continue;
                mbar_wait(&k_empty[ks], kph ^ 1);
                mbar_expect_tx(&k_full[ks], kTileBytes);
                load_tile(sK + ks * kTileBytes, &tm_k, &k_full[ks], int(x.krow0 + int64_t(x.tile) * kTile));
                if (++ks == kP2Stages) {
                    ks = 0;
                    kph ^= 1;
                }
                const int64_t hk = int64_t(x.l) * P.H + x.h;
                const bool reload = !resident || hk != head_key;
                head_key = hk;
                for (int c = 0; c < P.NQ; ++c, ++job) {
                    if (!reload) continue;
                    const int slot = resident ? c : int(job % kP2QSlots);
                    mbar_wait(&q_empty[slot], (qload[slot] & 1) ^ 1);
                    mbar_expect_tx(&q_full[slot], kTileBytes);
                    load_tile(sQ + slot * kTileBytes, &tm_q, &q_full[slot], int(hk / P.H * P.Hq * P.p) +
                              (x.h * P.G) * P.p + c * kTile);
                    ++qload[slot];
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer ----------------
            int ks = 0, ts = 0;
            uint32_t kph = 0, tph = 0;
            uint32_t qload[kP2QSlots] = {0, 0, 0, 0};
            int64_t head_key = -1;
            int64_t job = 0;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const P2Item x = p2_item(P, it);
                if (!x.live()) continue;
                const int64_t hk = int64_t(x.l) * P.H + x.h;
                const bool reload = !resident || hk != head_key;
                if (resident && reload && head_key >= 0)
                    for (int c = 0; c < P.NQ; ++c) mma_commit(&q_empty[c]);  // old head's Q retires
                head_key = hk;
                mbar_wait(&k_full[ks], kph);
                for (int c = 0; c < P.NQ; ++c, ++job) {
                    const int slot = resident ? c : int(job % kP2QSlots);
                    if (reload) {
                        mbar_wait(&q_full[slot], qload[slot] & 1);
                        ++qload[slot];
                    }
                    mbar_wait(&t_empty[ts], tph ^ 1);
                    tc_fence_after();
                    mma_tile(tmem + uint32_t(ts * kTile), sK + ks * kTileBytes, sQ + slot * kTileBytes);
                    mma_commit(&t_full[ts]);
                    if (!resident) mma_commit(&q_empty[slot]);
                    if (++ts == 4) {
                        ts = 0;
                        tph ^= 1;
                    }
                }
                mma_commit(&k_empty[ks]);
                if (++ks == kP2Stages) {
                    ks = 0;
                    kph ^= 1;
                }
            }
        }
    } else {  // ---------------- epilogue: one cache row per thread ----------------
        const int quarter = warp & 3;
        const int j_local = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const int etid = threadIdx.x - 64;  // 0..127
        int ts = 0;
        uint32_t tph = 0;
        int64_t head_key = -1;
        const float inv_p = 1.0f / float(P.p);
        for (int64_t it = it_beg; it < it_end; ++it) {
            const P2Item x = p2_item(P, it);
            if (!x.live()) continue;
            const int64_t hk = int64_t(x.l) * P.H + x.h;
            if (hk != head_key) {
                named_bar_sync(1, 128);
                for (int r = etid; r < P.NQ * kTile; r += 128) s_lse[r] = P.lse2[hk * (P.NQ * kTile) + r];
                named_bar_sync(1, 128);
                head_key = hk;
            }
            float best = -INFINITY, acc = 0.f;
            for (int c = 0; c < P.NQ; ++c) {
                mbar_wait(&t_full[ts], tph);
                tc_fence_after();
#pragma unroll 1
                for (int sub = 0; sub < 4; ++sub) {
                    float v[32];
                    tmem_ld32(tmem + lane_addr + uint32_t(ts * kTile + sub * 32), v);
                    const float* lse = s_lse + c * kTile + sub * 32;
                    if (P.agg_max) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            const float4 l4 = *reinterpret_cast<const float4*>(lse + i);
                            best = fmaxf(best, fmaf(v[i], P.c2, -l4.x));
                            best = fmaxf(best, fmaf(v[i + 1], P.c2, -l4.y));
                            best = fmaxf(best, fmaf(v[i + 2], P.c2, -l4.z));
                            best = fmaxf(best, fmaf(v[i + 3], P.c2, -l4.w));
                        }
                    } else {
                        for (int i = 0; i < 32; ++i) {
                            const int rq = c * kTile + sub * 32 + i;
                            if (rq >= P.Gp) break;
                            acc += ex2(fmaf(v[i], P.c2, -lse[i]));
                            if (rq % P.p == P.p - 1) {
                                best = fmaxf(best, acc * inv_p);
                                acc = 0.f;
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&t_empty[ts]);
                if (++ts == 4) {
                    ts = 0;
                    tph ^= 1;
                }
            }
            const int j = x.tile * kTile + j_local;
            if (j < x.n_h) P.scores[x.krow0 + j] = P.agg_max ? ex2(best) : best;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static int make_map(CUtensorMap* m, const void* base, int64_t rows) {
    auto enc = get_encode();
    if (!enc) return fail(EPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cuuint64_t(kD), cuuint64_t(std::max<int64_t>(rows, 1))};
    cuuint64_t strides[1] = {cuuint64_t(kD * 2)};
    cuuint32_t box[2] = {64, cuuint32_t(kTile)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(EPK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return EPK_OK;
}

int launch_score_tc(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int hq, int p, int agg_max,
                    int64_t n_max, float* scores) {
    if (c->dtype != EPK_BF16) return fail(EPK_ERR_ARG, "score(tensor core): cache dtype must be BF16");
    if (c->head_dim != kD) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): head_dim must be 128");
    const int H = c->kv_heads;
    if (hq % H != 0) return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
    TcParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.L = c->layers;
    P.H = H;
    P.Hq = hq;
    P.G = hq / H;
    P.p = p;
    P.Gp = P.G * p;
    P.NQ = (P.Gp + kTile - 1) / kTile;
    if (P.NQ > 16) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): group*prompt_len must be <= 2048");
    P.tiles_max = int(std::max<int64_t>(1, (n_max + kTile - 1) / kTile));
    P.splits = (P.tiles_max + kSplitTiles - 1) / kSplitTiles;
    P.prompt_tiles = (p + kTile - 1) / kTile;
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.c2 = float((1.0 / std::sqrt(double(kD))) * 1.4426950408889634);
    P.scores = scores;
    P.agg_max = agg_max;
    const int64_t rows = int64_t(P.L) * H * P.NQ * kTile;
    rc = ws_require(ctx, rows * P.splits * 8 + rows * 4 + 4096);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.part_m = carve.take<float>(rows * P.splits);
    P.part_z = carve.take<float>(rows * P.splits);
    P.lse2 = carve.take<float>(rows);

    CUtensorMap tm_k, tm_q, tm_kp;
    if ((rc = make_map(&tm_k, c->k, c->layer_base[c->layers]))) return rc;
    if ((rc = make_map(&tm_q, q, int64_t(P.L) * hq * p))) return rc;
    if ((rc = make_map(&tm_kp, kp, int64_t(P.L) * H * p))) return rc;

    const int smem1 = 1024 + kTileBytes + kP1Stages * kTileBytes + 256;
    const int smem2 = 1024 + kP2QSlots * kTileBytes + kP2Stages * kTileBytes + P.NQ * kTile * 4 + 256;
    static bool attr_set = false;
    if (!attr_set) {
        EPK_CUDA_CHECK(cudaFuncSetAttribute(tc_rowstats_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem1));
        EPK_CUDA_CHECK(cudaFuncSetAttribute(tc_colscore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            1024 + kP2QSlots * kTileBytes + kP2Stages * kTileBytes + 16 * kTile * 4 + 256));
        attr_set = true;
    }
    P.items = int64_t(P.L) * H * P.NQ * P.splits;
    int grid1 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p1_rowstats");
    tc_rowstats_kernel<<<grid1, kThreads, smem1, ctx->stream>>>(P, tm_k, tm_q, tm_kp);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "p1_merge");
    tc_merge_kernel<<<unsigned((rows + 255) / 256), 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    P.items = int64_t(P.L) * H * P.tiles_max;
    int grid2 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p2_colscore");
    tc_colscore_kernel<<<grid2, kThreads, smem2, ctx->stream>>>(P, tm_k, tm_q);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
