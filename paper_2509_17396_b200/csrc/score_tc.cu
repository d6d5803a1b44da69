// score_tc.cu -- K1: the tensor-core patched-prompt scorer (bf16 in, fp32
// accumulate), tcgen05 MMAs with TMEM accumulators fed by TMA.
//
// Computes the quantity of score_f32.cu / score_with_prompt
// (scoring.hpp:80-128 over the attention weights of toymodel.hpp:327-391):
//   score(j) = max_{g,t} exp(l_{g,t,j} - lse_{g,t})            (Aggregation::Max)
//   score(j) = max_g (1/p) sum_t exp(l_{g,t,j} - lse_{g,t})    (Aggregation::Avg)
// with l = q.k d^-1/2 and lse_{g,t} the log-sum-exp of query row (g,t) over
// the n_h cache columns plus the causal prompt columns 0..t.  The attention
// grid never exists in memory; K is streamed twice (P1, P2), Q stays in
// shared memory.
//
// One persistent kernel template, two modes.  An ITEM is (layer, kv-head,
// split of 8 K tiles [, query-chunk group]); the producer streams the item's
// 128-row K tiles once (TMA, 128-byte swizzle) and, per K tile, the MMA warp
// issues one 128x128x128 tcgen05.mma per resident 128-row query chunk:
//   STATS (P1): D[query row][cache col] = Q_c . K_t^T  -> epilogue lanes own a
//               query row, keep an online (max, sum exp2) -> partial (m, Z)
//               per (row, split, warpgroup); tc_merge_kernel folds them into
//               lse2 = log2 sum 2^(x - m) + m.
//   SCORE (P2): D[cache row][query row] = K_t . Q_c^T  -> epilogue lanes own a
//               cache row, reduce max_r (x c2 - lse2[r]) across the query
//               chunks -> one exp2 per cache row = its score.
// TMEM: 4 accumulator slots of 128 fp32 columns; epilogue warpgroup g (4 warps,
// one per TMEM lane quarter) owns slots {2g, 2g+1} and every other K tile, so
// two warps per SM sub-partition overlap TMEM loads, FMA and MUFU work.
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2-9 epilogue.  Items are dealt to CTAs in contiguous ranges,
// so a CTA loads a head's Q once and reuses it across that head's splits.
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
constexpr int kSplitTiles = 8;  // K tiles per item (1024 cache columns)
constexpr int kQSlots = 4;      // resident query chunks (<= 512 query rows)
constexpr int kEpiWarps = 8;
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr uint32_t kIdesc = idesc_bf16_f32(128, 128);

enum { MODE_STATS = 0, MODE_SCORE = 1 };

struct TcParams {
    LayerTable lt;
    int L, H, Hq, G, p, Gp, NQ;
    int tiles_max;     // ceil(n_max / 128)
    int splits;        // ceil(tiles_max / kSplitTiles)
    int cgroups;       // STATS: query-chunk groups of <= kQSlots chunks
    int prompt_tiles;  // ceil(p / 128)
    int qslots;        // resident Q slots allocated in smem
    int kstages;       // K ring depth
    const int32_t* head_off;
    const int32_t* head_len;
    float c2;       // d^-1/2 * log2(e)
    float* part_m;  // [L*H*NQ*128][2*splits]
    float* part_z;
    float* lse2;  // [L*H*NQ*128]
    float* scores;
    int agg_max;
    int64_t items;
};

// One 128x128x128 MMA: 8 K-steps of 16 elements (32 bytes) over the two
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

struct Item {
    int l, h, s, cg;
    int n_h;
    int64_t krow0;  // first K row of the head (global)
    int t0, nc, np;  // first cache tile, cache tiles, prompt tiles
    int c0, nq;      // first query chunk, chunks
    __device__ int ntiles() const { return nc + np; }
    __device__ int64_t qkey() const { return (int64_t(l) * 4096 + h) * 64 + cg; }
};

template <int MODE>
__device__ __forceinline__ Item decode(const TcParams& P, int64_t it) {
    Item x;
    if (MODE == MODE_STATS) {
        x.cg = int(it % P.cgroups);
        it /= P.cgroups;
    } else {
        x.cg = 0;
    }
    x.s = int(it % P.splits);
    const int64_t r = it / P.splits;
    x.h = int(r % P.H);
    x.l = int(r / P.H);
    x.n_h = P.head_len[x.l * P.H + x.h];
    x.krow0 = P.lt.base[x.l] + P.head_off[x.l * (P.H + 1) + x.h];
    const int tiles = (x.n_h + kTile - 1) / kTile;
    x.t0 = x.s * kSplitTiles;
    x.nc = max(0, min(tiles, x.t0 + kSplitTiles) - x.t0);
    x.np = (MODE == MODE_STATS && x.s == P.splits - 1) ? P.prompt_tiles : 0;
    if (MODE == MODE_STATS) {
        x.c0 = x.cg * kQSlots;
        x.nq = min(kQSlots, P.NQ - x.c0);
    } else {
        x.c0 = 0;
        x.nq = P.NQ;
    }
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_score_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + P.qslots * kTileBytes;
    float* s_lse = reinterpret_cast<float*>(sK + P.kstages * kTileBytes);  // SCORE: 2 x NQ*128
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lse + (MODE == MODE_SCORE ? 2 * P.NQ * kTile : 0));
    uint64_t* k_full = bars;
    uint64_t* k_empty = k_full + P.kstages;
    uint64_t* q_full = k_empty + P.kstages;
    uint64_t* q_empty = q_full + kQSlots;
    uint64_t* t_full = q_empty + kQSlots;
    uint64_t* t_empty = t_full + 4;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = (P.items + gridDim.x - 1) / gridDim.x;
    const int64_t it_beg = int64_t(blockIdx.x) * per;
    const int64_t it_end = min(P.items, it_beg + per);
    const bool resident = MODE == MODE_STATS || P.NQ <= P.qslots;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_q);
        if (MODE == MODE_STATS) tma_prefetch(&tm_kp);
        for (int s = 0; s < P.kstages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], 1);
        }
        for (int s = 0; s < kQSlots; ++s) {
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
        if (lane == 0) {  // ------------------------- TMA producer -------------------------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kQSlots] = {0, 0, 0, 0};
            int64_t key = -1, qjob = 0;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const Item x = decode<MODE>(P, it);
                if (x.ntiles() == 0) continue;
                const int qrow0 = (x.l * P.Hq + x.h * P.G) * P.p;
                if (resident && x.qkey() != key) {
                    key = x.qkey();
                    for (int c = 0; c < x.nq; ++c) {
                        mbar_wait(&q_empty[c], (qload[c] & 1) ^ 1);
                        mbar_expect_tx(&q_full[c], kTileBytes);
                        load_tile(sQ + c * kTileBytes, &tm_q, &q_full[c], qrow0 + (x.c0 + c) * kTile);
                        ++qload[c];
                    }
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    mbar_wait(&k_empty[ks], kph ^ 1);
                    mbar_expect_tx(&k_full[ks], kTileBytes);
                    if (t < x.nc)
                        load_tile(sK + ks * kTileBytes, &tm_k, &k_full[ks], int(x.krow0 + int64_t(x.t0 + t) * kTile));
                    else
                        load_tile(sK + ks * kTileBytes, &tm_kp, &k_full[ks],
                                  (x.l * P.H + x.h) * P.p + (t - x.nc) * kTile);
                    if (++ks == P.kstages) {
                        ks = 0;
                        kph ^= 1;
                    }
                    if (!resident) {
                        for (int c = 0; c < x.nq; ++c, ++qjob) {
                            const int slot = int(qjob % P.qslots);
                            mbar_wait(&q_empty[slot], (qload[slot] & 1) ^ 1);
                            mbar_expect_tx(&q_full[slot], kTileBytes);
                            load_tile(sQ + slot * kTileBytes, &tm_q, &q_full[slot], qrow0 + c * kTile);
                            ++qload[slot];
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ------------------------- MMA issuer ---------------------------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kQSlots] = {0, 0, 0, 0};
            uint32_t gj[2] = {0, 0};
            int64_t key = -1, qjob = 0, tcount = 0;
            int held = 0;  // resident chunks of the current key
            for (int64_t it = it_beg; it < it_end; ++it) {
                const Item x = decode<MODE>(P, it);
                if (x.ntiles() == 0) continue;
                bool fresh = false;
                if (resident && x.qkey() != key) {
                    for (int c = 0; c < held; ++c) mma_commit(&q_empty[c]);  // old Q retires with its MMAs
                    key = x.qkey();
                    held = x.nq;
                    fresh = true;
                }
                for (int t = 0; t < x.ntiles(); ++t, ++tcount) {
                    mbar_wait(&k_full[ks], kph);
                    const int g = int(tcount & 1);
                    for (int c = 0; c < x.nq; ++c) {
                        int slot = c;
                        if (!resident) {
                            slot = int(qjob % P.qslots);
                            ++qjob;
                            mbar_wait(&q_full[slot], qload[slot] & 1);
                            ++qload[slot];
                        } else if (fresh && t == 0) {
                            mbar_wait(&q_full[slot], qload[slot] & 1);
                            ++qload[slot];
                        }
                        const int ts = 2 * g + int(gj[g] & 1);
                        mbar_wait(&t_empty[ts], ((gj[g] >> 1) & 1) ^ 1);
                        tc_fence_after();
                        const uint32_t d = tmem + uint32_t(ts * kTile);
                        if (MODE == MODE_STATS)
                            mma_tile(d, sQ + slot * kTileBytes, sK + ks * kTileBytes);
                        else
                            mma_tile(d, sK + ks * kTileBytes, sQ + slot * kTileBytes);
                        mma_commit(&t_full[ts]);
                        if (!resident) mma_commit(&q_empty[slot]);
                        ++gj[g];
                    }
                    mma_commit(&k_empty[ks]);
                    if (++ks == P.kstages) {
                        ks = 0;
                        kph ^= 1;
                    }
                }
            }
        }
    } else {  // ------------------------- epilogue warpgroups --------------------------
        const int g = (warp - 2) >> 2;
        const int quarter = warp & 3;
        const int r_local = quarter * 32 + lane;  // TMEM lane owned by this thread
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const int gtid = (warp - 2 - 4 * g) * 32 + lane;  // 0..127 within the group
        uint32_t gj = 0;
        int64_t tcount = 0, lkey = -1;
        float* my_lse = s_lse + g * P.NQ * kTile;
        const float inv_p = 1.0f / float(P.p);
        for (int64_t it = it_beg; it < it_end; ++it) {
            const Item x = decode<MODE>(P, it);
            if (MODE == MODE_STATS) {
                float m[kQSlots], z[kQSlots];
#pragma unroll
                for (int c = 0; c < kQSlots; ++c) {
                    m[c] = -INFINITY;
                    z[c] = 0.f;
                }
                for (int t = 0; t < x.ntiles(); ++t, ++tcount) {
                    if (int(tcount & 1) != g) continue;
#pragma unroll
                    for (int c = 0; c < kQSlots; ++c) {
                        if (c >= x.nq) break;
                        const int rq = (x.c0 + c) * kTile + r_local;  // query row of the head (g*p + t)
                        int lim;
                        if (t < x.nc)
                            lim = x.n_h - (x.t0 + t) * kTile;
                        else
                            lim = min(P.p, rq % P.p + 1) - (t - x.nc) * kTile;
                        const int ts = 2 * g + int(gj & 1);
                        mbar_wait(&t_full[ts], (gj >> 1) & 1);
                        tc_fence_after();
#pragma unroll 1
                        for (int half = 0; half < 2; ++half) {
                            float v[64];
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * kTile + half * 64), v);
                            if (half == 1) {  // TMEM slot free: the last values are in registers
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&t_empty[ts]);
                            }
                            const int hl = lim - half * 64;
                            float mx = -INFINITY;
                            if (hl >= 64) {
#pragma unroll
                                for (int i = 0; i < 64; ++i) mx = fmaxf(mx, v[i]);
                            } else {
#pragma unroll
                                for (int i = 0; i < 64; ++i) {
                                    v[i] = (i < hl) ? v[i] : -INFINITY;
                                    mx = fmaxf(mx, v[i]);
                                }
                            }
                            mx *= P.c2;
                            if (mx > m[c]) {
                                z[c] *= ex2(m[c] - mx);
                                m[c] = mx;
                            }
                            if (m[c] != -INFINITY) {
                                const float mc = m[c];
                                float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
                                for (int i = 0; i < 64; i += 4) {
                                    s0 += ex2(fmaf(v[i], P.c2, -mc));
                                    s1 += ex2(fmaf(v[i + 1], P.c2, -mc));
                                    s2 += ex2(fmaf(v[i + 2], P.c2, -mc));
                                    s3 += ex2(fmaf(v[i + 3], P.c2, -mc));
                                }
                                z[c] += (s0 + s1) + (s2 + s3);
                            }
                        }
                        ++gj;
                    }
                }
                // partial (m, Z) of this warpgroup for each query row of the item
#pragma unroll
                for (int cc = 0; cc < kQSlots; ++cc) {
                    if (cc < x.nq) {
                        const int rq = (x.c0 + cc) * kTile + r_local;
                        const int64_t o = ((int64_t(x.l) * P.H + x.h) * (P.NQ * kTile) + rq) * (2 * P.splits) +
                                          2 * x.s + g;
                        P.part_m[o] = m[cc];
                        P.part_z[o] = z[cc];
                    }
                }
            } else {
                if (x.ntiles() == 0) continue;
                const int64_t hk = int64_t(x.l) * P.H + x.h;
                for (int t = 0; t < x.ntiles(); ++t, ++tcount) {
                    if (int(tcount & 1) != g) continue;
                    if (hk != lkey) {  // this group's copy of the head's lse2
                        named_bar_sync(1 + g, 128);
                        for (int r = gtid; r < P.NQ * kTile; r += 128) my_lse[r] = P.lse2[hk * (P.NQ * kTile) + r];
                        named_bar_sync(1 + g, 128);
                        lkey = hk;
                    }
                    float best = -INFINITY, acc = 0.f;
                    for (int c = 0; c < x.nq; ++c) {
                        const int ts = 2 * g + int(gj & 1);
                        mbar_wait(&t_full[ts], (gj >> 1) & 1);
                        tc_fence_after();
#pragma unroll 1
                        for (int half = 0; half < 2; ++half) {
                            float v[64];
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * kTile + half * 64), v);
                            if (half == 1) {
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&t_empty[ts]);
                            }
                            const float* lse = my_lse + c * kTile + half * 64;
                            if (P.agg_max) {
                                float b0 = best, b1 = -INFINITY, b2 = -INFINITY, b3 = -INFINITY;
#pragma unroll
                                for (int i = 0; i < 64; i += 4) {
                                    const float4 l4 = *reinterpret_cast<const float4*>(lse + i);
                                    b0 = fmaxf(b0, fmaf(v[i], P.c2, -l4.x));
                                    b1 = fmaxf(b1, fmaf(v[i + 1], P.c2, -l4.y));
                                    b2 = fmaxf(b2, fmaf(v[i + 2], P.c2, -l4.z));
                                    b3 = fmaxf(b3, fmaf(v[i + 3], P.c2, -l4.w));
                                }
                                best = fmaxf(fmaxf(b0, b1), fmaxf(b2, b3));
                            } else {
#pragma unroll
                                for (int i = 0; i < 64; ++i) {
                                    const int rq = c * kTile + half * 64 + i;
                                    if (rq < P.Gp) {  // pad rows have lse2 = +inf -> exp2 = 0
                                        acc += ex2(fmaf(v[i], P.c2, -lse[i]));
                                        if (rq % P.p == P.p - 1) {
                                            best = fmaxf(best, acc * inv_p);
                                            acc = 0.f;
                                        }
                                    }
                                }
                            }
                        }
                        ++gj;
                    }
                    const int j = (x.t0 + t) * kTile + r_local;
                    if (j < x.n_h) P.scores[x.krow0 + j] = P.agg_max ? ex2(best) : best;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// lse2 per query row = log2 sum_s Z_s 2^(m_s - M) + M over the partials.
__global__ void tc_merge_kernel(const __grid_constant__ TcParams P) {
    const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t rows = int64_t(P.L) * P.H * P.NQ * kTile;
    if (idx >= rows) return;
    const int rq = int(idx % (P.NQ * kTile));
    if (rq >= P.Gp) {
        P.lse2[idx] = INFINITY;
        return;
    }
    const int np = 2 * P.splits;
    float M = -INFINITY;
    for (int s = 0; s < np; ++s) M = fmaxf(M, P.part_m[idx * np + s]);
    float Z = 0.f;
    if (M != -INFINITY)
        for (int s = 0; s < np; ++s) {
            const float ms = P.part_m[idx * np + s];
            if (ms != -INFINITY) Z += P.part_z[idx * np + s] * ex2(ms - M);
        }
    P.lse2[idx] = M + log2f(Z);
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

static int smem_bytes(const TcParams& P, int mode) {
    return 1024 + (P.qslots + P.kstages) * kTileBytes + (mode == MODE_SCORE ? 2 * P.NQ * kTile * 4 : 0) +
           (2 * P.kstages + 2 * kQSlots + 8) * 8 + 16;
}

static void fit_stages(TcParams& P, int mode, int limit) {
    P.qslots = std::min(P.NQ, kQSlots);
    P.kstages = 2;
    while (P.kstages < 4) {
        ++P.kstages;
        if (smem_bytes(P, mode) > limit) {
            --P.kstages;
            break;
        }
    }
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
    P.cgroups = (P.NQ + kQSlots - 1) / kQSlots;
    P.prompt_tiles = (p + kTile - 1) / kTile;
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.c2 = float((1.0 / std::sqrt(double(kD))) * 1.4426950408889634);
    P.scores = scores;
    P.agg_max = agg_max;
    const int64_t rows = int64_t(P.L) * H * P.NQ * kTile;
    rc = ws_require(ctx, rows * 2 * P.splits * 8 + rows * 4 + 4096);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.part_m = carve.take<float>(rows * 2 * P.splits);
    P.part_z = carve.take<float>(rows * 2 * P.splits);
    P.lse2 = carve.take<float>(rows);

    CUtensorMap tm_k, tm_q, tm_kp;
    if ((rc = make_map(&tm_k, c->k, c->layer_base[c->layers]))) return rc;
    if ((rc = make_map(&tm_q, q, int64_t(P.L) * hq * p))) return rc;
    if ((rc = make_map(&tm_kp, kp, int64_t(P.L) * H * p))) return rc;

    // Dynamic shared memory limit: the per-block opt-in maximum minus the
    // kernel's static/reserved shared memory.
    static int limit = 0;
    if (!limit) {
        int optin = 0;
        EPK_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
        cudaFuncAttributes fa0, fa1;
        EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa0, tc_score_kernel<MODE_STATS>));
        EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa1, tc_score_kernel<MODE_SCORE>));
        limit = optin - int(std::max(fa0.sharedSizeBytes, fa1.sharedSizeBytes));
        EPK_CUDA_CHECK(cudaFuncSetAttribute(tc_score_kernel<MODE_STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            limit));
        EPK_CUDA_CHECK(cudaFuncSetAttribute(tc_score_kernel<MODE_SCORE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            limit));
    }
    // P1: query-chunk groups of <= 4 resident chunks, K ring fills the rest.
    fit_stages(P, MODE_STATS, limit);
    P.items = int64_t(P.L) * H * P.splits * P.cgroups;
    const int grid1 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p1_rowstats");
    tc_score_kernel<MODE_STATS><<<grid1, kThreads, smem_bytes(P, MODE_STATS), ctx->stream>>>(P, tm_k, tm_q, tm_kp);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "p1_merge");
    tc_merge_kernel<<<unsigned((rows + 255) / 256), 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);
    // P2: all query chunks resident when they fit, else streamed through 4 slots.
    fit_stages(P, MODE_SCORE, limit);
    P.items = int64_t(P.L) * H * P.splits;
    const int grid2 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p2_colscore");
    tc_score_kernel<MODE_SCORE><<<grid2, kThreads, smem_bytes(P, MODE_SCORE), ctx->stream>>>(P, tm_k, tm_q, tm_kp);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk
