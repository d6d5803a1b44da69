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
// One persistent kernel template, two modes; every MMA is 128 x 256 x 128
// (the shape that keeps tcgen05 at ~94% of issue peak -- 128 x 128 tiles
// saturate shared-memory operand bandwidth at ~69%, see
// profiles/mma_rate_r01.txt):
//   STATS (P1): A = 128-row query chunk (resident), B = 256-row K stage,
//               D[query row][cache col] -> epilogue lanes own a query row and
//               keep an online (max, sum exp2) per chunk -> partial (m, Z) per
//               (row, split, column half); tc_merge_kernel folds them into
//               lse2 = log2 sum 2^(x - m) + m.
//   SCORE (P2): A = 128-row K stage, B = two query chunks (256 query rows),
//               D[cache row][query row] -> epilogue lanes own a cache row and
//               reduce max_r (x c2 - lse2[r]) -> one exp2 per cache row.
// Shared memory keeps Q as [d-half][all query rows] (128-byte swizzled rows,
// 8-row groups 1024 B apart) so any two consecutive 128-row chunks form one
// 256-row B operand.  TMEM: two 256-column accumulator slots.
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2-9 epilogue (warp e: TMEM lane quarter e & 3, column half
// e >> 2 of every job).  Items = (layer, kv-head, 1024-column split [,
// query-chunk group]) dealt to CTAs in contiguous ranges, so a CTA loads a
// head's Q once.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "epk_internal.cuh"
#include "sm100.cuh"

namespace epk {

using namespace sm100;

constexpr int kD = 128;
constexpr int kRowB = 128;        // bytes of one d-half row (64 bf16)
constexpr int kChunk = 128;       // query rows per chunk (MMA M in P1)
constexpr int kSplitCols = 1024;  // cache columns per item
constexpr int kEpiWarps = 8;
constexpr int kMmaWarps = 2;  // MMA issuers alternate jobs: one issues while the other synchronises
constexpr int kThreads = 32 * (1 + kMmaWarps + kEpiWarps);
constexpr int kMaxQRes = 4;       // resident query chunks (P1: per chunk group)

enum { MODE_STATS = 0, MODE_SCORE = 1 };

struct TcParams {
    LayerTable lt;
    int L, H, Hq, G, p, Gp, NQ;
    int splits;        // ceil(n_max / 1024)
    int cgroups;       // STATS: query-chunk groups
    int cg_chunks;     // STATS: chunks per group
    int krows;         // K stage rows: 256 (STATS) / 128 (SCORE)
    int kstages;       // K ring depth
    int qcap;          // rows per d-half in the Q region
    int resident;      // SCORE: all query chunks resident (else streamed pairs)
    const int32_t* head_off;
    const int32_t* head_len;
    float c2;       // d^-1/2 * log2(e)
    float* part_m;  // [L*H*NQ*128][2*splits]
    float* part_z;
    float* lse2;  // [L*H*NQ*128]
    float* scores;
    int agg_max;
    int64_t items;
    unsigned long long* trace;  // diagnostics (EPK_TC_TRACE): CTA 0 timeline records
};

// Timeline record for CTA 0: per-role private regions of 60000 records,
// plain stores (no atomics): (event << 56) | clock low 56 bits.
#define EPK_TRACE(P, role, ev)                                                                          \
    do {                                                                                                \
        if ((P).trace && blockIdx.x == 0 && tr_n < 60000)                                               \
            (P).trace[1 + (role) * 60000 + tr_n++] = (uint64_t(ev) << 56) | (uint64_t(clock64()) & 0xFFFFFFFFFFFFFFull); \
    } while (0)

// D (+)= A * B^T over K = 128: 8 K-steps of 16 across the two 64-wide
// d-halves.  a_half / b_half: byte distance between the operands' d-halves.
__device__ __forceinline__ void mma_128xN(uint32_t d_tmem, uint32_t a, uint32_t a_half, uint32_t b, uint32_t b_half,
                                          uint32_t idesc) {
    // desc(addr + off) == desc(addr) + (off >> 4): shared addresses < 256 KB
    // never carry out of the 14-bit start-address field.
    const uint64_t da = sdesc_k_sw128(a), db = sdesc_k_sw128(b);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t k = uint32_t((kk & 3) * 32);
        const uint32_t h = uint32_t(kk >> 2);
        mma_bf16_ss(d_tmem, da + ((h * a_half + k) >> 4), db + ((h * b_half + k) >> 4), idesc, kk > 0 ? 1u : 0u);
    }
}

// Loads `rows` rows (both d-halves) of a [*, 128] bf16 tensor into a
// [d-half][rows] region whose halves are `half_bytes` apart.
__device__ __forceinline__ void load_rows(uint8_t* dst, uint32_t half_bytes, const CUtensorMap* map, uint64_t* bar,
                                          int row) {
    tma_load_2d(dst, map, bar, 0, row);
    tma_load_2d(dst + half_bytes, map, bar, 64, row);
}

struct Item {
    int l, h, s, cg;
    int n_h;
    int64_t krow0;   // first K row of the head (global)
    int t0, nc, np;  // first cache tile, cache tiles, prompt tiles (tiles of krows)
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
    const int per = kSplitCols / P.krows;
    const int tiles = (x.n_h + P.krows - 1) / P.krows;
    x.t0 = x.s * per;
    x.nc = max(0, min(tiles, x.t0 + per) - x.t0);
    x.np = (MODE == MODE_STATS && x.s == P.splits - 1) ? (P.p + P.krows - 1) / P.krows : 0;
    if (MODE == MODE_STATS) {
        x.c0 = x.cg * P.cg_chunks;
        x.nq = min(P.cg_chunks, P.NQ - x.c0);
    } else {
        x.c0 = 0;
        x.nq = P.NQ;
    }
    return x;
}

// SCORE epilogue on W columns of one cache row (query rows r0 .. r0+W):
// Max: best = max(best, x c2 - lse2); Avg: per-window sums of 2^(x c2 - lse2)
// accumulated per query head in shared memory.
template <int W>
__device__ __forceinline__ void score_cols(const float (&v)[W], const float* lse, int r0, const TcParams& P,
                                           float& best, float* s_avg, int r_local) {
    if (P.agg_max) {
        float b0 = best, b1 = -INFINITY, b2 = -INFINITY, b3 = -INFINITY;
#pragma unroll
        for (int i = 0; i < W; i += 4) {
            const float4 l4 = *reinterpret_cast<const float4*>(lse + i);
            b0 = fmaxf(b0, fmaf(v[i], P.c2, -l4.x));
            b1 = fmaxf(b1, fmaf(v[i + 1], P.c2, -l4.y));
            b2 = fmaxf(b2, fmaf(v[i + 2], P.c2, -l4.z));
            b3 = fmaxf(b3, fmaf(v[i + 3], P.c2, -l4.w));
        }
        best = fmaxf(fmaxf(b0, b1), fmaxf(b2, b3));
    } else {
        float acc = 0.f;
        int gcur = r0 / P.p;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const int rq = r0 + i;
            if (rq < P.Gp) {
                const int gg = rq / P.p;
                if (gg != gcur) {
                    atomicAdd(&s_avg[gcur * kChunk + r_local], acc);
                    acc = 0.f;
                    gcur = gg;
                }
                acc += ex2(fmaf(v[i], P.c2, -lse[i]));
            }
        }
        if (gcur < P.G) atomicAdd(&s_avg[gcur * kChunk + r_local], acc);
    }
}

// STATS epilogue on W columns of one query row, `lim` of them valid:
// online (max, sum 2^(x c2 - max)) update of (m, z).
template <int W>
__device__ __forceinline__ void stats_cols(float (&v)[W], int lim, float c2, float& m, float& z) {
    float mx = -INFINITY;
    if (lim >= W) {
#pragma unroll
        for (int i = 0; i < W; ++i) mx = fmaxf(mx, v[i]);
    } else {
#pragma unroll
        for (int i = 0; i < W; ++i) {
            v[i] = (i < lim) ? v[i] : -INFINITY;
            mx = fmaxf(mx, v[i]);
        }
    }
    mx *= c2;
    if (mx > m) {
        z *= ex2(m - mx);
        m = mx;
    }
    if (m != -INFINITY) {
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int i = 0; i < W; i += 4) {
            s0 += ex2(fmaf(v[i], c2, -m));
            s1 += ex2(fmaf(v[i + 1], c2, -m));
            s2 += ex2(fmaf(v[i + 2], c2, -m));
            s3 += ex2(fmaf(v[i + 3], c2, -m));
        }
        z += (s0 + s1) + (s2 + s3);
    }
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_score_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (SWIZZLE_128B atoms), derived from smem_raw by pointer
    // arithmetic so the compiler keeps shared-space (LDS/STS) addressing.
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t q_half = uint32_t(P.qcap) * kRowB;   // Q d-half stride
    const uint32_t k_half = uint32_t(P.krows) * kRowB;  // K d-half stride
    const uint32_t k_stage = 2 * k_half;
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + 2 * q_half;
    float* s_lse = reinterpret_cast<float*>(sK + P.kstages * k_stage);     // SCORE: NQ*128 lse2
    float* s_pair = s_lse + (MODE == MODE_SCORE ? P.NQ * kChunk : 0);     // SCORE: 128 half maxima
    float* s_avg = s_pair + (MODE == MODE_SCORE ? kChunk : 0);            // SCORE avg: G*128 sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_avg + (MODE == MODE_SCORE && !P.agg_max ? P.G * kChunk : 0));
    uint64_t* k_full = bars;
    uint64_t* k_empty = k_full + P.kstages;
    uint64_t* q_full = k_empty + P.kstages;  // per resident chunk, or per streamed pair slot
    uint64_t* q_empty = q_full + kMaxQRes;
    uint64_t* t_full = q_empty + kMaxQRes;
    uint64_t* t_empty = t_full + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t per = (P.items + gridDim.x - 1) / gridDim.x;
    const int64_t it_beg = int64_t(blockIdx.x) * per;
    const int64_t it_end = min(P.items, it_beg + per);
    const bool resident = MODE == MODE_STATS || P.resident;
    int tr_n = 0;  // EPK_TRACE record count of this thread

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_q);
        if (MODE == MODE_STATS) tma_prefetch(&tm_kp);
        for (int s = 0; s < P.kstages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], kMmaWarps);  // every MMA warp releases every stage
        }
        for (int s = 0; s < kMaxQRes; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], resident ? kMmaWarps : 1);  // streamed slots belong to one MMA warp
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&t_full[s], 1);
            mbar_init(&t_empty[s], kEpiWarps);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    if (MODE == MODE_SCORE && !P.agg_max)
        for (int i = threadIdx.x; i < P.G * kChunk; i += blockDim.x) s_avg[i] = 0.f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 0) {
        const bool leader = elect_one_sync();
        {  // ------------------------- TMA producer (warp-wide, one lane issues) -----------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kMaxQRes] = {0, 0, 0, 0};
            int64_t key = -1, pj = 0;
            const int npairs = (P.NQ + 1) / 2;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const Item x = decode<MODE>(P, it);
                if (x.ntiles() == 0) continue;
                const int qrow0 = (x.l * P.Hq + x.h * P.G) * P.p;
                if (resident && x.qkey() != key) {
                    key = x.qkey();
                    for (int c = 0; c < x.nq; ++c) {
                        mbar_wait(&q_empty[c], (qload[c] & 1) ^ 1);
                        if (leader) {
                            mbar_expect_tx(&q_full[c], 2 * kChunk * kRowB);
                            load_rows(sQ + c * kChunk * kRowB, q_half, &tm_q, &q_full[c], qrow0 + (x.c0 + c) * kChunk);
                        }
                        __syncwarp();
                        ++qload[c];
                    }
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    if (leader) EPK_TRACE(P, 0, 1);
                    mbar_wait(&k_empty[ks], kph ^ 1);
                    if (leader) EPK_TRACE(P, 0, 2);
                    if (leader) {
                        mbar_expect_tx(&k_full[ks], k_stage);
                        if (t < x.nc)
                            load_rows(sK + ks * k_stage, k_half, &tm_k, &k_full[ks],
                                      int(x.krow0 + int64_t(x.t0 + t) * P.krows));
                        else
                            load_rows(sK + ks * k_stage, k_half, &tm_kp, &k_full[ks],
                                      (x.l * P.H + x.h) * P.p + (t - x.nc) * P.krows);
                    }
                    __syncwarp();
                    if (++ks == P.kstages) {
                        ks = 0;
                        kph ^= 1;
                    }
                    if (!resident) {  // SCORE, streamed: query chunk pairs through 2 slots
                        for (int j = 0; j < npairs; ++j, ++pj) {
                            const int slot = int(pj & 1);
                            const int nch = min(2, P.NQ - 2 * j);
                            mbar_wait(&q_empty[slot], (qload[slot] & 1) ^ 1);
                            if (leader) {
                                mbar_expect_tx(&q_full[slot], nch * 2 * kChunk * kRowB);
                                for (int cc = 0; cc < nch; ++cc)
                                    load_rows(sQ + (slot * 2 + cc) * kChunk * kRowB, q_half, &tm_q, &q_full[slot],
                                              qrow0 + (2 * j + cc) * kChunk);
                            }
                            __syncwarp();
                            ++qload[slot];
                        }
                    }
                }
            }
        }
    } else if (warp <= kMmaWarps) {
        // MMA warp mw issues the jobs with (job & 1) == mw into TMEM slot mw;
        // both walk the same item/tile sequence and both release every K stage.
        const uint32_t mw = uint32_t(warp - 1);
        const bool leader = elect_one_sync();
        {  // ------------------------- MMA issuers (warp-wide, one lane issues) ------------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kMaxQRes] = {0, 0, 0, 0};
            uint32_t job = 0;
            int64_t key = -1;
            int held = 0;
            const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK);
            const bool tr = leader && mw == 0;
            for (int64_t it = it_beg; it < it_end; ++it) {
                const Item x = decode<MODE>(P, it);
                if (x.ntiles() == 0) continue;
                bool fresh = false;
                if (resident && x.qkey() != key) {
                    if (leader)
                        for (int c = 0; c < held; ++c) mma_commit(&q_empty[c]);  // old Q retires with its MMAs
                    __syncwarp();
                    key = x.qkey();
                    held = x.nq;
                    fresh = true;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    if (tr) EPK_TRACE(P, 1, 3);
                    mbar_wait(&k_full[ks], kph);
                    if (tr) EPK_TRACE(P, 1, 4);
                    const uint32_t kst = k0 + uint32_t(ks) * k_stage;
                    if (MODE == MODE_STATS) {
                        for (int c = 0; c < x.nq; ++c, ++job) {
                            if (fresh && t == 0) {
                                mbar_wait(&q_full[c], qload[c] & 1);
                                ++qload[c];
                            }
                            if ((job & 1) != mw) continue;
                            const int ts = int(mw);
                            mbar_wait(&t_empty[ts], ((job >> 1) & 1) ^ 1);
                            tc_fence_after();
                            if (leader) {
                                mma_128xN(tmem + uint32_t(ts * 256), q0 + uint32_t(c * kChunk * kRowB), q_half, kst,
                                          k_half, idesc_bf16_f32(128, 256));
                                mma_commit(&t_full[ts]);
                            }
                            __syncwarp();
                        }
                    } else {
                        for (int j = 0; 2 * j < x.nq; ++j, ++job) {
                            const int nch = min(2, x.nq - 2 * j);
                            if (resident && fresh && t == 0)
                                for (int cc = 0; cc < nch; ++cc) {
                                    mbar_wait(&q_full[2 * j + cc], qload[2 * j + cc] & 1);
                                    ++qload[2 * j + cc];
                                }
                            if ((job & 1) != mw) continue;
                            uint32_t qb;
                            const int slot = int(mw);  // streamed pair slot == TMEM slot == this warp
                            if (resident) {
                                qb = q0 + uint32_t(2 * j * kChunk * kRowB);
                            } else {
                                mbar_wait(&q_full[slot], qload[slot] & 1);
                                ++qload[slot];
                                qb = q0 + uint32_t(slot * 2 * kChunk * kRowB);
                            }
                            const int ts = int(mw);
                            if (tr) EPK_TRACE(P, 1, 5);
                            mbar_wait(&t_empty[ts], ((job >> 1) & 1) ^ 1);
                            if (tr) EPK_TRACE(P, 1, 6);
                            tc_fence_after();
                            if (leader) {
                                mma_128xN(tmem + uint32_t(ts * 256), kst, k_half, qb, q_half,
                                          idesc_bf16_f32(128, uint32_t(nch * kChunk)));
                                mma_commit(&t_full[ts]);
                                if (!resident) mma_commit(&q_empty[slot]);
                            }
                            __syncwarp();
                            if (tr) EPK_TRACE(P, 1, 7);
                        }
                    }
                    if (leader) mma_commit(&k_empty[ks]);
                    __syncwarp();
                    if (++ks == P.kstages) {
                        ks = 0;
                        kph ^= 1;
                    }
                }
            }
        }
    } else {  // ------------------------- epilogue (8 warps) -------------------------
        const int e = warp - 1 - kMmaWarps;
        const int quarter = warp & 3;  // TMEM lanes this warp may read
        const int half = e >> 2;       // column half of every job
        const int r_local = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const int etid = e * 32 + lane;
        uint32_t job = 0;
        int64_t lkey = -1;
        const float inv_p = 1.0f / float(P.p);
        for (int64_t it = it_beg; it < it_end; ++it) {
            const Item x = decode<MODE>(P, it);
            if (MODE == MODE_STATS) {
                float m[kMaxQRes], z[kMaxQRes];
#pragma unroll
                for (int c = 0; c < kMaxQRes; ++c) {
                    m[c] = -INFINITY;
                    z[c] = 0.f;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
#pragma unroll
                    for (int c = 0; c < kMaxQRes; ++c) {
                        if (c >= x.nq) break;
                        const int rq = (x.c0 + c) * kChunk + r_local;  // query row of the head (g*p + t)
                        int lim;  // valid columns of this job from its first column
                        if (t < x.nc)
                            lim = x.n_h - (x.t0 + t) * P.krows;
                        else
                            lim = min(P.p, rq % P.p + 1) - (t - x.nc) * P.krows;
                        const int ts = int(job & 1);
                        mbar_wait(&t_full[ts], (job >> 1) & 1);
                        tc_fence_after();
                        {
                            float v[128];
                            tmem_ld128(tmem + lane_addr + uint32_t(ts * 256 + half * 128), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);  // slot free: values are in registers
                            stats_cols<128>(v, lim - half * 128, P.c2, m[c], z[c]);
                        }
                        ++job;
                    }
                }
                // partial (m, Z) of this column half for each query row of the item
#pragma unroll
                for (int cc = 0; cc < kMaxQRes; ++cc) {
                    if (cc < x.nq) {
                        const int rq = (x.c0 + cc) * kChunk + r_local;
                        const int64_t o = ((int64_t(x.l) * P.H + x.h) * (P.NQ * kChunk) + rq) * (2 * P.splits) +
                                          2 * x.s + half;
                        P.part_m[o] = m[cc];
                        P.part_z[o] = z[cc];
                    }
                }
            } else {
                if (x.ntiles() == 0) continue;
                const int64_t hk = int64_t(x.l) * P.H + x.h;
                if (hk != lkey) {  // the head's lse2 (all 8 warps)
                    named_bar_sync(1, 32 * kEpiWarps);
                    for (int r = etid; r < P.NQ * kChunk; r += 32 * kEpiWarps)
                        s_lse[r] = P.lse2[hk * (P.NQ * kChunk) + r];
                    named_bar_sync(1, 32 * kEpiWarps);
                    lkey = hk;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    float best = -INFINITY;
                    for (int j = 0; 2 * j < x.nq; ++j) {
                        const int ncols = min(2, x.nq - 2 * j) * kChunk;  // query rows of the job
                        const int hw = ncols / 2;                         // columns per warp half
                        const int ts = int(job & 1);
                        if (lane == 0 && e == 0) EPK_TRACE(P, 2, 8);
                        mbar_wait(&t_full[ts], (job >> 1) & 1);
                        if (lane == 0 && e == 0) EPK_TRACE(P, 2, 9);
                        tc_fence_after();
                        const int r0 = 2 * j * kChunk + half * hw;  // first query row of this warp's columns
                        if (hw == 128) {
                            float v[128];
                            tmem_ld128(tmem + lane_addr + uint32_t(ts * 256 + half * hw), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);  // slot free: values are in registers
                            if (lane == 0 && e == 0) EPK_TRACE(P, 2, 10);
                            score_cols<128>(v, s_lse + r0, r0, P, best, s_avg, r_local);
                        } else {
                            float v[64];
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * hw), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);
                            if (lane == 0 && e == 0) EPK_TRACE(P, 2, 10);
                            score_cols<64>(v, s_lse + r0, r0, P, best, s_avg, r_local);
                        }
                        ++job;
                    }
                    if (lane == 0 && e == 0) EPK_TRACE(P, 2, 11);
                    // combine the two column halves of each cache row
                    const int jrow = (x.t0 + t) * P.krows + r_local;
                    if (P.agg_max) {
                        if (half == 1) s_pair[r_local] = best;
                        named_bar_sync(2 + quarter, 64);
                        if (half == 0 && jrow < x.n_h) P.scores[x.krow0 + jrow] = ex2(fmaxf(best, s_pair[r_local]));
                        named_bar_sync(2 + quarter, 64);
                    } else {
                        named_bar_sync(2 + quarter, 64);
                        if (half == 0) {
                            float b = -INFINITY;
                            for (int gg = 0; gg < P.G; ++gg) {
                                b = fmaxf(b, s_avg[gg * kChunk + r_local] * inv_p);
                                s_avg[gg * kChunk + r_local] = 0.f;
                            }
                            if (jrow < x.n_h) P.scores[x.krow0 + jrow] = b;
                        }
                        named_bar_sync(2 + quarter, 64);
                    }
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
    const int64_t rows = int64_t(P.L) * P.H * P.NQ * kChunk;
    if (idx >= rows) return;
    const int rq = int(idx % (P.NQ * kChunk));
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

static int make_map(CUtensorMap* m, const void* base, int64_t rows, int box_rows) {
    auto enc = get_encode();
    if (!enc) return fail(EPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {cuuint64_t(kD), cuuint64_t(std::max<int64_t>(rows, 1))};
    cuuint64_t strides[1] = {cuuint64_t(kD * 2)};
    cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(EPK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return EPK_OK;
}

static int smem_bytes(const TcParams& P, int mode) {
    return 1024 + 2 * P.qcap * kRowB + P.kstages * 2 * P.krows * kRowB +
           (mode == MODE_SCORE ? (P.NQ + 1 + (P.agg_max ? 0 : P.G)) * kChunk * 4 : 0) +
           (2 * P.kstages + 2 * kMaxQRes + 4) * 8 + 16;
}

int launch_score_tc(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int hq, int p, int agg_max,
                    int64_t n_max, float* scores) {
    if (c->dtype != EPK_BF16) return fail(EPK_ERR_ARG, "score(tensor core): cache dtype must be BF16");
    if (c->head_dim != kD) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): head_dim must be 128");
    const int H = c->kv_heads;
    if (hq % H != 0) return fail(EPK_ERR_DIM, "score_with_prompt: attention grid shape mismatch");
    if (p > 256) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): prompt_len must be <= 256");
    TcParams P;
    int rc = make_layer_table(c, &P.lt);
    if (rc) return rc;
    P.L = c->layers;
    P.H = H;
    P.Hq = hq;
    P.G = hq / H;
    P.p = p;
    P.Gp = P.G * p;
    P.NQ = (P.Gp + kChunk - 1) / kChunk;
    if (P.NQ > 16) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): group*prompt_len must be <= 2048");
    P.splits = int(std::max<int64_t>(1, (n_max + kSplitCols - 1) / kSplitCols));
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.c2 = float((1.0 / std::sqrt(double(kD))) * 1.4426950408889634);
    P.scores = scores;
    P.agg_max = agg_max;
    P.trace = nullptr;
    static unsigned long long* trace_buf = nullptr;
    if (std::getenv("EPK_TC_TRACE")) {
        if (!trace_buf) EPK_CUDA_CHECK(cudaMalloc(&trace_buf, 8 * 180001));
        EPK_CUDA_CHECK(cudaMemsetAsync(trace_buf, 0, 8 * 180001, ctx->stream));
        P.trace = trace_buf;
    }
    const int64_t rows = int64_t(P.L) * H * P.NQ * kChunk;
    rc = ws_require(ctx, rows * 2 * P.splits * 8 + rows * 4 + 4096);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.part_m = carve.take<float>(rows * 2 * P.splits);
    P.part_z = carve.take<float>(rows * 2 * P.splits);
    P.lse2 = carve.take<float>(rows);

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

    CUtensorMap tm_k1, tm_k2, tm_q, tm_kp;
    if ((rc = make_map(&tm_k1, c->k, c->layer_base[c->layers], 256))) return rc;
    if ((rc = make_map(&tm_k2, c->k, c->layer_base[c->layers], 128))) return rc;
    if ((rc = make_map(&tm_q, q, int64_t(P.L) * hq * p, kChunk))) return rc;
    if ((rc = make_map(&tm_kp, kp, int64_t(P.L) * H * p, 256))) return rc;

    // P1: 256-row K stages; query chunks in groups sized so two stages fit.
    P.krows = 256;
    P.resident = 1;
    P.cg_chunks = std::min(P.NQ, kMaxQRes);
    for (;;) {
        P.qcap = P.cg_chunks * kChunk;
        P.kstages = 2;
        if (smem_bytes(P, MODE_STATS) <= limit || P.cg_chunks == 1) break;
        --P.cg_chunks;
    }
    while (P.kstages < 4) {
        ++P.kstages;
        if (smem_bytes(P, MODE_STATS) > limit) {
            --P.kstages;
            break;
        }
    }
    if (const char* ks = std::getenv("EPK_P1_KSTAGES")) P.kstages = std::max(1, std::min(P.kstages, std::atoi(ks)));
    if (smem_bytes(P, MODE_STATS) > limit) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): shared memory");
    P.cgroups = (P.NQ + P.cg_chunks - 1) / P.cg_chunks;
    P.items = int64_t(P.L) * H * P.splits * P.cgroups;
    if (std::getenv("EPK_TC_VERBOSE"))
        fprintf(stderr, "P1: NQ=%d cg_chunks=%d kstages=%d smem=%d limit=%d items=%lld\n", P.NQ, P.cg_chunks,
                P.kstages, smem_bytes(P, MODE_STATS), limit, (long long)P.items);
    const int grid1 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p1_rowstats");
    tc_score_kernel<MODE_STATS><<<grid1, kThreads, smem_bytes(P, MODE_STATS), ctx->stream>>>(P, tm_k1, tm_q, tm_kp);
    EPK_LAUNCH_CHECK(ctx);
    EPK_PROF(ctx, "p1_merge");
    tc_merge_kernel<<<unsigned((rows + 255) / 256), 256, 0, ctx->stream>>>(P);
    EPK_LAUNCH_CHECK(ctx);

    // P2: 128-row K stages; all query chunks resident when they fit, else
    // streamed as chunk pairs through two 256-row slots.
    P.krows = 128;
    P.resident = P.NQ <= kMaxQRes;
    P.qcap = P.resident ? P.NQ * kChunk : 4 * kChunk;
    P.kstages = 1;
    while (P.kstages < 4) {
        ++P.kstages;
        if (smem_bytes(P, MODE_SCORE) > limit) {
            --P.kstages;
            break;
        }
    }
    if (const char* ks = std::getenv("EPK_P2_KSTAGES")) P.kstages = std::max(2, std::min(P.kstages, std::atoi(ks)));
    if (P.kstages < 2 || smem_bytes(P, MODE_SCORE) > limit)
        return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): shared memory");
    P.cgroups = 1;
    P.cg_chunks = P.NQ;
    P.items = int64_t(P.L) * H * P.splits;
    if (std::getenv("EPK_TC_VERBOSE"))
        fprintf(stderr, "P2: NQ=%d resident=%d kstages=%d smem=%d items=%lld\n", P.NQ, P.resident, P.kstages,
                smem_bytes(P, MODE_SCORE), (long long)P.items);
    const int grid2 = int(std::min<int64_t>(P.items, ctx->num_sms));
    EPK_PROF(ctx, "p2_colscore");
    tc_score_kernel<MODE_SCORE><<<grid2, kThreads, smem_bytes(P, MODE_SCORE), ctx->stream>>>(P, tm_k2, tm_q, tm_kp);
    EPK_LAUNCH_CHECK(ctx);
    if (P.trace) {  // dump CTA 0's P2 timeline
        static std::vector<unsigned long long> h(180001);
        EPK_CUDA_CHECK(cudaMemcpyAsync(h.data(), trace_buf, 8 * 180001, cudaMemcpyDeviceToHost, ctx->stream));
        EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (FILE* f = std::fopen(std::getenv("EPK_TC_TRACE"), "wb")) {
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    return EPK_OK;
}

}  // namespace epk
