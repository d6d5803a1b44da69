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
// One persistent kernel template, two modes, 128-row K tiles:
//   STATS (P1): A = 128-row query chunk (resident), B = K tile, MMA 128 x 128
//               x 128 per (tile, chunk) job, D[query row][cache col] ->
//               epilogue lanes own a query row and keep an online (max, sum
//               exp2) per chunk (13/16 of the exp2 on MUFU, 3/16 as an FMA-pipe
//               polynomial) -> one partial (m, Z) per (row, CTA segment,
//               epilogue group).  P1 is bound by the exp2 rate, not the MMA.
//   merge       tc_bias_kernel, one CTA per head: each query row's lse2 from
//               its partials, written as P2's bias operand row.
//   SCORE (P2): A = K tile, B = the head's query rows (<= 512 resident, as
//               MMA jobs of N <= 256, 384 -> 2 x 192), D[cache row][query
//               row]; the lse subtraction rides in the MMA as one extra
//               16-wide K-step (bias rows), so the epilogue lanes (a cache row
//               each) reduce a bare max over query rows -> one exp2 per cache
//               row.  More query chunks than fit: Max runs one launch per
//               resident query group carrying each row's running max; Avg
//               streams chunk pairs through two slots per K tile.
//
// Work partition (tile-balanced): a mode's work is the sequence of RUNS
// (STATS: (layer, kv-head, query-chunk group); SCORE: (layer, kv-head)), each
// a run of 128-row K tiles (STATS: ceil(n_h/128) cache tiles + the causal
// prompt tiles; SCORE: ceil(n_h/128)).  Every CTA computes the run prefix from the
// device-resident head lengths (ragged after pooled eviction) and takes the
// contiguous global tile range [T b/grid, T (b+1)/grid); a run cut by a CTA
// boundary becomes two segments whose softmax partials P2 combines.  So the
// makespan is within one tile of the mean for any layer group and any
// per-head raggedness.
//
// Shared memory keeps Q as [d-half][resident query rows] (128-byte swizzled
// rows, 8-row groups 1024 B apart) so consecutive 128-row chunks form one
// B operand of up to 256 rows.  TMEM (512 columns): STATS three 128-column
// accumulator slots, each owned by one epilogue group and one MMA warp (job
// j -> slot j mod 3); SCORE two 256-column slots.
// Warp roles: warp 0 TMA producer; STATS (512 threads): warps 1-3 MMA issuers
// (one per slot), warps 4-15 epilogue in three groups of four; SCORE (352
// threads): warps 1-2 MMA issuers (alternate jobs), warps 3-10 epilogue
// (warp e: TMEM lane quarter warp & 3, column half of every job).  Warp 1
// owns the TMEM allocation.  One elected lane issues per MMA warp.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "tc_common.cuh"

namespace epk {

using namespace sm100;

constexpr int kEpiWarps = 8;      // SCORE epilogue warps (two column halves)
#ifndef EPK_STATS_EPI_WARPS
#define EPK_STATS_EPI_WARPS 12
#endif
constexpr int kEpiWarpsStats = EPK_STATS_EPI_WARPS;  // STATS epilogue warps: job groups of four
constexpr int kStatGroups = kEpiWarpsStats / 4;
// STATS TMEM slots (128 columns each): a multiple of the group count so every
// slot belongs to ONE epilogue group, and STATS jobs go to the MMA warp of
// their SLOT (slot % kMmaWarpsStats) -- every slot's full/empty barriers are then
// waited on by one warp in phase order, so a parity wait can never alias two
// phases apart (with slot = job % 4 and three groups a group could reach its
// next job on a slot while another group's job there was still in flight; with
// three slots and jobs alternating MMA warps an MMA warp could skip a phase).
#ifdef EPK_STATS_SLOTS
constexpr int kStatSlots = EPK_STATS_SLOTS;
#else
constexpr int kStatSlots = kStatGroups == 2 ? 4 : kStatGroups;
#endif
static_assert(kStatSlots * 128 <= 512, "STATS TMEM slots");
constexpr int kMmaWarps = 2;  // SCORE: MMA issuers alternate jobs: one issues while the other synchronises
#ifndef EPK_STATS_MMA_WARPS
#define EPK_STATS_MMA_WARPS 3
#endif
// STATS: one MMA issuer per TMEM slot, so a slot whose group lags never
// holds back the MMA of another slot (no head-of-line blocking; 16 warps x 128
// registers = the whole register file; P1 0.285 -> 0.277 ms at cfg2)
constexpr int kMmaWarpsStats = EPK_STATS_MMA_WARPS;
// more slots than groups (a group's jobs rotate over the slots): one MMA warp
// issues every job in order, so a slot's phases complete in job order and a
// group can never wait on a phase two ahead of the slot's barrier
static_assert(kStatSlots % kStatGroups == 0 || kMmaWarpsStats == 1, "STATS slots/groups/MMA warps");
template <int MODE>
constexpr int mma_warps() { return MODE == 0 ? kMmaWarpsStats : kMmaWarps; }
constexpr int kThreads = 32 * (1 + kMmaWarps + kEpiWarps);
constexpr int kThreadsStats = 32 * (1 + kMmaWarpsStats + kEpiWarpsStats);
constexpr int kMaxQRes = 4;  // resident query chunks (P1: per chunk group)

enum { MODE_STATS = 0, MODE_SCORE = 1 };

struct TcParams {
    LayerTable lt;
    int L, H, Hq, G, p, Gp, NQ;
    int cgroups;    // STATS query-chunk groups (SCORE: P1's, for the merge)
    int cg_chunks;  // chunks per group
    int krows;      // K tile rows: 256 (STATS) / 128 (SCORE)
    int kstages;    // K ring depth
    int qcap;       // rows per d-half in the Q region
    int resident;   // SCORE: the launch's query chunks resident (else streamed pairs)
    int qg0, qgn;   // SCORE: the launch's query chunks [qg0, qg0 + qgn) (a query group when NQ > kMaxQRes)
    int qgroups;    // SCORE: resident query groups (0: streamed pairs)
    // SCORE over several query groups (Max, NQ > kMaxQRes): per cache row the
    // running max of x - lse2/c2 over the groups done so far; the launch of
    // a non-last group writes it, of a non-first group reads it, and only the
    // last group emits the score
    float* best_io;
    int best_read, best_write;
    int runs;       // runs of this launch
    int ptiles;     // STATS: causal prompt tiles per run
    int p1_grid;    // STATS grid (SCORE reads it to locate the partials)
    int p1_runs;    // STATS runs
    int slots;      // partial slots per query row (kStatGroups per STATS CTA)
    int hk_base;    // global (layer, head) index of this launch's first head (rows of part_m / part_z)
    int run_hk_base;  // SCORE: heads of the P1 launch (its layer range) before this launch's first head
    const int32_t* head_off;
    const int32_t* head_len;
    int32_t* p1_pre;  // [p1_runs + 1] run prefix of the STATS launch over this layer range (its CTA 0 writes it)
    float c2;         // d^-1/2 * log2(e)
    float* part_m;    // [slots][prow]: slot-major, so P1's writes and the merge's reads coalesce over rows
    float* part_z;
    int64_t prow;     // query rows of the whole plan (L*H*NQ*128)
    int sj, sj_n0, sj_nl;  // SCORE MMA jobs per K tile: count, N of all but the last, N of the last
    // SCORE: per (head, query row) -lse2/c2 split into three bf16 terms, in
    // the no-swizzle K-major operand layout of a 16-wide MMA K-step (32 B per
    // row; tc_bias_kernel writes it between the passes, P2 loads it next to
    // each query chunk):
    // the lse subtraction runs inside the MMA as one extra K-step.
    const uint8_t* bias;  // [L*H][NQ*128 rows][32 B]
    uint8_t* bias_out;    // tc_bias_kernel's output (the same buffer)
    float* scores;
    int agg_max;
    // SCORE, fused selection histogram (threshold select, select.cu): per
    // live row its order-preserving key, and per layer a 65536-bin histogram
    // of float_bits(score) >> 14 plus a 256-bin coarse one (bin >> 8).
    uint32_t* keys;         // [rows] or null
    uint32_t* hist_fine;    // [L][65536]
    uint32_t* hist_coarse;  // [L][256]
    int* err_flag;          // EPK_ERR_NAN on a NaN score
};

// ---- tile-balanced partition ------------------------------------------------
// CTA b owns global tiles [B(b), B(b+1)), B(b) = floor(T b / grid).
__device__ __forceinline__ int part_bound(int64_t T, int grid, int b) { return int(T * b / grid); }
// number of CTAs b in [0, grid) with B(b) <= x  (the CTA holding tile x is cnt(x) - 1)
__device__ __forceinline__ int part_cnt(int64_t T, int grid, int64_t x) {
    return int(min(int64_t(grid), ((x + 1) * grid + T - 1) / T));
}

template <int MODE>
__device__ __forceinline__ int run_tiles(const TcParams& P, int r) {
    if (MODE == MODE_STATS) {
        const int n = P.head_len[r / P.cgroups];
        return n > 0 ? (n + 127) / 128 + P.ptiles : 0;
    }
    return (P.head_len[r] + 127) / 128;
}

// Exclusive prefix of run tiles into s_pre[0..runs] (warp 0).
template <int MODE>
__device__ void run_prefix(const TcParams& P, int32_t* s_pre) {
    const int lane = threadIdx.x & 31;
    const int per = (P.runs + 31) / 32;
    const int a = min(P.runs, lane * per), b = min(P.runs, a + per);
    int sum = 0;
    for (int i = a; i < b; ++i) sum += run_tiles<MODE>(P, i);
    int incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    int run = incl - sum;
    for (int i = a; i < b; ++i) {
        s_pre[i] = run;
        run += run_tiles<MODE>(P, i);
    }
    if (lane == 31) s_pre[P.runs] = incl;
}

struct Seg {
    int r, hk, l, h, cg;
    int n_h;
    int64_t krow0;       // first K row of the head (global)
    int t0, nc, np, p0;  // first cache tile, cache tiles, prompt tiles, first prompt tile
    int c0, nq;          // first query chunk, chunks
    int slot;            // STATS: 2 * (this CTA - first CTA of the run)
    __device__ int ntiles() const { return nc + np; }
};

// The segment of this CTA's range that starts at global tile g.
template <int MODE>
__device__ __forceinline__ Seg seg_at(const TcParams& P, const int32_t* s_pre, int g, int g_end, int64_t T) {
    int lo = 0, hi = P.runs - 1;
    while (lo < hi) {  // last run with s_pre[r] <= g (skips empty runs)
        const int mid = (lo + hi + 1) >> 1;
        if (s_pre[mid] <= g) lo = mid; else hi = mid - 1;
    }
    Seg x;
    x.r = lo;
    const int R0 = s_pre[lo], R1 = s_pre[lo + 1];
    const int ta = g - R0, tb = min(R1, g_end) - R0;
    if (MODE == MODE_STATS) {
        x.hk = lo / P.cgroups;
        x.cg = lo % P.cgroups;
    } else {
        x.hk = lo;
        x.cg = 0;
    }
    x.l = x.hk / P.H;
    x.h = x.hk % P.H;
    x.n_h = P.head_len[x.hk];
    x.krow0 = P.lt.base[x.l] + P.head_off[x.l * (P.H + 1) + x.h];
    const int ntc = (x.n_h + P.krows - 1) / P.krows;
    x.t0 = ta;
    x.nc = max(0, min(tb, ntc) - ta);
    const int pa = max(ta, ntc);
    x.np = max(0, tb - pa);
    x.p0 = pa - ntc;
    if (MODE == MODE_STATS) {
        x.c0 = x.cg * P.cg_chunks;
        x.nq = min(P.cg_chunks, P.NQ - x.c0);
        x.slot = kStatGroups * (int(blockIdx.x) - (part_cnt(T, gridDim.x, R0) - 1));
    } else {
        x.c0 = P.qg0;
        x.nq = P.qgn;
        x.slot = 0;
    }
    return x;
}

// SCORE output of one live row: the score, and (fused selection) its key and
// histogram counts.
__device__ __forceinline__ void emit_score(const TcParams& P, int layer, int64_t row, float sc, uint32_t* s_coarse) {
    if (sc != sc) atomicCAS(P.err_flag, 0, EPK_ERR_NAN);  // non-finite inputs: the selection has no order for NaN
    if (P.scores) P.scores[row] = sc;  // null: a fused step whose caller wants no scores (the keys carry them)
    if (P.keys) {
        P.keys[row] = desc_key(sc);
        const uint32_t b = min(__float_as_uint(sc) >> 14, 65535u);
        atomicAdd(&P.hist_fine[int64_t(layer) * 65536 + b], 1u);
        atomicAdd(&s_coarse[b >> 8], 1u);
    }
}

// Adds the CTA's coarse histogram of `layer` to the global one and clears it
// (the 256 epilogue threads, after a barrier).
__device__ __forceinline__ void flush_coarse(const TcParams& P, int layer, uint32_t* s_coarse, int etid) {
    const uint32_t v = s_coarse[etid];
    if (v) {
        atomicAdd(&P.hist_coarse[layer * 256 + etid], v);
        s_coarse[etid] = 0;
    }
}

// lse2 of STATS query row rq of head hk (launch-local) from the partials of
// every P1 CTA that covered the row's run: `pre` = the P1 launch's run prefix,
// `grid` its CTAs, `run_hk_base` its heads before this launch's first.  The
// partials of other CTAs are read through L2 (ld.cg).
__device__ float merge_lse2(const TcParams& P, const int32_t* pre, int grid, int run_hk_base, int hk, int rq,
                            int64_t T1) {
    const int cg = (rq / kChunk) / P.cg_chunks;
    const int run = (hk + run_hk_base) * P.cgroups + cg;
    const int R0 = pre[run], R1 = pre[run + 1];
    if (R1 <= R0) return INFINITY;
    const int b0 = part_cnt(T1, grid, R0) - 1, b1 = part_cnt(T1, grid, R1 - 1) - 1;
    const int64_t row = int64_t(hk + P.hk_base) * (P.NQ * kChunk) + rq;
    const float* pm = P.part_m + row;
    const float* pz = P.part_z + row;
    float M = -INFINITY;
    for (int b = b0; b <= b1; ++b) {
        const int lo = max(R0, part_bound(T1, grid, b)), hi = min(R1, part_bound(T1, grid, b + 1));
        if (lo >= hi) continue;
        const int s = kStatGroups * (b - b0);
        for (int u = 0; u < kStatGroups; ++u) M = fmaxf(M, __ldcg(pm + (s + u) * P.prow));
    }
    if (M == -INFINITY) return INFINITY;
    float Z = 0.f;
    for (int b = b0; b <= b1; ++b) {
        const int lo = max(R0, part_bound(T1, grid, b)), hi = min(R1, part_bound(T1, grid, b + 1));
        if (lo >= hi) continue;
        const int s = kStatGroups * (b - b0);
#pragma unroll
        for (int u = 0; u < kStatGroups; ++u) {
            const float mu = __ldcg(pm + (s + u) * P.prow);
            if (mu != -INFINITY) Z += __ldcg(pz + (s + u) * P.prow) * ex2(mu - M);
        }
    }
    return M + log2f(Z);
}

// P2's bias operand row of (head hk, query row rq) from its lse2:
// -lse2/c2 = h + m + l (bf16 parts; each residual is exact in fp32, so the sum
// carries ~24 bits).  Padding rows (>= G*p) and rows with no live column get
// h = -1e30 (finite: the zero K elements of A' multiply it), so their columns
// never win the max.
__device__ void write_bias_row(const TcParams& P, int hk, int rq, float lse2) {
    float h = -1e30f, m = 0.f, l = 0.f;
    if (rq < P.Gp) {
        if (lse2 != lse2) atomicCAS(P.err_flag, 0, EPK_ERR_NAN);  // a NaN logit poisoned the row's sum
        if (lse2 != INFINITY) {
            const float v = __fdiv_rn(-lse2, P.c2);
            const __nv_bfloat16 bh = __float2bfloat16_rn(v);
            const float r1 = __fsub_rn(v, __bfloat162float(bh));
            const __nv_bfloat16 bm = __float2bfloat16_rn(r1);
            const float r2 = __fsub_rn(r1, __bfloat162float(bm));
            h = __bfloat162float(bh);
            m = __bfloat162float(bm);
            l = __bfloat162float(__float2bfloat16_rn(r2));
        }
    }
    const __nv_bfloat162 hm = __floats2bfloat162_rn(h, m), l0 = __floats2bfloat162_rn(l, 0.f);
    uint8_t* row = P.bias_out + int64_t(hk + P.hk_base) * (P.NQ * kChunk) * kBiasRowB + bias_off(rq);
    *reinterpret_cast<uint4*>(row) =
        make_uint4(*reinterpret_cast<const uint32_t*>(&hm), *reinterpret_cast<const uint32_t*>(&l0), 0u, 0u);
    *reinterpret_cast<uint4*>(row + 128) = make_uint4(0u, 0u, 0u, 0u);  // K elements 8..15
}

// Between P1 and P2, one CTA per head (NQ*128 threads, a query row each): the
// row's lse2 from its P1 partials, written as its bias operand row.  The
// covering P1 CTAs of each chunk group (the partial slots to merge) are
// listed once per CTA, so the per-row work is the merge loads alone.
constexpr int kBiasMaxCov = 32;
__global__ void tc_bias_kernel(const __grid_constant__ TcParams P) {
    __shared__ int s_cov[16][kBiasMaxCov];  // per chunk group: slot base of each covering P1 CTA
    __shared__ int s_ncov[16];
    TL_BEGIN();
    pdl_wait();
    TL_GO();
    const int hk = blockIdx.x;
    const int64_t T1 = P.p1_pre[P.p1_runs];
    if (threadIdx.x < P.cgroups) {
        const int run = (hk + P.run_hk_base) * P.cgroups + threadIdx.x;
        const int R0 = P.p1_pre[run], R1 = P.p1_pre[run + 1];
        int n = 0;
        if (R1 > R0) {
            const int b0 = part_cnt(T1, P.p1_grid, R0) - 1, b1 = part_cnt(T1, P.p1_grid, R1 - 1) - 1;
            for (int b = b0; b <= b1 && n >= 0; ++b) {
                if (max(R0, part_bound(T1, P.p1_grid, b)) >= min(R1, part_bound(T1, P.p1_grid, b + 1))) continue;
                if (n == kBiasMaxCov) n = -1;  // more covering CTAs than listed: the general merge
                else s_cov[threadIdx.x][n++] = kStatGroups * (b - b0);
            }
        }
        s_ncov[threadIdx.x] = n;
    }
    __syncthreads();
    for (int rq = threadIdx.x; rq < P.NQ * kChunk; rq += blockDim.x) {
    float lse2 = INFINITY;
    if (rq < P.Gp) {
        const int cg = (rq / kChunk) / P.cg_chunks;
        const int n = s_ncov[cg];
        if (n < 0) {
            lse2 = merge_lse2(P, P.p1_pre, P.p1_grid, P.run_hk_base, hk, rq, T1);
        } else if (n > 0) {
            const int64_t row = int64_t(hk + P.hk_base) * (P.NQ * kChunk) + rq;
            float M = -INFINITY;
            for (int i = 0; i < n; ++i)
#pragma unroll
                for (int u = 0; u < kStatGroups; ++u) M = fmaxf(M, P.part_m[(s_cov[cg][i] + u) * P.prow + row]);
            if (M != -INFINITY) {
                float Z = 0.f;
                for (int i = 0; i < n; ++i)
#pragma unroll
                    for (int u = 0; u < kStatGroups; ++u) {
                        const int64_t o = (s_cov[cg][i] + u) * P.prow + row;
                        const float mu = P.part_m[o];
                        if (mu != -INFINITY) Z += P.part_z[o] * ex2(mu - M);
                    }
                lse2 = M + log2f(Z);
            }
        }
    }
    write_bias_row(P, hk, rq, lse2);
    }
    TL_END(3);
}

// <= 128 registers (45K of the SM's 64K) and <= kSmemBudget of shared memory,
// so the side stream's select/compaction CTAs can co-reside with a scorer CTA.
#ifdef EPK_P1_PROF
#define P1PROF(...) __VA_ARGS__
#else
#define P1PROF(...)
#endif
#ifdef EPK_P2_PROF
#define P2PROF(...) __VA_ARGS__
#else
#define P2PROF(...)
#endif
#if defined(EPK_P1_PROF) || defined(EPK_P2_PROF)
#define MPROF(...) __VA_ARGS__
#else
#define MPROF(...)
#endif
#ifdef EPK_NO_BACKOFF
#define mbar_wait_pm mbar_wait
#else
#define mbar_wait_pm mbar_wait_backoff
#endif

template <int MODE>
__global__ void __maxnreg__(128)
    tc_score_kernel(const __grid_constant__ TcParams P, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp) {
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte aligned (SWIZZLE_128B atoms), derived from smem_raw by pointer
    // arithmetic so the compiler keeps shared-space (LDS/STS) addressing.
    TL_BEGIN();
    pdl_wait();  // every input may come from the previous kernel in the stream
    TL_GO();
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t q_half = uint32_t(P.qcap) * kRowB;   // Q d-half stride
    const uint32_t k_half = uint32_t(P.krows) * kRowB;  // K d-half stride
    const uint32_t k_stage = 2 * k_half;
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + 2 * q_half;
    uint8_t* s_bias = sK + P.kstages * k_stage;  // SCORE: bias rows of the Q region's chunks
    uint8_t* s_aone = s_bias + (MODE == MODE_SCORE ? P.qcap * kBiasRowB : 0);  // SCORE: A' = [1 1 1 0..] x 128 rows
    float* s_pair = reinterpret_cast<float*>(s_aone + (MODE == MODE_SCORE ? kBiasChunkB : 0));  // SCORE: [2][128] half maxima
    float* s_avg = s_pair + (MODE == MODE_SCORE ? 2 * kChunk : 0);     // SCORE avg: G*128 sums
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_avg + (MODE == MODE_SCORE && !P.agg_max ? P.G * kChunk : 0));
    uint64_t* k_full = bars;
    uint64_t* k_empty = k_full + P.kstages;
    uint64_t* q_full = k_empty + P.kstages;  // per resident chunk, or per streamed pair slot
    uint64_t* q_empty = q_full + kMaxQRes;
    uint64_t* t_full = q_empty + kMaxQRes;
    uint64_t* t_empty = t_full + 4;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(t_empty + 4);
    int32_t* s_pre = reinterpret_cast<int32_t*>(tmem_holder + 4);  // [runs + 1]

    __shared__ uint32_t s_coarse[256];      // SCORE: coarse histogram of the current layer
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool resident = MODE == MODE_STATS || P.resident;

    if (warp == 0) {
        run_prefix<MODE>(P, s_pre);
        if (lane == 0) {
            tma_prefetch(&tm_k);
            tma_prefetch(&tm_q);
            if (MODE == MODE_STATS) tma_prefetch(&tm_kp);
            for (int s = 0; s < P.kstages; ++s) {
                mbar_init(&k_full[s], 1);
                mbar_init(&k_empty[s], mma_warps<MODE>());  // every MMA warp releases every stage
            }
            for (int s = 0; s < kMaxQRes; ++s) {
                mbar_init(&q_full[s], 1);
                mbar_init(&q_empty[s], resident ? mma_warps<MODE>() : 1);  // streamed slots belong to one MMA warp
            }
            for (int s = 0; s < 4; ++s) {
                mbar_init(&t_full[s], 1);
                // STATS: a slot is drained by the 4 warps of the job's group;
                // SCORE: by all 8 (two column halves)
                mbar_init(&t_empty[s], MODE == MODE_STATS ? 4 : kEpiWarps);
            }
            fence_barrier_init();
        }
    }
    if (MODE == MODE_STATS && P.hist_fine) {
        // the fused selection's score histograms start every step at zero:
        // P1 clears them (its CTAs are SFU-bound, the stores are free) for the
        // P2 launch that fills them; the previous step's select read them
        // before this launch's pdl_wait returned
        const int64_t n4 = int64_t(P.L) * (65536 / 4), per = (n4 + gridDim.x - 1) / gridDim.x;
        uint4* hf4 = reinterpret_cast<uint4*>(P.hist_fine);
        for (int64_t i = blockIdx.x * per + threadIdx.x; i < min(n4, (blockIdx.x + 1) * per); i += blockDim.x)
            hf4[i] = make_uint4(0, 0, 0, 0);
        if (blockIdx.x == 0)
            for (int i = threadIdx.x; i < P.L * 256; i += blockDim.x) P.hist_coarse[i] = 0;
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    if (MODE == MODE_SCORE && !P.agg_max)
        for (int i = threadIdx.x; i < P.G * kChunk; i += blockDim.x) s_avg[i] = 0.f;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_coarse[i] = 0;
    if (MODE == MODE_SCORE) {
        // A' rows: bf16 1.0 in K elements 0..2, zeros elsewhere (written by
        // threads, read by the tensor core: async-proxy fence before the barrier)
        for (int i = threadIdx.x; i < kBiasChunkB / 4; i += blockDim.x) {
            const int byte = i * 4, kb = byte & 15, khi = byte & 128;  // every row of the chunk alike
            uint32_t w = 0;
            if (!khi && kb == 0) w = 0x3F803F80u;  // K 0, 1
            if (!khi && kb == 4) w = 0x00003F80u;  // K 2
            reinterpret_cast<uint32_t*>(s_aone)[i] = w;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const int64_t T = s_pre[P.runs];
    if (MODE == MODE_STATS && blockIdx.x == 0)
        for (int i = threadIdx.x; i <= P.runs; i += blockDim.x) P.p1_pre[i] = s_pre[i];
    const int it_beg = part_bound(T, gridDim.x, blockIdx.x);
    const int it_end = part_bound(T, gridDim.x, blockIdx.x + 1);

    if (warp == 0) {
        const bool leader = elect_one_sync();
        {  // ------------------------- TMA producer (warp-wide, one lane issues) -----------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kMaxQRes] = {0, 0, 0, 0};
            int key = -1;
            int64_t pj = 0;
            const int npairs = (P.NQ + 1) / 2;
            MPROF(long long pw = 0; const long long p_beg = clock64());
            for (int g = it_beg; g < it_end;) {
                const Seg x = seg_at<MODE>(P, s_pre, g, it_end, T);
                g += x.ntiles();
                const int qrow0 = (x.l * P.Hq + x.h * P.G) * P.p;
                if (resident && x.r != key) {
                    key = x.r;
                    for (int c = 0; c < x.nq; ++c) {
                        mbar_wait_pm(&q_empty[c], (qload[c] & 1) ^ 1);
                        if (leader) {
                            mbar_expect_tx(&q_full[c], 2 * kChunk * kRowB + (MODE == MODE_SCORE ? kBiasChunkB : 0));
                            load_rows(sQ + c * kChunk * kRowB, q_half, &tm_q, &q_full[c], qrow0 + (x.c0 + c) * kChunk);
                            if (MODE == MODE_SCORE)
                                bulk_load_1d(s_bias + c * kBiasChunkB,
                                             P.bias + (int64_t(x.hk + P.hk_base) * P.NQ + x.c0 + c) * kBiasChunkB,
                                             kBiasChunkB, &q_full[c]);
                        }
                        __syncwarp();
                        ++qload[c];
                    }
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    MPROF(long long c0 = clock64());
                    mbar_wait_pm(&k_empty[ks], kph ^ 1);
                    MPROF(pw += clock64() - c0);
                    if (leader) {
                        mbar_expect_tx(&k_full[ks], k_stage);
                        if (t < x.nc)
                            load_rows(sK + ks * k_stage, k_half, &tm_k, &k_full[ks],
                                      int(x.krow0 + int64_t(x.t0 + t) * P.krows));
                        else
                            load_rows(sK + ks * k_stage, k_half, &tm_kp, &k_full[ks],
                                      (x.l * P.H + x.h) * P.p + (x.p0 + t - x.nc) * P.krows);
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
                            mbar_wait_pm(&q_empty[slot], (qload[slot] & 1) ^ 1);
                            if (leader) {
                                mbar_expect_tx(&q_full[slot], nch * (2 * kChunk * kRowB + kBiasChunkB));
                                for (int cc = 0; cc < nch; ++cc) {
                                    load_rows(sQ + (slot * 2 + cc) * kChunk * kRowB, q_half, &tm_q, &q_full[slot],
                                              qrow0 + (2 * j + cc) * kChunk);
                                    bulk_load_1d(s_bias + (slot * 2 + cc) * kBiasChunkB,
                                                 P.bias + (int64_t(x.hk + P.hk_base) * P.NQ + 2 * j + cc) * kBiasChunkB,
                                                 kBiasChunkB, &q_full[slot]);
                                }
                            }
                            __syncwarp();
                            ++qload[slot];
                        }
                    }
                }
            }
            MPROF(if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
                      printf("%sPROF cta %d producer total %lld wait_kempty %lld\n", MODE == MODE_SCORE ? "P2" : "P1",
                             blockIdx.x, clock64() - p_beg, pw));
        }
    } else if (warp <= mma_warps<MODE>()) {
        // STATS: MMA warp mw issues the jobs of slot mw (job % 3); SCORE: the
        // jobs with (job & 1) == mw.  All MMA warps walk the same segment/tile
        // sequence and each releases every K stage.
        const uint32_t mw = uint32_t(warp - 1);
        const bool leader = elect_one_sync();
        {  // ------------------------- MMA issuers (warp-wide, one lane issues) ------------
            int ks = 0;
            uint32_t kph = 0;
            uint32_t qload[kMaxQRes] = {0, 0, 0, 0};
            uint32_t job = 0;
            int key = -1;
            int held = 0;
            const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK);
            MPROF(long long wk = 0, wt = 0, m_beg = clock64(); int ntile = 0);
            for (int g = it_beg; g < it_end;) {
                const Seg x = seg_at<MODE>(P, s_pre, g, it_end, T);
                g += x.ntiles();
                bool fresh = false;
                if (resident && x.r != key) {
                    if (leader)
                        for (int c = 0; c < held; ++c) mma_commit(&q_empty[c]);  // old Q retires with its MMAs
                    __syncwarp();
                    key = x.r;
                    held = x.nq;
                    fresh = true;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
                    MPROF(long long c0 = clock64());
                    mbar_wait_pm(&k_full[ks], kph);
                    MPROF(wk += clock64() - c0; ++ntile);
                    const uint32_t kst = k0 + uint32_t(ks) * k_stage;
                    if (MODE == MODE_STATS) {
                        for (int c = 0; c < x.nq; ++c, ++job) {
                            if (fresh && t == 0) {
                                mbar_wait_pm(&q_full[c], qload[c] & 1);
                                ++qload[c];
                            }
                            const int ts = int(job % kStatSlots);  // 128-column slots, one group each
                            if (ts % mma_warps<MODE>() != int(mw)) continue;
                            MPROF(long long c1 = clock64());
                            mbar_wait_pm(&t_empty[ts], ((job / kStatSlots) & 1) ^ 1);
                            MPROF(wt += clock64() - c1);
                            tc_fence_after();
                            if (leader) {
#if !defined(EPK_XP_NOMMA)  // experiment: P1 without its MMAs (wrong values)
                                mma_128xN(tmem + uint32_t(ts * 128), q0 + uint32_t(c * kChunk * kRowB), q_half, kst,
                                          k_half, idesc_bf16_f32(128, 128));
#endif
                                mma_commit(&t_full[ts]);
                            }
                            __syncwarp();
                        }
                    } else {
                        if (resident && fresh && t == 0)
                            for (int c = 0; c < x.nq; ++c) {
                                mbar_wait_pm(&q_full[c], qload[c] & 1);
                                ++qload[c];
                            }
                        for (int j = 0; j < P.sj; ++j, ++job) {
                            const int jn = j + 1 < P.sj ? P.sj_n0 : P.sj_nl;  // query rows (MMA N) of the job
                            if ((job & 1) != mw) continue;
                            uint32_t qb, bb;
                            const int slot = int(mw);  // streamed pair slot == TMEM slot == this warp
                            if (resident) {
                                const int row0 = j * P.sj_n0;
                                qb = q0 + uint32_t(row0 * kRowB);
                                bb = smem_u32(s_bias) + uint32_t(bias_off(row0));
                            } else {
                                mbar_wait_pm(&q_full[slot], qload[slot] & 1);
                                ++qload[slot];
                                qb = q0 + uint32_t(slot * 2 * kChunk * kRowB);
                                bb = smem_u32(s_bias) + uint32_t(slot * 2 * kBiasChunkB);
                            }
                            const int ts = int(mw);
                            P2PROF(long long c1 = clock64());
                            mbar_wait_pm(&t_empty[ts], ((job >> 1) & 1) ^ 1);
                            P2PROF(wt += clock64() - c1);
                            tc_fence_after();
                            if (leader) {
                                mma_128xN_bias(tmem + uint32_t(ts * 256), kst, k_half, qb, q_half, smem_u32(s_aone), bb,
                                               idesc_bf16_f32(128, uint32_t(jn)));
                                mma_commit(&t_full[ts]);
                                if (!resident) mma_commit(&q_empty[slot]);
                            }
                            __syncwarp();
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
            MPROF(if (lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
                       printf("%sPROF cta %d mma%d tiles %d total %lld wait_k %lld wait_tempty %lld\n",
                              MODE == MODE_SCORE ? "P2" : "P1", blockIdx.x, mw, ntile, clock64() - m_beg, wk, wt));
        }
    } else {  // ------------------------- epilogue warps -------------------------
        const int e = warp - 1 - mma_warps<MODE>();
        const int quarter = warp & 3;  // TMEM lanes this warp may read
        const int half = e >> 2;       // SCORE: column half of every job; STATS: job group (job % 3)
        const int r_local = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const int etid = e * 32 + lane;
        uint32_t job = 0;
        uint32_t tcount = 0;  // SCORE: tiles done (emitting half, partial buffer)
        int lkey = -1;
        const float inv_p = 1.0f / float(P.p);
        P2PROF(long long ewf = 0, ebar = 0, ehead = 0; int etiles = 0; const long long e_beg = clock64());
        P1PROF(long long pw = 0, pl = 0, pc = 0, pj = 0, po = 0, pfirst = 0; const long long p_beg = clock64(); long long c_prev = p_beg;
               uint64_t g_beg; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_beg)));
        for (int g = it_beg; g < it_end;) {
            const Seg x = seg_at<MODE>(P, s_pre, g, it_end, T);
            g += x.ntiles();
            if (MODE == MODE_STATS) {
                float m[kMaxQRes], z[kMaxQRes];
#pragma unroll
                for (int c = 0; c < kMaxQRes; ++c) {
                    m[c] = -INFINITY;
                    z[c] = 0.f;
                }
                // Group `half` takes the jobs (tile, chunk) with job % 3 ==
                // half -- TMEM slot `half` -- whole (128 columns), so the three
                // epilogue warps sharing an SM sub-partition work on different
                // jobs and their max / exp2 phases interleave on the SFU.
                for (int t = 0; t < x.ntiles(); ++t) {
#pragma unroll
                    for (int c = 0; c < kMaxQRes; ++c) {
                        if (c >= x.nq) break;
                        if (int(job % kStatGroups) != half) {
                            ++job;
                            continue;
                        }
                        const int rq = (x.c0 + c) * kChunk + r_local;  // query row of the head (g*p + t)
                        int lim;  // valid columns of this job from its first column
                        if (t < x.nc)
                            lim = x.n_h - (x.t0 + t) * P.krows;
                        else
                            lim = min(P.p, rq % P.p + 1) - (x.p0 + t - x.nc) * P.krows;
                        const int ts = int(job % kStatSlots);
                        P1PROF(long long c_0 = clock64(); po += c_0 - c_prev);
                        mbar_wait(&t_full[ts], (job / kStatSlots) & 1);
                        tc_fence_after();
                        {
                            float v[64];
                            P1PROF(long long c_1 = clock64());
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 128), v);
                            P1PROF(long long c_2 = clock64());
                            stats_cols<64>(v, lim, P.c2, m[c], z[c]);
                            P1PROF(long long c_3 = clock64());
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 128 + 64), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);  // slot free: values are in registers
                            P1PROF(long long c_4 = clock64());
                            stats_cols<64>(v, lim - 64, P.c2, m[c], z[c]);
                            P1PROF(long long c_5 = clock64(); pw += c_1 - c_0; pl += (c_2 - c_1) + (c_4 - c_3);
                                   pc += (c_3 - c_2) + (c_5 - c_4); if (pj == 0) pfirst = c_1 - p_beg; ++pj; c_prev = c_5);
                        }
                        ++job;
                    }
                }
                // partial (m, Z) of this column half for each query row of the segment
#pragma unroll
                for (int cc = 0; cc < kMaxQRes; ++cc) {
                    if (cc < x.nq) {
                        const int rq = (x.c0 + cc) * kChunk + r_local;
                        const int64_t o = int64_t(x.slot + half) * P.prow + int64_t(x.hk + P.hk_base) * (P.NQ * kChunk) + rq;
                        P.part_m[o] = m[cc];
                        P.part_z[o] = z[cc];
                    }
                }
            } else {
                P2PROF(long long ch = clock64());
                if (P.keys && x.l != lkey) {  // a new layer: flush the previous layer's coarse histogram
                    named_bar_sync(1, 32 * kEpiWarps);
                    if (lkey >= 0) flush_coarse(P, lkey, s_coarse, etid);
                    named_bar_sync(1, 32 * kEpiWarps);
                    lkey = x.l;
                }
                P2PROF(ehead += clock64() - ch);
                for (int t = 0; t < x.ntiles(); ++t) {
                    P2PROF(++etiles);
                    float best = -INFINITY;
                    for (int j = 0; j < P.sj; ++j) {
                        const int hw = (j + 1 < P.sj ? P.sj_n0 : P.sj_nl) / 2;  // columns per warp half: 32..128
                        const int ts = int(job & 1);
                        P2PROF(long long c0 = clock64());
                        mbar_wait(&t_full[ts], (job >> 1) & 1);
                        P2PROF(ewf += clock64() - c0);
                        tc_fence_after();
                        const int r0 = j * P.sj_n0 + half * hw;  // first query row of this warp's columns
                        const uint32_t ta = tmem + lane_addr + uint32_t(ts * 256 + half * hw);
                        if (hw >= 64) {
                            float v[64];
                            tmem_ld64(ta, v);
                            if (hw == 64) {
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&t_empty[ts]);  // slot free: values are in registers
                            }
                            score_cols<64>(v, r0, P, best, s_avg, r_local);
                            if (hw == 128) {
                                tmem_ld64(ta + 64, v);
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&t_empty[ts]);
                                score_cols<64>(v, r0 + 64, P, best, s_avg, r_local);
                            } else if (hw == 96) {
                                float w[32];
                                tmem_ld32(ta + 64, w);
                                tc_fence_before();
                                __syncwarp();
                                if (lane == 0) mbar_arrive(&t_empty[ts]);
                                score_cols<32>(w, r0 + 64, P, best, s_avg, r_local);
                            }
                        } else {
                            float w[32];
                            tmem_ld32(ta, w);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);
                            score_cols<32>(w, r0, P, best, s_avg, r_local);
                        }
                        ++job;
                    }
                    // combine the two column halves of each cache row
                    const int jrow = (x.t0 + t) * P.krows + r_local;
                    if (P.agg_max) {
                        // the halves take turns emitting (tile parity) and the
                        // partials are double-buffered, so one barrier per tile
                        // suffices: buffer b is rewritten two tiles later, past
                        // a barrier the reading half reaches only after its read
                        const int em = int(tcount & 1);
                        float* sp = s_pair + em * kChunk;
                        if (half != em) sp[r_local] = best;
                        P2PROF(long long cb = clock64());
                        named_bar_sync(2 + quarter, 64);
                        P2PROF(ebar += clock64() - cb);
                        if (half == em && jrow < x.n_h) {
                            const int64_t row = x.krow0 + jrow;
                            float b2 = fmaxf(best, sp[r_local]);
                            if (P.best_read) b2 = fmaxf(b2, __ldcg(P.best_io + row));
                            if (P.best_write)
                                P.best_io[row] = b2;  // a later query group's launch finishes the row
                            else
                                emit_score(P, x.l, row, ex2(b2 * P.c2), s_coarse);
                        }
                        ++tcount;
                    } else {
                        named_bar_sync(2 + quarter, 64);
                        if (half == 0) {
                            float b = -INFINITY;
                            for (int gg = 0; gg < P.G; ++gg) {
                                b = fmaxf(b, s_avg[gg * kChunk + r_local] * inv_p);
                                s_avg[gg * kChunk + r_local] = 0.f;
                            }
                            if (jrow < x.n_h) emit_score(P, x.l, x.krow0 + jrow, b, s_coarse);
                        }
                        named_bar_sync(2 + quarter, 64);
                    }
                }
            }
        }
        if (MODE == MODE_SCORE && P.keys && lkey >= 0) {  // last layer's coarse histogram
            named_bar_sync(1, 32 * kEpiWarps);
            flush_coarse(P, lkey, s_coarse, etid);
        }
        P2PROF(if (MODE == MODE_SCORE && lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
                   printf("P2PROF cta %d epi%d tiles %d total %lld wait_tfull %lld bar %lld head %lld\n", blockIdx.x, e,
                          etiles, clock64() - e_beg, ewf, ebar, ehead));
        P1PROF(uint64_t g_end; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end)); const long long p_end = clock64();
               if (MODE == MODE_STATS && lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77))
                   printf("P1PROF cta %d warp %2d jobs %lld total %lld wait %lld ld %lld compute %lld between %lld first %lld\n",
                          blockIdx.x, warp, pj, p_end - p_beg, pw, pl, pc, po, pfirst);
               if (MODE == MODE_STATS && lane == 0 && warp == 1 + kMmaWarpsStats) {
                   uint32_t smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                   printf("P1GT %d %llu %llu %u %lld %lld %lld %d %d\n", blockIdx.x, (unsigned long long)g_beg, (unsigned long long)g_end, smid, pj, pw, p_end - p_beg, it_beg, it_end);
               });
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
    TL_END(MODE == MODE_STATS ? 1 : 2);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int smem_bytes(const TcParams& P, int mode) {
    return 1024 + 2 * P.qcap * kRowB + P.kstages * 2 * P.krows * kRowB +
           (mode == MODE_SCORE ? (2 + (P.agg_max ? 0 : P.G)) * kChunk * 4 + P.qcap * kBiasRowB + kBiasChunkB : 0) +
           (2 * P.kstages + 2 * kMaxQRes + 8) * 8 + 16 + (P.runs + 1) * 4;
}

// SCORE launch of query group g (chunks [g kMaxQRes, ...)): its query rows
// (64-row units) split evenly over <= 256-row MMA jobs (384 -> 2 x 192).
static void p2_group_jobs(TcParams* P, int g) {
    P->qg0 = g * kMaxQRes;
    P->qgn = P->qgroups <= 1 ? P->NQ : std::min(kMaxQRes, P->NQ - P->qg0);
    const int rows = std::min(P->Gp - P->qg0 * kChunk, P->qgn * kChunk);
    const int R = (rows + 63) / 64 * 64;
    P->sj = (R + 255) / 256;
    P->sj_n0 = (R / 64 + P->sj - 1) / P->sj * 64;
    P->sj_nl = R - (P->sj - 1) * P->sj_n0;
}

// A tensor-core scoring launch plan.  P1 and P2 run per layer range [l0, l1)
// (a step's layer group): P1 of a range, then P2 of the same range, so the
// range's K tiles are re-read from L2 and a finished group's selection /
// compaction can overlap the next group's scoring.
struct TcPlan {
    TcParams P1, P2;
    CUtensorMap tm_k, tm_q, tm_kp;
    int smem1, smem2;
    int grid;  // persistent CTAs of both passes
    float* best_buf;  // P2 in query groups: the running max per cache row
    void (*stats_fn)(TcParams, CUtensorMap, CUtensorMap, CUtensorMap);
    void (*score_fn)(TcParams, CUtensorMap, CUtensorMap, CUtensorMap);
    const void* q;
    const void* kp;
    int64_t qlayer;   // bytes of one layer's query rows
    int64_t kplayer;  // bytes of one layer's prompt-key rows
    int32_t* p1_pre_all;  // run prefixes: range [l0, l1) at p1_pre_all + l0 * (H * cgroups + 1)
    epk_cache_desc c;
};

static int tc_plan(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int hq, int p, int agg_max,
                   float* scores, const FusedSelect* fs, TcPlan* out) {
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
    if (int64_t(P.L) * H * 16 > (1 << 20)) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): too many heads");
    P.head_off = c->head_off;
    P.head_len = c->head_len;
    P.c2 = float((1.0 / std::sqrt(double(kD))) * 1.4426950408889634);
    P.scores = scores;
    P.agg_max = agg_max;
    P.err_flag = ctx->err_flag;
    P.keys = fs ? fs->keys : nullptr;
    P.hist_fine = fs ? fs->hist_fine : nullptr;
    P.hist_coarse = fs ? fs->hist_coarse : nullptr;
    P.ptiles = (p + 127) / 128;
    P.hk_base = 0;
    P.run_hk_base = 0;
    P.qgroups = 1;
    P.qg0 = P.qgn = 0;
    P.best_io = nullptr;
    P.best_read = P.best_write = 0;
    const int grid = score_grid(ctx);  // persistent: one CTA per SM, tile-balanced ranges

    using KernelFn = void (*)(TcParams, CUtensorMap, CUtensorMap, CUtensorMap);
    const KernelFn stats_fn = tc_score_kernel<MODE_STATS>;
    const KernelFn score_fn = tc_score_kernel<MODE_SCORE>;
    // Dynamic shared memory limit: the per-block opt-in maximum minus the
    // kernels' static shared memory.  Function attributes are per device, so
    // the opt-in is made once per device (contexts of several GPUs may share
    // a process and call from several threads).
    static std::mutex attr_mu;
    static int dev_limit[kMaxDevices] = {};
    if (ctx->device < 0 || ctx->device >= kMaxDevices) return fail(EPK_ERR_UNSUPPORTED, "device ordinal too large");
    int limit = 0;
    {
        std::lock_guard<std::mutex> attr_lock(attr_mu);
        if (!dev_limit[ctx->device]) {
            int optin = 0;
            EPK_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
            cudaFuncAttributes fa0;
            EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa0, reinterpret_cast<const void*>(stats_fn)));
            const size_t stat = fa0.sharedSizeBytes;
            cudaFuncAttributes fa1;
            EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa1, reinterpret_cast<const void*>(score_fn)));
            const int lim = optin - int(std::max(stat, fa1.sharedSizeBytes));
            EPK_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(stats_fn),
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
            EPK_CUDA_CHECK(cudaFuncSetAttribute(reinterpret_cast<const void*>(score_fn),
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, lim));
            dev_limit[ctx->device] = lim;  // only once every attribute is set
        }
        limit = dev_limit[ctx->device];
    }
    // Shared-memory budget: leave ~30 KB of the SM for co-resident side-stream
    // kernels (EPK_TC_SMEM_KB overrides, for experiments).
    int budget = std::min(limit, 200 * 1024);
    if (const char* e = std::getenv("EPK_TC_SMEM_KB")) budget = std::min(limit, std::atoi(e) * 1024);
    TcPlan& T = *out;
    if ((rc = make_map(&T.tm_k, c->k, c->layer_base[c->layers], 128))) return rc;
    if ((rc = make_map(&T.tm_q, q, int64_t(P.L) * hq * p, kChunk))) return rc;
    if ((rc = make_map(&T.tm_kp, kp, int64_t(P.L) * H * p, 128))) return rc;

    // P1: 128-row K tiles (the MMA N = 128 is enough: P1 is bound by the
    // SFU exp2 rate, not the tensor pipe); query chunks in groups sized so
    // >= 2 K stages fit the budget.
    P.krows = 128;
    P.resident = 1;
    P.cg_chunks = std::min(P.NQ, kMaxQRes);
    for (;;) {
        P.cgroups = (P.NQ + P.cg_chunks - 1) / P.cg_chunks;
        P.runs = P.L * H * P.cgroups;
        P.qcap = P.cg_chunks * kChunk;
        P.kstages = 2;
        if (smem_bytes(P, MODE_STATS) <= budget || P.cg_chunks == 1) break;
        --P.cg_chunks;
    }
    while (P.kstages < 4) {
        ++P.kstages;
        if (smem_bytes(P, MODE_STATS) > budget) {
            --P.kstages;
            break;
        }
    }
    if (smem_bytes(P, MODE_STATS) > limit) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): shared memory");
    P.p1_grid = grid;
    P.p1_runs = P.runs;
    P.slots = kStatGroups * grid;
    const int64_t rows = int64_t(P.L) * H * P.NQ * kChunk;
    const int64_t pre_n = int64_t(P.L) * (int64_t(H) * P.cgroups + 1) + 1;
    const int64_t cache_rows = c->layer_base[c->layers];
    const bool multi_group = P.NQ > kMaxQRes && agg_max;  // P2 in query groups: a running max per cache row
    rc = ws_require(ctx, 2 * rows * P.slots * 4 + pre_n * 4 + rows * kBiasRowB + 4096 +
                             (multi_group ? cache_rows * 4 + 256 : 0));
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.prow = rows;
    P.part_m = carve.take<float>(rows * P.slots);
    P.part_z = carve.take<float>(rows * P.slots);
    P.p1_pre = carve.take<int32_t>(pre_n);
    P.bias_out = carve.take<uint8_t>(rows * kBiasRowB);
    P.bias = P.bias_out;
    float* best_buf = multi_group ? carve.take<float>(cache_rows) : nullptr;
    out->p1_pre_all = P.p1_pre;
    out->grid = grid;
    T.P1 = P;
    T.smem1 = smem_bytes(P, MODE_STATS);
    T.stats_fn = stats_fn;
    if (std::getenv("EPK_TC_VERBOSE"))
        fprintf(stderr, "P1: NQ=%d cg_chunks=%d cgroups=%d kstages=%d smem=%d limit=%d runs=%d\n", P.NQ, P.cg_chunks,
                P.cgroups, P.kstages, T.smem1, limit, P.runs);

    // P2: 128-row K tiles; all query chunks resident when they fit, else
    // streamed as chunk pairs through two 256-row slots.  cgroups/cg_chunks
    // stay P1's (the merge maps query rows to P1 runs).
    P.krows = 128;
    P.runs = P.L * H;
    // more query chunks than fit: Max runs one launch per query group of <=
    // kMaxQRes resident chunks (K streamed once per group, the running max
    // carried in best_io); Avg streams chunk pairs through two slots per K tile
    P.qgroups = P.NQ <= kMaxQRes ? 1 : (agg_max ? (P.NQ + kMaxQRes - 1) / kMaxQRes : 0);
    P.resident = P.qgroups > 0;
    P.qg0 = 0;
    P.qgn = P.NQ;
    P.best_io = nullptr;
    P.best_read = P.best_write = 0;
    P.qcap = P.NQ <= kMaxQRes ? P.NQ * kChunk : 4 * kChunk;
    if (P.resident) {
        p2_group_jobs(&P, 0);
    } else {  // streamed chunk pairs
        P.sj = (P.NQ + 1) / 2;
        P.sj_n0 = 256;
        P.sj_nl = (P.NQ & 1) ? 128 : 256;
    }
    P.kstages = 1;
    // P2 keeps three K stages next to the resident queries and their bias
    // rows (a little over the P1 co-residency budget)
    const int budget2 = std::min(limit, std::max(budget, 216 * 1024));
    while (P.kstages < 3) {
        ++P.kstages;
        if (smem_bytes(P, MODE_SCORE) > budget2) {
            --P.kstages;
            break;
        }
    }
    if (P.kstages < 2) P.kstages = 2;  // over the co-residency budget: use the whole opt-in limit
    if (smem_bytes(P, MODE_SCORE) > limit) return fail(EPK_ERR_UNSUPPORTED, "score(tensor core): shared memory");
    T.best_buf = best_buf;
    T.P2 = P;
    T.smem2 = smem_bytes(P, MODE_SCORE);
    T.score_fn = score_fn;
    T.q = q;
    T.kp = kp;
    T.qlayer = int64_t(hq) * p * kD * 2;
    T.kplayer = int64_t(H) * p * kD * 2;
    T.c = *c;
    if (std::getenv("EPK_TC_VERBOSE"))
        fprintf(stderr, "P2: NQ=%d resident=%d kstages=%d smem=%d runs=%d\n", P.NQ, P.resident, P.kstages, T.smem2,
                P.runs);
    return EPK_OK;
}

// The plan's parameters of one pass restricted to layers [l0, l1), with its
// query (and, for P1, prompt-key) tensor maps re-based to layer l0.  A P2
// view names the layer range [p0, p1) of the P1 launch whose partials it reads
// (P1 may cover more layers than one P2 launch).
static int tc_view(const TcPlan& T, int mode, int l0, int l1, int p0, int p1, TcParams* out, CUtensorMap* tm_q,
                   CUtensorMap* tm_kp) {
    TcParams P = mode == MODE_STATS ? T.P1 : T.P2;
    *tm_q = T.tm_q;
    *tm_kp = T.tm_kp;
    if (mode == MODE_STATS) {
        p0 = l0;
        p1 = l1;
    }
    P.hk_base = l0 * P.H;
    P.run_hk_base = (l0 - p0) * P.H;
    P.p1_pre = T.p1_pre_all + int64_t(p0) * (int64_t(P.H) * P.cgroups + 1);
    P.p1_runs = (p1 - p0) * P.H * P.cgroups;
    if (l0 > 0 || l1 < P.L) {
        epk_cache_desc v = T.c;
        v.layers = l1 - l0;
        v.layer_base = T.c.layer_base + l0;
        int rc = make_layer_table(&v, &P.lt);
        if (rc) return rc;
        P.L = l1 - l0;
        P.runs = mode == MODE_STATS ? P.p1_runs : P.L * P.H;
        P.head_off = T.c.head_off + int64_t(l0) * (P.H + 1);
        P.head_len = T.c.head_len + int64_t(l0) * P.H;
        if (P.hist_fine) {
            P.hist_fine += int64_t(l0) * 65536;
            P.hist_coarse += int64_t(l0) * 256;
        }
        if ((rc = make_map(tm_q, static_cast<const char*>(T.q) + l0 * T.qlayer, int64_t(P.L) * P.Hq * P.p, kChunk)))
            return rc;
        if (mode == MODE_STATS &&
            (rc = make_map(tm_kp, static_cast<const char*>(T.kp) + l0 * T.kplayer, int64_t(P.L) * P.H * P.p, 128)))
            return rc;
    }
    *out = P;
    return EPK_OK;
}

// P1 over layers [l0, l1) of the plan's cache.
static int tc_launch_p1(epk_ctx* ctx, const TcPlan& T, int l0, int l1) {
    TcParams P;
    CUtensorMap tm_q, tm_kp;
    int rc = tc_view(T, MODE_STATS, l0, l1, l0, l1, &P, &tm_q, &tm_kp);
    if (rc) return rc;
    EPK_PROF(ctx, "p1_rowstats");
    EPK_CUDA_CHECK(launch_pdl(T.stats_fn, dim3(T.grid), dim3(kThreadsStats), T.smem1, ctx->stream, P, T.tm_k, tm_q,
                              tm_kp));
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// P2 over layers [l0, l1), after the P1 launch over [p0, p1) (a superset).
static int tc_launch_p2(epk_ctx* ctx, const TcPlan& T, int l0, int l1, int p0, int p1) {
    TcParams P;
    CUtensorMap tm_q, tm_kp;
    int rc = tc_view(T, MODE_SCORE, l0, l1, p0, p1, &P, &tm_q, &tm_kp);
    if (rc) return rc;
    EPK_PROF(ctx, "p2_bias");
    EPK_CUDA_CHECK(launch_pdl(tc_bias_kernel, dim3(unsigned(P.L * P.H)), dim3(unsigned(std::min(P.NQ * kChunk, 1024))), 0, ctx->stream,
                              P));
    EPK_LAUNCH_CHECK(ctx);
    const int groups = std::max(1, P.qgroups);
    for (int g = 0; g < groups; ++g) {
        if (P.qgroups > 1) {
            p2_group_jobs(&P, g);
            P.best_io = T.best_buf;
            P.best_read = g > 0;
            P.best_write = g + 1 < groups;
        }
        EPK_PROF(ctx, "p2_colscore");
        EPK_CUDA_CHECK(launch_pdl(T.score_fn, dim3(T.grid), dim3(kThreads), T.smem2, ctx->stream, P, T.tm_k, tm_q,
                                  T.tm_kp));
        EPK_LAUNCH_CHECK(ctx);
    }
    return EPK_OK;
}

int launch_score_tc(epk_ctx* ctx, const epk_cache_desc* c, const void* q, const void* kp, int hq, int p, int agg_max,
                    int64_t n_max, float* scores, const FusedSelect* fs) {
    (void)n_max;  // the tile partition reads the live head lengths on the device
    TcPlan T;
    int rc = tc_plan(ctx, c, q, kp, hq, p, agg_max, scores, fs, &T);
    if (rc) return rc;
    if ((rc = tc_launch_p1(ctx, T, 0, c->layers))) return rc;
    return tc_launch_p2(ctx, T, 0, c->layers, 0, c->layers);
}

// One tensor-core block step with the fused selection: P1 over every layer
// (one tile-balanced launch: the partition, hence the bits, do not depend on
// the grouping), then per layer group P2 -> threshold select on the context
// stream and count/plan/gather on `side` (when given) so a group's compaction
// overlaps the next group's scoring.  (P1 per group -- its K re-read by P2
// from L2 -- measured slower: every launch pays the ~25 us CTA-speed tail.)
int launch_step_tc_grouped(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out, const void* q,
                           const void* kp, int hq, int p, int agg_max, const int64_t* budgets, int group,
                           cudaStream_t side, cudaEvent_t ev_fork, int out_slack, float* scores, uint8_t* keep,
                           const FusedSelect& fs_all, uint64_t* thr, int32_t* kept,
                           int (*select_fn)(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, int,
                                            const FusedSelect*, const int64_t*, uint64_t*, int32_t*),
                           int (*compact_fn)(epk_ctx*, const epk_cache_desc*, const epk_cache_desc*, const uint8_t*,
                                             int, const uint32_t*, const uint64_t*, uint32_t*, uint32_t*),
                           epk_cache_desc (*view_fn)(const epk_cache_desc*, int, int)) {
    TcPlan T;
    int rc = tc_plan(ctx, in, q, kp, hq, p, agg_max, scores, &fs_all, &T);
    if (rc) return rc;
    const int L = in->layers;
    cudaStream_t main = ctx->stream;
    if ((rc = tc_launch_p1(ctx, T, 0, L))) return rc;
    for (int l0 = 0; l0 < L; l0 += group) {
        const int l1 = std::min(L, l0 + group);
        if ((rc = tc_launch_p2(ctx, T, l0, l1, 0, L))) return rc;
        const epk_cache_desc vin = view_fn(in, l0, l1), vout = view_fn(out, l0, l1);
        const FusedSelect fs{fs_all.keys,
                             fs_all.hist_fine + int64_t(l0) * 65536,
                             fs_all.hist_coarse + int64_t(l0) * 256,
                             fs_all.cand + int64_t(l0) * 1024,
                             fs_all.cand_n + l0,
                             fs_all.done + l0};
        if ((rc = select_fn(ctx, &vin, &vout, out_slack, &fs, budgets + l0, thr + 2 * l0, kept ? kept + l0 : nullptr)))
            return rc;
        if (side) {
            EPK_CUDA_CHECK(cudaEventRecord(ev_fork, main));
            EPK_CUDA_CHECK(cudaStreamWaitEvent(side, ev_fork, 0));
            ctx->stream = side;
        }
        // the last group's compaction has no scoring left to overlap: all SMs
        const int saved_ctas = ctx->gather_ctas;
        if (l1 == L) ctx->gather_ctas = 0;
        rc = compact_fn(ctx, &vin, &vout, keep, out_slack, fs.keys, thr + 2 * l0, fs.hist_fine, fs.hist_coarse);
        ctx->gather_ctas = saved_ctas;
        ctx->stream = main;
        if (rc) return rc;
    }
    return EPK_OK;
}

}  // namespace epk
