// step.cu -- the fused tensor-core block step: ONE persistent cooperative
// kernel per block step that scores, selects and compacts every layer,
// overlapping the HBM-bound compaction of early layers with the SFU/tensor
// bound scoring of later ones (a layer-ordered dataflow inside the kernel).
//
// Same results as the multi-launch path (epk_evict_step with layer groups):
// score_with_prompt (scoring.hpp:80-128) over the attention weights of
// toymodel.hpp:327-391, evict_to_budget's pooled selection (kvcache.hpp:
// 142-190) and its stable output loop (:192-199), written out of place.
//
// Warp roles (480 threads, one CTA per SM, all CTAs co-resident):
//   warp 0      scheduler + TMA producer: takes scoring items from a global
//               queue (atomic counter) in a fixed order and streams their
//               query chunks and 128-row K tiles;
//   warps 1-2   tcgen05 MMA issuers (alternate jobs, two 256-column TMEM slots);
//   warps 3-10  scoring epilogue:
//                 P1 item (layer, head, split): online (max, sum exp2) of the
//                   split's columns per query row -> partial (m, Z);
//                 P2 item (layer, head, split): waits for the head's P1 items,
//                   merges lse2, scores the split's rows, writes score, key
//                   and the layer's score histograms (fine 65536 bins of
//                   float_bits >> 14, coarse 256);
//   warps 11-14 evict: take evict items from a second queue, per layer in
//               order: collect (threshold bin from the histograms; the bin's
//               candidates -> a list), select (exact threshold key T and
//               tiebreak U from the list), count (keep[] + per-chunk counts),
//               plan (chunk prefix, output head offsets), gather (kept K/V
//               rows + positions to the output cache, 16-byte vectors).
// Item order: P1(l) items, then P2(l - lag) items, slot by slot, so a P2
// item's P1 inputs were dispensed `lag` slots earlier; evict items of layer l
// wait on per-layer counters.  Every wait is bounded (a timeout raises
// EPK_ERR_CUDA through the context error flag instead of hanging).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

namespace epk {

constexpr int kSEpi = 8;
constexpr int kSMma = 2;
constexpr int kSEvict = 4;
// Four warpgroups: WG0 = producer, 2 MMA issuers, 1 idle (setmaxnreg down to
// 48), WG1-2 = 8 epilogue warps (128), WG3 = 4 evict warps (setmaxnreg up to
// 208, so a warp keeps a whole 32-row group of K and V -- 32 KB -- in flight).
constexpr int kSThreads = 512;
constexpr int kEpiWarp0 = 4;
constexpr int kEvictWarp0 = 12;
constexpr int kSMaxQ = 4;       // query chunks resident (G * p <= 512)
constexpr int kEvRows = 4096;   // rows per evict chunk
constexpr int kCandCap = 1024;  // threshold-bin candidates resolved in shared memory
constexpr int kEvBar = 6;       // named barrier of the evict warps
constexpr int kEpiBar = 1;      // named barrier of the scoring epilogue warps
constexpr int kSMaxHeads = 64;

// Control block (zeroed before every launch): queue counters and the
// per-layer / per-(layer, head) progress counters of the dataflow.
struct StepCtl {
    unsigned* base;
    int L, H;
    __device__ unsigned* q_score() const { return base; }
    __device__ unsigned* q_evict() const { return base + 1; }
    __device__ unsigned* p2_done(int l) const { return base + 2 + l; }
    __device__ unsigned* cand_n(int l) const { return base + 2 + L + l; }
    __device__ unsigned* collect_done(int l) const { return base + 2 + 2 * L + l; }
    __device__ unsigned* thr_ready(int l) const { return base + 2 + 3 * L + l; }
    __device__ unsigned* count_done(int l) const { return base + 2 + 4 * L + l; }
    __device__ unsigned* plan_ready(int l) const { return base + 2 + 5 * L + l; }
    __device__ unsigned* p1_done(int hk) const { return base + 2 + 6 * L + hk; }
    __device__ unsigned* head_cnt(int hk) const { return base + 2 + 6 * L + L * H + hk; }
    static int64_t words(int L, int H) { return 2 + 6 * int64_t(L) + 2 * int64_t(L) * H; }
};

struct StepParams {
    LayerTable lt_in, lt_out;
    int64_t budget[kMaxLayers];
    int L, H, Hq, G, p, Gp, NQ;
    int Smax;         // partial slots per query row / 2 (>= splits of any head)
    int split_tiles;  // 128-row tiles per split (a head of n rows has ceil(n / (128 * split_tiles)) splits)
    int ptiles;       // causal prompt tiles (last P1 split of a head)
    int lag;          // P2 of layer l is dispensed after P1 of layer l + lag
    int C;            // evict chunks per layer
    int ev_items;     // evict items
    int kstages;
    int slack;
    int agg_max;
    float c2;
    const int32_t* in_off;
    const int32_t* in_len;
    const int32_t* in_pos;
    const uint4* in_k;
    const uint4* in_v;
    int32_t* out_off;
    int32_t* out_len;
    int32_t* out_pos;
    uint4* out_k;
    uint4* out_v;
    float* part_m;  // [L*H*NQ*128][2*S]
    float* part_z;
    float* scores;  // [rows] in-cache rows
    uint32_t* keys;
    uint32_t* hist_fine;    // [L][65536]
    uint32_t* hist_coarse;  // [L][256]
    uint8_t* keep;          // [rows]
    uint64_t* thr;          // [L][2]
    int32_t* chunk_cnt;     // [L][C]
    int32_t* chunk_pre;     // [L][C]
    uint4* cand;            // [L][kCandCap] {key, 0, tiebreak lo, tiebreak hi}
    int32_t* kept_per_layer;
    StepCtl ctl;
    int* err_flag;
    unsigned long long* trace;  // EPK_STEP_TRACE: per evict item {item, cta, t0, t1}, [0] = count; per CTA scoring end
    int debug;  // EPK_STEP_DEBUG bits (timing experiments only): 1 skip evict, 2 skip gather copies, 4 no L2 prefetch
};

// ---- cross-CTA waits ----------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Spins until *c >= target (bounded: ~2 s); on timeout flags the error and
// returns so the kernel can never hang the device.
__device__ __forceinline__ void wait_ge(const unsigned* c, unsigned target, int* err) {
    for (long it = 0; ld_acquire(c) < target; ++it) {
        if (it > (1l << 24)) {
            atomicCAS(err, 0, EPK_ERR_CUDA);
            return;
        }
        __nanosleep(100);
    }
}

// ---- scoring items --------------------------------------------------------------
struct SItem {
    int mode, l, h, s;
    int n_h;
    int64_t krow0;
    int t0, nc, np;
    __device__ int ntiles() const { return nc + np; }
};

// Item tables (shared memory, built from the live head lengths at kernel
// start): hpre[l*(H+1) + h] = splits of layer l's heads before h (so
// hpre[l*(H+1) + H] = U_l, the layer's items per pass), spre[k] = items
// dispensed before slot k, where slot k holds P1(k) (k < L) then P2(k - lag)
// (k >= lag).
struct ItemTables {
    const int* hpre;
    const int* spre;
    __device__ int U(const StepParams& P, int l) const { return hpre[l * (P.H + 1) + P.H]; }
    __device__ int splits(const StepParams& P, int hk) const {
        const int l = hk / P.H, h = hk % P.H;
        return hpre[l * (P.H + 1) + h + 1] - hpre[l * (P.H + 1) + h];
    }
    __device__ int items(const StepParams& P) const { return spre[P.L + P.lag]; }
};

__device__ __forceinline__ void build_tables(const StepParams& P, int* hpre, int* spre) {
    // every thread of the CTA takes part; caller synchronises
    const int split_rows = P.split_tiles * 128;
    for (int l = threadIdx.x; l < P.L; l += blockDim.x) {
        int acc = 0;
        for (int h = 0; h < P.H; ++h) {
            hpre[l * (P.H + 1) + h] = acc;
            acc += (P.in_len[l * P.H + h] + split_rows - 1) / split_rows;
        }
        hpre[l * (P.H + 1) + P.H] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int k = 0; k < P.L + P.lag; ++k) {
            spre[k] = acc;
            if (k < P.L) acc += hpre[k * (P.H + 1) + P.H];
            if (k >= P.lag) acc += hpre[(k - P.lag) * (P.H + 1) + P.H];
        }
        spre[P.L + P.lag] = acc;
    }
}

__device__ __forceinline__ SItem decode_item(const StepParams& P, const ItemTables& T, int i) {
    int lo = 0, hi = P.L + P.lag - 1;
    while (lo < hi) {  // slot: last k with spre[k] <= i
        const int mid = (lo + hi + 1) >> 1;
        if (T.spre[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int k = lo;
    int r = i - T.spre[k];
    SItem x;
    const int u1 = k < P.L ? T.U(P, k) : 0;
    if (r < u1) {
        x.mode = 0;
        x.l = k;
    } else {
        x.mode = 1;
        x.l = k - P.lag;
        r -= u1;
    }
    const int* hp = T.hpre + x.l * (P.H + 1);
    lo = 0;
    hi = P.H - 1;
    while (lo < hi) {  // head: last h with hp[h] <= r (skips empty heads)
        const int mid = (lo + hi + 1) >> 1;
        if (hp[mid] <= r) lo = mid; else hi = mid - 1;
    }
    x.h = lo;
    x.s = r - hp[lo];
    const int nsplit = hp[lo + 1] - hp[lo];
    x.n_h = P.in_len[x.l * P.H + x.h];
    x.krow0 = P.lt_in.base[x.l] + P.in_off[x.l * (P.H + 1) + x.h];
    const int ntc = (x.n_h + 127) / 128;
    x.t0 = x.s * P.split_tiles;
    x.nc = max(0, min(ntc, x.t0 + P.split_tiles) - x.t0);
    x.np = (x.mode == 0 && x.s == nsplit - 1) ? P.ptiles : 0;
    return x;
}

// ---- evict helpers (128 threads, named barrier kEvBar) ------------------------
struct EvShared {
    int32_t off[kSMaxHeads + 1];
    int32_t len[kSMaxHeads];
    uint32_t tot[256];
    uint32_t hist[256];
    uint32_t ck[kCandCap];
    uint64_t ct[kCandCap];
    int64_t red[kSEvict];
    int bucket;
    int64_t before, eq;
    int item;
    int wcnt[kSEvict];
    int ncand;
    uint32_t hcnt[kSMaxHeads];
    uint32_t ccnt[512];  // prep: kept rows per evict chunk (C <= 512)
    uint32_t gbal[kEvRows / 32];  // gather: keep ballot of each 32-row group of the chunk
    alignas(16) uint8_t keepb[kEvRows];  // gather: the chunk's keep bytes
    uint8_t gsrc[kSEvict][2][32]; // gather: lane of each kept rank (per warp, 2 groups in flight)
    int32_t gdst[kSEvict][2][32]; // gather: destination row (layer-relative) of each kept rank
    int cur_layer;                // layer whose off/len are loaded
    int gpre[kEvRows / 32];       // gather: kept rows of the chunk before each group
};

__device__ __forceinline__ void ev_sync() { named_bar_sync(kEvBar, 32 * kSEvict); }

// Bucket of tot[0..nbins) (nbins <= 256) holding the k-th smallest (1-based).
__device__ __forceinline__ void ev_find_bucket(EvShared& E, const uint32_t* tot, int nbins, int64_t k, int et) {
    const int lane = et & 31, w = et >> 5;
    const int b0 = et * 2;
    const int64_t mine = (b0 < nbins ? tot[b0] : 0) + (b0 + 1 < nbins ? tot[b0 + 1] : 0);
    int64_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    ev_sync();
    if (lane == 31) E.red[w] = incl;
    ev_sync();
    int64_t excl = incl - mine;
    for (int q = 0; q < w; ++q) excl += E.red[q];
    if (mine > 0 && excl < k && k <= excl + mine) {
        const int64_t t0 = b0 < nbins ? tot[b0] : 0;
        if (excl + t0 >= k) {
            E.bucket = b0;
            E.before = excl;
            E.eq = t0;
        } else {
            E.bucket = b0 + 1;
            E.before = excl + t0;
            E.eq = tot[b0 + 1];
        }
    }
    ev_sync();
}

__device__ __forceinline__ int ev_head_of(const EvShared& E, int H, int r) {
    int lo = 0, hi = H - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (E.off[mid] <= r) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// The layer's threshold bin from the score histograms: key prefix kb (keys
// with key >> 14 == kb), slots left in it (k_rem) and its size (eq).
__device__ __forceinline__ void ev_threshold_bin(const StepParams& P, EvShared& E, int l, int64_t limit, int et, uint32_t& kb,
                                 int64_t& k_rem, int64_t& eq) {
    k_rem = limit;
    for (int i = et; i < 256; i += 32 * kSEvict) E.tot[i] = __ldcg(P.hist_coarse + l * 256 + 255 - i);
    ev_sync();
    ev_find_bucket(E, E.tot, 256, k_rem, et);
    k_rem -= E.before;
    const int cb = 255 - E.bucket;
    for (int i = et; i < 256; i += 32 * kSEvict)
        E.tot[i] = __ldcg(P.hist_fine + int64_t(l) * 65536 + cb * 256 + 255 - i);
    ev_sync();
    ev_find_bucket(E, E.tot, 256, k_rem, et);
    k_rem -= E.before;
    eq = E.eq;
    kb = uint32_t(0x1FFFF - (cb * 256 + 255 - E.bucket));
}

__device__ __forceinline__ void ev_load_layer(const StepParams& P, EvShared& E, int l, int et) {
    if (E.cur_layer == l) return;  // uniform: written before the last ev_sync
    for (int i = et; i <= P.H; i += 32 * kSEvict) E.off[i] = P.in_off[l * (P.H + 1) + i];
    for (int i = et; i < P.H; i += 32 * kSEvict) E.len[i] = P.in_len[l * P.H + i];
    ev_sync();
    if (et == 0) E.cur_layer = l;
    ev_sync();
}

// Exact (T, U) among candidates with key >> 14 == kb: 8-bit radix on the
// remaining key bits, then on the 40-bit tiebreak.  for_each(f) calls
// f(key, tiebreak) for every candidate (shared list or global rows).
template <typename ForEach>
__device__ __forceinline__ void ev_resolve(EvShared& E, ForEach& for_each, uint32_t kb, int64_t k_rem, int64_t eq, int et,
                           uint32_t& T, uint64_t& U) {
    uint32_t prefix = kb << 14, mask = 0xFFFFC000u;
    int lo = 14;
    while (lo > 0) {
        const int hi = lo;
        lo = hi > 8 ? hi - 8 : 0;
        const uint32_t dmask = (1u << (hi - lo)) - 1;
        for (int i = et; i < 256; i += 32 * kSEvict) E.hist[i] = 0;
        ev_sync();
        for_each([&](uint32_t k, uint64_t) {
            if (((k ^ prefix) & mask) == 0) atomicAdd(&E.hist[(k >> lo) & dmask], 1u);
        });
        ev_sync();
        ev_find_bucket(E, E.hist, int(dmask) + 1, k_rem, et);
        k_rem -= E.before;
        eq = E.eq;
        prefix |= uint32_t(E.bucket) << lo;
        mask |= dmask << lo;
    }
    T = prefix;
    U = ~uint64_t(0);
    if (eq > k_rem) {
        uint64_t tp = 0, tm = 0;
        for (int shift = 32; shift >= 0; shift -= 8) {
            for (int i = et; i < 256; i += 32 * kSEvict) E.hist[i] = 0;
            ev_sync();
            for_each([&](uint32_t k, uint64_t tb) {
                if (k == T && ((tb ^ tp) & tm) == 0) atomicAdd(&E.hist[(tb >> shift) & 0xFF], 1u);
            });
            ev_sync();
            ev_find_bucket(E, E.hist, 256, k_rem, et);
            k_rem -= E.before;
            tp |= uint64_t(E.bucket) << shift;
            tm |= uint64_t(0xFF) << shift;
        }
        U = tp;
    }
}

// ---- the kernel ---------------------------------------------------------------
__global__ void __launch_bounds__(kSThreads, 1)
    step_kernel(const __grid_constant__ StepParams P, const __grid_constant__ CUtensorMap tm_k,
                const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kp) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t q_half = uint32_t(P.NQ * kChunk) * kRowB;
    const uint32_t k_half = uint32_t(128) * kRowB;
    const uint32_t k_stage = 2 * k_half;
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + 2 * q_half;
    float* s_lse = reinterpret_cast<float*>(sK + P.kstages * k_stage);  // NQ*128
    float* s_pair = s_lse + P.NQ * kChunk;                              // 128
    float* s_avg = s_pair + kChunk;                                     // G*128
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_avg + P.G * kChunk);
    uint64_t* k_full = bars;
    uint64_t* k_empty = k_full + P.kstages;
    uint64_t* q_full = k_empty + P.kstages;
    uint64_t* q_empty = q_full + kSMaxQ;
    uint64_t* t_full = q_empty + kSMaxQ;
    uint64_t* t_empty = t_full + 2;
    uint64_t* it_full = t_empty + 2;
    uint64_t* it_empty = it_full + 2;
    int* s_item = reinterpret_cast<int*>(it_empty + 2);
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_item + 2);
    int* s_hpre = reinterpret_cast<int*>(tmem_holder + 4);  // [L*(H+1)]
    int* s_spre = s_hpre + P.L * (P.H + 1);                  // [L+lag+1]
    __shared__ uint32_t s_coarse[256];
    __shared__ EvShared E;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const StepCtl& ctl = P.ctl;
    if (P.trace && threadIdx.x == 0) P.trace[8 + 4 * 60000 + 512 + blockIdx.x] = gtimer();

    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_kp);
        for (int s = 0; s < P.kstages; ++s) {
            mbar_init(&k_full[s], 1);
            mbar_init(&k_empty[s], kSMma);
        }
        for (int s = 0; s < kSMaxQ; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], kSMma);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&t_full[s], 1);
            mbar_init(&t_empty[s], kSEpi);
            mbar_init(&it_full[s], 1);
            mbar_init(&it_empty[s], kSMma + kSEpi);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(tmem_holder, 512);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_coarse[i] = 0;
    for (int i = threadIdx.x; i < P.G * kChunk; i += blockDim.x) s_avg[i] = 0.f;
    build_tables(P, s_hpre, s_spre);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;
    const ItemTables IT{s_hpre, s_spre};
    const int n_items = IT.items(P);

    if (warp < kEpiWarp0) asm volatile("setmaxnreg.dec.sync.aligned.u32 48;\n" ::: "memory");
    if (warp >= kEvictWarp0) asm volatile("setmaxnreg.inc.sync.aligned.u32 208;\n" ::: "memory");
    if (warp == 0) {  // ------------------- scheduler + TMA producer -------------------
        const bool leader = elect_one_sync();
        int ks = 0;
        uint32_t kph = 0;
        uint32_t qn = 0;  // Q loads so far (all chunks of an item load together)
        for (uint32_t n = 0;; ++n) {
            int i = 0;
            if (leader) i = int(atomicAdd(ctl.q_score(), 1u));
            i = __shfl_sync(0xffffffffu, i, __ffs(__ballot_sync(0xffffffffu, leader)) - 1);
            const int slot = int(n & 1);
            mbar_wait(&it_empty[slot], ((n >> 1) & 1) ^ 1);
            if (leader) {
                s_item[slot] = i < n_items ? i : -1;
                mbar_arrive(&it_full[slot]);
            }
            __syncwarp();
            if (i >= n_items) break;
            const SItem x = decode_item(P, IT, i);
            if (x.ntiles() == 0) continue;
            const int qrow0 = (x.l * P.Hq + x.h * P.G) * P.p;
            for (int c = 0; c < P.NQ; ++c) {
                mbar_wait(&q_empty[c], (qn & 1) ^ 1);
                if (leader) {
                    mbar_expect_tx(&q_full[c], 2 * kChunk * kRowB);
                    load_rows(sQ + c * kChunk * kRowB, q_half, &tm_q, &q_full[c], qrow0 + c * kChunk);
                }
                __syncwarp();
            }
            ++qn;
            for (int t = 0; t < x.ntiles(); ++t) {
                mbar_wait(&k_empty[ks], kph ^ 1);
                if (leader) {
                    mbar_expect_tx(&k_full[ks], k_stage);
                    if (t < x.nc)
                        load_rows(sK + ks * k_stage, k_half, &tm_k, &k_full[ks], int(x.krow0 + int64_t(x.t0 + t) * 128));
                    else
                        load_rows(sK + ks * k_stage, k_half, &tm_kp, &k_full[ks],
                                  (x.l * P.H + x.h) * P.p + (t - x.nc) * 128);
                }
                __syncwarp();
                if (++ks == P.kstages) {
                    ks = 0;
                    kph ^= 1;
                }
            }
        }
    } else if (warp <= kSMma) {  // ------------------- MMA issuers -------------------
        const uint32_t mw = uint32_t(warp - 1);
        const bool leader = elect_one_sync();
        int ks = 0;
        uint32_t kph = 0;
        uint32_t qn = 0;
        uint32_t job = 0;
        int held = 0;
        const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK);
        for (uint32_t n = 0;; ++n) {
            const int slot = int(n & 1);
            mbar_wait(&it_full[slot], (n >> 1) & 1);
            const int i = s_item[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[slot]);
            if (i < 0) break;
            const SItem x = decode_item(P, IT, i);
            if (x.ntiles() == 0) continue;
            if (leader)
                for (int c = 0; c < held; ++c) mma_commit(&q_empty[c]);  // previous Q retires with its MMAs
            __syncwarp();
            held = P.NQ;
            const uint32_t qph = qn & 1;
            ++qn;
            for (int t = 0; t < x.ntiles(); ++t) {
                mbar_wait(&k_full[ks], kph);
                const uint32_t kst = k0 + uint32_t(ks) * k_stage;
                if (x.mode == 0) {
                    for (int c = 0; c < P.NQ; ++c, ++job) {
                        if (t == 0) {
                            mbar_wait(&q_full[c], qph);
                        }
                        if ((job & 1) != mw) continue;
                        const int ts = int(mw);
                        mbar_wait(&t_empty[ts], ((job >> 1) & 1) ^ 1);
                        tc_fence_after();
                        if (leader) {
                            mma_128xN(tmem + uint32_t(ts * 256), q0 + uint32_t(c * kChunk * kRowB), q_half, kst, k_half,
                                      idesc_bf16_f32(128, 128));
                            mma_commit(&t_full[ts]);
                        }
                        __syncwarp();
                    }
                } else {
                    for (int j = 0; 2 * j < P.NQ; ++j, ++job) {
                        const int nch = min(2, P.NQ - 2 * j);
                        if (t == 0)
                            for (int cc = 0; cc < nch; ++cc) {
                                mbar_wait(&q_full[2 * j + cc], qph);
                            }
                        if ((job & 1) != mw) continue;
                        const int ts = int(mw);
                        mbar_wait(&t_empty[ts], ((job >> 1) & 1) ^ 1);
                        tc_fence_after();
                        if (leader) {
                            mma_128xN(tmem + uint32_t(ts * 256), kst, k_half, q0 + uint32_t(2 * j * kChunk * kRowB), q_half,
                                      idesc_bf16_f32(128, uint32_t(nch * kChunk)));
                            mma_commit(&t_full[ts]);
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
    } else if (warp < kEpiWarp0) {
        // idle warp of WG0
    } else if (warp < kEvictWarp0) {  // ------------------- scoring epilogue -------------------
        const int e = warp - kEpiWarp0;
        const int quarter = warp & 3;
        const int half = e >> 2;
        const int r_local = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        const int etid = e * 32 + lane;
        uint32_t job = 0;
        const float inv_p = 1.0f / float(P.p);
        const int rows_q = P.NQ * kChunk;
        for (uint32_t n = 0;; ++n) {
            const int slot = int(n & 1);
            mbar_wait(&it_full[slot], (n >> 1) & 1);
            const int i = s_item[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&it_empty[slot]);
            if (i < 0) break;
            const SItem x = decode_item(P, IT, i);
            const int hk = x.l * P.H + x.h;
            if (x.mode == 0) {  // ---- P1: partial softmax stats of the split
                float m[kSMaxQ], z[kSMaxQ];
#pragma unroll
                for (int c = 0; c < kSMaxQ; ++c) {
                    m[c] = -INFINITY;
                    z[c] = 0.f;
                }
                for (int t = 0; t < x.ntiles(); ++t) {
#pragma unroll
                    for (int c = 0; c < kSMaxQ; ++c) {
                        if (c >= P.NQ) break;
                        const int rq = c * kChunk + r_local;
                        int lim;
                        if (t < x.nc)
                            lim = x.n_h - (x.t0 + t) * 128;
                        else
                            lim = min(P.p, rq % P.p + 1) - (t - x.nc) * 128;
                        const int ts = int(job & 1);
                        mbar_wait(&t_full[ts], (job >> 1) & 1);
                        tc_fence_after();
                        float v[64];
                        tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * 64), v);
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&t_empty[ts]);
                        stats_cols<64, 0>(v, lim - half * 64, P.c2, m[c], z[c]);
                        ++job;
                    }
                }
#pragma unroll
                for (int c = 0; c < kSMaxQ; ++c) {
                    if (c < P.NQ) {
                        const int64_t o = (int64_t(hk) * rows_q + c * kChunk + r_local) * (2 * P.Smax) + 2 * x.s + half;
                        P.part_m[o] = m[c];
                        P.part_z[o] = z[c];
                    }
                }
                __threadfence();
                named_bar_sync(kEpiBar, 32 * kSEpi);
                if (etid == 0) atomicAdd(ctl.p1_done(hk), 1u);
            } else {  // ---- P2: column scores of the split
                if (x.ntiles() > 0) {
                    const int ns = IT.splits(P, hk);
                    if (etid == 0) wait_ge(ctl.p1_done(hk), unsigned(ns), P.err_flag);
                    named_bar_sync(kEpiBar, 32 * kSEpi);
                    for (int r = etid; r < rows_q; r += 32 * kSEpi) {
                        float v = INFINITY;
                        if (r < P.Gp) {
                            const float* pm = P.part_m + (int64_t(hk) * rows_q + r) * (2 * P.Smax);
                            const float* pz = P.part_z + (int64_t(hk) * rows_q + r) * (2 * P.Smax);
                            float M = -INFINITY;
                            for (int q = 0; q < 2 * ns; ++q) M = fmaxf(M, __ldcg(pm + q));
                            float Z = 0.f;
                            if (M != -INFINITY)
                                for (int q = 0; q < 2 * ns; ++q) {
                                    const float mq = __ldcg(pm + q);
                                    if (mq != -INFINITY) Z += __ldcg(pz + q) * ex2(mq - M);
                                }
                            v = M == -INFINITY ? INFINITY : M + log2f(Z);
                        }
                        s_lse[r] = -v;  // negated: the epilogue adds it with FFMA2
                    }
                    named_bar_sync(kEpiBar, 32 * kSEpi);
                }
                for (int t = 0; t < x.nc; ++t) {
                    float best = -INFINITY;
                    for (int j = 0; 2 * j < P.NQ; ++j) {
                        const int ncols = min(2, P.NQ - 2 * j) * kChunk;
                        const int hw = ncols / 2;
                        const int ts = int(job & 1);
                        mbar_wait(&t_full[ts], (job >> 1) & 1);
                        tc_fence_after();
                        const int r0 = 2 * j * kChunk + half * hw;
                        if (hw == 128) {
                            float v[64];
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * hw), v);
                            score_cols<64>(v, s_lse + r0, r0, P, best, s_avg, r_local);
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * hw + 64), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);
                            score_cols<64>(v, s_lse + r0 + 64, r0 + 64, P, best, s_avg, r_local);
                        } else {
                            float v[64];
                            tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * hw), v);
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&t_empty[ts]);
                            score_cols<64>(v, s_lse + r0, r0, P, best, s_avg, r_local);
                        }
                        ++job;
                    }
                    const int jrow = (x.t0 + t) * 128 + r_local;
                    float sc = 0.f;
                    bool have = false;
                    if (P.agg_max) {
                        if (half == 1) s_pair[r_local] = best;
                        named_bar_sync(2 + quarter, 64);
                        if (half == 0 && jrow < x.n_h) {
                            sc = ex2(fmaxf(best, s_pair[r_local]));
                            have = true;
                        }
                        named_bar_sync(2 + quarter, 64);
                    } else {
                        named_bar_sync(2 + quarter, 64);
                        if (half == 0) {
                            float b = -INFINITY;
                            for (int gg = 0; gg < P.G; ++gg) {
                                b = fmaxf(b, s_avg[gg * kChunk + r_local] * inv_p);
                                s_avg[gg * kChunk + r_local] = 0.f;
                            }
                            sc = b;
                            have = jrow < x.n_h;
                        }
                        named_bar_sync(2 + quarter, 64);
                    }
                    if (have) {
                        const int64_t row = x.krow0 + jrow;
                        P.scores[row] = sc;
                        P.keys[row] = desc_key(sc);
                        const uint32_t b = min(__float_as_uint(sc) >> 14, 65535u);
                        if (!(P.debug & 64)) atomicAdd(&P.hist_fine[int64_t(x.l) * 65536 + b], 1u);
                        atomicAdd(&s_coarse[b >> 8], 1u);
                    }
                }
                // publish: coarse histogram, then the item counter
                named_bar_sync(kEpiBar, 32 * kSEpi);
                {
                    const uint32_t v = s_coarse[etid];
                    if (v) {
                        atomicAdd(&P.hist_coarse[x.l * 256 + etid], v);
                        s_coarse[etid] = 0;
                    }
                }
                __threadfence();
                named_bar_sync(kEpiBar, 32 * kSEpi);
                if (etid == 0) atomicAdd(ctl.p2_done(x.l), 1u);
            }
        }
    } else {  // ------------------- evict warps -------------------
        const int et = threadIdx.x - 32 * kEvictWarp0;
        const int ew = et >> 5;
        if (P.debug & 1) goto evict_done;
        if (et == 0) E.cur_layer = -1;
        ev_sync();

        for (;;) {
            if (et == 0) E.item = int(atomicAdd(ctl.q_evict(), 1u));
            ev_sync();
            const int j = E.item;
            ev_sync();
            if (j >= P.ev_items) break;
            const unsigned long long t_item0 = P.trace ? gtimer() : 0;
            unsigned long long t_ready = t_item0;
            unsigned long long tp[4] = {0, 0, 0, 0};  // prep phase marks (trace only)
            // Dispatch order: round t carries prep(t) then gather(t-1) x C, so a
            // gather's prep was dispensed a round earlier.
            int l = 0, c = -1;  // c < 0: prep item
            if (j > 0) {
                const int jp = j - 1;
                const int t = 1 + jp / (P.C + 1), q = jp % (P.C + 1);
                if (t <= P.L - 1) {
                    l = q == 0 ? t : t - 1;
                    c = q - 1;
                } else {  // last round: the last layer's gathers
                    l = P.L - 1;
                    c = jp - (P.L - 1) * (P.C + 1);
                }
            }
            const int64_t limit = int64_t(P.H) * P.budget[l];
            const int64_t base = P.lt_in.base[l];
            const int32_t* pos = P.in_pos + base;
            uint8_t* keep = P.keep + base;
            if (c < 0) {  // ---- prep: threshold, keep[], chunk/head counts, output plan of layer l
                if (et == 0) wait_ge(ctl.p2_done(l), unsigned(IT.U(P, l)), P.err_flag);
                ev_sync();
                if (P.trace) t_ready = gtimer();
                ev_load_layer(P, E, l, et);
                int64_t n_live = 0;
                for (int h = 0; h < P.H; ++h) n_live += E.len[h];
                const int region = E.off[P.H];
                bool all = true;
                uint32_t T = 0;
                uint64_t U = ~uint64_t(0);
                // loads one thread's kSpan-row span of keys (rows >= region -> 0):
                // kSpan / 4 independent 16-byte loads, one memory round trip
                constexpr int kSpan = 64;
                auto load16 = [&](int r0, uint32_t (&kv)[kSpan]) {
                    const uint32_t* src = P.keys + base + r0;
                    if (r0 + kSpan <= region && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
                        for (int q4 = 0; q4 < kSpan / 4; ++q4) {
                            const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src) + q4);
                            kv[4 * q4] = v.x;
                            kv[4 * q4 + 1] = v.y;
                            kv[4 * q4 + 2] = v.z;
                            kv[4 * q4 + 3] = v.w;
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < kSpan; ++u) kv[u] = r0 + u < region ? __ldcg(src + u) : 0u;
                    }
                };
                if (n_live > limit) {
                    all = false;
                    uint32_t kb;
                    int64_t k_rem, eq;
                    ev_threshold_bin(P, E, l, limit, et, kb, k_rem, eq);
                    if (P.trace) tp[0] = gtimer();
                    // the threshold bin's candidates -> shared list
                    if (et == 0) E.ncand = 0;
                    ev_sync();
                    for (int b0 = 0; b0 < region; b0 += kSpan * 32 * kSEvict) {
                        const int r0 = b0 + et * kSpan;
                        if (r0 >= region) continue;
                        uint32_t kv[kSpan];
                        load16(r0, kv);
                        int h = ev_head_of(E, P.H, r0);
                        int live_end = E.off[h] + E.len[h], head_end = E.off[h + 1];  // register-cached bounds
#pragma unroll
                        for (int u = 0; u < kSpan; ++u) {
                            const int rr = r0 + u;
                            if (rr >= region) break;
                            while (rr >= head_end) {
                                ++h;
                                live_end = E.off[h] + E.len[h];
                                head_end = E.off[h + 1];
                            }
                            if (rr < live_end && (kv[u] >> 14) == kb) {
                                const int at = atomicAdd(&E.ncand, 1);
                                if (at < kCandCap) {
                                    E.ck[at] = kv[u];
                                    E.ct[at] = (uint64_t(uint32_t(pos[rr])) << 8) | uint64_t(h);
                                }
                            }
                        }
                    }
                    ev_sync();
                    if (P.trace) tp[1] = gtimer();
                    const int n = E.ncand;
                    if (int64_t(n) == eq && n <= kCandCap) {
                        auto each = [&](auto&& f) {
                            for (int i = et; i < n; i += 32 * kSEvict) f(E.ck[i], E.ct[i]);
                        };
                        ev_resolve(E, each, kb, k_rem, eq, et, T, U);
                    } else {  // list overflow: resolve over the layer's rows in global memory
                        auto each = [&](auto&& f) {
                            for (int rr = et; rr < region; rr += 32 * kSEvict) {
                                const int h = ev_head_of(E, P.H, rr);
                                if (rr - E.off[h] >= E.len[h]) continue;
                                const uint32_t key = __ldcg(P.keys + base + rr);
                                if ((key >> 14) != kb) continue;
                                f(key, (uint64_t(uint32_t(pos[rr])) << 8) | uint64_t(h));
                            }
                        };
                        ev_resolve(E, each, kb, k_rem, eq, et, T, U);
                    }
                }
                if (P.trace) tp[2] = gtimer();
                // keep[] + kept rows per evict chunk and per head
                for (int i = et; i < P.C; i += 32 * kSEvict) E.ccnt[i] = 0;
                for (int i = et; i < P.H; i += 32 * kSEvict) E.hcnt[i] = 0;
                ev_sync();
                for (int b0 = 0; b0 < region; b0 += kSpan * 32 * kSEvict) {
                    const int r0 = b0 + et * kSpan;
                    if (r0 >= region) continue;
                    uint32_t kv[kSpan];
                    load16(r0, kv);
                    int h = ev_head_of(E, P.H, r0);
                    int live_end = E.off[h] + E.len[h], head_end = E.off[h + 1];
                    uint64_t kbits = 0;
                    int cnt = 0, hrun = 0;
#pragma unroll
                    for (int u = 0; u < kSpan; ++u) {
                        const int rr = r0 + u;
                        if (rr >= region) break;
                        while (rr >= head_end) {
                            if (hrun) atomicAdd(&E.hcnt[h], uint32_t(hrun));
                            hrun = 0;
                            ++h;
                            live_end = E.off[h] + E.len[h];
                            head_end = E.off[h + 1];
                        }
                        bool k = false;
                        if (rr < live_end)
                            k = all || kv[u] < T ||
                                (kv[u] == T && ((uint64_t(uint32_t(pos[rr])) << 8) | uint64_t(h)) <= U);
                        if (k) {
                            kbits |= uint64_t(1) << u;
                            ++cnt;
                            ++hrun;
                        }
                    }
                    if (hrun) atomicAdd(&E.hcnt[h], uint32_t(hrun));
                    if (cnt) atomicAdd(&E.ccnt[r0 / kEvRows], uint32_t(cnt));  // kEvRows % kSpan == 0
                    uint8_t* dstk = keep + r0;
                    if (r0 + kSpan <= region && (reinterpret_cast<uintptr_t>(dstk) & 15) == 0) {
#pragma unroll
                        for (int q16 = 0; q16 < kSpan / 16; ++q16) {
                            uint32_t w[4];
#pragma unroll
                            for (int q4 = 0; q4 < 4; ++q4) {
                                w[q4] = 0;
#pragma unroll
                                for (int b = 0; b < 4; ++b)
                                    w[q4] |= uint32_t((kbits >> (16 * q16 + 4 * q4 + b)) & 1u) << (8 * b);
                            }
                            reinterpret_cast<uint4*>(dstk)[q16] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    } else {
                        for (int u = 0; u < kSpan && r0 + u < region; ++u) dstk[u] = uint8_t((kbits >> u) & 1u);
                    }
                }
                __threadfence();
                ev_sync();
                if (P.trace) tp[3] = gtimer();
                if (ew == 0) {  // plan: chunk prefix (one warp), output head offsets
                    int run = 0;
                    for (int c0 = 0; c0 < P.C; c0 += 32) {
                        const int cc = c0 + lane;
                        const int v = cc < P.C ? int(E.ccnt[cc]) : 0;
                        int incl = v;
                        for (int o = 1; o < 32; o <<= 1) {
                            const int u = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += u;
                        }
                        if (cc < P.C) P.chunk_pre[l * P.C + cc] = run + incl - v;
                        run += __shfl_sync(0xffffffffu, incl, 31);
                    }
                    if (lane == 0) {
                        const int64_t cap = P.lt_out.base[l + 1] - P.lt_out.base[l];
                        int64_t acc = 0;
                        for (int h = 0; h < P.H; ++h) {
                            const int64_t nh = E.hcnt[h];
                            P.out_off[l * (P.H + 1) + h] = int32_t(acc + int64_t(P.slack) * h);
                            P.out_len[l * P.H + h] = int32_t(nh);
                            acc += nh;
                        }
                        P.out_off[l * (P.H + 1) + P.H] = int32_t(acc + int64_t(P.slack) * P.H);
                        if (acc + int64_t(P.slack) * P.H > cap) atomicCAS(P.err_flag, 0, EPK_ERR_ARG);
                        if (P.kept_per_layer) P.kept_per_layer[l] = int32_t(acc);
                        __threadfence();
                        atomicExch(ctl.plan_ready(l), 1u);
                    }
                }
                ev_sync();
            } else {  // ---- gather chunk c: kept K/V rows and positions
                if (et == 0) wait_ge(ctl.plan_ready(l), 1u, P.err_flag);
                ev_sync();
                if (P.trace) t_ready = gtimer();
                ev_load_layer(P, E, l, et);
                const int64_t out_base = P.lt_out.base[l];
                const int r_beg = c * kEvRows, r_end = min(E.off[P.H], r_beg + kEvRows);
                const int run = __ldcg(P.chunk_pre + l * P.C + c);
                const int hl = lane >> 4, cl = lane & 15;
                const int nrows = r_end - r_beg;
                const int ngrp = (nrows + 31) / 32;
                if (P.debug & 2) goto gather_done;
                for (int r0 = et * 16; r0 < nrows; r0 += 16 * 32 * kSEvict) {  // keep bytes -> shared memory
                    {
                        const uint8_t* src = P.keep + base + r_beg + r0;
                        if (r0 + 16 <= nrows && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                            *reinterpret_cast<uint4*>(E.keepb + r0) = __ldcg(reinterpret_cast<const uint4*>(src));
                        } else {
                            for (int u = 0; u < 16; ++u) E.keepb[r0 + u] = r0 + u < nrows ? __ldcg(src + u) : 0;
                        }
                    }
                }
                ev_sync();
                for (int g = ew; g < ngrp; g += kSEvict) {  // keep ballot of every 32-row group
                    const int i = g * 32 + lane;
                    const unsigned bal = __ballot_sync(0xffffffffu, i < nrows && E.keepb[i] != 0);
                    if (lane == 0) E.gbal[g] = bal;
                }
                ev_sync();
                if (ew == 0) {  // kept rows of the chunk before each group
                    int acc = run;
                    for (int g0 = 0; g0 < ngrp; g0 += 32) {
                        const int g = g0 + lane;
                        const int v = g < ngrp ? __popc(E.gbal[g]) : 0;
                        int incl = v;
                        for (int o = 1; o < 32; o <<= 1) {
                            const int u = __shfl_up_sync(0xffffffffu, incl, o);
                            if (lane >= o) incl += u;
                        }
                        if (g < ngrp) E.gpre[g] = acc + incl - v;
                        acc += __shfl_sync(0xffffffffu, incl, 31);
                    }
                }
                ev_sync();
                {
                    // Each warp copies its groups (32 rows, <= 32 kept) as pairs
                    // of 16-row halves, software-pipelined: the loads of pair j
                    // are issued before the stores of pair j-1, so ~16 KB per
                    // warp stay in flight.  Half-warp per row, 16-byte vectors.
                    const int ngw = ngrp > ew ? (ngrp - ew + kSEvict - 1) / kSEvict : 0;
                    uint4 ka[8], va[8], kb2[8], vb[8];
                    int32_t da[8], db[8];  // destination rows relative to out_base
                    int32_t pos_pending = 0;
                    int64_t pos_dst = -1;
                    auto prep = [&](int i) {  // rank tables of group i; its positions
                        const int g = ew + i * kSEvict;
                        const unsigned bal = E.gbal[g];
                        const int rr = r_beg + g * 32 + lane;
                        if ((bal >> lane) & 1u) {
                            const int rank = __popc(bal & ((1u << lane) - 1u));
                            int32_t dst = E.gpre[g] + rank;
                            if (P.slack) dst += P.slack * ev_head_of(E, P.H, rr);
                            E.gsrc[ew][i & 1][rank] = uint8_t(lane);
                            E.gdst[ew][i & 1][rank] = dst;
                            pos_pending = P.in_pos[base + rr];
                            pos_dst = out_base + dst;
                        } else {
                            pos_dst = -1;
                        }
                        __syncwarp();
                    };
                    auto load_pair = [&](int j, uint4 (&kk)[8], uint4 (&vv2)[8], int32_t (&dd)[8]) {
                        const int i = j >> 1, hf = j & 1;
                        const int g = ew + i * kSEvict;
                        const int nk = __popc(E.gbal[g]);
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            const int rank = 16 * hf + 2 * v + hl;
                            dd[v] = -1;
                            if (rank < nk) {
                                const int srcl = E.gsrc[ew][i & 1][rank];
                                dd[v] = E.gdst[ew][i & 1][rank];
                                const int64_t src = (base + r_beg + g * 32 + srcl) * 16 + cl;
                                kk[v] = __ldg(P.in_k + src);
                                vv2[v] = __ldg(P.in_v + src);
                            }
                        }
                    };
                    uint4* ok = P.out_k + out_base * 16 + cl;
                    uint4* ov = P.out_v + out_base * 16 + cl;
                    auto store_pair = [&](uint4 (&kk)[8], uint4 (&vv2)[8], int32_t (&dd)[8]) {
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            if (dd[v] >= 0) {
                                ok[int64_t(dd[v]) * 16] = kk[v];
                                ov[int64_t(dd[v]) * 16] = vv2[v];
                            }
                        }
                    };
                    const int npair = 2 * ngw;
                    for (int j = 0; j < npair + 1; j += 2) {
                        // even pair j -> buffer a; store odd pair j-1 from buffer b
                        if (j < npair) {
                            if (pos_dst >= 0) P.out_pos[pos_dst] = pos_pending;  // previous group's positions
                            prep(j >> 1);
                            load_pair(j, ka, va, da);
                        }
                        if (j >= 1) store_pair(kb2, vb, db);
                        if (j + 1 < npair) load_pair(j + 1, kb2, vb, db);
                        if (j < npair) store_pair(ka, va, da);
                    }
                    if (pos_dst >= 0) P.out_pos[pos_dst] = pos_pending;
                }
            gather_done:
                // this chunk's share of the layer's histogram reset (read by
                // collect/select, which precede plan_ready)
                const int per = (65536 + P.C - 1) / P.C;
                uint32_t* hf = P.hist_fine + int64_t(l) * 65536;
                for (int b = c * per + et; b < min(65536, (c + 1) * per); b += 32 * kSEvict) hf[b] = 0;
                if (c == 0)
                    for (int b = et; b < 256; b += 32 * kSEvict) P.hist_coarse[l * 256 + b] = 0;
            }
            if (P.trace && et == 0) {
                const unsigned long long t1 = gtimer();
                const unsigned slot = atomicAdd(reinterpret_cast<unsigned*>(P.trace), 1u);
                if (slot < 60000) {
                    unsigned long long* rec = P.trace + 8 + 4 * uint64_t(slot);
                if (c < 0 && slot < 1000) {
                    unsigned long long* px = P.trace + 8 + 4 * 60000 + 2048 + 4 * uint64_t(l);
                    for (int q = 0; q < 4; ++q) px[q] = tp[q] ? tp[q] - t_item0 : 0;
                }
                    rec[0] = uint64_t(j) | (uint64_t(l) << 32);
                    rec[1] = blockIdx.x | ((t_ready - t_item0) << 16);
                    rec[2] = t_item0;
                    rec[3] = t1;
                }
            }
        }
    }
evict_done:
    if (P.trace && threadIdx.x == 32 * kEpiWarp0)  // scoring epilogue finished (warp 4 exits its loop)
        P.trace[8 + 4 * 60000 + blockIdx.x] = gtimer();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int step_smem(int NQ, int G, int kstages, int L, int H, int lag) {
    return 1024 + 2 * NQ * kChunk * kRowB + kstages * 2 * 128 * kRowB + (NQ * kChunk + kChunk + G * kChunk) * 4 +
           (2 * kstages + 2 * kSMaxQ + 8) * 8 + 2 * 4 + 16 + (L * (H + 1) + L + lag + 1) * 4;
}

// Shapes the fused step supports (else epk_evict_step uses the layer-group
// path): bf16, head_dim 128, G * p <= 512, <= 64 kv heads, no pins.
bool step_fused_supported(const epk_cache_desc* in, int q_heads, int p, int n_pins) {
    if (in->dtype != EPK_BF16 || in->head_dim != kD || n_pins != 0 || in->kv_heads > kSMaxHeads) return false;
    if (q_heads % in->kv_heads != 0 || p < 1 || p > 256) return false;
    if ((q_heads / in->kv_heads) * p > kSMaxQ * kChunk) return false;
    return std::getenv("EPK_STEP_UNFUSED") == nullptr;
}

int launch_step_fused(epk_ctx* ctx, const epk_cache_desc* in, const epk_cache_desc* out, const void* q,
                      const void* kp, int hq, int p, const int64_t* budgets, int agg_max, int64_t n_max, int slack,
                      float* scores, uint32_t* keys, uint32_t* hist_f, uint32_t* hist_c, uint8_t* keep, uint64_t* thr,
                      int32_t* kept) {
    StepParams P;
    int rc = make_layer_table(in, &P.lt_in);
    if (rc) return rc;
    if ((rc = make_layer_table(out, &P.lt_out))) return rc;
    if (in->layers != out->layers || in->kv_heads != out->kv_heads || in->head_dim != out->head_dim ||
        in->dtype != out->dtype)
        return fail(EPK_ERR_DIM, "evict_step: in/out cache shapes differ");
    for (int l = 0; l < in->layers; ++l) {
        if (budgets[l] < 0) return fail(EPK_ERR_ARG, "select: negative budget");
        P.budget[l] = budgets[l];
    }
    const int H = in->kv_heads, L = in->layers;
    P.L = L;
    P.H = H;
    P.Hq = hq;
    P.G = hq / H;
    P.p = p;
    P.Gp = P.G * p;
    P.NQ = (P.Gp + kChunk - 1) / kChunk;
    P.ptiles = (p + 127) / 128;
    (void)n_max;  // items follow the live head lengths on the device
    int64_t max_region = 0;
    for (int l = 0; l < L; ++l) max_region = std::max<int64_t>(max_region, P.lt_in.base[l + 1] - P.lt_in.base[l]);
    // splits of 20 tiles (2560 rows): items large enough to amortise the Q
    // reload, small enough to balance ~10 items per CTA at cfg2
    P.split_tiles = 20;
    P.Smax = int(std::max<int64_t>(1, (max_region + P.split_tiles * 128 - 1) / (P.split_tiles * 128)));
    // lag: P2(l) goes out ~2 waves of items after P1(l) (estimated from the
    // layers' largest possible item count)
    {
        int64_t tot = 0;
        for (int l = 0; l < L; ++l) tot += std::min<int64_t>(int64_t(H) * P.Smax, (P.lt_in.base[l + 1] - P.lt_in.base[l]) / (P.split_tiles * 128) + H);
        const int64_t per_layer = std::max<int64_t>(1, tot / L);
        P.lag = int(std::max<int64_t>(1, std::min<int64_t>(L, (2 * ctx->num_sms + per_layer - 1) / per_layer + 1)));
    }
    P.C = int(std::max<int64_t>(1, (max_region + kEvRows - 1) / kEvRows));
    P.ev_items = L * (P.C + 1);
    if (P.C > 512) return fail(EPK_ERR_UNSUPPORTED, "evict_step(fused): layer region too large");
    P.slack = slack;
    P.agg_max = agg_max;
    P.c2 = float((1.0 / std::sqrt(double(kD))) * 1.4426950408889634);
    P.in_off = in->head_off;
    P.in_len = in->head_len;
    P.in_pos = in->pos;
    P.in_k = static_cast<const uint4*>(in->k);
    P.in_v = static_cast<const uint4*>(in->v);
    P.out_off = out->head_off;
    P.out_len = out->head_len;
    P.out_pos = out->pos;
    P.out_k = static_cast<uint4*>(out->k);
    P.out_v = static_cast<uint4*>(out->v);
    P.scores = scores;
    P.keys = keys;
    P.hist_fine = hist_f;
    P.hist_coarse = hist_c;
    P.keep = keep;
    P.thr = thr;
    P.kept_per_layer = kept;
    P.err_flag = ctx->err_flag;
    P.debug = std::getenv("EPK_STEP_DEBUG") ? std::atoi(std::getenv("EPK_STEP_DEBUG")) : 0;
    static unsigned long long* trace_buf = nullptr;
    const size_t trace_words = 8 + 4 * 60000 + 2048 + 4 * 128;
    P.trace = nullptr;
    if (std::getenv("EPK_STEP_TRACE")) {
        if (!trace_buf) EPK_CUDA_CHECK(cudaMalloc(&trace_buf, trace_words * 8));
        EPK_CUDA_CHECK(cudaMemsetAsync(trace_buf, 0, trace_words * 8, ctx->stream));
        P.trace = trace_buf;
    }
    // workspace: partials, chunk counts/prefix, candidates, control block
    const int64_t qrows = int64_t(L) * H * P.NQ * kChunk;
    const int64_t ws = 2 * qrows * 2 * P.Smax * 4 + 2 * int64_t(L) * P.C * 4 + int64_t(L) * kCandCap * 16 +
                       StepCtl::words(L, H) * 4 + 8 * 256;
    rc = ws_require(ctx, ws);
    if (rc) return rc;
    WsCarver carve(ctx->ws);
    P.part_m = carve.take<float>(qrows * 2 * P.Smax);
    P.part_z = carve.take<float>(qrows * 2 * P.Smax);
    P.chunk_cnt = carve.take<int32_t>(int64_t(L) * P.C);
    P.chunk_pre = carve.take<int32_t>(int64_t(L) * P.C);
    P.cand = carve.take<uint4>(int64_t(L) * kCandCap);
    P.ctl.base = carve.take<unsigned>(StepCtl::words(L, H));
    P.ctl.L = L;
    P.ctl.H = H;

    static int limit = 0;
    if (!limit) {
        int optin = 0;
        EPK_CUDA_CHECK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
        cudaFuncAttributes fa;
        EPK_CUDA_CHECK(cudaFuncGetAttributes(&fa, step_kernel));
        limit = optin - int(fa.sharedSizeBytes);
        EPK_CUDA_CHECK(cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
    }
    P.kstages = 4;
    while (P.kstages > 2 && step_smem(P.NQ, P.G, P.kstages, L, H, P.lag) > limit) --P.kstages;
    const int smem = step_smem(P.NQ, P.G, P.kstages, L, H, P.lag);
    if (smem > limit) return fail(EPK_ERR_UNSUPPORTED, "evict_step(fused): shared memory");
    int per_sm = 0;
    EPK_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, step_kernel, kSThreads, smem));
    if (per_sm < 1) return fail(EPK_ERR_UNSUPPORTED, "evict_step(fused): kernel does not fit an SM");

    CUtensorMap tm_k, tm_q, tm_kp;
    if ((rc = make_map(&tm_k, in->k, in->layer_base[L], 128))) return rc;
    if ((rc = make_map(&tm_q, q, int64_t(L) * hq * p, kChunk))) return rc;
    if ((rc = make_map(&tm_kp, kp, int64_t(L) * H * p, 128))) return rc;

    EPK_CUDA_CHECK(cudaMemsetAsync(P.ctl.base, 0, size_t(StepCtl::words(L, H)) * 4, ctx->stream));
    if (std::getenv("EPK_TC_VERBOSE"))
        fprintf(stderr, "step: L=%d H=%d NQ=%d Smax=%d split_tiles=%d lag=%d C=%d ev_items=%d kstages=%d smem=%d\n",
                L, H, P.NQ, P.Smax, P.split_tiles, P.lag, P.C, P.ev_items, P.kstages, smem);
    void* args[] = {&P, &tm_k, &tm_q, &tm_kp};
    EPK_PROF(ctx, "step_fused");
    EPK_CUDA_CHECK(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(step_kernel), dim3(ctx->num_sms),
                                               dim3(kSThreads), args, size_t(smem), ctx->stream));
    EPK_LAUNCH_CHECK(ctx);
    if (P.trace) {  // diagnostics: dump the evict-item timeline
        std::vector<unsigned long long> h(trace_words);
        EPK_CUDA_CHECK(cudaMemcpyAsync(h.data(), trace_buf, trace_words * 8, cudaMemcpyDeviceToHost, ctx->stream));
        EPK_CUDA_CHECK(cudaStreamSynchronize(ctx->stream));
        if (FILE* f = std::fopen(std::getenv("EPK_STEP_TRACE"), "wb")) {
            const uint32_t meta[4] = {uint32_t(P.C), uint32_t(L), uint32_t(ctx->num_sms), 0};
            std::fwrite(meta, 4, 4, f);
            std::fwrite(h.data(), 8, h.size(), f);
            std::fclose(f);
        }
    }
    return EPK_OK;
}

}  // namespace epk
