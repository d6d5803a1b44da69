// epk_internal.cuh -- shared device/host helpers for the sm_100a kernels.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <string>
#include <utility>

#include "epk/epk.h"

#include <vector>

struct epk_prof_rec {
    char name[32];
    cudaEvent_t start, stop;
    int side;  // 1: launched on the context's side stream
};

struct epk_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;  // grow-only workspace (scoring, selection)
    int64_t ws_bytes = 0;
    void* ws2 = nullptr;  // grow-only workspace (compaction; may run on `side`)
    int64_t ws2_bytes = 0;
    cudaStream_t side = nullptr;  // second stream: compaction overlaps the next layer group's scoring
    cudaStream_t hi = nullptr;    // overlap mode: scoring + select at the highest stream priority
    cudaEvent_t ev_hi = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    cudaStream_t aux = nullptr;  // highest priority: concurrent consumer kernels (K5 chain)
    cudaEvent_t ev_aux_fork = nullptr, ev_aux_join = nullptr;
    int layer_group = 0;  // layers per group in epk_evict_step (0 = auto: group K fits in L2)
    int overlap = 1;      // run each group's compaction on `side`
    int pool_kernel = 1;  // EPK_OPT_POOL_KERNEL: opt-in max-pool smoothing of the scores (1 = off, the reference)
    void* step_buf = nullptr;  // epk_evict_step scores + keep mask
    int64_t step_bytes = 0;
    int* err_flag = nullptr;  // deferred device-side error code (device int)
    int64_t launches = 0;
    int num_sms = 148;
    int gather_sms = 0;     // SMs left to the compaction gather while the scorer runs (0: scorer takes all)
    int gather_ctas = 0;    // gather launch: persistent CTAs (0: one warp per 128-row chunk)
    int gather_threads = 128;
    int gather_smem = 0;    // dynamic shared memory reserved per gather CTA (keeps it off scorer SMs)
    bool profiling = false;  // record CUDA events around every kernel launch
    std::vector<epk_prof_rec> prof;
};

namespace epk {

// Persistent CTAs of the tensor-core scorer passes.
inline int score_grid(const epk_ctx* c) { return c->num_sms - c->gather_sms; }

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

// Workspace carve-up: returns a pointer into ctx->ws (grows the workspace when
// needed; growing is not allowed while the stream is being captured).
int ws_require(epk_ctx* ctx, int64_t bytes);
// Creates the context's aux stream and its fork/join events on first use.
int ensure_aux_stream(epk_ctx* ctx);
int ws2_require(epk_ctx* ctx, int64_t bytes);

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct WsCarver {
    char* base;
    int64_t off = 0;
    explicit WsCarver(void* b) : base(static_cast<char*>(b)) {}
    template <typename T>
    T* take(int64_t count) {
        off = align_up(off, 256);
        T* p = reinterpret_cast<T*>(base + off);
        off += count * int64_t(sizeof(T));
        return p;
    }
};

inline int dtype_size(int dt) { return dt == EPK_F64 ? 8 : (dt == EPK_F32 ? 4 : 2); }

#define EPK_CUDA_CHECK(expr)                                      \
    do {                                                          \
        cudaError_t _e = (expr);                                  \
        if (_e != cudaSuccess) return ::epk::cuda_fail(_e, #expr); \
    } while (0)

#define EPK_LAUNCH_CHECK(ctx)                                                \
    do {                                                                     \
        (ctx)->launches++;                                                   \
        ::epk::prof_end(ctx);                                                \
        cudaError_t _e = cudaGetLastError();                                 \
        if (_e != cudaSuccess) return ::epk::cuda_fail(_e, "kernel launch"); \
    } while (0)

// Live per-kernel timing (epk_ctx_profile): events on the launching stream.
void prof_begin(epk_ctx* ctx, const char* name);
void prof_end(epk_ctx* ctx);
#define EPK_PROF(ctx, name) ::epk::prof_begin(ctx, name)

// Programmatic dependent launch: the step's kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization so the next grid's launch
// is staged while its predecessor drains; every such kernel calls pdl_wait()
// before its first global access (a no-op without the attribute).  No early
// griddepcontrol.launch_dependents: dependents holding SM slots while the
// primary drains measured slower (0.84 -> 0.86 ms/step); implicit completion
// gives ~0.5 %.  EPK_NO_PDL=1 disables the attribute.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Experiment builds only (-DEPK_TIMELINE): lane 0 of every warp records its
// kernel's globaltimer at entry, after pdl_wait, and at exit into a device
// ring read back by epk_debug_timeline (scripts/tl_step.py prints the step's
// per-kernel critical path).
#ifdef EPK_TIMELINE
// one ring per translation unit (no relocatable device code), each reader
// registered with epk_api.cu's epk_debug_timeline at load time
constexpr int kTlMax = 1 << 15;
static __device__ unsigned long long g_tl[kTlMax][4];  // {kernel id << 32 | cta << 8 | warp, entry, go, end}
static __device__ unsigned int g_tl_n;
int tl_register(int (*reader)(int, unsigned long long*, int));
static int tl_read_local(int reset, unsigned long long* out, int max_records) {
    unsigned int n = 0;
    cudaMemcpyFromSymbol(&n, g_tl_n, sizeof(n));
    n = n < unsigned(kTlMax) ? n : unsigned(kTlMax);
    const unsigned m = n < unsigned(max_records > 0 ? max_records : 0) ? n : unsigned(max_records > 0 ? max_records : 0);
    if (out && m) cudaMemcpyFromSymbol(out, g_tl, size_t(m) * 32);
    if (reset) {
        const unsigned z = 0;
        cudaMemcpyToSymbol(g_tl_n, &z, sizeof(z));
    }
    return int(m);
}
static const int tl_registered = tl_register(tl_read_local);
__device__ __forceinline__ uint64_t tl_now() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TL_BEGIN() const uint64_t tl_t0 = tl_now()
#define TL_GO() const uint64_t tl_t1 = tl_now()
#define TL_END(id)                                                                                        \
    do {                                                                                                  \
        if ((threadIdx.x & 31) == 0) {                                                                    \
            const unsigned i_ = atomicAdd(&g_tl_n, 1u);                                                   \
            if (i_ < unsigned(kTlMax)) {                                                                  \
                g_tl[i_][0] = (uint64_t(id) << 32) | (uint64_t(blockIdx.x + blockIdx.y * gridDim.x) << 8) | \
                              uint64_t(threadIdx.x >> 5);                                                 \
                g_tl[i_][1] = tl_t0;                                                                      \
                g_tl[i_][2] = tl_t1;                                                                      \
                g_tl[i_][3] = tl_now();                                                                   \
            }                                                                                             \
        }                                                                                                 \
    } while (0)
#else
#define TL_BEGIN()
#define TL_GO()
#define TL_END(id)
#endif

bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Per-device host state (function attributes) is kept for ordinals < kMaxDevices.
constexpr int kMaxDevices = 64;

// Layer table passed by value to kernels (host layer_base copied in).
constexpr int kMaxLayers = 128;
struct LayerTable {
    int64_t base[kMaxLayers + 1];
};

int make_layer_table(const epk_cache_desc* c, LayerTable* t);

// Compaction plan buffers (compact.cu), per launch in the context's second
// workspace: per (layer, 128-row chunk) kept counts and their exclusive
// prefix, and a per-layer "does not fit the output" flag.  The threshold
// select (select.cu) fills them itself for the tensor-core step; the generic
// path's count/plan kernels fill them otherwise.
constexpr int kChunkRows = 128;
struct CompactWs {
    int32_t* chunk_cnt;     // [layers][max_chunks]
    int32_t* chunk_prefix;  // [layers][max_chunks]
    int32_t* layer_bad;     // [layers]
    int max_chunks;
};
int compact_ws(epk_ctx* ctx, const epk_cache_desc* in, CompactWs* w);

// Threshold-select buffers the tensor-core scorer fills in its SCORE pass
// (select.cu select_threshold_kernel consumes them).  Pointers are for the
// launch's first layer.
struct FusedSelect {
    uint32_t* keys;         // [rows] per global cache row
    uint32_t* hist_fine;    // [layers][65536] counts of float_bits(score) >> 14
    uint32_t* hist_coarse;  // [layers][256] counts of that bin >> 8
    uint4* cand;            // [layers][1024] threshold-bin candidates (select)
    unsigned* cand_n;       // [layers] candidate counts (zero between steps)
    unsigned* done;         // [layers] select arrival counters (zero between steps)
};

// ---------------------------------------------------------------------------
// Order-preserving score keys.  Selection sorts ascending on
//   (desc_key(score), position, head)
// desc_key maps larger scores to smaller keys; -0.0 is canonicalised to +0.0
// because the reference compares with != (kvcache.hpp:182), under which
// -0.0 == +0.0 and the tie falls through to the position.
// ---------------------------------------------------------------------------
__host__ __device__ inline uint32_t desc_key(float s) {
    uint32_t u;
#ifdef __CUDA_ARCH__
    u = __float_as_uint(s);
#else
    memcpy(&u, &s, 4);
#endif
    if (u == 0x80000000u) u = 0;
    const uint32_t ord = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ~ord;
}

__host__ __device__ inline uint64_t desc_key(double s) {
    uint64_t u;
#ifdef __CUDA_ARCH__
    u = static_cast<uint64_t>(__double_as_longlong(s));
#else
    memcpy(&u, &s, 8);
#endif
    if (u == 0x8000000000000000ull) u = 0;
    const uint64_t ord = (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
    return ~ord;
}

}  // namespace epk
