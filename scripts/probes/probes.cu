// probes.cu -- diagnostics, not on the product path:
//   epk_debug_tma_stream: TMA streaming bandwidth of the scorer's K-tile
//     producer with a trivial consumer (sizes the K ring);
//   epk_debug_mma_rate: tcgen05.mma issue ceiling for 128xN bf16 tiles from
//     resident shared memory, optionally drained by epilogue warps.
#include <cudaTypedefs.h>

#include <algorithm>

#include "epk_internal.cuh"
#include "sm100.cuh"
#include "tc_common.cuh"

namespace epk {
using namespace sm100;

__global__ void __launch_bounds__(64, 1) tma_stream_kernel(const __grid_constant__ CUtensorMap tm, int64_t rows,
                                                           int box_rows, int stages, unsigned* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int tile_bytes = box_rows * 256;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * tile_bytes);
    uint64_t* empty = full + stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int64_t tiles = rows / box_rows;
    const int64_t per = (tiles + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
    if (warp == 0 && lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], tile_bytes);
            tma_load_2d(smem + s * tile_bytes, &tm, &full[s], 0, int(t * box_rows));
            tma_load_2d(smem + s * tile_bytes + tile_bytes / 2, &tm, &full[s], 64, int(t * box_rows));
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1 && lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        unsigned acc = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&full[s], ph);
            acc += smem[s * tile_bytes + (t & 255)];
            mbar_arrive(&empty[s]);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
        if (acc == 0xFFFFFFFFu) *sink = acc;
    }
}

int launch_tma_stream(epk_ctx* ctx, const void* base, int64_t rows, int box_rows, int stages, int grid) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {128, cuuint64_t(rows)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(EPK_ERR_CUDA, "tensor map");
    const int smem = 1024 + stages * box_rows * 256 + 2 * stages * 8;
    EPK_CUDA_CHECK(cudaFuncSetAttribute(tma_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    unsigned* sink = reinterpret_cast<unsigned*>(ctx->err_flag);
    EPK_PROF(ctx, "tma_stream");
    tma_stream_kernel<<<grid, 64, smem, ctx->stream>>>(m, rows, box_rows, stages, sink);
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// 128 x N x 128 bf16 MMAs (8 K-steps) from resident smem into a ring of
// TMEM slots; with `drain`, 4 epilogue warps tcgen05.ld each result (64
// columns at a time) before the slot is reused.
template <int N>
__global__ void __launch_bounds__(192, 1) mma_rate_kernel(int iters, int drain, unsigned* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;                  // 128 x 128 bf16 (two swizzled halves)
    uint8_t* sB = smem + 32768;          // N x 128
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + N * 256);
    uint64_t* empty = full + 8;
    uint32_t* holder = reinterpret_cast<uint32_t*>(empty + 8);
    constexpr int kSlots = 512 / N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (32768 + N * 256) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(holder, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    if (warp == 1 && lane == 0) {
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int it = 0; it < iters; ++it) {
            const int s = it % kSlots;
            const uint32_t ph = (it / kSlots) & 1;
            if (drain) mbar_wait(&empty[s], ph ^ 1);
            else if (it >= kSlots) mbar_wait(&full[s], ph ^ 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t aoff = uint32_t((kk >> 2) * 16384 + (kk & 3) * 32);
                const uint32_t boff = uint32_t((kk >> 2) * (N * 128) + (kk & 3) * 32);
                mma_bf16_ss(tmem + uint32_t(s * N), sdesc_k_sw128(a0 + aoff), sdesc_k_sw128(b0 + boff), idesc, kk > 0);
            }
            mma_commit(&full[s]);
        }
    } else if (warp >= 2 && drain) {
        const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
        float acc = 0.f;
        for (int it = 0; it < iters; ++it) {
            const int s = it % kSlots;
            mbar_wait(&full[s], (it / kSlots) & 1);
            tc_fence_after();
            for (int c = 0; c < N; c += 64) {
                float v[64];
                tmem_ld64(tmem + lane_addr + uint32_t(s * N + c), v);
                acc += v[0] + v[63];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 12345.f) *sink = 1;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

int launch_mma_rate(epk_ctx* ctx, int n, int iters, int drain) {
    const int smem = 1024 + 32768 + n * 256 + 256;
    unsigned* sink = reinterpret_cast<unsigned*>(ctx->err_flag);
    EPK_PROF(ctx, "mma_rate");
    auto run = [&](auto kern) -> int {
        EPK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        kern<<<ctx->num_sms, 192, smem, ctx->stream>>>(iters, drain, sink);
        return EPK_OK;
    };
    int rc;
    switch (n) {
        case 64: rc = run(mma_rate_kernel<64>); break;
        case 128: rc = run(mma_rate_kernel<128>); break;
        case 192: rc = run(mma_rate_kernel<192>); break;
        case 256: rc = run(mma_rate_kernel<256>); break;
        default: return fail(EPK_ERR_ARG, "mma_rate: n must be 64, 128, 192 or 256");
    }
    if (rc) return rc;
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// Two-SM variant: tcgen05.mma.cta_group::2 (M = 256: each CTA of the pair
// supplies its 128 A rows and N/2 B rows from its own shared memory at the
// same offsets; D lands in both CTAs' TMEM, 128 lanes x N each).  The leader
// CTA issues; commits multicast to both CTAs' barriers.  Measures whether
// the pair runs N = 128 / 256 jobs at the tensor pipe's rate (the one-SM
// N = 128 jobs reach 69 %, see mma_rate_kernel).
template <int N>
__global__ void __launch_bounds__(64, 1) mma2sm_rate_kernel(int iters, unsigned* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = smem;          // 128 x 128 bf16 (this CTA's half of A)
    uint8_t* sB = smem + 32768;  // N/2 x 128 (this CTA's half of B)
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + (N / 2) * 256);
    uint32_t* holder = reinterpret_cast<uint32_t*>(full + 8);
    constexpr int kSlots = 512 / N;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < (32768 + (N / 2) * 256) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kSlots; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(holder))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = *holder;
    constexpr uint32_t idesc = idesc_bf16_f32(256, N);
    if (rank == 0 && warp == 0 && lane == 0) {
        const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
        for (int it = 0; it < iters; ++it) {
            const int s = it % kSlots;
            if (it >= kSlots) mbar_wait(&full[s], ((it / kSlots) & 1) ^ 1);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const uint32_t aoff = uint32_t((kk >> 2) * 16384 + (kk & 3) * 32);
                const uint32_t boff = uint32_t((kk >> 2) * ((N / 2) * 128) + (kk & 3) * 32);
                const uint64_t ad = sdesc_k_sw128(a0 + aoff), bd = sdesc_k_sw128(b0 + boff);
                const uint32_t acc = kk > 0 ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + uint32_t(s * N)),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
                    : "memory");
            }
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&full[s])),
                "h"(uint16_t(3))
                : "memory");
        }
        // drain: the last commit of every slot
        for (int it = iters; it < iters + kSlots; ++it) {
            const int s = it % kSlots;
            if (it >= kSlots) mbar_wait(&full[s], ((it / kSlots) & 1) ^ 1);
        }
    }
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    if (threadIdx.x == 0 && iters < 0) *sink = tmem;
}

int launch_mma2sm_rate(epk_ctx* ctx, int n, int iters) {
    const int smem = 1024 + 32768 + (n / 2) * 256 + 256;
    unsigned* sink = reinterpret_cast<unsigned*>(ctx->err_flag);
    auto run = [&](auto kern) -> int {
        EPK_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctx->num_sms & ~1);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        EPK_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, iters, sink));
        return EPK_OK;
    };
    EPK_PROF(ctx, "mma2sm_rate");
    int rc;
    switch (n) {
        case 128: rc = run(mma2sm_rate_kernel<128>); break;
        case 256: rc = run(mma2sm_rate_kernel<256>); break;
        default: return fail(EPK_ERR_ARG, "mma2sm_rate: n must be 128 or 256");
    }
    if (rc) return rc;
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// TMA gather (round-2 evidence for an overlapped compaction): `sms` CTAs of 4
// warps walk 128-row chunks; the kept rows' indices (from keep[]) feed
// tile::gather4 loads (4 arbitrary rows of K / V per op) into a packed shared
// buffer, and one 1-D bulk store per tensor writes the chunk's kept rows to
// their contiguous destination (prefix[chunk]).  Two buffers: a chunk's
// stores drain while the next chunk's gathers land.  No registers hold the
// bytes in flight, so a few SMs can keep HBM busy.
__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int col, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
        : "memory");
}
__device__ __forceinline__ void bulk_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(reinterpret_cast<uint64_t>(dst)),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

template <int NB>
__global__ void __launch_bounds__(128) tma_gather_kernel(const __grid_constant__ CUtensorMap tk,
                                                         const __grid_constant__ CUtensorMap tv,
                                                         const uint8_t* keep, const int32_t* prefix, int nchunks,
                                                         uint8_t* kout, uint8_t* vout) {
    // NB chunks in flight per CTA: chunk i's gathers are issued, then chunk
    // i-(NB-1)'s (long landed) rows are stored
    extern __shared__ __align__(128) uint8_t smem_raw[];
    uint8_t* buf = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);  // [NB][K 32 KB | V 32 KB]
    __shared__ uint64_t full[NB];
    __shared__ int s_idx[NB][128];
    __shared__ int s_n[NB], s_c[NB];
    __shared__ int s_wc[4];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NB; ++i) mbar_init(&full[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int mine = nchunks > int(blockIdx.x) ? (nchunks - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
    for (int it = 0; it < mine + NB - 1; ++it) {
        const int b = it % NB;
        if (it < mine) {
            const int c = int(blockIdx.x) + it * int(gridDim.x);
            const int r = c * 128 + warp * 32 + lane;
            const bool k = keep[r] != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, k);
            if (lane == 0) s_wc[warp] = __popc(bal);
            __syncthreads();
            int base = 0;
            for (int w = 0; w < warp; ++w) base += s_wc[w];
            if (k) s_idx[b][base + __popc(bal & ((1u << lane) - 1u))] = r;
            if (threadIdx.x == 0) {
                s_n[b] = s_wc[0] + s_wc[1] + s_wc[2] + s_wc[3];
                s_c[b] = c;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                const int n = s_n[b];
                uint8_t* sk = buf + b * 65536;
                uint8_t* sv = sk + 32768;
                // buffer b's previous stores (chunk it-NB) must have read it
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(NB - 2) : "memory");
                const int groups = (n + 3) / 4;
                mbar_expect_tx(&full[b], uint32_t(groups * 4 * 256 * 2));
                for (int g = 0; g < groups; ++g) {
                    const int* ix = s_idx[b] + 4 * g;
                    const int i0 = ix[0], i1 = 4 * g + 1 < n ? ix[1] : i0, i2 = 4 * g + 2 < n ? ix[2] : i0,
                              i3 = 4 * g + 3 < n ? ix[3] : i0;
                    tma_gather4(sk + g * 1024, &tk, &full[b], 0, i0, i1, i2, i3);
                    tma_gather4(sv + g * 1024, &tv, &full[b], 0, i0, i1, i2, i3);
                }
            }
        }
        const int jt = it - (NB - 1);  // the chunk whose rows are stored now
        if (threadIdx.x == 0 && jt >= 0) {
            const int bj = jt % NB;
            mbar_wait(&full[bj], uint32_t((jt / NB) & 1));
            const int n = s_n[bj];
            if (n) {
                const int64_t dst = int64_t(prefix[s_c[bj]]) * 256;
                bulk_store_1d(kout + dst, buf + bj * 65536, uint32_t(n * 256));
                bulk_store_1d(vout + dst, buf + bj * 65536 + 32768, uint32_t(n * 256));
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int launch_tma_gather(epk_ctx* ctx, const void* k, const void* v, int64_t rows, const uint8_t* keep,
                      const int32_t* prefix, void* kout, void* vout, int sms) {
    auto enc = get_encode();
    if (!enc) return fail(EPK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap mk, mv;
    cuuint64_t dims[2] = {128, cuuint64_t(rows)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t es[2] = {1, 1};
    for (int t = 0; t < 2; ++t) {
        CUresult r = enc(t ? &mv : &mk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(t ? v : k), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(EPK_ERR_CUDA, "tma_gather: tensor map (" + std::to_string(int(r)) + ")");
    }
    constexpr int NB = 3;
    const int smem = NB * 65536 + 128;
    EPK_CUDA_CHECK(cudaFuncSetAttribute(tma_gather_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    EPK_PROF(ctx, "tma_gather");
    tma_gather_kernel<NB><<<std::max(1, std::min(sms, ctx->num_sms)), 128, smem, ctx->stream>>>(
        mk, mv, keep, prefix, int(rows / 128), static_cast<uint8_t*>(kout), static_cast<uint8_t*>(vout));
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

// TMA-streamed 256-row K stages (`stages`-deep ring) feeding `nq` resident
// 128-row A chunks: per stage nq MMAs of 128 x 256 x 128 into two TMEM slots,
// drained by 8 epilogue warps (tcgen05.ld, no math).  The P1 pipeline
// without its softmax epilogue.
__global__ void __launch_bounds__(320, 1) mma_stream_kernel(const __grid_constant__ CUtensorMap tm, int64_t rows,
                                                            int nq, int stages, int drain, unsigned* sink) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t q_half = uint32_t(nq) * 128 * 128;
    uint8_t* sQ = smem;
    uint8_t* sK = smem + 2 * q_half;
    const uint32_t k_half = 256 * 128, k_stage = 2 * k_half;
    uint64_t* full = reinterpret_cast<uint64_t*>(sK + stages * k_stage);
    uint64_t* empty = full + stages;
    uint64_t* tfull = empty + stages;
    uint64_t* tempty = tfull + 2;
    uint32_t* holder = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < int(2 * q_half / 4); i += blockDim.x) reinterpret_cast<uint32_t*>(sQ)[i] = 0x3c003c00u;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], 8);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc(holder, 512);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    const int64_t tiles = rows / 256;
    const int64_t per = (tiles + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = blockIdx.x * per, t1 = min(tiles, t0 + per);
    if (warp == 0 && lane == 0) {
        int s = 0;
        uint32_t ph = 0;
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_expect_tx(&full[s], k_stage);
            tma_load_2d(sK + s * k_stage, &tm, &full[s], 0, int(t * 256));
            tma_load_2d(sK + s * k_stage + k_half, &tm, &full[s], 64, int(t * 256));
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp == 1 && lane == 0) {
        int s = 0;
        uint32_t ph = 0, job = 0;
        const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK);
        for (int64_t t = t0; t < t1; ++t) {
            mbar_wait(&full[s], ph);
            for (int c = 0; c < nq; ++c) {
                const int ts = int(job & 1);
                if (drain) mbar_wait(&tempty[ts], ((job >> 1) & 1) ^ 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint32_t k = uint32_t((kk & 3) * 32), h = uint32_t(kk >> 2);
                    mma_bf16_ss(tmem + uint32_t(ts * 256), sdesc_k_sw128(q0 + uint32_t(c) * 16384 + h * q_half + k),
                                sdesc_k_sw128(k0 + uint32_t(s) * k_stage + h * k_half + k), idesc_bf16_f32(128, 256),
                                kk > 0);
                }
                mma_commit(&tfull[ts]);
                ++job;
            }
            mma_commit(&empty[s]);
            if (++s == stages) {
                s = 0;
                ph ^= 1;
            }
        }
    } else if (warp >= 2 && drain) {
        const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
        const int half = (warp - 2) >> 2;
        float acc = 0.f;
        uint32_t job = 0;
        for (int64_t t = t0; t < t1; ++t)
            for (int c = 0; c < nq; ++c, ++job) {
                const int ts = int(job & 1);
                mbar_wait(&tfull[ts], (job >> 1) & 1);
                tc_fence_after();
                for (int q4 = 0; q4 < 2; ++q4) {
                    float v[64];
                    tmem_ld64(tmem + lane_addr + uint32_t(ts * 256 + half * 128 + q4 * 64), v);
                    acc += v[0] + v[63];
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[ts]);
            }
        if (acc == 12345.f) *sink = 1;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

int launch_mma_stream(epk_ctx* ctx, const void* base, int64_t rows, int nq, int stages, int drain) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
        enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    CUtensorMap m;
    cuuint64_t dims[2] = {128, cuuint64_t(rows)};
    cuuint64_t strides[1] = {256};
    cuuint32_t box[2] = {64, 256};
    cuuint32_t es[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return fail(EPK_ERR_CUDA, "tensor map");
    const int smem = 1024 + 2 * nq * 128 * 128 + stages * 65536 + 256;
    EPK_CUDA_CHECK(cudaFuncSetAttribute(mma_stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    EPK_PROF(ctx, "mma_stream");
    mma_stream_kernel<<<ctx->num_sms, 320, smem, ctx->stream>>>(m, rows, nq, stages, drain,
                                                                reinterpret_cast<unsigned*>(ctx->err_flag));
    EPK_LAUNCH_CHECK(ctx);
    return EPK_OK;
}

}  // namespace epk

extern "C" int epk_debug_mma_stream(epk_ctx* ctx, const void* k, int64_t rows, int32_t nq, int32_t stages,
                                    int32_t drain) {
    return epk::launch_mma_stream(ctx, k, rows, nq, stages, drain);
}

extern "C" int epk_debug_mma_rate(epk_ctx* ctx, int32_t n, int32_t iters, int32_t drain) {
    return epk::launch_mma_rate(ctx, n, iters, drain);
}

extern "C" int epk_debug_tma_gather(epk_ctx* ctx, const void* k, const void* v, int64_t rows, const uint8_t* keep,
                                    const int32_t* prefix, void* kout, void* vout, int32_t sms) {
    return epk::launch_tma_gather(ctx, k, v, rows, keep, prefix, kout, vout, sms);
}

extern "C" int epk_debug_mma2sm_rate(epk_ctx* ctx, int32_t n, int32_t iters) {
    return epk::launch_mma2sm_rate(ctx, n, iters);
}

extern "C" int epk_debug_tma_stream(epk_ctx* ctx, const void* base, int64_t rows, int32_t box_rows, int32_t stages,
                                    int32_t grid) {
    return epk::launch_tma_stream(ctx, base, rows, box_rows, stages, grid);
}
