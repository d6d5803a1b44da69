// tc_common.cuh -- device and host helpers shared by the tensor-core scorer
// (score_tc.cu) and the fused step kernel (step.cu): the 128 x N x 128 bf16
// tcgen05 MMA over SWIZZLE_128B operands, the TMA row loads, the two
// epilogues (STATS: online max / sum exp2 per query row; SCORE: max over query
// rows of x c2 - lse2), and the K-major bf16 tensor-map encoder.
#pragma once

#include <cudaTypedefs.h>

#include <cmath>
#include <string>

#include "epk_internal.cuh"
#include "sm100.cuh"

namespace epk {

using namespace sm100;

constexpr int kD = 128;
constexpr int kRowB = 128;   // bytes of one d-half row (64 bf16)
constexpr int kChunk = 128;  // query rows per chunk (MMA M in P1)

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

// ---- the lse bias K-step (P2) ---------------------------------------------------
// P2 needs x - lse2/c2 for every (cache row, query row).  The query-side term
// -lse2_r/c2 = h + m + l (three bf16 parts, exact to ~2^-24 relative) rides
// in an extra 16-wide MMA K-step: A' = [1 1 1 0 ...] for every cache row, B' =
// [h m l 0 ...] for every query row, so D = bias + q.k accumulates in fp32 and
// the epilogue is a bare max.  Both operands use the no-swizzle K-major layout:
// row r of a 128-row chunk at (r/8)*256 + (r%8)*16, K elements 8..15 at +128.
constexpr int kBiasRowB = 32;                    // bytes per row (16 bf16)
constexpr int kBiasChunkB = kChunk * kBiasRowB;  // 4 KB per 128 rows
constexpr uint32_t kBiasLbo = 128, kBiasSbo = 256;
__host__ __device__ constexpr int bias_off(int r) { return (r >> 3) * 256 + (r & 7) * 16; }

// D = A' B'^T (bias) + A B^T over K = 128: the bias K-step first, then the 8
// K-steps of mma_128xN accumulating onto it.
__device__ __forceinline__ void mma_128xN_bias(uint32_t d_tmem, uint32_t a, uint32_t a_half, uint32_t b,
                                               uint32_t b_half, uint32_t a_bias, uint32_t b_bias, uint32_t idesc) {
    mma_bf16_ss(d_tmem, sdesc_k_none(a_bias, kBiasLbo, kBiasSbo), sdesc_k_none(b_bias, kBiasLbo, kBiasSbo), idesc, 0u);
    const uint64_t da = sdesc_k_sw128(a), db = sdesc_k_sw128(b);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const uint32_t k = uint32_t((kk & 3) * 32);
        const uint32_t h = uint32_t(kk >> 2);
        mma_bf16_ss(d_tmem, da + ((h * a_half + k) >> 4), db + ((h * b_half + k) >> 4), idesc, 1u);
    }
}

// Loads `rows` rows (both d-halves) of a [*, 128] bf16 tensor into a
// [d-half][rows] region whose halves are `half_bytes` apart.
__device__ __forceinline__ void load_rows(uint8_t* dst, uint32_t half_bytes, const CUtensorMap* map, uint64_t* bar,
                                          int row) {
    tma_load_2d(dst, map, bar, 0, row);
    tma_load_2d(dst + half_bytes, map, bar, 64, row);
}

// SCORE epilogue on W columns of one cache row (query rows r0 .. r0+W); the
// values are x - lse2/c2 (bias K-step): Max: best = max(best, x) as three-input
// max chains (0.5 issue slots per column); Avg: per-window sums of 2^(x c2)
// accumulated per query head in shared memory.
template <int W, typename PT>
__device__ __forceinline__ void score_cols(const float (&v)[W], int r0, const PT& P, float& best, float* s_avg,
                                           int r_local) {
    if (P.agg_max) {
        // four independent three-input-max chains (short dependency chains)
        float b[4] = {best, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int i = 0; i < W; i += 8) {
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = fmaxf(fmaxf(b[j], v[i + 2 * j]), v[i + 2 * j + 1]);
        }
        best = fmaxf(fmaxf(b[0], b[1]), fmaxf(b[2], b[3]));
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
                acc += ex2(v[i] * P.c2);
            }
        }
        if (gcur < P.G) atomicAdd(&s_avg[gcur * kChunk + r_local], acc);
    }
}

// EPK_P1_POLY3 (0 = off): that many column pairs of every EPK_P1_POLY3_OF take
// their exp2 on the FMA pipe -- Cody-Waite split t = j + f (j by the 1.5*2^23
// magic add, f in [-1/2, 1/2]), degree-3 minimax for 2^f (max rel. error
// 7.5e-5, mean 5e-6), j added to the exponent bits -- so the SFU, the bound of
// P1, carries the rest.  t is clamped at -126 (masked columns), NaN kept.
#ifndef EPK_P1_POLY3
#define EPK_P1_POLY3 3
#endif
#ifndef EPK_P1_POLY3_OF
#define EPK_P1_POLY3_OF 16
#endif
__device__ __forceinline__ float clamp_lo_nan(float t) { return t < -126.f ? -126.f : t; }
__device__ __forceinline__ uint64_t exp2_poly3x2(uint64_t t2) {
    float a, b;
    f2_unpack(t2, a, b);
    const uint64_t t = f2_pack(clamp_lo_nan(a), clamp_lo_nan(b));
    const uint64_t magic = f2_pack(12582912.f, 12582912.f);
    const uint64_t r = fadd2(t, magic);
    const uint64_t j = fadd2(r, f2_pack(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(j, f2_pack(-1.f, -1.f), t);
    uint64_t p = ffma2(f2_pack(0x1.c3f76p-5f, 0x1.c3f76p-5f), f, f2_pack(0x1.f0de1ap-3f, 0x1.f0de1ap-3f));
    p = ffma2(p, f, f2_pack(0x1.62f31ap-1f, 0x1.62f31ap-1f));
    p = ffma2(p, f, f2_pack(0x1.fff692p-1f, 0x1.fff692p-1f));
    float p0, p1, r0, r1;
    f2_unpack(p, p0, p1);
    f2_unpack(r, r0, r1);
    return f2_pack(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(r0) << 23)),
                   __uint_as_float(__float_as_uint(p1) + (__float_as_uint(r1) << 23)));
}

// STATS epilogue on W columns of one query row, `lim` of them valid:
// online (max, sum 2^(x c2 - max)) update of (m, z).  Pairs of columns go
// through FFMA2/FADD2; the exp2 of EPK_P1_POLY3 of every EPK_P1_POLY3_OF pairs
// through exp2_poly3x2 on the FMA pipe, the rest through MUFU.EX2 (the bound
// of this pass; 3/16 measured best, profiles/p1_variants_r02c.txt).
template <int W>
__device__ __forceinline__ void stats_cols(float (&v)[W], int lim, float c2, float& m, float& z) {
    float mx = -INFINITY;
    if (lim >= W) {
        // max as eight independent three-input-max chains + a tree, not one
        // W-deep dependency chain (the chain was the epilogue's top stall)
        constexpr int C = W >= 16 ? 8 : W / 2;
        float t[C];
#pragma unroll
        for (int j = 0; j < C; ++j) t[j] = fmaxf(v[2 * j], v[2 * j + 1]);
#pragma unroll
        for (int i = 2 * C; i < W; i += 2 * C)
#pragma unroll
            for (int j = 0; j < C; ++j) t[j] = fmaxf(fmaxf(t[j], v[i + 2 * j]), v[i + 2 * j + 1]);
#pragma unroll
        for (int w = C / 2; w >= 1; w /= 2)
#pragma unroll
            for (int j = 0; j < w; ++j) t[j] = fmaxf(t[j], t[j + w]);
        mx = t[0];
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
        const uint64_t c2x2 = f2_pack(c2, c2), nm2 = f2_pack(-m, -m);
        uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
#pragma unroll
        for (int i = 0; i < W; i += 4) {
            const uint64_t t0 = ffma2(f2_pack(v[i], v[i + 1]), c2x2, nm2);
            const uint64_t t1 = ffma2(f2_pack(v[i + 2], v[i + 3]), c2x2, nm2);
            uint64_t e[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (((i / 2 + q) % EPK_P1_POLY3_OF) >= EPK_P1_POLY3_OF - EPK_P1_POLY3) {
                    e[q] = exp2_poly3x2(q ? t1 : t0);
                } else {
                    float a, b;
                    f2_unpack(q ? t1 : t0, a, b);
                    e[q] = f2_pack(ex2(a), ex2(b));
                }
            }
            acc0 = fadd2(acc0, e[0]);
            acc1 = fadd2(acc1, e[1]);
        }
        float a0, a1, b0, b1;
        f2_unpack(acc0, a0, a1);
        f2_unpack(acc1, b0, b1);
        z += (a0 + a1) + (b0 + b1);
    }
}

// ---- host: K-major bf16 [rows, 128] tensor maps with SWIZZLE_128B boxes -----
inline PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
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

inline int make_map(CUtensorMap* m, const void* base, int64_t rows, int box_rows) {
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

}  // namespace epk
