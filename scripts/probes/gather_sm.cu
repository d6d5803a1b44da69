// gather_sm.cu -- probe: how much HBM bandwidth can the K/V compaction gather
// draw from S SMs?  Decides whether compaction can run on a subset of SMs
// next to the scorer (SM-partitioned step) or must share every SM.
//
// Data: R rows of K and V (256 B each, bf16 d = 128), ~80 % kept at random
// (the cfg2 steady state keeps 8192 of 10240 per head), chunk prefix per
// 128 rows precomputed.  Three gathers, each persistent over S CTAs:
//   lsu   warps copy kept rows with 16-B loads/stores (compact_gather's
//         scheme: half-warp per row, U rows in flight per half-warp);
//   tma   one producer lane streams 64-row K and V chunks into a shared ring
//         with 1-D bulk copies; 4 consumer warps copy the kept rows
//         shared -> global with 16-B stores;
//   bulk  as tma, but the kept RUNS go shared -> global as bulk copies.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_sm gather_sm.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA %s at %s:%d: %s\n", cudaGetErrorString(e), __FILE__, __LINE__, #x); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int RV = 16;  // uint4 per row
constexpr int CH = 128; // rows per prefix chunk

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(512) lsu_gather(const uint4* __restrict__ ik, const uint4* __restrict__ iv,
                                                  const uint8_t* __restrict__ keep, const int* __restrict__ pre,
                                                  uint4* ok, uint4* ov, int nchunks) {
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int hl = lane >> 4, cl = lane & 15;
    for (int chunk = blockIdx.x * wpb + (threadIdx.x >> 5); chunk < nchunks; chunk += gridDim.x * wpb) {
        int run = pre[chunk];
        const int64_t r0 = int64_t(chunk) * CH;
        for (int sc = 0; sc < CH / 32; ++sc) {
            const int64_t rs = r0 + sc * 32;
            const bool k = keep[rs + lane];
            const unsigned bal = __ballot_sync(~0u, k);
            const int64_t dst = run + __popc(bal & ((1u << lane) - 1u));
            run += __popc(bal);
            for (int k0 = 0; k0 < 32; k0 += 16) {
                uint4 kv[8], vv[8];
                int64_t d[8];
                bool okk[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int idx = k0 + 2 * u + hl;
                    okk[u] = (bal >> idx) & 1u;
                    d[u] = __shfl_sync(~0u, dst, idx);
                    if (okk[u]) {
                        kv[u] = __ldg(ik + (rs + idx) * RV + cl);
                        vv[u] = __ldg(iv + (rs + idx) * RV + cl);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (okk[u]) {
                        ok[d[u] * RV + cl] = kv[u];
                        ov[d[u] * RV + cl] = vv[u];
                    }
            }
        }
    }
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
            su32(b)),
        "r"(ph)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(su32(src)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int SR = 64;  // rows per stage

// MODE 0: consumers copy with 16-B stores; MODE 1: bulk s2g per kept run
template <int MODE>
__global__ void __launch_bounds__(160) tma_gather(const uint4* __restrict__ ik, const uint4* __restrict__ iv,
                                                  const uint8_t* __restrict__ keep, const int* __restrict__ pre,
                                                  uint4* ok, uint4* ov, int nchunks, int nst) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm);
    uint64_t* empty = full + 16;
    uint8_t* ring = sm + 1024;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nsub = nchunks * (CH / SR);  // 64-row sub-chunks
    if (warp == 0) {
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int c = blockIdx.x; c < nsub; c += gridDim.x) {
                mbar_wait(&empty[s], ph ^ 1);
                mbar_expect_tx(&full[s], 2 * SR * 256);
                uint8_t* st = ring + size_t(s) * 2 * SR * 256;
                bulk_g2s(st, ik + int64_t(c) * SR * RV, SR * 256, &full[s]);
                bulk_g2s(st + SR * 256, iv + int64_t(c) * SR * RV, SR * 256, &full[s]);
                if (++s == nst) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    } else {
        const int cw = warp - 1;  // consumer warp 0..3: rows [16 cw, 16 cw + 16) of every stage
        int s = 0;
        uint32_t ph = 0;
        for (int c = blockIdx.x; c < nsub; c += gridDim.x) {
            mbar_wait(&full[s], ph);
            const uint4* st = reinterpret_cast<const uint4*>(ring + size_t(s) * 2 * SR * 256);
            const int chunk = c / (CH / SR), half = c % (CH / SR);
            const int64_t r0 = int64_t(chunk) * CH;
            // kept before this warp's 16 rows: chunk prefix + rows of the chunk before
            const uint32_t b0 = __ballot_sync(~0u, keep[r0 + lane]);
            const uint32_t b1 = __ballot_sync(~0u, keep[r0 + 32 + lane]);
            const uint32_t b2 = __ballot_sync(~0u, keep[r0 + 64 + lane]);
            const uint32_t b3 = __ballot_sync(~0u, keep[r0 + 96 + lane]);
            const uint32_t bb[4] = {b0, b1, b2, b3};
            const int first = half * SR + cw * 16;  // row within the 128-row chunk
            int before = pre[chunk];
            for (int i = 0; i < first / 32; ++i) before += __popc(bb[i]);
            const uint32_t word = bb[first / 32];
            const int sh = first % 32;
            before += __popc(word & ((1u << sh) - 1u));
            const uint32_t m16 = (word >> sh) & 0xFFFFu;
            if (MODE == 0) {
                const int hl = lane >> 4, cl = lane & 15;
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int i = 2 * u + hl;
                    if ((m16 >> i) & 1u) {
                        const int64_t d = before + __popc(m16 & ((1u << i) - 1u));
                        const int lr = cw * 16 + i;
                        ok[d * RV + cl] = st[lr * RV + cl];
                        ov[d * RV + cl] = st[SR * RV + lr * RV + cl];
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            } else {
                // lane i < 16 owns row i; a row starting a run issues the run's copies
                if (lane < 16) {
                    const bool kept = (m16 >> lane) & 1u;
                    const bool start = kept && (lane == 0 || !((m16 >> (lane - 1)) & 1u));
                    if (start) {
                        int len = 1;
                        while (lane + len < 16 && ((m16 >> (lane + len)) & 1u)) ++len;
                        const int64_t d = before + __popc(m16 & ((1u << lane) - 1u));
                        const int lr = cw * 16 + lane;
                        bulk_s2g(ok + d * RV, st + lr * RV, uint32_t(len) * 256);
                        bulk_s2g(ov + d * RV, st + SR * RV + lr * RV, uint32_t(len) * 256);
                        bulk_commit();
                        bulk_wait_read0();
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (++s == nst) {
                s = 0;
                ph ^= 1;
            }
        }
        if (MODE == 1) bulk_wait0();
    }
}

__global__ void fill(uint4* x, int64_t R, uint32_t salt) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < R * RV; i += int64_t(gridDim.x) * blockDim.x)
        x[i] = make_uint4(uint32_t(i / RV), uint32_t(i % RV), salt, uint32_t(i) ^ salt);
}

int main(int argc, char** argv) {
    const int64_t R = argc > 1 ? atoll(argv[1]) : 28LL * 8 * 10240;  // cfg2 rows per step
    const double keep_frac = 0.8;
    const int nchunks = int(R / CH);
    std::vector<uint8_t> keep(R);
    std::vector<int> pre(nchunks);
    std::mt19937_64 g(1);
    std::bernoulli_distribution bd(keep_frac);
    int64_t kept = 0;
    for (int c = 0; c < nchunks; ++c) {
        pre[c] = int(kept);
        for (int i = 0; i < CH; ++i) {
            keep[c * CH + i] = bd(g);
            kept += keep[c * CH + i];
        }
    }
    uint4 *ik, *iv, *ok, *ov;
    uint8_t* dk;
    int* dp;
    CK(cudaMalloc(&ik, R * 256));
    CK(cudaMalloc(&iv, R * 256));
    CK(cudaMalloc(&ok, R * 256));
    CK(cudaMalloc(&ov, R * 256));
    CK(cudaMalloc(&dk, R));
    CK(cudaMalloc(&dp, nchunks * 4));
    fill<<<1024, 256>>>(ik, R, 1);
    fill<<<1024, 256>>>(iv, R, 2);
    CK(cudaMemcpy(dk, keep.data(), R, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dp, pre.data(), nchunks * 4, cudaMemcpyHostToDevice));
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const double bytes = double(kept) * 256 * 2 * 2;
    printf("rows %lld kept %lld bytes/launch %.3f GB sms %d\n", (long long)R, (long long)kept, bytes / 1e9, nsm);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    // reference: the product's launch shape (4 warps per CTA, one chunk per warp)
    auto timeit = [&](auto launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            CK(cudaEventRecord(a));
            launch();
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        return best;
    };
    {
        float ms = timeit([&] { lsu_gather<<<(nchunks + 3) / 4, 128>>>(ik, iv, dk, dp, ok, ov, nchunks); });
        printf("lsu   full-grid (128 thr CTAs)        %.4f ms  %.0f GB/s\n", ms, bytes / ms / 1e6);
    }
    const int nst = 6;
    const int smem = 1024 + nst * 2 * SR * 256;
    CK(cudaFuncSetAttribute(tma_gather<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(tma_gather<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    int Ss[] = {8, 16, 24, 32, 40, 48, 64, 96, 148};
    for (int S : Ss) {
        if (S > nsm) continue;
        float m1 = timeit([&] { lsu_gather<<<S, 512>>>(ik, iv, dk, dp, ok, ov, nchunks); });
        float m1b = timeit([&] { lsu_gather<<<2 * S, 512>>>(ik, iv, dk, dp, ok, ov, nchunks); });
        float m2 = timeit([&] { tma_gather<0><<<S, 160, smem>>>(ik, iv, dk, dp, ok, ov, nchunks, nst); });
        float m3 = timeit([&] { tma_gather<1><<<S, 160, smem>>>(ik, iv, dk, dp, ok, ov, nchunks, nst); });
        printf("S=%3d  lsu(1x512) %6.0f GB/s (%5.1f/SM)  lsu(2x512) %6.0f (%5.1f/SM)  tma+stg %6.0f (%5.1f/SM)  "
               "tma+bulk %6.0f (%5.1f/SM)\n",
               S, bytes / m1 / 1e6, bytes / m1 / 1e6 / S, bytes / m1b / 1e6, bytes / m1b / 1e6 / S,
               bytes / m2 / 1e6, bytes / m2 / 1e6 / S, bytes / m3 / 1e6, bytes / m3 / 1e6 / S);
    }
    // check: tma+stg output equals lsu output
    std::vector<uint4> h1(kept * RV), h2(kept * RV);
    CK(cudaMemset(ok, 0, R * 256));
    lsu_gather<<<148, 512>>>(ik, iv, dk, dp, ok, ov, nchunks);
    CK(cudaMemcpy(h1.data(), ok, kept * 256, cudaMemcpyDeviceToHost));
    CK(cudaMemset(ok, 0, R * 256));
    tma_gather<1><<<148, 160, smem>>>(ik, iv, dk, dp, ok, ov, nchunks, nst);
    CK(cudaMemcpy(h2.data(), ok, kept * 256, cudaMemcpyDeviceToHost));
    printf("bulk == lsu: %s\n", memcmp(h1.data(), h2.data(), kept * 256) == 0 ? "yes" : "NO");
    return 0;
}
