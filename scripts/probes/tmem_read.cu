// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM, for the
// 32x32b shape at x32 / x64 / x128 columns, with 4..16 warps per CTA (one CTA
// per SM, 512 TMEM columns).  Bounds the scorer epilogues, which read every
// fp32 logit of the S tile from TMEM once per pass.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2509_17396_b200/csrc/sm100.cuh"
using namespace epk::sm100;

template <int X>
__device__ __forceinline__ float ld_sum(uint32_t addr);
template <>
__device__ __forceinline__ float ld_sum<32>(uint32_t addr) {
    float v[32];
    tmem_ld32(addr, v);
    return v[0] + v[31];  // the asm is volatile: every column is loaded regardless
}
template <>
__device__ __forceinline__ float ld_sum<64>(uint32_t addr) {
    float v[64];
    tmem_ld64(addr, v);
    return v[0] + v[63];
}
template <>
__device__ __forceinline__ float ld_sum<128>(uint32_t addr) {
    float v[128];
    tmem_ld128(addr, v);
    return v[0] + v[127];
}

template <int X>
__global__ void __launch_bounds__(X == 128 ? 384 : 512, 1) k_tmem(float* out, long long* cyc, int iters) {
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&holder, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    float acc = 0.f;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = uint32_t((it * X + (warp >> 2) * 128) & 511);
        acc += ld_sum<X>(tmem + lane_addr + col);
    }
    const long long c1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, sms * 512 * sizeof(float));
    long long* cyc; cudaMalloc(&cyc, sms * sizeof(long long));
    long long hc[1024];
    for (int x : {32, 64, 128})
        for (int warps : {1, 2, 4, 8, 12, 16}) {
            if (x == 128 && warps > 12) continue;
            const int iters = 4096 * 64 / x;
            auto launch = [&] {
                if (x == 32) k_tmem<32><<<sms, warps * 32>>>(out, cyc, iters);
                else if (x == 64) k_tmem<64><<<sms, warps * 32>>>(out, cyc, iters);
                else k_tmem<128><<<sms, warps * 32>>>(out, cyc, iters);
            };
            launch();
            cudaDeviceSynchronize();
            launch();
            cudaDeviceSynchronize();
            cudaMemcpy(hc, cyc, sms * sizeof(long long), cudaMemcpyDeviceToHost);
            double avg = 0;
            for (int i = 0; i < sms; ++i) avg += hc[i];
            avg /= sms;
            const double bytes = double(warps) * 32 * 4 * x * iters;  // per CTA
            printf("x%-3d warps=%2d: %.1f B/clk/SM (TMEM read), %.0f clk per warp-ld\n", x, warps, bytes / avg,
                   avg / iters);
        }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
