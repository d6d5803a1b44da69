// Microbenchmark: 2-input vs 3-input fp32 max (FMNMX / FMNMX3) throughput,
// and the P2 epilogue inner loop (FFMA2 + max per column pair, lse from smem).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2509_17396_b200/csrc/sm100.cuh"
using namespace epk::sm100;

template <int MODE>  // 0: fmaxf(fmaxf()) pairs (FMNMX3 expected), 1: single fmaxf chains, 2: P2-like loop
__global__ void k_max(float* out, int iters) {
    __shared__ float s_l[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_l[i] = -0.01f * i;
    __syncthreads();
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = 0.001f * ((threadIdx.x * 7 + i * 13) & 255);
    float b[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = -1e30f;
    const uint64_t c2x2 = f2_pack(1.0001f, 1.0001f);
    for (int it = 0; it < iters; ++it) {
        const float sh = 1e-7f * b[it & 7];
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 64; i += 2) b[(i / 2) & 7] = fmaxf(fmaxf(b[(i / 2) & 7], v[i] + sh), v[i + 1]);
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 64; ++i) b[i & 7] = fmaxf(b[i & 7], v[i] + sh);
        } else {
            const float* nl = s_l + (it & 3) * 64;
#pragma unroll
            for (int i = 0; i < 64; i += 4) {
                const float4 l4 = *reinterpret_cast<const float4*>(nl + i);
                float a0, a1, a2, a3;
                f2_unpack(ffma2(f2_pack(v[i], v[i + 1]), c2x2, f2_pack(l4.x + sh, l4.y)), a0, a1);
                f2_unpack(ffma2(f2_pack(v[i + 2], v[i + 3]), c2x2, f2_pack(l4.z, l4.w)), a2, a3);
                const int j = (i / 4) & 1;
                b[2 * j] = fmaxf(fmaxf(b[2 * j], a0), a1);
                b[2 * j + 1] = fmaxf(fmaxf(b[2 * j + 1], a2), a3);
            }
        }
    }
    float r = -1e30f;
    for (int j = 0; j < 8; ++j) r = fmaxf(r, b[j]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; cudaMalloc(&out, sms * 1024 * sizeof(float));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        launch(); cudaDeviceSynchronize();
        cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); return ms;
    };
    for (int warps : {2, 4, 8, 16}) {
        const int th = warps * 32, iters = 4096;
        const double el = double(sms) * th * iters * 64;
        const float m0 = timeit([&] { k_max<0><<<sms, th>>>(out, iters); });
        const float m1 = timeit([&] { k_max<1><<<sms, th>>>(out, iters); });
        const float m2 = timeit([&] { k_max<2><<<sms, th>>>(out, iters); });
        printf("warps/SM=%2d: max3 pairs %.1f col/clk/SM, max2 %.1f col/clk/SM, P2 loop %.1f col/clk/SM (at 1.965 GHz)\n",
               warps, el / (m0 * 1e-3) / sms / 1.965e9, el / (m1 * 1e-3) / sms / 1.965e9,
               el / (m2 * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
