// Microbenchmark of the P1 row-statistics inner loop alone (registers only,
// no TMEM): elements/clk/SM for the SFU-only form and for forms that move a
// share of the exp2 onto the FMA pipe (polynomial), plus FFMA2 throughput.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2509_17396_b200/csrc/sm100.cuh"
using namespace epk::sm100;

// degree-3 minimax-ish 2^f on [-0.5, 0.5] (FA4-style), exponent add
__device__ __forceinline__ uint64_t exp2_poly3(uint64_t t) {
    const uint64_t magic = f2_pack(12582912.f, 12582912.f);
    const uint64_t r = fadd2(t, magic);
    const uint64_t j = fadd2(r, f2_pack(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(j, f2_pack(-1.f, -1.f), t);
    uint64_t p = ffma2(f2_pack(0x1.c6b348p-5f, 0x1.c6b348p-5f), f, f2_pack(0x1.ebfbe0p-3f, 0x1.ebfbe0p-3f));
    p = ffma2(p, f, f2_pack(0x1.62e430p-1f, 0x1.62e430p-1f));
    p = ffma2(p, f, f2_pack(1.f, 1.f));
    float p0, p1, r0, r1;
    f2_unpack(p, p0, p1);
    f2_unpack(r, r0, r1);
    return f2_pack(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(r0) << 23)),
                   __uint_as_float(__float_as_uint(p1) + (__float_as_uint(r1) << 23)));
}

template <int MODE>  // 0: all SFU; 1: 1/4 poly5; 2: 1/4 poly3; 3: 1/2 poly3; 4: 3/8 poly3
__global__ void k_mix(float* out, int iters, float c2) {
    float v[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = -0.01f * ((threadIdx.x + i * 7) & 127);
    uint64_t acc0 = f2_pack(0.f, 0.f), acc1 = acc0;
    const uint64_t c2x2 = f2_pack(c2, c2);
    for (int it = 0; it < iters; ++it) {
        float a0_, a1_;
        f2_unpack(acc0, a0_, a1_);
        const float sh = -float(it & 7) - 1e-30f * a0_;  // depends on the running sum: no hoisting
        const uint64_t nm2 = f2_pack(sh, sh);
#pragma unroll
        for (int i = 0; i < 64; i += 4) {
            const uint64_t t0 = ffma2(f2_pack(v[i], v[i + 1]), c2x2, nm2);
            const uint64_t t1 = ffma2(f2_pack(v[i + 2], v[i + 3]), c2x2, nm2);
            uint64_t e[2];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const uint64_t t = q ? t1 : t0;
                const int pr = (i / 2 + q) & 7;  // pair index mod 8
                bool poly = MODE == 1 ? (pr & 3) == 3 : MODE == 2 ? (pr & 3) == 3 : MODE == 3 ? (pr & 1) : MODE == 4 ? (pr % 8 == 1 || pr % 8 == 4 || pr % 8 == 6) : false;
                if (poly) {
                    e[q] = MODE == 1 ? exp2_poly2(t) : exp2_poly3(t);
                } else {
                    float a, b;
                    f2_unpack(t, a, b);
                    e[q] = f2_pack(ex2(a), ex2(b));
                }
            }
            acc0 = fadd2(acc0, e[0]);
            acc1 = fadd2(acc1, e[1]);
        }
    }
    float a0, a1, b0, b1;
    f2_unpack(acc0, a0, a1);
    f2_unpack(acc1, b0, b1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + b0 + b1;
}

__global__ void k_ffma2(float* out, int iters) {
    uint64_t a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = f2_pack(0.001f * (threadIdx.x + i), 0.002f * i);
    const uint64_t m = f2_pack(0.999f, 0.998f), c = f2_pack(1e-4f, 2e-4f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 16; ++i) a[i] = ffma2(a[i], m, c);
    float s = 0;
    for (int i = 0; i < 16; ++i) { float x, y; f2_unpack(a[i], x, y); s += x + y; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
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
    for (int warps : {8, 12, 16}) {
        const int th = warps * 32, iters = 2048;
        const double el = double(sms) * th * iters * 64;
        float ms[5];
        ms[0] = timeit([&] { k_mix<0><<<sms, th>>>(out, iters, 0.1f); });
        ms[1] = timeit([&] { k_mix<1><<<sms, th>>>(out, iters, 0.1f); });
        ms[2] = timeit([&] { k_mix<2><<<sms, th>>>(out, iters, 0.1f); });
        ms[3] = timeit([&] { k_mix<3><<<sms, th>>>(out, iters, 0.1f); });
        ms[4] = timeit([&] { k_mix<4><<<sms, th>>>(out, iters, 0.1f); });
        const char* nm[5] = {"sfu only", "1/4 poly5", "1/4 poly3", "1/2 poly3", "3/8 poly3"};
        for (int m = 0; m < 5; ++m)
            printf("warps/SM=%2d %-10s: %.3f ms, %.2f elem/clk/SM at 1.965 GHz\n", warps, nm[m], ms[m],
                   el / (ms[m] * 1e-3) / sms / 1.965e9);
        const float f = timeit([&] { k_ffma2<<<sms, th>>>(out, iters * 8); });
        printf("warps/SM=%2d ffma2     : %.2f FFMA2 lane-ops/clk/SM (x2 flops each)\n", warps,
               double(sms) * th * iters * 8 * 16 / (f * 1e-3) / sms / 1.965e9);
    }
    return 0;
}
