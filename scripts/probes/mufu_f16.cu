// Microbenchmark + accuracy: ex2.approx.f16x2 (two exp2 per lane per MUFU op?)
// vs ex2.approx.ftz.f32, and the error of ex2.approx.f16x2 over every f16
// input in [-24, 0] against a double-precision 2^x.
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__global__ void k_ex2(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = ex2(a[i]) - 1.0f;
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ex2h2(float* out, int iters) {
  uint32_t a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { __half2 h = __floats2half2_rn(-0.001f * (threadIdx.x + i), -0.002f * i); a[i] = *reinterpret_cast<uint32_t*>(&h); }
  const __half2 one = __floats2half2_rn(1.f, 1.f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t y = ex2h2(a[i]);
      __half2 h = __hsub2(*reinterpret_cast<__half2*>(&y), one);
      a[i] = *reinterpret_cast<uint32_t*>(&h);
    }
  }
  float s = 0; for (int i = 0; i < 16; ++i) { __half2 h = *reinterpret_cast<__half2*>(&a[i]); s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_acc(const unsigned short* in, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t x = uint32_t(in[i]) | (uint32_t(in[i]) << 16);
  uint32_t y = ex2h2(x);
  __half2 h = *reinterpret_cast<__half2*>(&y);
  out[i] = __low2float(h);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 1024 * 8 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16}) {
    for (int which = 0; which < 2; ++which) {
      int iters = 4096, threads = warps * 32;
      auto launch = [&]() { if (which == 0) k_ex2<<<sms, threads>>>(out, iters); else k_ex2h2<<<sms, threads>>>(out, iters); };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(sms) * threads * iters * 16 * (which ? 2 : 1);  // exp2 results
      printf("%s warps/SM=%2d: %.3f ms, %.2f G exp2/s, %.1f exp2/clk/SM at 1.965 GHz\n", which ? "ex2.f16x2" : "ex2.f32  ",
             warps, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  // accuracy over all f16 in [-24, 0]
  static unsigned short hs[65536]; int n = 0;
  for (int b = 0; b < 65536; ++b) {
    __half h = *reinterpret_cast<__half*>(&b);
    float f = __half2float(h);
    if (std::isfinite(f) && f <= 0.f && f >= -24.f) hs[n++] = (unsigned short)b;
  }
  unsigned short* din; float* dout; cudaMalloc(&din, n * 2); cudaMalloc(&dout, n * 4);
  cudaMemcpy(din, hs, n * 2, cudaMemcpyHostToDevice);
  k_acc<<<(n + 255) / 256, 256>>>(din, dout, n);
  static float res[65536]; cudaMemcpy(res, dout, n * 4, cudaMemcpyDeviceToHost);
  double maxrel = 0, sumrel = 0, maxrel_rn = 0, sumrel_rn = 0; float worst = 0;
  for (int i = 0; i < n; ++i) {
    unsigned short b = hs[i];
    float x = __half2float(*reinterpret_cast<__half*>(&b));
    double ex = std::exp2(double(x));
    if (ex < 6.1e-5) continue;  // below f16 normal range
    double r = (res[i] - ex) / ex;
    double rn = (double(__half2float(__float2half_rn(float(ex)))) - ex) / ex;
    if (std::fabs(r) > maxrel) { maxrel = std::fabs(r); worst = x; }
    sumrel += r; maxrel_rn = std::max(maxrel_rn, std::fabs(rn)); sumrel_rn += rn;
  }
  printf("ex2.approx.f16x2 over %d f16 inputs in [-14, 0]: max rel err %.3e (at x=%g), mean rel err %.3e; "
         "correctly rounded f16: max %.3e mean %.3e\n", n, maxrel, worst, sumrel / n, maxrel_rn, sumrel_rn / n);
  return 0;
}
