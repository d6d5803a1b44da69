// Microbenchmark: MUFU.EX2 and FFMA throughput per SM on this GPU (calibrates
// the SFU bound of the P1 row-statistics pass).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
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
__global__ void k_ffma(float* out, int iters) {
  float a[16];
  #pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], 0.999f, 0.0001f);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sms * 1024 * 8 * sizeof(float));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    for (int which = 0; which < 2; ++which) {
      int iters = 4096, threads = warps * 32;
      auto launch = [&]() { if (which == 0) k_ex2<<<sms, threads>>>(out, iters); else k_ffma<<<sms, threads>>>(out, iters); };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops = double(sms) * threads * iters * 16;
      printf("%s warps/SM=%2d: %.3f ms, %.2f Gop/s, %.1f op/clk/SM at 1.965 GHz\n", which ? "ffma" : "ex2 ",
             warps, ms, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
    }
  }
  return 0;
}
