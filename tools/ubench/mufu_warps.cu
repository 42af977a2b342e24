// MUFU throughput of the softmax instruction mix (per element pair: FFMA2, 2x MUFU.EX2, FADD2, F2FP
// pack) with 1, 2, 3 or 4 warps per SM sub-partition: can ONE warp keep MUFU busy while its partner
// is in a non-exp phase?   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_warps mufu_warps.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t pk2(float lo, float hi) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
constexpr int NIT = 512;
__global__ void k(long long* out, float* sink) {
  const int lane = threadIdx.x & 31;
  float x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = -0.001f * (i + lane);
  const uint64_t sc = pk2(1.0001f, 1.0001f), nm = pk2(-0.01f, -0.01f);
  uint64_t acc = pk2(0.f, 0.f);
  uint32_t pk = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < NIT; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const uint64_t y = fma2(pk2(x[2 * i], x[2 * i + 1]), sc, nm);
      float y0, y1;
      up2(y, y0, y1);
      const float p0 = ex2(y0), p1 = ex2(y1);
      acc = add2(acc, pk2(p0, p1));
      uint32_t b;
      asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(b) : "f"(p1), "f"(p0));
      pk ^= b;
      x[2 * i] = y0 * 0.5f;
    }
  }
  long long t1 = clock64();
  float a0, a1;
  up2(acc, a0, a1);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + __uint_as_float(pk);
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main() {
  long long* d; float* s;
  cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 148 * 1024 * 4);
  for (int wps = 1; wps <= 4; ++wps) {
    const int threads = 128 * wps;  // wps warps per SM sub-partition
    k<<<148, threads>>>(d, s);
    k<<<148, threads>>>(d, s);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double exps = double(threads) * NIT * 32;  // per SM
    printf("%d warp(s) per SMSP: %.2f exp2/clk/SM (MUFU peak 16)\n", wps, exps / h);
  }
  return 0;
}
