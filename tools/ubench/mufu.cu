// Microbenchmark: MUFU ex2 throughput per SM for f32, f16x2, bf16x2 (results per clock per SM).
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cstdint>
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  uint32_t h0 = 0x3c003c00u ^ threadIdx.x, h1 = h0 + 1, h2 = h0 + 2, h3 = h0 + 3;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a3));
    } else if (MODE == 1) {
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h3));
    } else {
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h2)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h3));
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + __uint_as_float(h0 ^ h1 ^ h2 ^ h3);
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int threads : {128, 256, 512, 1024}) {
      auto kern = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      kern<<<148, threads>>>(out, iters, cyc);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      double ops = double(threads) * iters * 4 * (mode ? 2 : 1);  // exps per SM
      printf("mode %s threads %4d: %.2f exps/clk/SM (%.2f instr-lanes/clk)\n", mode == 0 ? "f32   " : mode == 1 ? "f16x2 " : "bf16x2",
             threads, ops / h, double(threads) * iters * 4 / h);
    }
  }
  cudaError_t e = cudaGetLastError(); printf("%s\n", cudaGetErrorString(e));
}
