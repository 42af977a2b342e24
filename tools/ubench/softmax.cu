// Microbenchmark: per-warp throughput of the softmax inner loop (64 column pairs per row) with
// one warp per SM sub-partition, from registers (no TMEM).  Variants drop parts of the mix.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk2(float lo, float hi) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }

template <int V>
__global__ void k(float* out, uint32_t* outp, int iters, long long* cyc) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = (threadIdx.x + i) * 1e-3f;
  const uint64_t sc2 = pk2(1.44f, 1.44f);
  uint64_t nm2 = pk2(-0.5f, -0.5f);
  float tot = 0.f; uint32_t px = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
    float m0 = -1e30f, m1 = -1e30f;
    uint32_t pk[64];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
      float s0 = s[2 * i], s1 = s[2 * i + 1];
      if (V != 3) { if (i & 1) m1 = fmax3(m1, s0, s1); else m0 = fmax3(m0, s0, s1); }
      const uint64_t x = fma2(pk2(s0, s1), sc2, nm2);
      float x0, x1; up2(x, x0, x1);
      float p0 = ex2(x0), p1 = ex2(x1);
      if (V != 1) { if (i & 1) acc1 = add2(acc1, pk2(p0, p1)); else acc0 = add2(acc0, pk2(p0, p1)); }
      if (V != 2) pk[i] = pack(p0, p1); else pk[i] = __float_as_uint(p0);
    }
    float a, b, c, d; up2(acc0, a, b); up2(acc1, c, d);
    tot += a + b + c + d + m0 + m1;
#pragma unroll
    for (int i = 0; i < 64; ++i) px ^= pk[i];
    nm2 = pk2(-0.5f + tot * 1e-30f, -0.5f);  // loop-carried dependency
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot;
  outp[blockIdx.x * blockDim.x + threadIdx.x] = px;
}
int main() {
  float* out; uint32_t* op; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&op, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 256;
  const char* names[] = {"full mix", "no row sum", "no bf16 pack", "no max"};
  for (int v = 0; v < 4; ++v)
    for (int threads : {128, 256}) {
      auto kern = v == 0 ? k<0> : v == 1 ? k<1> : v == 2 ? k<2> : k<3>;
      kern<<<148, threads>>>(out, op, iters, cyc);
      cudaDeviceSynchronize();
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("%-14s warps/SMSP %d: %.0f clk per 128-col row-tile per warp (MUFU floor 1024 x warps/SMSP)\n", names[v], threads / 128, double(h) / iters);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
