// Per-tile softmax time for a 128-row x 128-key tile on ONE SM sub-partition set, from registers:
// COLS columns per warp (128: one warp per row group; 64: two column-split warps per row group),
// EMU of every 8 column pairs through the FMA-pipe polynomial exp2.  Reports cycles per tile.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint64_t pk2(float lo, float hi) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) { uint64_t d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) { uint64_t d; asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t pack(float lo, float hi) { uint32_t r; asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo)); return r; }
__device__ __forceinline__ float fmax3(float a, float b, float c) { float d; asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1; up2(x2, x0, x1);
  x0 = fmaxf(x0, -125.f); x1 = fmaxf(x1, -125.f);
  const uint64_t xc = pk2(x0, x1);
  const uint64_t magic = pk2(12582912.f, 12582912.f), nmagic = pk2(-12582912.f, -12582912.f);
  const uint64_t t = add2(xc, magic), j = add2(t, nmagic), f = fma2(j, pk2(-1.f, -1.f), xc);
  uint64_t pp = fma2(f, pk2(0.0095828f, 0.0095828f), pk2(0.0559064f, 0.0559064f));
  pp = fma2(f, pp, pk2(0.240241f, 0.240241f)); pp = fma2(f, pp, pk2(0.693124f, 0.693124f)); pp = fma2(f, pp, pk2(1.f, 1.f));
  float p0, p1, t0, t1; up2(pp, p0, p1); up2(t, t0, t1);
  return pk2(__int_as_float(__float_as_int(t0) * (1 << 23) + __float_as_int(p0)), __int_as_float(__float_as_int(t1) * (1 << 23) + __float_as_int(p1)));
}
template <int COLS, int EMU>
__global__ void k(float* out, uint32_t* outp, int iters, long long* cyc) {
  float s[COLS];
#pragma unroll
  for (int i = 0; i < COLS; ++i) s[i] = (threadIdx.x + i) * 1e-3f;
  const uint64_t sc2 = pk2(1.44f, 1.44f);
  uint64_t nm2 = pk2(-0.5f, -0.5f);
  float tot = 0.f; uint32_t px = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
    float m0 = -1e30f, m1 = -1e30f;
#pragma unroll
    for (int i = 0; i < COLS / 2; ++i) {
      float s0 = s[2 * i], s1 = s[2 * i + 1];
      if (i & 1) m1 = fmax3(m1, s0, s1); else m0 = fmax3(m0, s0, s1);
      const uint64_t x = fma2(pk2(s0, s1), sc2, nm2);
      float p0, p1;
      if ((i & 7) < EMU) { up2(exp2_poly2(x), p0, p1); } else { float x0, x1; up2(x, x0, x1); p0 = ex2(x0); p1 = ex2(x1); }
      if (i & 1) acc1 = add2(acc1, pk2(p0, p1)); else acc0 = add2(acc0, pk2(p0, p1));
      px ^= pack(p0, p1);
    }
    float a, b, c, d; up2(acc0, a, b); up2(acc1, c, d);
    tot += a + b + c + d + m0 + m1;
    nm2 = pk2(-0.5f + tot * 1e-30f, -0.5f);
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot; outp[blockIdx.x * blockDim.x + threadIdx.x] = px;
}
template <int COLS, int EMU> void run(float* out, uint32_t* op, long long* cyc) {
  const int iters = 256, threads = 128 * (128 / COLS);  // one 128x128 tile per block per iter
  k<COLS, EMU><<<148, threads>>>(out, op, iters, cyc); cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("cols/warp %3d warps/SMSP %d EMU %d: %6.0f clk per 128x128 tile\n", COLS, 128 / COLS, EMU, double(h) / iters);
}
int main() {
  float* out; uint32_t* op; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&op, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  run<128, 0>(out, op, cyc); run<128, 2>(out, op, cyc); run<128, 3>(out, op, cyc); run<128, 4>(out, op, cyc);
  run<64, 0>(out, op, cyc); run<64, 2>(out, op, cyc); run<64, 3>(out, op, cyc); run<64, 4>(out, op, cyc);
  run<32, 0>(out, op, cyc); run<32, 3>(out, op, cyc);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
