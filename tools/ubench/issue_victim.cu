// Does the tcgen05.mma issuer (or a warp spinning on an mbarrier) steal MUFU / issue throughput
// from the softmax warps of its SM sub-partition?  Warp 0 (SMSP 0) runs MODE:
//   0: idle                 1: back-to-back SS MMAs 128x64x16 (issue-bound, 32 pipe cycles each)
//   2: SS MMAs 128x128x16   3: spin on an mbarrier that never completes (try_wait loop)
//   4: same spin with a suspend-time hint
// Victims: warps 4, 8 (SMSP 0, with the issuer) and warps 1, 5 (SMSP 1, control) each run a
// softmax-like throughput loop: per element pair FFMA2, 2x MUFU.EX2, F2FP pack, FADD2.
// Reported: victim elements per clock per SMSP.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o issue_victim issue_victim.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
  uint64_t d = 0;
  d |= uint64_t((a & 0x3FFFFu) >> 4);
  d |= uint64_t(16 >> 4) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) { asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v)); }
__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
constexpr int NIT = 256;
template <int MODE>
__global__ void k(long long* out, float* sink, int n_mma) {
  __shared__ __align__(1024) uint8_t sm[40960];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (w == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(sm + 40000);
  if (w == 0) {
    if (MODE == 1 || MODE == 2) {
      if (lane == 0) {
        const uint32_t N = MODE == 1 ? 64 : 128;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
        for (int i = 0; i < n_mma; ++i) {
          uint64_t a = sdesc(smem_u32(sm) + (i & 3) * 32), b = sdesc(smem_u32(sm + 16384) + (i & 3) * 32);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                       "l"(a), "l"(b), "r"(idesc), "r"(i & 7));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[0])));
        asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar[0])));
      }
    } else if (MODE == 3 || MODE == 4) {
      // spin until the victims are done (they set *stop); bar[1] never completes
      while (*stop == 0) {
        if (MODE == 3)
          asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t}" ::"r"(smem_u32(&bar[1])));
        else
          asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0, %1;\n\t}" ::"r"(smem_u32(&bar[1])), "r"(20000u));
      }
    }
  } else if (w == 4 || w == 8 || w == 1 || w == 5) {
    float x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) x[i] = -0.001f * (i + lane);
    const uint64_t sc = pk2(1.0001f, 1.0001f), nm = pk2(-0.01f, -0.01f);
    uint64_t acc = pk2(0.f, 0.f);
    uint32_t pk = 0;
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
        x[2 * i] = y0 * 0.5f;  // keep the inputs changing
      }
    }
    long long t1 = clock64();
    float a0, a1;
    up2(acc, a0, a1);
    sink[threadIdx.x] = a0 + a1 + __uint_as_float(pk);
    if (lane == 0) out[w] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x == 128) *stop = 1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
int main() {
  long long* d; float* s;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&s, 4096 * 4);
  const char* names[] = {"idle", "SS MMA N=64 stream", "SS MMA N=128 stream", "mbarrier spin", "mbarrier spin+hint"};
  for (int mode = 0; mode < 5; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(d, 0, 64 * 8);
      const int n_mma = 3000;
      switch (mode) {
        case 0: k<0><<<1, 384>>>(d, s, n_mma); break;
        case 1: k<1><<<1, 384>>>(d, s, n_mma); break;
        case 2: k<2><<<1, 384>>>(d, s, n_mma); break;
        case 3: k<3><<<1, 384>>>(d, s, n_mma); break;
        case 4: k<4><<<1, 384>>>(d, s, n_mma); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[64]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      if (rep == 1) {
        const double el = 32.0 * 32 * NIT;  // elements per victim warp
        printf("%-22s SMSP0 victims (w4, w8): %.2f %.2f elem/clk   SMSP1 control (w1, w5): %.2f %.2f elem/clk\n",
               names[mode], el / h[4], el / h[8], el / h[1], el / h[5]);
      }
    }
  }
  return 0;
}
