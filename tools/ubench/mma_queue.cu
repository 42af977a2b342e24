// How deep is the tcgen05.mma issue queue, and does an issuer blocked on a full queue stall the
// other warps of its SM sub-partition?  Warp 0 (one lane) issues NMMA back-to-back 128x128x16 SS
// MMAs (64 pipe cycles each) and stamps clock64 after each issue; warp 4 (same sub-partition) runs
// a dependent FFMA chain and stamps every 64 iterations; warp 1 (another sub-partition) does the
// same as a control.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_queue mma_queue.cu
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
constexpr int NMMA = 48, NV = 64;
__global__ void k(long long* out, float* sink) {
  __shared__ __align__(1024) uint8_t sm[40960];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (w == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(128 >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  if (w == 0) {
    if (lane == 0) {
      long long t0 = clock64();
      for (int i = 0; i < NMMA; ++i) {
        uint64_t a = sdesc(smem_u32(sm) + (i & 3) * 32), b = sdesc(smem_u32(sm + 16384) + (i & 3) * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                     "l"(a), "l"(b), "r"(idesc), "r"(i));
        out[i] = clock64() - t0;
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
      asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar)));
      out[NMMA] = clock64() - t0;
    }
  } else if (w == 4 || w == 1) {
    float x = 1.0f + lane;
    long long t0 = clock64();
    const uint32_t taddr = tmem + (uint32_t((w & 3) * 32) << 16) + 64;
    for (int i = 0; i < NV; ++i) {
#if VICTIM_LDTM
      uint32_t r[32];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                     "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int q = 0; q < 32; ++q) x += __uint_as_float(r[q]);
#else
#pragma unroll
      for (int r = 0; r < 64; ++r) x = fmaf(x, 1.0000001f, 0.5f);
#endif
      if (lane == 0) out[64 + (w == 4 ? 0 : NV) + i] = clock64() - t0;
    }
    sink[threadIdx.x] = x;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
int main() {
  long long* d; float* s;
  cudaMalloc(&d, 512 * 8); cudaMalloc(&s, 4096);
  cudaMemset(d, 0, 512 * 8);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 256>>>(d, s);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  long long h[512]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("issue-done clock per MMA:"); for (int i = 0; i < NMMA; ++i) printf(" %lld", h[i]); printf("\nall complete: %lld\n", h[NMMA]);
  printf("victim (same SMSP) per iter:"); for (int i = 0; i < NV; ++i) printf(" %lld", i ? h[64 + i] - h[63 + i] : h[64]); printf("\n");
  printf("control (other SMSP) per iter:"); for (int i = 0; i < NV; ++i) printf(" %lld", i ? h[64 + NV + i] - h[63 + NV + i] : h[64 + NV]); printf("\n");
  return 0;
}
