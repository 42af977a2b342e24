// Issue cost of tcgen05.mma from one thread: time to issue NMMA back-to-back MMAs (no stamps in
// between) for N = 256 / 128 / 64 / 32 (pipe time 128 / 64 / 32 / 16 cycles per 128xNx16 MMA),
// and the time until all complete.  If issuing is slower than the pipe, small-N MMAs show it.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_issue mma_issue.cu
#include <cstdio>
#include <cstdlib>
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
template <int N, int NMMA, int NW = 1>
__global__ void k(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar_[4];
  uint64_t& bar = bar_[0];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = 0x3c003c00u;
  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  const int iw = (w == 0) ? 0 : (w >= 2 ? w - 1 : -1);  // issuing warps: 0, 2, 3 (warp 1 owns TMEM)
  if (iw >= 0 && iw < NW && lane == 0) {
    uint64_t a[4], b[4];
    for (int i = 0; i < 4; ++i) { a[i] = sdesc(smem_u32(sm) + i * 32); b[i] = sdesc(smem_u32(sm + 32768) + i * 32); }
    long long t0 = clock64();
#pragma unroll
    for (int i = 0; i < NMMA; ++i)
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + iw * N),
                   "l"(a[i & 3]), "l"(b[i & 3]), "r"(idesc), "r"(i));
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar + iw)));
    asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(smem_u32(&bar + iw)));
    long long t2 = clock64();
    if (iw == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
template <int N, int NMMA, int NW = 1>
void run() {
  long long* d; cudaMalloc(&d, 64);
  cudaFuncSetAttribute(k<N, NMMA, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<N, NMMA, NW><<<1, 128, 65536>>>(d); k<N, NMMA, NW><<<1, 128, 65536>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("NW=%d N=%3d NMMA=%3d: issue %6lld cyc (%.1f/MMA), complete %6lld cyc (%.1f/MMA), pipe model %d/MMA\n", NW, N, NMMA,
         h[0], double(h[0]) / NMMA, h[1], double(h[1]) / NMMA, N / 2);
  cudaFree(d);
}
int main() {
  run<64, 64>(); run<64, 64, 2>(); run<64, 64, 3>(); run<32, 64>(); run<32, 64, 2>(); run<32, 64, 3>(); run<128, 64>(); run<128, 64, 2>();
  return 0;
}
