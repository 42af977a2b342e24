// TMEM read bandwidth of tcgen05.ld.32x32b.x32 per SM: W warps (W/4 per sub-partition), each loops
// NIT times over 4 back-to-back x32 loads (16 KB per warp per iteration) + wait::ld.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define R8(a, i) "=r"(a[i]), "=r"(a[i + 1]), "=r"(a[i + 2]), "=r"(a[i + 3]), "=r"(a[i + 4]), "=r"(a[i + 5]), "=r"(a[i + 6]), "=r"(a[i + 7])
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : R8(r, 0), R8(r, 8), R8(r, 16), R8(r, 24) : "r"(taddr));
}
template <int NIT>
__global__ void k(long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int w = threadIdx.x >> 5;
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot + (uint32_t((w & 3) * 32) << 16) + (w >> 2) * 128;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < NIT; ++it) {
    uint32_t a[32], b[32], c[32], d[32];
    ld32(t, a); ld32(t + 32, b); ld32(t + 64, c); ld32(t + 96, d);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    acc += __uint_as_float(a[it & 31]) + __uint_as_float(b[3]) + __uint_as_float(c[7]) + __uint_as_float(d[9]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
  sink[threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}
int main() {
  long long* d; float* s;
  cudaMalloc(&d, 64); cudaMalloc(&s, 4096 * 4);
  for (int W : {1, 4, 8, 12, 16}) {
    k<256><<<1, 32 * W>>>(d, s); k<256><<<1, 32 * W>>>(d, s);
    cudaError_t e = cudaDeviceSynchronize();
    if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double bytes = 256.0 * W * 16384;
    printf("warps %2d: %lld cycles, %.1f B/clk per SM, %.0f cycles per 16 KB warp-load\n", W, h, bytes / h, double(h) / 256);
  }
  return 0;
}
