// pipefusion.cu -- SURVEY §8(f) NEXT 3: PipeFusion's patch step on a synthetic DiT stack
// (§4.1.2; reading R4).
//
// One synthetic DiT block applied to one patch of the latent (stage-local work of a PipeFusion
// micro-step):
//   pf_prep_kernel     : q = h * wq into the workspace; the patch's FRESH k = h * wk, v = h * wv
//                        written into rows [off, off + n) of the block's KV buffer [2][B][H][S][D]
//                        (the other rows keep the stale K,V of the previous step -- "uses stale
//                        activations from the previous timestep to provide context");
//   attention          : the tcgen05 kernel (bf16) / SIMT kernel (fp32) of the USP path, queries = the
//                        patch, keys/values = the whole KV buffer (head-major strides, read by TMA);
//   pf_residual_kernel : h <- h + g * o (fp32 math, one rounding to h's dtype).
// pf_sampler_kernel: x <- x - sigma * eps (the synthetic sampler step of R4).
// Elementwise kernels are HBM-bound: 16-byte vectors, one thread per vector, grid-stride.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "xdit_internal.h"

namespace xdit {
namespace {

int pf_grid(int64_t n) {
  const int nsm = device_sm_count();
  const int64_t blocks = (n + 255) / 256;
  return int(blocks < int64_t(nsm) * 8 ? (blocks > 0 ? blocks : 1) : int64_t(nsm) * 8);
}

// 8 bf16 <-> 8 floats
__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const float2 t = __bfloat1622float2(b[k]);
    f[2 * k] = t.x;
    f[2 * k + 1] = t.y;
  }
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&f)[8]) {
  uint4 u;
  __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int k = 0; k < 4; ++k) b[k] = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
  *reinterpret_cast<uint4*>(p) = u;
}
__device__ __forceinline__ void ld8(const float* p, float (&f)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}
__device__ __forceinline__ void st8(float* p, const float (&f)[8]) {
  *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
  *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
}

// h [B][n][H][D] -> q [B][n][H][D]; K, V rows [off, off+n) of kv [2][B][H][S][D].  8 elements per thread.
template <typename T>
__global__ void pf_prep_kernel(const T* __restrict__ h, const float* __restrict__ w, T* __restrict__ q,
                               T* __restrict__ kv, int B, int n, int H, int S, int off, int D) {
  const int vd = D / 8;
  const int64_t total = int64_t(B) * n * H * vd;
  const int64_t half = int64_t(B) * H * S * D;
  const int HD = H * D;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int dv = int(i % vd);
    int64_t r = i / vd;
    const int hh = int(r % H);
    r /= H;
    const int t = int(r % n);
    const int b = int(r / n);
    const int64_t e = i * 8;  // element offset in h / q
    const int c = hh * D + dv * 8;  // channel in [H][D]
    float x[8], y[8];
    ld8(h + e, x);
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = x[k] * w[c + k];
    st8(q + e, y);
    const int64_t kvo = ((int64_t(b) * H + hh) * S + off + t) * D + dv * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = x[k] * w[HD + c + k];
    st8(kv + kvo, y);
#pragma unroll
    for (int k = 0; k < 8; ++k) y[k] = x[k] * w[2 * HD + c + k];
    st8(kv + half + kvo, y);
  }
}

// h <- h + g * o  (o [B][n][H][D]: fp32 from pf_block's attention, or h's dtype from the USP call)
template <typename T, typename O>
__global__ void pf_residual_kernel(T* __restrict__ h, const O* __restrict__ o, const float* __restrict__ g,
                                   int64_t n8, int HD) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const int c = int((i * 8) % HD);
    float x[8], a[8];
    ld8(h + i * 8, x);
    ld8(o + i * 8, a);
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(g[c + k], a[k], x[k]);
    st8(h + i * 8, x);
  }
}

// q, k, v <- h * wq, h * wk, h * wv  (all [B][n][H][D]; the hybrid's USP call does the KV placement)
template <typename T>
__global__ void pf_qkv_kernel(const T* __restrict__ h, const float* __restrict__ w, T* __restrict__ q,
                              T* __restrict__ k, T* __restrict__ v, int64_t n8, int HD) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const int c = int((i * 8) % HD);
    float x[8], y[8];
    ld8(h + i * 8, x);
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = x[e] * w[c + e];
    st8(q + i * 8, y);
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = x[e] * w[HD + c + e];
    st8(k + i * 8, y);
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = x[e] * w[2 * HD + c + e];
    st8(v + i * 8, y);
  }
}

// x <- x - sigma * eps
template <typename T>
__global__ void pf_sampler_kernel(T* __restrict__ x, const T* __restrict__ eps, int64_t n8, float sigma) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    float a[8], e[8];
    ld8(x + i * 8, a);
    ld8(eps + i * 8, e);
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fmaf(-sigma, e[k], a[k]);
    st8(x + i * 8, a);
  }
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

size_t pf_workspace_bytes(int B, int n, int H, int D, int dtype) {
  const size_t elems = size_t(B) * n * H * D;
  const size_t eb = dtype == 0 ? 2 : 4;
  return al256(elems * eb) + al256(elems * 4) + (dtype == 0 ? attn_scratch_floats(D) * sizeof(float) : 0);
}

cudaError_t launch_pf_block(void* h, void* kv, const float* w, void* work, int B, int H, int S, int off, int n,
                            int D, int dtype, cudaStream_t st) {
  if (B == 0 || n == 0) return cudaSuccess;
  const size_t elems = size_t(B) * n * H * D;
  const size_t eb = dtype == 0 ? 2 : 4;
  char* q = static_cast<char*>(work);
  float* o = reinterpret_cast<float*>(q + al256(elems * eb));
  float* scratch = reinterpret_cast<float*>(reinterpret_cast<char*>(o) + al256(elems * 4));
  const int64_t n8 = int64_t(elems / 8);
  if (dtype == 0)
    pf_prep_kernel<__nv_bfloat16><<<pf_grid(n8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(h), w,
                                                               reinterpret_cast<__nv_bfloat16*>(q),
                                                               static_cast<__nv_bfloat16*>(kv), B, n, H, S, off, D);
  else
    pf_prep_kernel<float><<<pf_grid(n8), 256, 0, st>>>(static_cast<const float*>(h), w, reinterpret_cast<float*>(q),
                                                       static_cast<float*>(kv), B, n, H, S, off, D);
  note_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  // attention of the patch's queries over the whole (partly stale) KV buffer
  AttnArgs a{};
  a.q = q;
  a.k = kv;
  a.v = static_cast<char*>(kv) + size_t(B) * H * S * D * eb;
  a.o = o;
  a.lse = nullptr;
  a.B = B; a.H = H; a.Sq = n; a.Skv = S; a.D = D;
  a.q_b = int64_t(n) * H * D; a.q_s = int64_t(H) * D; a.q_h = D;
  a.kv_b = int64_t(H) * S * D; a.kv_s = D; a.kv_h = int64_t(S) * D;
  xdit_rowmap m{};
  m.nseg = 1;
  m.seg_off[1] = n;
  for (int s = 2; s < 9; ++s) m.seg_off[s] = n;
  m.o_b = int64_t(n) * H * D; m.o_s = int64_t(H) * D; m.o_h = D;
  a.omap = m;
  a.out_f32 = 1;
  if (dtype == 0) {
    a.scratch = scratch;
    a.scratch_floats = attn_scratch_floats(D);
    e = launch_attn_fwd_bf16(a, st);
  } else {
    e = launch_attn_fwd_f32(a, st);
  }
  if (e != cudaSuccess) return e;
  if (dtype == 0)
    pf_residual_kernel<__nv_bfloat16, float><<<pf_grid(n8), 256, 0, st>>>(static_cast<__nv_bfloat16*>(h), o,
                                                                          w + 3 * H * D, n8, H * D);
  else
    pf_residual_kernel<float, float><<<pf_grid(n8), 256, 0, st>>>(static_cast<float*>(h), o, w + 3 * H * D, n8,
                                                                  H * D);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_pf_sampler(void* x, const void* eps, int64_t n, float sigma, int dtype, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (dtype == 0)
    pf_sampler_kernel<__nv_bfloat16><<<pf_grid(n / 8), 256, 0, st>>>(
        static_cast<__nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(eps), n / 8, sigma);
  else
    pf_sampler_kernel<float><<<pf_grid(n / 8), 256, 0, st>>>(static_cast<float*>(x), static_cast<const float*>(eps),
                                                             n / 8, sigma);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_pf_qkv(const void* h, const float* w, void* q, void* k, void* v, int B, int n, int H, int D,
                          int dtype, cudaStream_t st) {
  const int64_t n8 = int64_t(B) * n * H * D / 8;
  if (n8 == 0) return cudaSuccess;
  if (dtype == 0) {
    using T = __nv_bfloat16;
    pf_qkv_kernel<T><<<pf_grid(n8), 256, 0, st>>>(static_cast<const T*>(h), w, static_cast<T*>(q), static_cast<T*>(k),
                                                  static_cast<T*>(v), n8, H * D);
  } else {
    pf_qkv_kernel<float><<<pf_grid(n8), 256, 0, st>>>(static_cast<const float*>(h), w, static_cast<float*>(q),
                                                      static_cast<float*>(k), static_cast<float*>(v), n8, H * D);
  }
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_pf_residual(void* h, const void* o, const float* w, int B, int n, int H, int D, int dtype,
                               cudaStream_t st) {
  const int64_t n8 = int64_t(B) * n * H * D / 8;
  if (n8 == 0) return cudaSuccess;
  if (dtype == 0) {
    using T = __nv_bfloat16;
    pf_residual_kernel<T, T><<<pf_grid(n8), 256, 0, st>>>(static_cast<T*>(h), static_cast<const T*>(o), w + 3 * H * D,
                                                          n8, H * D);
  } else {
    pf_residual_kernel<float, float><<<pf_grid(n8), 256, 0, st>>>(static_cast<float*>(h), static_cast<const float*>(o),
                                                                  w + 3 * H * D, n8, H * D);
  }
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace xdit
