// next_ops.cu -- the two SURVEY §8(f) NEXT rows built on the USP path.
//
// * kv_place_kernel (NEXT 1, reading R2): copy a K/V block the rank
//   holds during a USP call -- its ring block after the Ulysses all-to-all, or an incoming ring
//   block -- into the caller's KV buffer [2][B][Hh][S_total][D], so the rank keeps the K,V "of the
//   sequence within the SP group" for its heads instead of discarding them: at one sequence offset
//   (xdit_usp_attention_kv, SP-shard order) or scattered by a segment table to the tokens' global
//   rows (xdit_usp_attention_buf, the hybrid PipeFusion x SP buffer, reading R6).  Pure data
//   movement: HBM-bound, 16-byte vectors, one thread per vector, K and V in one launch.
// * cfg_combine_kernel (NEXT 2, reading R3):
//   eps = eps_u + g * (eps_c - eps_u), evaluated in fp32 as g*eps_c + (1-g)*eps_u (one FMA after
//   one multiply: exact at both endpoints g = 0 and g = 1, which the eps_u + g*(eps_c - eps_u) form
//   is not when |eps_c| << |eps_u|), rounded once (RNE) to the output dtype.  HBM-bound.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "xdit_internal.h"

namespace xdit {
namespace {

// src element (b, t, h, d) at src + b*sb + t*ss + h*sh + d (elements of eb bytes) -> dst
// [B][Hh][S_total][D] at row segs.dst[k] + t - segs.src[k] for the segment k holding block row t
// (segments cover [0, S_blk) in increasing order).  vec = D*eb/16 16-byte vectors per row;
// blockIdx.y = 0 copies K, 1 copies V (the V half of dst starts `half` bytes in).
__global__ void kv_place_kernel(const uint8_t* __restrict__ srck, const uint8_t* __restrict__ srcv,
                                uint8_t* __restrict__ dst, size_t half, int B, int Hh, int S_blk, int S_total,
                                KvSegs segs, int vec, int64_t sb, int64_t ss, int64_t sh, int eb) {
  const uint8_t* src = blockIdx.y ? srcv : srck;
  uint8_t* out = dst + (blockIdx.y ? half : 0);
  const int64_t n = int64_t(B) * Hh * S_blk * vec;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < n;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int v = int(idx % vec);
    int64_t r = idx / vec;
    const int t = int(r % S_blk);
    r /= S_blk;
    const int h = int(r % Hh);
    const int b = int(r / Hh);
    int k = 0;
    for (int x = 1; x < segs.n; ++x)
      if (t >= segs.src[x]) k = x;
    const int row = segs.dst[k] + t - segs.src[k];
    const uint4* s = reinterpret_cast<const uint4*>(src + (b * sb + t * ss + h * sh) * eb) + v;
    uint4* d = reinterpret_cast<uint4*>(out + ((int64_t(b) * Hh + h) * S_total + row) * int64_t(vec) * 16) + v;
    *d = __ldg(s);
  }
}

__global__ void cfg_combine_bf16(const uint4* __restrict__ c, const uint4* __restrict__ u, uint4* __restrict__ o,
                                 int64_t n8, float g) {
  const float gu = 1.f - g;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n8; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 cv = c[i], uv = u[i];
    const __nv_bfloat162* cp = reinterpret_cast<const __nv_bfloat162*>(&cv);
    const __nv_bfloat162* up = reinterpret_cast<const __nv_bfloat162*>(&uv);
    uint4 ov;
    __nv_bfloat162* op = reinterpret_cast<__nv_bfloat162*>(&ov);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 cf = __bfloat1622float2(cp[k]), uf = __bfloat1622float2(up[k]);
      op[k] = __floats2bfloat162_rn(fmaf(g, cf.x, gu * uf.x), fmaf(g, cf.y, gu * uf.y));
    }
    o[i] = ov;
  }
}

__global__ void cfg_combine_f32(const float4* __restrict__ c, const float4* __restrict__ u, float4* __restrict__ o,
                                int64_t n4, float g) {
  const float gu = 1.f - g;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 cv = c[i], uv = u[i];
    o[i] = make_float4(fmaf(g, cv.x, gu * uv.x), fmaf(g, cv.y, gu * uv.y), fmaf(g, cv.z, gu * uv.z),
                       fmaf(g, cv.w, gu * uv.w));
  }
}

int grid_for(int64_t n) {
  const int nsm = device_sm_count();
  const int64_t blocks = (n + 255) / 256;
  return int(blocks < int64_t(nsm) * 8 ? (blocks > 0 ? blocks : 1) : int64_t(nsm) * 8);
}

}  // namespace

cudaError_t launch_kv_place(const void* k, const void* v, void* kv, int B, int Hh, int S_blk, int S_total,
                            const KvSegs& segs, int D, int64_t sb, int64_t ss, int64_t sh, int eb, cudaStream_t st) {
  if (B == 0 || S_blk == 0) return cudaSuccess;
  const int vec = D * eb / 16;
  const int64_t n = int64_t(B) * Hh * S_blk * vec;
  const size_t half = size_t(B) * Hh * S_total * D * eb;
  kv_place_kernel<<<dim3(grid_for(n), 2), 256, 0, st>>>(static_cast<const uint8_t*>(k), static_cast<const uint8_t*>(v),
                                                        static_cast<uint8_t*>(kv), half, B, Hh, S_blk, S_total, segs,
                                                        vec, sb, ss, sh, eb);
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_kv_retain(const void* k, const void* v, void* kv_keep, int B, int Hh, int S_blk, int S_total,
                             int seq_off, int D, int64_t sb, int64_t ss, int64_t sh, int eb, cudaStream_t st) {
  KvSegs one{};
  one.n = 1;
  one.dst[0] = seq_off;
  return launch_kv_place(k, v, kv_keep, B, Hh, S_blk, S_total, one, D, sb, ss, sh, eb, st);
}

cudaError_t launch_cfg_combine(const void* c, const void* u, void* o, int64_t n, float g, int dtype,
                               cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  if (dtype == 0) {
    cfg_combine_bf16<<<grid_for(n / 8), 256, 0, st>>>(static_cast<const uint4*>(c), static_cast<const uint4*>(u),
                                                       static_cast<uint4*>(o), n / 8, g);
  } else {
    cfg_combine_f32<<<grid_for(n / 4), 256, 0, st>>>(static_cast<const float4*>(c), static_cast<const float4*>(u),
                                                      static_cast<float4*>(o), n / 4, g);
  }
  note_launches(1);
  return cudaGetLastError();
}

}  // namespace xdit
