// attn_fwd_f32.cu -- fp32-input attention forward on the SIMT (FFMA) pipes: the fp32 mode of the
// ABI (xdit_usp_attention_f32), SURVEY §8(a) step a6 in fp32 throughout (reading C10: "The fp32
// mode computes in fp32 throughout").  O = softmax(Q K^T / sqrt(D)) V with LSE (§4.1.2;
// readings C1, C2), streamed over KV tiles with the online-softmax recurrence (§4.1.1).
//
// Layout of the work: a CTA of 128 threads owns 32 query rows of one (b, h); each query row is
// handled by 4 consecutive lanes that split the head dim (lane c owns d = c, c+4, ...), reduce
// partial dot products with two shuffles, and keep their quarter of the fp32 O row in registers.
// K/V tiles of 32 keys are staged in shared memory (row-contiguous, read as broadcasts).
#include <cuda_runtime.h>

#include <cmath>

#include "xdit_internal.h"

namespace xdit {
namespace {

constexpr int kRows = 32;     // query rows per CTA
constexpr int kKeys = 32;     // keys per smem tile
constexpr int kThreads = 128;

template <int DQ>  // DQ = max head-dim elements per lane (D <= 4*DQ)
__global__ void __launch_bounds__(kThreads)
    attn_fwd_f32_kernel(const float* __restrict__ q, const float* __restrict__ k,
                        const float* __restrict__ v, AttnArgs a, float scale) {
  extern __shared__ float sm[];
  const int D = a.D;
  float* sK = sm;                 // [kKeys][D]
  float* sV = sm + kKeys * D;     // [kKeys][D]
  const int h = blockIdx.y, b = blockIdx.z;
  const int r_loc = threadIdx.x >> 2, c = threadIdx.x & 3;
  const int row = blockIdx.x * kRows + r_loc;
  const bool row_ok = row < a.Sq;

  float qr[DQ], o[DQ];
#pragma unroll
  for (int i = 0; i < DQ; ++i) {
    const int d = c + 4 * i;
    qr[i] = (row_ok && d < D) ? q[b * a.q_b + int64_t(row) * a.q_s + h * a.q_h + d] * scale : 0.f;
    o[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j0 = 0; j0 < a.Skv; j0 += kKeys) {
    const int nk = min(kKeys, a.Skv - j0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < nk * D; idx += kThreads) {
      const int jj = idx / D, d = idx - jj * D;
      const int64_t off = b * a.kv_b + int64_t(j0 + jj) * a.kv_s + h * a.kv_h + d;
      sK[jj * D + d] = k[off];
      sV[jj * D + d] = v[off];
    }
    __syncthreads();
#pragma unroll 1
    for (int jj = 0; jj < nk; ++jj) {
      float part = 0.f;
#pragma unroll
      for (int i = 0; i < DQ; ++i) {
        const int d = c + 4 * i;
        if (d < D) part = fmaf(qr[i], sK[jj * D + d], part);
      }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      if (part > m) {  // online-softmax rescale (uniform across the row's 4 lanes)
        const float alpha = expf(m - part);  // exp(-inf) = 0 on the first key
        l *= alpha;
#pragma unroll
        for (int i = 0; i < DQ; ++i) o[i] *= alpha;
        m = part;
      }
      const float pj = expf(part - m);
      l += pj;
#pragma unroll
      for (int i = 0; i < DQ; ++i) {
        const int d = c + 4 * i;
        if (d < D) o[i] = fmaf(pj, sV[jj * D + d], o[i]);
      }
    }
  }
  if (!row_ok) return;
  const RowDst dst = rowmap_dst(a.omap, b, row, h);
  float* out = static_cast<float*>(a.o) + dst.o_off;
  const float inv_l = 1.f / l;
#pragma unroll
  for (int i = 0; i < DQ; ++i) {
    const int d = c + 4 * i;
    if (d < D) out[d] = o[i] * inv_l;
  }
  if (c == 0 && a.lse) a.lse[dst.l_off] = m + logf(l);
}

template <int DQ>
cudaError_t launch_dq(const AttnArgs& a, cudaStream_t st) {
  const size_t smem = size_t(2) * kKeys * a.D * sizeof(float);
  static DeviceFlags attr;
  if (!attr.test()) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_f32_kernel<DQ>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kKeys * 256 * 4);
    if (e != cudaSuccess) return e;
    attr.set();
  }
  dim3 grid((a.Sq + kRows - 1) / kRows, a.H, a.B);
  attn_fwd_f32_kernel<DQ><<<grid, kThreads, smem, st>>>(
      static_cast<const float*>(a.q), static_cast<const float*>(a.k),
      static_cast<const float*>(a.v), a, float(1.0 / std::sqrt(double(a.D)))); note_launches(1);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_fwd_f32(const AttnArgs& a, cudaStream_t st) {
  if (a.Sq == 0 || a.B == 0) return cudaSuccess;
  if (a.D <= 64) return launch_dq<16>(a, st);
  if (a.D <= 128) return launch_dq<32>(a, st);
  if (a.D <= 256) return launch_dq<64>(a, st);
  return cudaErrorInvalidValue;
}

}  // namespace xdit
