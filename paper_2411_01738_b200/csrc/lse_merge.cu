// lse_merge.cu -- merge of two partial attention results over disjoint key blocks by their
// log-sum-exp: SURVEY §8(a) step a7, the step that makes Ring attention "a parallel version of
// Flash Attention" (§4.1.1).  For one query row with partials (O_a, L_a), (O_b, L_b):
//     M = max(L_a, L_b),  L = M + log(exp(L_a - M) + exp(L_b - M)),
//     O = exp(L_a - L) * O_a + exp(L_b - L) * O_b                        (reading C9, fp32)
// HBM-bound: each row reads 2*D*4 bytes and writes D*4 (or D*2 for the final bf16 cast).  One warp
// per (b, row, head) row; lanes move float4 vectors.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "xdit_internal.h"

namespace xdit {
namespace {

constexpr int kWarps = 8;

__global__ void __launch_bounds__(kWarps * 32)
    lse_merge_kernel(float* __restrict__ o_acc, float* __restrict__ lse_acc,
                     const float* __restrict__ o_s, const float* __restrict__ lse_s, int B, int S,
                     int Hh, int D, void* fin, float* fin_lse, xdit_rowmap fmap, int fin_dtype) {
  const int64_t nrows = int64_t(B) * S * Hh;
  const int lane = threadIdx.x & 31;
  for (int64_t r = int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5); r < nrows;
       r += int64_t(gridDim.x) * kWarps) {
    // row r = ((b * S) + t) * Hh + hh  (O layout [B][S][Hh][D]); LSE layout [B][Hh][S]
    const int hh = int(r % Hh);
    const int64_t bt = r / Hh;
    const int t = int(bt % S), b = int(bt / S);
    const int64_t li = (int64_t(b) * Hh + hh) * S + t;
    const float la = lse_acc[li], lb = lse_s[li];
    const float M = fmaxf(la, lb);
    const float L = M + logf(expf(la - M) + expf(lb - M));
    const float wa = expf(la - L), wb = expf(lb - L);
    float* pa = o_acc + r * D;
    const float* pb = o_s + r * D;
    if (fin == nullptr) {
      for (int d = lane * 4; d < D; d += 128) {
        const float4 x = *reinterpret_cast<const float4*>(pa + d);
        const float4 y = *reinterpret_cast<const float4*>(pb + d);
        *reinterpret_cast<float4*>(pa + d) =
            make_float4(wa * x.x + wb * y.x, wa * x.y + wb * y.y, wa * x.z + wb * y.z, wa * x.w + wb * y.w);
      }
      if (lane == 0) lse_acc[li] = L;
    } else {
      const RowDst dst = rowmap_dst(fmap, b, t, hh);
      for (int d = lane * 4; d < D; d += 128) {
        const float4 x = *reinterpret_cast<const float4*>(pa + d);
        const float4 y = *reinterpret_cast<const float4*>(pb + d);
        const float4 z = make_float4(wa * x.x + wb * y.x, wa * x.y + wb * y.y, wa * x.z + wb * y.z,
                                     wa * x.w + wb * y.w);
        if (fin_dtype == 0) {
          __nv_bfloat162* q = reinterpret_cast<__nv_bfloat162*>(static_cast<__nv_bfloat16*>(fin) + dst.o_off + d);
          q[0] = __floats2bfloat162_rn(z.x, z.y);
          q[1] = __floats2bfloat162_rn(z.z, z.w);
        } else {
          *reinterpret_cast<float4*>(static_cast<float*>(fin) + dst.o_off + d) = z;
        }
      }
      if (lane == 0 && fin_lse) fin_lse[dst.l_off] = L;
    }
  }
}

}  // namespace

cudaError_t launch_lse_merge(float* o_acc, float* lse_acc, const float* o_s, const float* lse_s,
                             int B, int S, int Hh, int D, void* fin, float* fin_lse,
                             const xdit_rowmap* fmap, int fin_dtype, cudaStream_t st) {
  const int64_t nrows = int64_t(B) * S * Hh;
  if (nrows == 0) return cudaSuccess;
  const int nsm = device_sm_count();
  int64_t blocks = (nrows + kWarps - 1) / kWarps;
  const int64_t cap = int64_t(nsm) * 8;  // grid-stride beyond 8 CTAs per SM
  if (blocks > cap) blocks = cap;
  xdit_rowmap m{};
  if (fmap) m = *fmap;
  lse_merge_kernel<<<unsigned(blocks), kWarps * 32, 0, st>>>(o_acc, lse_acc, o_s, lse_s, B, S, Hh, D, fin,
                                                             fin_lse, m, fin_dtype); note_launches(1);
  return cudaGetLastError();
}

}  // namespace xdit
