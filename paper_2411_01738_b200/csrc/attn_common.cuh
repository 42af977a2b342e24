// attn_common.cuh -- pieces of the bf16 attention kernel (attn_fwd_2sm.cu: persistent CTA pairs)
// kept apart from it: epilogue parameters, packed fp32x2 helpers, the FMA-pipe exp2, the tail-split
// merge kernel and the TMA tensor-map encoder.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>

#include "sm100_ptx.cuh"
#include "xdit_internal.h"

namespace xdit {
namespace {

constexpr int kRowsPerItem = 256;  // query rows per work item (tile pair / CTA pair)
// floats at the end of the attention scratch holding the persistent kernel's work-unit counter
constexpr size_t kCounterFloats = 4;

struct EpiParams {
  void* o;
  float* lse;
  xdit_rowmap map;
  int H, Sq, Skv, out_f32;
  float scale_log2;
  // Work decomposition (1-D grid): items are (query-tile pair, head, batch), query tile fastest.
  // Items [0, n_full) run over all keys; each of the remaining n_tail items is split into n_split
  // key ranges of kv_chunk keys whose normalised fp32 partials (O, LSE) go to `part` and are merged
  // by tail_merge_kernel -- this fills the last, partial wave of the grid.
  int n_qt, n_full, n_split, kv_chunk;
  float* part;  // [n_tail * n_split][256][D] fp32 O, then [n_tail * n_split][256] fp32 LSE
  // Persistent CTA pairs: n_units = n_full + n_tail * n_split work units; unit_counter (zeroed
  // before the launch, in the caller's scratch) hands them out dynamically, else round-robin.
  int n_units;
  unsigned* unit_counter;
  // Ring merge fused into the epilogue (a7, reading C9; CTA-pair kernel): merge = 1 combines this
  // launch's (O_s, LSE_s) row with the accumulator row (acc_o, acc_l_in; layout acc_map) by their
  // log-sum-exp; merge_final = 0 writes the result back to acc_o (in place) and acc_l_out, 1 writes
  // it to the final destination (o, lse through map, bf16 or fp32).
  int merge, merge_final;
  float* acc_o;
  const float* acc_l_in;
  float* acc_l_out;
  xdit_rowmap acc_map;
  int diag;  // profiling builds only (-DXDIT_PROFILE): 1 = the softmax does no math (skeleton)
  unsigned long long* trace;  // profiling builds only: per-iteration clock64 stamps of the first pair
};

__device__ __forceinline__ float u2f(uint32_t x) { return __uint_as_float(x); }
__device__ __forceinline__ uint32_t f2u(float x) { return __float_as_uint(x); }

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void up2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
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

// exp2 of two packed fp32 values on the FMA pipe (no MUFU): Cody-Waite split x = j + f with
// j = round(x) (magic-number add), f in [-0.5, 0.5]; 2^f by a degree-4 polynomial with p(0) = 1
// exactly (minimax on [-0.5, 0.5], max relative error 2.9e-6, mean 3e-7 -- far below the bf16
// rounding P gets anyway, and no bias on the row sum l); 2^j is added straight into the exponent
// field.  x is clamped to [-125, 127] so the result stays a normal number.
__device__ __forceinline__ uint64_t exp2_poly2(uint64_t x2) {
  float x0, x1;
  up2(x2, x0, x1);
  x0 = fminf(fmaxf(x0, -125.f), 127.f);  // 2^127 still flags the softmax's overflow test
  x1 = fminf(fmaxf(x1, -125.f), 127.f);
  const uint64_t xc = pk2(x0, x1);
  const uint64_t magic = pk2(12582912.f, 12582912.f), nmagic = pk2(-12582912.f, -12582912.f);
  const uint64_t t = add2(xc, magic);             // 1.5*2^23 + round(x)
  const uint64_t j = add2(t, nmagic);             // round(x)
  const uint64_t f = fma2(j, pk2(-1.f, -1.f), xc);  // x - round(x)
  uint64_t pp = fma2(f, pk2(0.009582849219441414f, 0.009582849219441414f),
                     pk2(0.055906426161527634f, 0.055906426161527634f));
  pp = fma2(f, pp, pk2(0.24024099111557007f, 0.24024099111557007f));
  pp = fma2(f, pp, pk2(0.6931241750717163f, 0.6931241750717163f));
  pp = fma2(f, pp, pk2(1.f, 1.f));
  float p0, p1, t0, t1;
  up2(pp, p0, p1);
  up2(t, t0, t1);
  // (bits(t) << 23) == round(x) << 23 (mod 2^32): the magic's own bits shift out
  const int r0 = __float_as_int(t0) * (1 << 23) + __float_as_int(p0);
  const int r1 = __float_as_int(t1) * (1 << 23) + __float_as_int(p1);
  return pk2(__int_as_float(r0), __int_as_float(r1));
}

// Merge of the split tail items (LSE-weighted, as the ring merge a7): one warp per (tail item, row).
template <int D>
__global__ void __launch_bounds__(256)
    tail_merge_kernel(const float* __restrict__ part, int n_tail, int n_split, int n_full, int n_qt,
                      int H, int Sq, EpiParams p) {
  const int w = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (w >= n_tail * kRowsPerItem) return;
  const int ti = w / kRowsPerItem, rr = w % kRowsPerItem;
  const int item = n_full + ti, hb = item / n_qt, h = hb % H, b = hb / H;
  const int row = (item % n_qt) * kRowsPerItem + rr;
  if (row >= Sq) return;
  const int64_t n_pieces = int64_t(n_tail) * n_split;
  const float* plse = part + n_pieces * kRowsPerItem * D;
  float M = -INFINITY;
  for (int s = 0; s < n_split; ++s) M = fmaxf(M, plse[(int64_t(ti) * n_split + s) * kRowsPerItem + rr]);
  float sum = 0.f;
  for (int s = 0; s < n_split; ++s) sum += expf(plse[(int64_t(ti) * n_split + s) * kRowsPerItem + rr] - M);
  const float Ls = M + logf(sum);  // LSE of this launch's key range
  float L = Ls;
  const RowDst dst = rowmap_dst(p.map, b, row, h);
  // fused ring merge (p.merge): combine with the accumulator row, as lse_merge_kernel does
  float wa = 0.f, wb = 1.f;
  RowDst ad{0, 0};
  if (p.merge) {
    ad = rowmap_dst(p.acc_map, b, row, h);
    const float la = p.acc_l_in[ad.l_off];
    const float M2 = fmaxf(la, L);
    const float L2 = M2 + logf(expf(la - M2) + expf(L - M2));
    wa = expf(la - L2);
    wb = expf(L - L2);
    L = L2;
  }
  for (int d = lane * 4; d < D; d += 128) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < n_split; ++s) {
      const int64_t pr = (int64_t(ti) * n_split + s) * kRowsPerItem + rr;
      const float wgt = expf(plse[pr] - Ls);
      const float4 x = *reinterpret_cast<const float4*>(part + pr * D + d);
      acc.x += wgt * x.x; acc.y += wgt * x.y; acc.z += wgt * x.z; acc.w += wgt * x.w;
    }
    if (p.merge) {
      const float4 y = *reinterpret_cast<const float4*>(p.acc_o + ad.o_off + d);
      acc = make_float4(wa * y.x + wb * acc.x, wa * y.y + wb * acc.y, wa * y.z + wb * acc.z, wa * y.w + wb * acc.w);
      if (!p.merge_final) {
        *reinterpret_cast<float4*>(p.acc_o + ad.o_off + d) = acc;
        continue;
      }
    }
    if (p.out_f32) {
      *reinterpret_cast<float4*>(static_cast<float*>(p.o) + dst.o_off + d) = acc;
    } else {
      uint2 v;
      v.x = ptx::pack_bf16x2(acc.x, acc.y);
      v.y = ptx::pack_bf16x2(acc.z, acc.w);
      *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(p.o) + dst.o_off + d) = v;
    }
  }
  if (lane == 0) {
    if (p.merge && !p.merge_final) p.acc_l_out[ad.l_off] = L;
    else if (p.lse) p.lse[dst.l_off] = L;
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qres;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) ==
            cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

// [B][S][H][D] bf16 view with element strides (sb, ss, sh); box = box_cols columns x box_rows rows
// with the swizzle of the box row: 64 columns / 128B, 32 columns / 64B (the CTA-pair kernel's D=64
// V halves), 16 columns / 32B (the D=72 tail atom).
bool make_map(CUtensorMap* map, const void* base, int B, int S, int H, int D, int64_t sb, int64_t ss,
              int64_t sh, int box_cols = 64, int box_rows = 128) {
  auto enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(H), cuuint64_t(S), cuuint64_t(B)};
  cuuint64_t strides[3] = {cuuint64_t(sh * 2), cuuint64_t(ss * 2), cuuint64_t(sb * 2)};
  cuuint32_t box[4] = {cuuint32_t(box_cols), 1, cuuint32_t(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_cols == 64 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : (box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace
}  // namespace xdit
