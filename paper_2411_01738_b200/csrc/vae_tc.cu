// vae_tc.cu -- SURVEY §8(f) NEXT 4 on the tensor cores: the decoder's 3x3 conv as an implicit GEMM
// on tcgen05 (§4.3; reading R5, §7.7).
//
// out[y][x][co] = b[co] + sum_{dy,dx} sum_ci w[co][ci][dy][dx] * in[y+dy][x+dx-1][ci]
// over a halo-extended row band in[H+2][W][Ci] (bf16, channels innermost), zero padding in x.
// GEMM view per (tap, 64-channel chunk): A = 128 consecutive pixels of one input row, shifted by the
// tap (TMA box (64 ch, 128 px) at (ci0, row y+dy, x0+dx-1); out-of-range pixels and channels are
// zero-filled by the TMA, which IS the zero padding), B = the tap's weights for COT output channels
// (wt[9][Co][Ci], K-major), D = pixels x COT channels in TMEM (fp32), accumulated over 9 taps x
// ceil(Ci/64) chunks, 4 MMAs (K = 16) each.  CTA PAIRS (cta_group::2, M = 256): a 2-CTA cluster
// takes output rows y, y+1 of one 128-pixel strip and COT (128 or 256) output channels; each CTA
// loads its own pixel tile and HALF of the weights.  Warp 4 = TMA producer (both CTAs), warp 5 = MMA
// issuer (leader), warps 0-3 = epilogue (thread = pixel = TMEM lane): bias, optional SiLU + nearest
// x2 upsample, bf16 [H'][W'][Co8] (Co rounded up to 8, the extra channels zero) written through
// shared memory with TMA stores.
// Every pixel's sum is the same MMA sequence whatever band it sits in, so the banded decode stays
// bit-identical to the whole-image decode.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "attn_common.cuh"

namespace xdit {
namespace {

constexpr int kPix = 128, kKC = 64;
constexpr int kTileA = kPix * kKC * 2;  // 16 KB
// TMA store of a 4-D box from shared memory (bulk-group completion) and its helpers.
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* smem_src, int c0, int c1, int c2,
                                             int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(ptx::smem_u32(smem_src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// CTA-pair variant (cta_group::2, M = 256): the two CTAs of a cluster take output rows y and y + 1
// of one 128-pixel strip (each its own A tile and TMEM accumulator rows) and split the COT output
// channels' weights (each loads COT/2 of them; the pair's MMA reads the other half from the peer).
// Per SM and K step that is 16 KB of pixels + COT*64 B of weights instead of 16 KB + COT*128 B,
// and the smaller stages allow a 3-4 deep pipeline at two CTAs per SM: the one-CTA kernel ran its
// 2 x 48 KB stages latency-bound (ncu: tensor pipe 43 %, L2 28 % of peak).
template <int COT>
struct TC2 {
  static constexpr int kCoT = COT, kCoHalf = COT / 2;
  static constexpr int kTileB = kCoHalf * kKC * 2;
  static constexpr int kStageBytes = kTileA + kTileB;
  // 3 / 4 stages keep two CTAs per SM (one CTA's epilogue overlaps the other's K loop); 4 stages of
  // 32 KB at one CTA per SM measured 23-33 % slower (profiles/r02_s3_ab_vae2.txt)
  static constexpr int kStages = COT == 256 ? 3 : 4;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static_assert(kStages * kStageBytes >= 2 * kPix * 32 * 2, "output staging fits in the stages");
};

template <int COT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 2)
    vae_conv_tc2_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmO, const float* __restrict__ bias, int Hout, int W,
                        int Ci, int Co, int act_up) {
  using T = TC2<COT>;
  constexpr int kCoT = T::kCoT, kStages = T::kStages, kStageBytes = T::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem;  // the operand stages are free once the last MMA has completed
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);  // leader: both halves landed
  uint64_t* empty = full + kStages;                                             // each CTA: MMAs done with s
  uint64_t* acc_full = empty + kStages;                                         // each CTA: accumulator done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int x0 = (blockIdx.x >> 1) * kPix, y = blockIdx.y * 2 + int(rank), co0 = blockIdx.z * kCoT;
  const int nkc = (Ci + kKC - 1) / kKC, nk = 9 * nkc;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(acc_full, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 5) {
    ptx::tmem_alloc_pair(tmem_slot, kCoT);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // both CTAs' barriers initialised and TMEM allocated before any remote use
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 4) {  // ---------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW);
      const uint64_t pol = ptx::policy_evict_last();
      for (int it = 0; it < nk; ++it) {
        const int s = it % kStages, round = it / kStages;
        if (round > 0) ptx::mbar_wait(&empty[s], (round - 1) & 1);
        const int tap = it / nkc, c0 = (it % nkc) * kKC, dy = tap / 3, dx = tap % 3;
        if (rank == 0) ptx::mbar_expect_tx(&full[s], 2 * kStageBytes);
        const uint32_t full_cl = ptx::mapa(&full[s], 0);
        uint8_t* st = smem + s * kStageBytes;
        ptx::tma_load_4d_pair(st, &tmX, full_cl, c0, y + dy, x0 + dx - 1, 0, pol);  // (ch, row, px)
        ptx::tma_load_4d_pair(st + kTileA, &tmW, full_cl, c0, tap, co0 + int(rank) * T::kCoHalf, 0, pol);
      }
    }
  } else if (warp == 5) {  // -------------------------------------------- MMA issuer (leader CTA)
    if (rank == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kPix, kCoT, 0, 0);
      const uint32_t sa = ptx::smem_u32(smem);
      for (int it = 0; it < nk; ++it) {
        const int s = it % kStages;
        ptx::mbar_wait(&full[s], (it / kStages) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t a = sa + s * kStageBytes, b = a + kTileA;
#pragma unroll
          for (int k = 0; k < kKC / 16; ++k)
            ptx::mma_ss_pair(tmem, ptx::sdesc_sw128(a + k * 32, 16, 1024), ptx::sdesc_sw128(b + k * 32, 16, 1024),
                             idesc, (it > 0 || k > 0) ? 1u : 0u);
          ptx::tc_commit_pair(&empty[s]);
          if (it == nk - 1) ptx::tc_commit_pair(acc_full);
        }
        __syncwarp();
      }
    }
  } else {  // ------------------------------------------------------------ epilogue (warps 0-3)
    ptx::mbar_wait_sleep(acc_full, 0);
    ptx::tc_fence_after();
    const int xl = warp * 32 + lane;
    const uint32_t tl = tmem + (uint32_t(warp * 32) << 16);
    float bz[32];
#pragma unroll 1
    for (int cb = 0; cb < kCoT; cb += 32) {
      uint32_t r[32];
      ptx::tmem_ld32(tl + cb, r);
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        const int co = co0 + cb + q;
        bz[q] = co < Co ? __ldg(bias + co) : 0.f;
      }
      ptx::tmem_ld_wait();
      float v[32];
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        v[q] = u2f(r[q]) + bz[q];
        // SiLU with the MUFU exp2 / reciprocal (the accurate expf and division made the epilogue,
        // which sits on the critical path at two CTAs per SM, 8-13 % slower; parity unchanged)
        if (act_up) v[q] = __fdividef(v[q], 1.f + __expf(-v[q]));
      }
      uint4 pk[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        pk[q] = make_uint4(ptx::pack_bf16x2(v[8 * q], v[8 * q + 1]), ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                           ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
      if (cb > 0) {
        if (threadIdx.x == 0) bulk_wait_read0();
        ptx::named_bar_sync(1, 128);
      }
      const int nrow = act_up ? 2 : 1;
      for (int rr = 0; rr < nrow; ++rr) {
        const int row = act_up ? 2 * xl + rr : xl;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(stage_out + row * 64 + ((q ^ ((row >> 1) & 3)) * 16)) = pk[q];
      }
      fence_proxy_async();
      ptx::named_bar_sync(1, 128);
      if (threadIdx.x == 0 && y < Hout) {
        if (act_up) {
          tma_store_4d(&tmO, stage_out, co0 + cb, 2 * y, 2 * x0, 0);
          tma_store_4d(&tmO, stage_out, co0 + cb, 2 * y + 1, 2 * x0, 0);
        } else {
          tma_store_4d(&tmO, stage_out, co0 + cb, y, x0, 0);
        }
        bulk_commit();
      }
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // the peer's smem / TMEM stay live until the leader's MMAs are done
  ptx::tc_fence_after();
  if (warp == 5) ptx::tmem_dealloc_pair(tmem, kCoT);
}

}  // namespace

namespace {
template <int COT>
cudaError_t launch_tc2(const CUtensorMap& mx, const void* wt, const CUtensorMap& mo, const float* b, int Hout, int Ci,
                       int W, int Co, int act_up, cudaStream_t st) {
  using T = TC2<COT>;
  CUtensorMap mw;
  if (!make_map(&mw, wt, 1, Co, 9, Ci, int64_t(9) * Co * Ci, Ci, int64_t(Co) * Ci, kKC, T::kCoHalf))
    return cudaErrorInvalidValue;
  static DeviceFlags attr;
  if (!attr.test()) {
    cudaError_t e = cudaFuncSetAttribute(vae_conv_tc2_kernel<COT>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::kSmem);
    if (e != cudaSuccess) return e;
    attr.set();
  }
  const dim3 grid(2 * ((W + kPix - 1) / kPix), (Hout + 1) / 2, (Co + COT - 1) / COT);
  vae_conv_tc2_kernel<COT><<<grid, 192, T::kSmem, st>>>(mx, mw, mo, b, Hout, W, Ci, Co, act_up);
  note_launches(1);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_vae_conv_tc(const void* in, int Hout, int Ci, int W, const void* wt, const float* b, void* out,
                               int Co, int act_up, cudaStream_t st) {
  if (Hout == 0 || W == 0) return cudaSuccess;
  CUtensorMap mx, mo;
  const int Co8 = (Co + 7) / 8 * 8;  // output channel stride (16-byte rows for the TMA store)
  // activations [Hout+2][W][Ci]: dims (Ci, rows->"H", pixels->"S"); box 64 channels x 128 pixels
  if (!make_map(&mx, in, 1, W, Hout + 2, Ci, int64_t(Hout + 2) * W * Ci, Ci, int64_t(W) * Ci, kKC, kPix) ||
      // output [H'][W'][Co8]: boxes of 32 channels (64B swizzle) x 128 (256 upsampled) pixels x 1 row
      !make_map(&mo, out, 1, act_up ? 2 * W : W, act_up ? 2 * Hout : Hout, Co8,
                int64_t(act_up ? 4 : 1) * Hout * W * Co8, Co8, int64_t(act_up ? 2 * W : W) * Co8, 32,
                act_up ? 2 * kPix : kPix))
    return cudaErrorInvalidValue;
  // 256 output channels per CTA for the wide layers (half the A-tile loads per FLOP), else 128
  // (profiles/r01_ab_vae_cot.txt)
  const bool wide = Co >= 256;
  return wide ? launch_tc2<256>(mx, wt, mo, b, Hout, Ci, W, Co, act_up, st)
              : launch_tc2<128>(mx, wt, mo, b, Hout, Ci, W, Co, act_up, st);
}

}  // namespace xdit
