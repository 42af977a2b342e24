// vae_tc.cu -- SURVEY §8(f) NEXT 4 on the tensor cores: the decoder's 3x3 conv as an implicit GEMM
// on tcgen05 (§4.3; reading R5, §7.7).
//
// out[y][x][co] = b[co] + sum_{dy,dx} sum_ci w[co][ci][dy][dx] * in[y+dy][x+dx-1][ci]
// over a halo-extended row band in[H+2][W][Ci] (bf16, channels innermost), zero padding in x.
// GEMM view: A = 128 consecutive pixels of input row y+dy shifted by dx-1, B = tap (dy, dx)'s weights
// for COT output channels (wt[9][Co][Ci], K-major), D = pixels x COT channels in TMEM (fp32),
// accumulated over 3 dy x ceil(Ci/64) channel chunks x 3 dx x 4 MMAs (K = 16).  One TMA box of 136
// pixels x 64 channels at (ci0, row y+dy, x0-1) serves all three dx taps (the shift is a 128-byte
// offset of the MMA descriptor into the 128B-swizzled tile); out-of-range pixels and channels are
// zero-filled by the TMA, which IS the zero padding.  CTA PAIRS (cta_group::2, M = 256): a 2-CTA
// cluster takes output rows y, y+1 of one 128-pixel strip and COT (128 or 256) output channels; each
// CTA loads its own pixel row and HALF of the weights.  Persistent: one cluster per TPC loops over
// the tiles, two TMEM accumulators.  Warp 4 = TMA producer (both CTAs), warp 5 = MMA issuer
// (leader), warps 0-3 = epilogue (thread = pixel = TMEM lane): bias, optional SiLU + nearest x2
// upsample, bf16 [H'][W'][Co8] (Co rounded up to 8, the extra channels zero) written through shared
// memory with TMA stores.
// Every pixel's sum is the same MMA sequence whatever band it sits in, so the banded decode stays
// bit-identical to the whole-image decode.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "attn_common.cuh"

namespace xdit {
namespace {

constexpr int kPix = 128, kKC = 64;
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

// CTA pairs (cta_group::2, M = 256): the two CTAs of a cluster take output rows y and y + 1 of one
// 128-pixel strip (each its own A tile and TMEM accumulator rows) and split the COT output channels'
// weights (each loads COT/2 of them; the pair's MMA reads the other half from the peer): per SM and K
// step 16 KB of pixels + COT*64 B of weights instead of 16 KB + COT*128 B (the one-CTA kernel of
// round 1 ran its 2 x 48 KB stages latency-bound: ncu tensor pipe 43 %, L2 28 % of peak).
// Persistent: one cluster per TPC loops over the tiles (row pair, 128-pixel strip,
// COT-channel block; round-robin), the operand ring runs on across tiles (3 / 4 stages of one pixel
// row + three taps' weights at one CTA per SM), and two TMEM accumulators let the epilogue of tile i
// (its own staging buffer) overlap the K loop of tile i + 1: acc_full[b] (MMA -> epilogue,
// multicast) / acc_empty[b] (the 8 epilogue warps of the pair -> the leader's MMA warp).
template <int COT>
struct TCP {
  static constexpr int kCoT = COT, kCoHalf = COT / 2;
  static constexpr int kTileB = kCoHalf * kKC * 2;
  // one pixel row per (dy, channel chunk) for all three dx taps: 136 pixels (x0-1 .. x0+134) and the
  // three taps' weight halves in one stage; the dx shift is a 128-byte start offset into the
  // 128B-swizzled pixel tile (the swizzle follows the absolute smem address bits, so the shifted
  // descriptor needs no base offset -- with base offset dx the parity tests fail)
  static constexpr int kRowsA = 136;
  static constexpr int kTileAX = kRowsA * kKC * 2;
  static constexpr int kStageBytes = (kTileAX + 1023) / 1024 * 1024 + 3 * kTileB;
  static constexpr int kStages = COT == 256 ? 3 : 4;
  static constexpr int kOutBytes = 2 * kPix * 64;  // 256 staging rows of 32 bf16 channels
  static constexpr int kSmem = kStages * kStageBytes + kOutBytes + 1024 + 256;
};

template <int COT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    vae_conv_tcp_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmO, const float* __restrict__ bias, int Hout, int W,
                        int Ci, int Co, int act_up) {
  using T = TCP<COT>;
  constexpr int kCoT = T::kCoT, kStages = T::kStages, kStageBytes = T::kStageBytes;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stage_out = smem + kStages * kStageBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(stage_out + T::kOutBytes);  // leader: both halves landed
  uint64_t* empty = full + kStages;                                        // each CTA: MMAs done with s
  uint64_t* acc_full = empty + kStages;                                    // each CTA [2]: accumulator b done
  uint64_t* acc_empty = acc_full + 2;                                      // leader [2]: accumulator b read out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const int nkc = (Ci + kKC - 1) / kKC;
  const int n_sx = (W + kPix - 1) / kPix, n_by = (Hout + 1) / 2, n_z = (Co + kCoT - 1) / kCoT;
  const int n_tiles = n_sx * n_by * n_z;
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  auto tile = [&](int t, int& x0, int& y, int& co0) {
    x0 = (t % n_sx) * kPix;
    const int r = t / n_sx;
    y = (r % n_by) * 2 + int(rank);
    co0 = (r / n_by) * kCoT;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&acc_full[b], 1);
      ptx::mbar_init(&acc_empty[b], 8);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 5) {
    ptx::tmem_alloc_pair(tmem_slot, 2 * kCoT);
    ptx::tmem_relinquish_pair();
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp == 4) {  // ---------------------------------------------------- TMA producer (both CTAs)
    if (lane == 0) {
      ptx::tma_prefetch_desc(&tmX);
      ptx::tma_prefetch_desc(&tmW);
      const uint64_t pol = ptx::policy_evict_last();
      uint32_t it = 0;
      for (int t = cid; t < n_tiles; t += ncl) {
        int x0, y, co0;
        tile(t, x0, y, co0);
        for (int k = 0; k < 3 * nkc; ++k, ++it) {  // (dy, chunk); the stage holds all three dx taps
          const int s = int(it % kStages);
          const uint32_t round = it / kStages;
          if (round > 0) ptx::mbar_wait(&empty[s], (round - 1) & 1);
          const int dy = k / nkc, c0 = (k % nkc) * kKC;
          if (rank == 0) ptx::mbar_expect_tx(&full[s], 2 * (T::kTileAX + 3 * T::kTileB));
          const uint32_t full_cl = ptx::mapa(&full[s], 0);
          uint8_t* st = smem + s * kStageBytes;
          ptx::tma_load_4d_pair(st, &tmX, full_cl, c0, y + dy, x0 - 1, 0, pol);
          uint8_t* sb = st + (T::kTileAX + 1023) / 1024 * 1024;
          for (int dx = 0; dx < 3; ++dx)
            ptx::tma_load_4d_pair(sb + dx * T::kTileB, &tmW, full_cl, c0, 3 * dy + dx,
                                  co0 + int(rank) * T::kCoHalf, 0, pol);
        }
      }
    }
  } else if (warp == 5) {  // -------------------------------------------- MMA issuer (leader CTA)
    if (rank == 0) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kPix, kCoT, 0, 0);
      const uint32_t sa = ptx::smem_u32(smem);
      uint32_t it = 0;
      int li = 0;
      for (int t = cid; t < n_tiles; t += ncl, ++li) {
        const int ab = li & 1;
        if (li >= 2) ptx::mbar_wait(&acc_empty[ab], ((li - 2) >> 1) & 1);
        const uint32_t d = tmem + uint32_t(ab * kCoT);
        for (int k = 0; k < 3 * nkc; ++k, ++it) {
          const int s = int(it % kStages);
          ptx::mbar_wait(&full[s], (it / kStages) & 1);
          ptx::tc_fence_after();
          if (ptx::elect_one()) {
            const uint32_t a = sa + s * kStageBytes, b = a + (T::kTileAX + 1023) / 1024 * 1024;
#pragma unroll
            for (int dx = 0; dx < 3; ++dx)
#pragma unroll
              for (int kk = 0; kk < kKC / 16; ++kk)  // pixel rows dx .. dx + 127: base offset dx
                ptx::mma_ss_pair(d, ptx::sdesc_sw128(a + dx * 128 + kk * 32, 16, 1024),
                                 ptx::sdesc_sw128(b + dx * T::kTileB + kk * 32, 16, 1024), idesc,
                                 (k > 0 || dx > 0 || kk > 0) ? 1u : 0u);
            ptx::tc_commit_pair(&empty[s]);
            if (k == 3 * nkc - 1) ptx::tc_commit_pair(&acc_full[ab]);
          }
          __syncwarp();
        }
      }
    }
  } else {  // ------------------------------------------------------------ epilogue (warps 0-3)
    const int xl = warp * 32 + lane;
    const uint32_t acc_empty_cl = ptx::mapa(&acc_empty[0], 0);
    bool first = true;
    int li = 0;
    for (int t = cid; t < n_tiles; t += ncl, ++li) {
      int x0, y, co0;
      tile(t, x0, y, co0);
      const int ab = li & 1;
      ptx::mbar_wait_sleep(&acc_full[ab], (li >> 1) & 1);
      ptx::tc_fence_after();
      const uint32_t tl = tmem + (uint32_t(warp * 32) << 16) + uint32_t(ab * kCoT);
#pragma unroll 1
      for (int cb = 0; cb < kCoT; cb += 32) {
        uint32_t r[32];
        ptx::tmem_ld32(tl + cb, r);
        float bz[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          const int co = co0 + cb + q;
          bz[q] = co < Co ? __ldg(bias + co) : 0.f;
        }
        ptx::tmem_ld_wait();
        if (cb + 32 >= kCoT) {  // the accumulator is read out: the MMA may start tile li + 2 in it
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(acc_empty_cl + uint32_t(ab * 8));
        }
        float v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          v[q] = u2f(r[q]) + bz[q];
          if (act_up) v[q] = __fdividef(v[q], 1.f + __expf(-v[q]));
        }
        uint4 pk[4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
          pk[q] = make_uint4(ptx::pack_bf16x2(v[8 * q], v[8 * q + 1]), ptx::pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                             ptx::pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), ptx::pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
        if (!first) {  // the previous chunk's TMA stores have read the staging buffer
          if (threadIdx.x == 0) bulk_wait_read0();
          ptx::named_bar_sync(1, 128);
        }
        first = false;
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
    }
    if (threadIdx.x == 0) bulk_wait0();
  }
  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 5) ptx::tmem_dealloc_pair(tmem, 2 * kCoT);
}

}  // namespace

namespace {
template <int COT>
cudaError_t launch_tcp(const CUtensorMap& mx, const void* wt, const CUtensorMap& mo, const float* b, int Hout, int Ci,
                       int W, int Co, int act_up, cudaStream_t st) {
  using T = TCP<COT>;
  CUtensorMap mw;
  if (!make_map(&mw, wt, 1, Co, 9, Ci, int64_t(9) * Co * Ci, Ci, int64_t(Co) * Ci, kKC, T::kCoHalf))
    return cudaErrorInvalidValue;
  static DeviceFlags attr;
  if (!attr.test()) {
    cudaError_t e = cudaFuncSetAttribute(vae_conv_tcp_kernel<COT>, cudaFuncAttributeMaxDynamicSharedMemorySize, T::kSmem);
    if (e != cudaSuccess) return e;
    attr.set();
  }
  const int n_tiles = ((W + kPix - 1) / kPix) * ((Hout + 1) / 2) * ((Co + COT - 1) / COT);
  const dim3 grid(2 * std::min(n_tiles, device_sm_count() / 2));
  vae_conv_tcp_kernel<COT><<<grid, 192, T::kSmem, st>>>(mx, mw, mo, b, Hout, W, Ci, Co, act_up);
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
  constexpr int kBoxPix = 136;  // x0-1 .. x0+134: the three dx taps of a 128-pixel strip
  if (!make_map(&mx, in, 1, W, Hout + 2, Ci, int64_t(Hout + 2) * W * Ci, Ci, int64_t(W) * Ci, kKC, kBoxPix) ||
      // output [H'][W'][Co8]: boxes of 32 channels (64B swizzle) x 128 (256 upsampled) pixels x 1 row
      !make_map(&mo, out, 1, act_up ? 2 * W : W, act_up ? 2 * Hout : Hout, Co8,
                int64_t(act_up ? 4 : 1) * Hout * W * Co8, Co8, int64_t(act_up ? 2 * W : W) * Co8, 32,
                act_up ? 2 * kPix : kPix))
    return cudaErrorInvalidValue;
  // 256 output channels per tile (half the pixel-tile loads per FLOP) for Co >= 512, else 128 --
  // the choice must not depend on the band height, so that a banded decode runs the same tiles as
  // the whole image (bit-identical).  A/B on the persistent grid (profiles/r02_s3_ab_vae_cot.txt):
  // the 512-channel layer at 128^2 px 1116 TFLOP/s with 256-channel tiles vs 963 with 128; the
  // 256-channel layer at 256^2 px 871 vs 949 (its 256 tiles of 256 channels leave a 4th round of 74
  // clusters half empty).
#ifdef XDIT_VAE_WIDE_MIN  // A/B builds: the smallest Co that takes 256-channel tiles
  const bool wide = Co >= XDIT_VAE_WIDE_MIN;
#else
  const bool wide = Co >= 512;
#endif
  return wide ? launch_tcp<256>(mx, wt, mo, b, Hout, Ci, W, Co, act_up, st)
              : launch_tcp<128>(mx, wt, mo, b, Hout, Ci, W, Co, act_up, st);
}

}  // namespace xdit
