// attn_fwd_sm100.cu -- flash-attention forward for B200 (sm_100a) on 5th-gen tensor cores.
//
// Computes, for one (Q block, KV block) pair of the USP ring loop:
//     O = softmax(Q K^T / sqrt(D)) V   and   LSE = log sum_j exp(q.k_j / sqrt(D))
// -- the "full attention" of PAPER P:257 §4.1.2 evaluated blockwise as in "a parallel version of
// Flash Attention" (§4.1.1); readings C1 (scale 1/sqrt(D)), C2 (natural-log LSE), C3 (no mask
// other than the ragged KV tail), C10 (bf16 inputs, fp32 scores/accumulators, P rounded RNE to
// bf16 before P.V, O rounded RNE to bf16 on the final write).
//
// Design (B200-first):
//   * one CTA = 2 query tiles of 128 rows of one (batch, head) sharing every K/V tile;
//   * warp 8 issues TMA (128B-swizzled boxes of 128 rows x 64 columns) for Q once and for the
//     K_j, V_j stream through a ring of smem stages (mbarrier full/empty pairs);
//   * warp 9 (one lane) issues tcgen05.mma: S_t = Q_t K_j^T (SS, fp32 in TMEM) and
//     O_t += P_t V_j (TS: P_t read straight from TMEM, V from smem, MN-major);
//   * warps 0-3 / 4-7 are the softmax warpgroups of tile 0 / tile 1 (thread = query row = TMEM lane):
//     tcgen05.ld the 128 scores, online softmax in base 2 with a lazily updated running max (O is
//     rescaled in TMEM only when the max grows by more than 2^8), tcgen05.st of P as bf16 pairs
//     over the consumed S columns, then the epilogue (O / l, LSE) written through an xdit_rowmap.
//   The two tiles ping-pong: while one warpgroup runs exp2 on its S, the tensor core runs the
//   other tile's QK^T / PV, so MUFU and tensor pipes overlap.
// TMEM (512 columns x 128 lanes x 32 bit): S0 [0,128) S1 [128,256) O0 [256,256+D) O1 [256+D,256+2D);
// P_t aliases the first 64 columns of S_t.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "attn_common.cuh"

namespace xdit {
namespace {

constexpr int kBlockM = 128;      // query rows per tile (= TMEM lanes)
constexpr int kQTiles = 2;        // query tiles per CTA
constexpr int kBlockN = 128;      // keys per KV tile
constexpr int kThreads = 384;     // 2 softmax warpgroups + 1 warpgroup {TMA, MMA, 2 spare warps}
constexpr uint32_t kRegsSoftmax = 216, kRegsOther = 72;  // setmaxnreg split of 384 x 168 registers
constexpr int kWarpTma = 8;
constexpr int kWarpMma = 9;
constexpr float kRescaleThresh = 8.0f;  // log2 units: rescale O only if the max grows by > 2^8
constexpr float kRedoThresh = 64.0f;    // log2 units: recompute a tile whose P would exceed 2^64
constexpr uint32_t kTmemCols = 512;
// exp2 pairs (of every 8) evaluated by polynomial on the FMA pipe: D=128 is tensor/MUFU balanced and
// gains nothing (profiles/r01_ncu_attn_flux.md), D <= 80 is MUFU-bound and gains ~12%.
constexpr int default_emu(int D) { return D >= 128 ? 0 : 2; }

template <int D>
struct Cfg {
  // Head dim layout in smem: D/64 atoms of 64 columns, 128-byte swizzle; D = 72 adds one atom of 16
  // columns with 32-byte swizzle whose last 8 columns TMA zero-fills (K padded to the MMA K step 16).
  static constexpr int kN128 = D / 64;
  static constexpr bool kTail16 = (D % 64) != 0;
  static constexpr int kDp = kN128 * 64 + (kTail16 ? 16 : 0);  // padded head dim (MMA K / PV N)
  static constexpr int kAtom128 = kBlockM * 128;  // 128 rows x 128 B
  static constexpr int kAtom32 = kBlockM * 32;    // 128 rows x 32 B
  static constexpr int kTileBytes = kN128 * kAtom128 + (kTail16 ? kAtom32 : 0);
  static constexpr int kStages = (D == 128) ? 4 : 8;  // also forces 1 CTA/SM (TMEM is 512 cols)
  static constexpr int kSmemQ = kQTiles * kTileBytes;
  static constexpr int kSmemKV = kStages * kTileBytes;
  static constexpr int kSmemBar = 256;
  static constexpr int kSmemBytes = kSmemQ + kSmemKV + kSmemBar + 1024;
  static_assert(D == 64 || D == 72 || D == 128, "head dim");
  static_assert(kTileBytes % 1024 == 0, "tiles must keep 1024-byte alignment for the swizzle");
  __host__ __device__ static constexpr uint32_t col_s(int t) { return uint32_t(t) * 128u; }
  __host__ __device__ static constexpr uint32_t col_o(int t) { return 256u + uint32_t(t) * kDp; }
};


constexpr int kTraceIters = 64, kTraceEv = 16;
static_assert(kQTiles * kBlockM == kRowsPerItem, "work item = one query-tile pair");
__device__ __forceinline__ void stamp(const EpiParams& p, int j, int ev) {
  if (p.trace && j < kTraceIters && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 &&
      (threadIdx.x & 31) == 0)
    p.trace[j * kTraceEv + ev] = clock64();
}


// Pass 1 of the softmax of one 128-key tile: the row max of the raw scores S[row, 0:128) read from
// TMEM (this thread's lane).  MASK: keys >= valid are excluded (ragged KV tail).  Four independent
// FMNMX3 chains keep the dependency depth at 16.
template <bool MASK>
__device__ __forceinline__ float row_max(uint32_t tS, int valid) {
  float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
  for (int c = 0; c < 4; c += 2) {
    uint32_t a[32], bq[32];
    ptx::tmem_ld32(tS + c * 32, a);
    ptx::tmem_ld32(tS + c * 32 + 32, bq);
    ptx::tmem_ld_wait();
    if (MASK) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (c * 32 + i >= valid) a[i] = f2u(-INFINITY);
        if (c * 32 + 32 + i >= valid) bq[i] = f2u(-INFINITY);
      }
    }
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      m0 = fmax3(m0, u2f(a[i]), u2f(a[i + 1]));
      m1 = fmax3(m1, u2f(a[i + 2]), u2f(a[i + 3]));
      m2 = fmax3(m2, u2f(bq[i]), u2f(bq[i + 1]));
      m3 = fmax3(m3, u2f(bq[i + 2]), u2f(bq[i + 3]));
    }
  }
  return fmax3(m0, m1, fmaxf(m2, m3));
}


// Pass 2: P = exp2(S * scale*log2e - m) for the tile, written back to TMEM as bf16 pairs over the
// first 64 columns of S (the A operand of the P.V MMA).  Returns the fp32 row sum of P.
// FFMA2 / FADD2 process two columns per instruction; MUFU.EX2 does the exponentials except for EMU
// of every 8 column pairs, which use exp2_poly2 on the FMA pipe so MUFU stops being the co-bottleneck.
template <bool MASK, int EMU>
__device__ __forceinline__ float exp_store_p(uint32_t tS, int valid, float sl2, float neg_m) {
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(neg_m, neg_m);
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t a[32], bq[32], pk[32];
    ptx::tmem_ld32(tS + half * 64, a);
    ptx::tmem_ld32(tS + half * 64 + 32, bq);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t* src = (i < 16) ? a : bq;
      const int e = (i & 15) * 2, col = half * 64 + (i < 16 ? 0 : 32) + e;
      const uint64_t x = fma2(pk2(u2f(src[e]), u2f(src[e + 1])), sc2, nm2);
      float p0, p1;
      if ((i & 7) < EMU) {
        up2(exp2_poly2(x), p0, p1);
      } else {
        float x0, x1;
        up2(x, x0, x1);
        p0 = ptx::ex2(x0);
        p1 = ptx::ex2(x1);
      }
      if (MASK) {
        if (col >= valid) p0 = 0.f;
        if (col + 1 >= valid) p1 = 0.f;
      }
      if (i & 1) acc1 = add2(acc1, pk2(p0, p1));
      else acc0 = add2(acc0, pk2(p0, p1));
      pk[i] = ptx::pack_bf16x2(p0, p1);
    }
    ptx::tmem_st32(tS + half * 32, pk);
  }
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  return (s0 + s1) + (s2 + s3);
}

// One pass over the tile: P = exp2(S * scale*log2e - m) for all 128 keys into 64 packed bf16x2
// registers (nothing is written to TMEM yet, so S stays intact for a redo), the fp32 row sum of P
// and the row max of the raw scores.  The two 64-column halves are read with two LDTM each.
template <bool MASK, int EMU>
__device__ __forceinline__ void exp_tile_regs(uint32_t tS, int valid, float sl2, float neg_m,
                                              uint32_t (&pk)[64], float& rs, float& mx) {
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(neg_m, neg_m);
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    uint32_t a[32], bq[32];
    ptx::tmem_ld32(tS + half * 64, a);
    ptx::tmem_ld32(tS + half * 64 + 32, bq);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const uint32_t* src = (i < 16) ? a : bq;
      const int e = (i & 15) * 2, col = half * 64 + (i < 16 ? 0 : 32) + e;
      float s0 = u2f(src[e]), s1 = u2f(src[e + 1]);
      if (MASK) {
        if (col >= valid) s0 = -INFINITY;
        if (col + 1 >= valid) s1 = -INFINITY;
      }
      if (i & 1) m1 = fmax3(m1, s0, s1);
      else m0 = fmax3(m0, s0, s1);
      const uint64_t x = fma2(pk2(s0, s1), sc2, nm2);
      float p0, p1;
      if (!MASK && (i & 7) < EMU) {
        up2(exp2_poly2(x), p0, p1);
      } else {
        float x0, x1;
        up2(x, x0, x1);
        p0 = ptx::ex2(x0);
        p1 = ptx::ex2(x1);
      }
      if (i & 1) acc1 = add2(acc1, pk2(p0, p1));
      else acc0 = add2(acc0, pk2(p0, p1));
      pk[half * 32 + i] = ptx::pack_bf16x2(p0, p1);
    }
  }
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  rs = (s0 + s1) + (s2 + s3);
  mx = fmaxf(m0, m1);
}

// One 64-column half of a 128-key tile: P = exp2(S * scale*log2e - m) for S columns
// [col0, col0 + 64) into 32 packed bf16x2 registers (nothing written to TMEM yet, so the half can be
// recomputed), the fp32 row sum of those P and the row max of the raw scores.
template <bool MASK, int EMU>
__device__ __forceinline__ void exp_regs64(const uint32_t (&a)[32], const uint32_t (&bq)[32], int col0,
                                           int valid, float sl2, float neg_m, uint32_t (&pk)[32],
                                           float& rs, float& mx) {
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(neg_m, neg_m);
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
  float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const uint32_t* src = (i < 16) ? a : bq;
    const int e = (i & 15) * 2, col = col0 + (i < 16 ? 0 : 32) + e;
    float s0 = u2f(src[e]), s1 = u2f(src[e + 1]);
    if (MASK) {
      if (col >= valid) s0 = -INFINITY;
      if (col + 1 >= valid) s1 = -INFINITY;
    }
    if (i & 1) m1 = fmax3(m1, s0, s1);
    else m0 = fmax3(m0, s0, s1);
    const uint64_t x = fma2(pk2(s0, s1), sc2, nm2);
    float p0, p1;
    if (!MASK && (i & 7) < EMU) {
      up2(exp2_poly2(x), p0, p1);
    } else {
      float x0, x1;
      up2(x, x0, x1);
      p0 = ptx::ex2(x0);
      p1 = ptx::ex2(x1);
    }
    if (i & 1) acc1 = add2(acc1, pk2(p0, p1));
    else acc0 = add2(acc0, pk2(p0, p1));
    pk[i] = ptx::pack_bf16x2(p0, p1);
  }
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  rs = (s0 + s1) + (s2 + s3);
  mx = fmaxf(m0, m1);
}

template <bool MASK, int EMU>
__device__ __forceinline__ void exp_half64(uint32_t tS, int col0, int valid, float sl2, float neg_m,
                                           uint32_t (&pk)[32], float& rs, float& mx) {
  uint32_t a[32], bq[32];
  ptx::tmem_ld32(tS + col0, a);
  ptx::tmem_ld32(tS + col0 + 32, bq);
  ptx::tmem_ld_wait();
  exp_regs64<MASK, EMU>(a, bq, col0, valid, sl2, neg_m, pk, rs, mx);
}

template <int D, int EMU>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_sm100_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmQ16,
                          const __grid_constant__ CUtensorMap tmK16,
                          const __grid_constant__ CUtensorMap tmV16, const EpiParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sKV = smem + C::kSmemQ;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kSmemKV);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;
  uint64_t* p_full = s_full + 2;             // [t][half]: P of keys [64 half, 64 half + 64) stored
  uint64_t* o_half = p_full + 4;             // [t]: PV of the first key half of tile t completed
  uint64_t* o_full = o_half + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int item = blockIdx.x, kv0 = 0, kv_len = p.Skv, piece = -1;
  if (item >= p.n_full) {  // tail item: one key range of a split (query-tile pair, head, batch)
    const int r = item - p.n_full;
    piece = r;
    item = p.n_full + r / p.n_split;
    kv0 = (r % p.n_split) * p.kv_chunk;
    kv_len = min(p.kv_chunk, p.Skv - kv0);
  }
  const int hb = item / p.n_qt, h = hb % p.H, b = hb / p.H;
  const int m0 = (item % p.n_qt) * (kQTiles * kBlockM);
  const int n_kv = (kv_len + kBlockN - 1) / kBlockN;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&p_full[2 * t], 4);  // one arrive per softmax warp
      ptx::mbar_init(&p_full[2 * t + 1], 4);
      ptx::mbar_init(&o_half[t], 1);
      ptx::mbar_init(&o_full[t], 1);
    }
    ptx::fence_mbar_init();
  }
  if (warp == kWarpMma) {
    ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tmem_relinquish();
  }
  if (warp == kWarpTma && lane == 0) {
    ptx::tma_prefetch_desc(&tmQ);
    ptx::tma_prefetch_desc(&tmK);
    ptx::tma_prefetch_desc(&tmV);
    if (C::kTail16) {
      ptx::tma_prefetch_desc(&tmQ16);
      ptx::tma_prefetch_desc(&tmK16);
      ptx::tma_prefetch_desc(&tmV16);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
   // warpgroup 2: TMA producer (warp 8), MMA issuer (warp 9), two spare warps -- few registers
   ptx::setmaxnreg_dec<kRegsOther>();
   if (warp == kWarpTma) {
    // ===================================================== TMA producer
    {  // converged warp; one elected lane issues (operands stay in the uniform datapath)
      const uint64_t pol_q = ptx::policy_evict_first();
      const uint64_t pol_kv = ptx::policy_evict_last();
      if (ptx::elect_one()) {
        ptx::mbar_expect_tx(q_full, kQTiles * C::kTileBytes);
        for (int t = 0; t < kQTiles; ++t) {
          for (int c = 0; c < C::kN128; ++c)
            ptx::tma_load_4d(sQ + t * C::kTileBytes + c * C::kAtom128, &tmQ, q_full, c * 64, h,
                             m0 + t * kBlockM, b, pol_q);
          if (C::kTail16)
            ptx::tma_load_4d(sQ + t * C::kTileBytes + C::kN128 * C::kAtom128, &tmQ16, q_full,
                             C::kN128 * 64, h, m0 + t * kBlockM, b, pol_q);
        }
      }
      __syncwarp();
      int it = 0;
      for (int j = 0; j < n_kv; ++j) {
        for (int kv = 0; kv < 2; ++kv, ++it) {
          const int stage = it % C::kStages, round = it / C::kStages;
          if (round > 0) ptx::mbar_wait(&kv_empty[stage], (round - 1) & 1);
          if (ptx::elect_one()) {
            ptx::mbar_expect_tx(&kv_full[stage], C::kTileBytes);
            for (int c = 0; c < C::kN128; ++c)
              ptx::tma_load_4d(sKV + stage * C::kTileBytes + c * C::kAtom128, kv ? &tmV : &tmK,
                               &kv_full[stage], c * 64, h, kv0 + j * kBlockN, b, pol_kv);
            if (C::kTail16)
              ptx::tma_load_4d(sKV + stage * C::kTileBytes + C::kN128 * C::kAtom128,
                               kv ? &tmV16 : &tmK16, &kv_full[stage], C::kN128 * 64, h, kv0 + j * kBlockN,
                               b, pol_kv);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == kWarpMma) {
    // ===================================================== MMA issuer (single thread)
    {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(kBlockM, kBlockN, 0, 0);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(kBlockM, C::kTail16 ? 64 : D, 0, 1);
      constexpr uint32_t idesc_pv16 = ptx::idesc_bf16_f32(kBlockM, 16, 0, 1);
      const uint32_t sQa = ptx::smem_u32(sQ), sKVa = ptx::smem_u32(sKV);
      // K-major operand (Q or K tile): 16-element K step k lives in 128B atom k/4 at byte 32*(k%4);
      // the D=72 tail step is the whole 32-byte row of the 32B-swizzled atom.
      auto kmaj = [&](uint32_t base, int k) -> uint64_t {
        if (C::kTail16 && k == C::kN128 * 4)
          return ptx::sdesc(base + C::kN128 * C::kAtom128, 16, 8 * 32, ptx::kLayoutSW32);
        return ptx::sdesc_sw128(base + (k >> 2) * C::kAtom128 + (k & 3) * 32, 16, 1024);
      };
      // MN-major V tile: 16-key step k starts at row 16k; 64-column atoms are kAtom128 apart.
      auto vdesc = [&](int stage, int k) -> uint64_t {
        return ptx::sdesc_sw128(sKVa + stage * C::kTileBytes + k * 16 * 128, C::kAtom128, 1024);
      };
      auto vdesc16 = [&](int stage, int k) -> uint64_t {  // D=72 tail: 16 columns, 32B swizzle
        return ptx::sdesc(sKVa + stage * C::kTileBytes + C::kN128 * C::kAtom128 + k * 16 * 32, 16,
                          8 * 32, ptx::kLayoutSW32);
      };
      auto kv_wait = [&](int idx) -> int {
        const int stage = idx % C::kStages;
        ptx::mbar_wait(&kv_full[stage], (idx / C::kStages) & 1);
        ptx::tc_fence_after();
        return stage;
      };
      auto qk = [&](int t, int sK) {
        const uint32_t qa = sQa + t * C::kTileBytes, ka = sKVa + sK * C::kTileBytes;
#pragma unroll
        for (int k = 0; k < C::kDp / 16; ++k)
          ptx::mma_ss(tmem + C::col_s(t), kmaj(qa, k), kmaj(ka, k), idesc_qk, k > 0 ? 1u : 0u);
      };
      // O_t += P_t V for key half hf (16-key steps 4hf .. 4hf+3)
      auto pv = [&](int t, int sV, bool acc, int hf) {
#pragma unroll
        for (int k = 4 * hf; k < 4 * hf + 4; ++k) {
          ptx::mma_ts(tmem + C::col_o(t), tmem + C::col_s(t) + k * 8, vdesc(sV, k), idesc_pv,
                      (acc || k > 0) ? 1u : 0u);
          if (C::kTail16)
            ptx::mma_ts(tmem + C::col_o(t) + 64, tmem + C::col_s(t) + k * 8, vdesc16(sV, k),
                        idesc_pv16, (acc || k > 0) ? 1u : 0u);
        }
      };

      // PV of tile t, step jj: first key half as soon as the softmax released it (then commit
      // o_half so a rare mid-tile O rescale can wait for it), second half when released.
      auto pv_tile = [&](int t, int sV, int jj) {
        if (p.diag < 2) ptx::mbar_wait(&p_full[2 * t], jj & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          pv(t, sV, jj > 0, 0);
          ptx::tc_commit(&o_half[t]);
        }
        __syncwarp();
        if (p.diag < 2) ptx::mbar_wait(&p_full[2 * t + 1], jj & 1);
        if (t == 0) stamp(p, jj, 14);
        ptx::tc_fence_after();
        if (ptx::elect_one()) pv(t, sV, true, 1);
        __syncwarp();
      };

      ptx::mbar_wait(q_full, 0);
      ptx::tc_fence_after();
      int sVprev = 0;
      for (int j = 0; j < n_kv; ++j) {
        stamp(p, j, 13);
        const int sK = kv_wait(2 * j);
        stamp(p, j, 0);
        if (ptx::elect_one()) {
          qk(0, sK);  // S0 = Q0 K_j^T
          ptx::tc_commit(&s_full[0]);
        }
        __syncwarp();
        stamp(p, j, 1);
        if (j > 0) {  // O1 += P1(j-1) V_{j-1}, key half by key half as the softmax releases them
          pv_tile(1, sVprev, j - 1);
          stamp(p, j, 2);
          if (ptx::elect_one()) ptx::tc_commit(&kv_empty[sVprev]);
          __syncwarp();
        }
        if (ptx::elect_one()) {
          qk(1, sK);  // S1 = Q1 K_j^T
          ptx::tc_commit(&s_full[1]);
          ptx::tc_commit(&kv_empty[sK]);
        }
        __syncwarp();
        const int sV = kv_wait(2 * j + 1);
        stamp(p, j, 3);
        pv_tile(0, sV, j);  // O0 += P0(j) V_j
        stamp(p, j, 4);
        if (j == n_kv - 1) {
          if (ptx::elect_one()) ptx::tc_commit(&o_full[0]);
          __syncwarp();
        }
        sVprev = sV;
      }
      pv_tile(1, sVprev, n_kv - 1);
      if (ptx::elect_one()) {
        ptx::tc_commit(&o_full[1]);
        ptx::tc_commit(&kv_empty[sVprev]);
      }
      __syncwarp();
    }
   }
  } else {
    ptx::setmaxnreg_inc<kRegsSoftmax>();
    // ===================================================== softmax warpgroups (tile t = warp/4)
    const int t = warp >> 2, wq = warp & 3;
    const int row_in_tile = wq * 32 + lane;
    const uint32_t lane_off = uint32_t(wq * 32) << 16;
    const uint32_t tS = tmem + C::col_s(t) + lane_off;
    const uint32_t tO = tmem + C::col_o(t) + lane_off;
    const float sl2 = p.scale_log2;
    float m_used = 0.f, m_next = 0.f, l = 0.f;
    // O and l <- O, l * 2^(m_used - m_new); m_used <- m_new (warp-collective TMEM ld/st of O).
    auto rescale_o = [&](float m_new) {
      const float alpha = ptx::ex2(m_used - m_new);
      l *= alpha;
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        ptx::tmem_ld32(tO + c * 32, o);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * alpha);
        ptx::tmem_st32(tO + c * 32, o);
      }
      if (D % 32) {  // D = 72: columns 64..71 (64..79 of the padded O hold zeros)
        uint32_t o[8];
        ptx::tmem_ld8(tO + (D / 32) * 32, o);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = f2u(u2f(o[i]) * alpha);
        ptx::tmem_st8(tO + (D / 32) * 32, o);
      }
      m_used = m_new;
    };
    for (int j = 0; j < n_kv; ++j) {
      ptx::mbar_wait(&s_full[t], j & 1);
      if ((warp & 3) == 0 && lane == 0) stamp(p, j, 5 + 2 * t);
      ptx::tc_fence_after();
      if (p.diag) {  // profiling: measure the MMA/TMA skeleton without the softmax
        __syncwarp();
        if (lane == 0) {
          ptx::mbar_arrive(&p_full[2 * t]);
          ptx::mbar_arrive(&p_full[2 * t + 1]);
        }
        continue;
      }
      const bool ragged = (j == n_kv - 1) && (kv_len - j * kBlockN < kBlockN);
      const int valid = kv_len - j * kBlockN;  // ragged KV tail of this key range (reading C16)
      // Reading R1 (lazy max): P of tile j is computed against the running reference m_used in ONE
      // pass over S (no separate max pass on the critical path); the tile max found on the way only
      // moves m_used -- and rescales O and l -- before the NEXT tile, when it grew by more than
      // 2^kRescaleThresh.  A tile whose max exceeds m_used by more than kRedoThresh (P would exceed
      // 2^kRedoThresh) is recomputed against its own max: S is still intact in TMEM at that point.
      if (j == 0) {
        m_used = (ragged ? row_max<true>(tS, valid) : row_max<false>(tS, valid)) * sl2;
      } else if (__any_sync(0xffffffffu, m_next > m_used)) {
        rescale_o(m_next);  // PV(j-1) is complete: s_full(j) was committed after it
      }
      // The tile is processed in two 64-key halves; P of the first half is stored and released to
      // the MMA warp (p_full[t][0]) before the second half is computed, so the tensor core runs
      // PV over keys 0..63 while the exps of keys 64..127 are still in flight.
      float m_tile;
      uint32_t s0a[32], s0b[32], s1a[32], s1b[32];  // all 128 scores, one TMEM round trip
      ptx::tmem_ld32(tS, s0a);
      ptx::tmem_ld32(tS + 32, s0b);
      ptx::tmem_ld32(tS + 64, s1a);
      ptx::tmem_ld32(tS + 96, s1b);
      ptx::tmem_ld_wait();
      if ((warp & 3) == 0 && lane == 0) stamp(p, j, 9 + 2 * t);
      {
        uint32_t pk[32];
        float rs, mx;
        if (ragged) exp_regs64<true, 0>(s0a, s0b, 0, valid, sl2, -m_used, pk, rs, mx);
        else exp_regs64<false, EMU>(s0a, s0b, 0, valid, sl2, -m_used, pk, rs, mx);
        if (__any_sync(0xffffffffu, mx * sl2 > m_used + kRedoThresh)) {  // rare: recompute
          rescale_o(fmaxf(m_used, mx * sl2));  // PV(j-1) complete; PV(j) not issued yet
          if (ragged) exp_half64<true, 0>(tS, 0, valid, sl2, -m_used, pk, rs, mx);
          else exp_half64<false, EMU>(tS, 0, valid, sl2, -m_used, pk, rs, mx);
        }
        l += rs;
        m_tile = mx * sl2;
        ptx::tmem_st32(tS, pk);  // P keys 0..63 -> packed columns 0..31 (their scores are consumed)
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[2 * t]);
        if ((warp & 3) == 0 && lane == 0) stamp(p, j, 10 + 2 * t);
      }
      {
        uint32_t pk[32];
        float rs, mx;
        if (ragged) exp_regs64<true, 0>(s1a, s1b, 64, valid, sl2, -m_used, pk, rs, mx);
        else exp_regs64<false, EMU>(s1a, s1b, 64, valid, sl2, -m_used, pk, rs, mx);
        if (__any_sync(0xffffffffu, mx * sl2 > m_used + kRedoThresh)) {  // rare: recompute
          // O already received PV over keys 0..63: wait for it (o_half completes once per step and
          // PV(j+1) cannot start before this warp arrives, so the parity wait is exact), then
          // rescale O and l together and recompute this half against the new reference.
          ptx::mbar_wait(&o_half[t], j & 1);
          ptx::tc_fence_after();
          rescale_o(fmaxf(m_used, mx * sl2));
          if (ragged) exp_half64<true, 0>(tS, 64, valid, sl2, -m_used, pk, rs, mx);
          else exp_half64<false, EMU>(tS, 64, valid, sl2, -m_used, pk, rs, mx);
        }
        l += rs;
        m_tile = fmaxf(m_tile, mx * sl2);
        ptx::tmem_st32(tS + 32, pk);  // P keys 64..127 -> packed columns 32..63
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&p_full[2 * t + 1]);
      }
      m_next = (m_tile > m_used + kRescaleThresh) ? m_tile : m_used;
      if ((warp & 3) == 0 && lane == 0) stamp(p, j, 6 + 2 * t);
    }
    // ------------------------------------------------- epilogue: O / l, LSE
    ptx::mbar_wait(&o_full[t], 0);
    ptx::tc_fence_after();
    const int row = m0 + t * kBlockM + row_in_tile;
    const float inv_l = 1.f / l;
    RowDst dst = rowmap_dst(p.map, b, row, h);
    void* obase = p.o;
    float* lbase = p.lse;
    int of32 = p.out_f32;
    if (piece >= 0) {  // split tail item: normalised fp32 partial for tail_merge_kernel
      const int64_t prow = int64_t(piece) * (kQTiles * kBlockM) + t * kBlockM + row_in_tile;
      const int64_t n_pieces = int64_t(gridDim.x) - p.n_full;
      obase = p.part;
      lbase = p.part + n_pieces * (kQTiles * kBlockM) * D;
      of32 = 1;
      dst.o_off = prow * D;
      dst.l_off = prow;
    }
    const bool valid = row < p.Sq;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      ptx::tmem_ld32(tO + c * 32, o);
      ptx::tmem_ld_wait();
      if (valid) {
        if (of32) {
          float4* dstp = reinterpret_cast<float4*>(static_cast<float*>(obase) + dst.o_off + c * 32);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            dstp[i] = make_float4(u2f(o[4 * i]) * inv_l, u2f(o[4 * i + 1]) * inv_l,
                                  u2f(o[4 * i + 2]) * inv_l, u2f(o[4 * i + 3]) * inv_l);
        } else {
          uint4* dstp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(obase) + dst.o_off + c * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dstp[i] = make_uint4(ptx::pack_bf16x2(u2f(o[8 * i]) * inv_l, u2f(o[8 * i + 1]) * inv_l),
                                 ptx::pack_bf16x2(u2f(o[8 * i + 2]) * inv_l, u2f(o[8 * i + 3]) * inv_l),
                                 ptx::pack_bf16x2(u2f(o[8 * i + 4]) * inv_l, u2f(o[8 * i + 5]) * inv_l),
                                 ptx::pack_bf16x2(u2f(o[8 * i + 6]) * inv_l, u2f(o[8 * i + 7]) * inv_l));
        }
      }
    }
    if (D % 32) {  // D = 72 tail columns 64..71
      uint32_t o[8];
      ptx::tmem_ld8(tO + (D / 32) * 32, o);
      ptx::tmem_ld_wait();
      if (valid) {
        if (of32) {
          float4* dstp = reinterpret_cast<float4*>(static_cast<float*>(obase) + dst.o_off + (D / 32) * 32);
          dstp[0] = make_float4(u2f(o[0]) * inv_l, u2f(o[1]) * inv_l, u2f(o[2]) * inv_l, u2f(o[3]) * inv_l);
          dstp[1] = make_float4(u2f(o[4]) * inv_l, u2f(o[5]) * inv_l, u2f(o[6]) * inv_l, u2f(o[7]) * inv_l);
        } else {
          uint4* dstp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(obase) + dst.o_off + (D / 32) * 32);
          dstp[0] = make_uint4(ptx::pack_bf16x2(u2f(o[0]) * inv_l, u2f(o[1]) * inv_l),
                               ptx::pack_bf16x2(u2f(o[2]) * inv_l, u2f(o[3]) * inv_l),
                               ptx::pack_bf16x2(u2f(o[4]) * inv_l, u2f(o[5]) * inv_l),
                               ptx::pack_bf16x2(u2f(o[6]) * inv_l, u2f(o[7]) * inv_l));
        }
      }
    }
    if (valid && lbase) lbase[dst.l_off] = (m_used + log2f(l)) * 0.69314718055994530942f;
  }
  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == kWarpMma) ptx::tmem_dealloc(tmem, kTmemCols);
}


// ------------------------------------------------------------------ host side

template <int D, int EMU>
cudaError_t launch_kernel(dim3 grid, const CUtensorMap* m, const EpiParams& p, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_sm100_kernel<D, EMU>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  attn_fwd_sm100_kernel<D, EMU><<<grid, kThreads, Cfg<D>::kSmemBytes, st>>>(m[0], m[1], m[2], m[3], m[4],
                                                                           m[5], p);
  note_launches(1);
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D>;
  CUtensorMap m[6];
  if (!make_map(&m[0], a.q, a.B, a.Sq, a.H, D, a.q_b, a.q_s, a.q_h) ||
      !make_map(&m[1], a.k, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h) ||
      !make_map(&m[2], a.v, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h))
    return cudaErrorInvalidValue;
  if (C::kTail16) {
    if (!make_map(&m[3], a.q, a.B, a.Sq, a.H, D, a.q_b, a.q_s, a.q_h, 16) ||
        !make_map(&m[4], a.k, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, 16) ||
        !make_map(&m[5], a.v, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, 16))
      return cudaErrorInvalidValue;
  } else {
    m[3] = m[0];
    m[4] = m[1];
    m[5] = m[2];
  }
  EpiParams p;
  p.o = a.o;
  p.lse = a.lse;
  p.map = a.omap;
  p.H = a.H;
  p.Sq = a.Sq;
  p.Skv = a.Skv;
  p.out_f32 = a.out_f32;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(D)));
  static const int diag = [] {
    const char* e = std::getenv("XDIT_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  p.diag = diag;
  static unsigned long long* trace = [] {
    unsigned long long* t = nullptr;
    if (std::getenv("XDIT_TRACE")) cudaMalloc(&t, sizeof(unsigned long long) * kTraceIters * kTraceEv);
    return t;
  }();
  p.trace = trace;
  if (trace) cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * kTraceIters * kTraceEv, st);
  // 1-D grid over (query-tile pair, head, batch) items; split the last partial wave over key
  // ranges when a scratch buffer is available (DESIGN.md §7.1 "tail split").
  p.n_qt = (a.Sq + kQTiles * kBlockM - 1) / (kQTiles * kBlockM);
  const int items = p.n_qt * a.H * a.B;
  p.n_full = items;
  p.n_split = 1;
  p.kv_chunk = a.Skv;
  p.part = nullptr;
  int n_tail = 0;
  static const int nsm = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  static const bool no_split = std::getenv("XDIT_NO_TAIL_SPLIT") != nullptr;
  if (a.scratch && !no_split && items > nsm && items % nsm) {
    const int rem = items % nsm, n_kv_tiles = (a.Skv + kBlockN - 1) / kBlockN;
    int ns = std::min(std::min(nsm / rem, 8), n_kv_tiles / 2);
    if (ns >= 2) {
      const int chunk = ((n_kv_tiles + ns - 1) / ns) * kBlockN;
      ns = (a.Skv + chunk - 1) / chunk;
      const size_t need = size_t(rem) * ns * (kQTiles * kBlockM) * (D + 1);
      if (ns >= 2 && need <= a.scratch_floats) {
        n_tail = rem;
        p.n_full = items - rem;
        p.n_split = ns;
        p.kv_chunk = chunk;
        p.part = a.scratch;
      }
    }
  }
  dim3 grid(p.n_full + n_tail * p.n_split);
  // fraction of exp2 moved to the FMA pipe: EMU of every 8 column pairs (XDIT_EXP_EMU overrides)
  static const int emu = [] {
    const char* e = std::getenv("XDIT_EXP_EMU");
    return e ? std::atoi(e) : -1;
  }();
  cudaError_t err;
  switch (emu >= 0 ? emu : default_emu(D)) {
    case 0: err = launch_kernel<D, 0>(grid, m, p, st); break;
    case 3: err = launch_kernel<D, 3>(grid, m, p, st); break;
    case 4: err = launch_kernel<D, 4>(grid, m, p, st); break;
    default: err = launch_kernel<D, 2>(grid, m, p, st); break;
  }
  if (err == cudaSuccess && n_tail) {
    const int rows = n_tail * kQTiles * kBlockM;
    tail_merge_kernel<D><<<(rows + 7) / 8, 256, 0, st>>>(p.part, n_tail, p.n_split, p.n_full, p.n_qt,
                                                          a.H, a.Sq, p);
    note_launches(1);
    err = cudaGetLastError();
  }
  if (trace) {  // profiling only: print CTA 0's stamps relative to its first K arrival
    unsigned long long h[kTraceIters * kTraceEv];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[0];
    fprintf(stderr, "j kready qk0iss p1seen p0wait p0seen | s0seen p0arr s1seen p1arr | ld0 h0arr ld1 h1arr\n");
    for (int j = 0; j < kTraceIters; ++j) {
      fprintf(stderr, "%d", j);
      for (int e = 0; e < 15; ++e)
        fprintf(stderr, " %lld", h[j * kTraceEv + e] ? (long long)(h[j * kTraceEv + e] - t0) : -1LL);
      fprintf(stderr, "\n");
    }
  }
  return err;
}

}  // namespace

size_t attn_scratch_floats(int D) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return size_t(nsm) * (kQTiles * kBlockM) * size_t(D + 1);
}

static bool force_1sm_kernel() {
  // XDIT_ATTN_KERNEL=1sm forces the one-CTA kernel where the CTA-pair kernel would run.
  static const bool force = [] {
    const char* e = std::getenv("XDIT_ATTN_KERNEL");
    return e && std::string(e) == "1sm";
  }();
  return force;
}

bool attn_fused_merge_supported(int D) { return !force_1sm_kernel() && attn_fwd_2sm_supports(D); }

cudaError_t launch_attn_fwd_sm100(const AttnArgs& a, cudaStream_t st) {
  if (a.Sq == 0 || a.B == 0) return cudaSuccess;
  const bool force_1sm = force_1sm_kernel();
  if (a.merge && (force_1sm || !attn_fwd_2sm_supports(a.D))) return cudaErrorInvalidValue;
  if (!force_1sm && attn_fwd_2sm_supports(a.D)) return launch_attn_fwd_2sm(a, st);
  switch (a.D) {
    case 64: return launch_d<64>(a, st);
    case 72: return launch_d<72>(a, st);
    case 128: return launch_d<128>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace xdit
