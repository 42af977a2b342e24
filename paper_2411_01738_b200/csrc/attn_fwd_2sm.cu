// attn_fwd_2sm.cu -- persistent flash-attention forward on CTA PAIRS (cta_group::2) for B200 (sm_100a).
//
// The bf16 attention of the hot path (§4.1.1 / P:257 §4.1.2;
// readings C1-C3, C10, R1): O = softmax(Q K^T / sqrt(D)) V and LSE for one (Q block, KV block),
// with the ring's LSE merge (a7) and the bf16 cast + reverse-all-to-all pack (a8) fused into the
// epilogue.
//
// Why a CTA pair: in a one-CTA kernel holding two query tiles the S_t / P_t TMEM
// columns alias, so QK^T of the next key tile of a query tile cannot start before the P.V of the
// current one -- every step of a tile is a serial chain softmax -> PV -> QK^T, and the tensor core
// idled ~40 % (round 1's one-CTA kernel, profiles/r01_ncu_attn_flux.md; retired in round 2, in git
// history).  Here the two SMs of a TPC run one 256-row work unit together with M = 256 MMAs, which
// frees TMEM for DOUBLE-BUFFERED S and P per SM:
//   * CTA rank r owns query rows [128 r, 128 r + 128) of the unit: its Q tile, its S/P/O in TMEM;
//   * each CTA loads HALF of every K tile (keys [64 r, 64 r + 64)) and HALF of every V tile
//     (head-dim columns [D/2 r, D/2 r + D/2)): the pair's MMAs read the other half from the peer SM,
//     so L2->SM traffic per SM equals the one-CTA kernel's (two query tiles per K/V load) and the
//     smem operand traffic per SM drops to 3/4 (QK^T) and 1/2 (PV);
//   * the leader's MMA warp issues QK^T(g+2) into S[g%2] as soon as the softmax has loaded S(g)
//     into registers -- before PV(g) -- so the tensor core has the next score tile queued while the
//     softmax of step g runs; P(g) goes to P[g%2], free once PV(g-2) has completed;
//   * 8 softmax warps per CTA, two per TMEM lane quarter, alternating key tiles (see the softmax
//     section): one runs its exp2 stream while the other loads its S; P is computed against a
//     reference max without a max pass and reconciled with the other warp's reference at the end of
//     the step (reading R1').
// PERSISTENT (round 2): one CTA pair per TPC loops over work units (a unit = 256 query rows of one
// (batch, head) against its key range), so the per-unit prologue (launch, barrier init, TMEM
// allocation, Q load latency, pipeline fill) and the drain are paid once per pair instead of once
// per unit (measured 5.5-6 us per unit in the non-persistent kernel, profiles/r02_sweep_items_nonpersistent.txt --
// 17 % of a PixArt/SD3-sized unit).  Q is double-buffered in smem, so the next unit's first two
// QK^T run while the current unit's last P.V and epilogue drain; the first P.V of a unit waits only
// until the previous unit's epilogue has read O out of TMEM (o_empty).  The K/V smem ring, the S/P
// TMEM buffers and every barrier phase continue across units (global tile counter g).  Units are
// handed out by an atomic counter in the caller's scratch (dynamic: pairs that start late -- e.g.
// behind a concurrent NCCL kernel of the ring's side stream -- simply take fewer units) or, without
// scratch, round-robin; the leader's TMA warp fetches each unit id and broadcasts it through a small
// smem ring into both CTAs.
// TMEM per SM (512 columns): S[0] [0,128) S[1] [128,256) P[0] [256,320) P[1] [320,384) O [384,384+D);
// at D = 64 also Q[0] [448,480) Q[1] [480,512) (QK^T reads Q from TMEM, copied in by tcgen05.cp).
// Head dims 128, 72 and 64 (the V halves of D = 64 are 32 columns: 64-byte swizzled rows).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "attn_common.cuh"

namespace xdit {
namespace {

namespace pair2 {

constexpr int kThreads = 384;      // 8 softmax warps, TMA warp, MMA warp, 2 idle warps
constexpr int kWarpTma = 8, kWarpMma = 9;

constexpr int kRows = 128;         // query rows per CTA (= TMEM lanes)
constexpr int kKeys = 128;         // keys per step
constexpr float kMoveThresh = 40.0f;    // log2 units: a reference jump above 2^40 moves it (R1')
constexpr uint32_t kTmemCols = 512;
constexpr int kRing = 8;           // work-unit broadcast ring depth (units in flight <= 5, see below)
// exp2 pairs (of every 8) the softmax evaluates with the FMA-pipe polynomial instead of MUFU.EX2:
// 1 (same-session A/B with the deferred reconciliation, profiles/r02_ab_softmax.txt: +1-4 % over 0
// at every head dim, 2 is slower).  A/B builds set it with -DXDIT_EXP_EMU=n.
#ifndef XDIT_EXP_EMU
#define XDIT_EXP_EMU 1
#endif
#ifdef XDIT_PROFILE
constexpr int kTraceIters = 96, kTraceEv = 8, kTraceWarps = 10;
#endif
// Profiling builds only (-DXDIT_PROFILE, tools/trace_attn.py): clock64 stamps of every warp role of
// the first CTA pair per global key tile g (XDIT_PROFILE_TRACE=<file>: raw dump after the launch)
// and the softmax-free skeleton (XDIT_PROFILE_DIAG=1).
__device__ __forceinline__ void stamp(const EpiParams& p, uint32_t g, int ev) {
#ifdef XDIT_PROFILE
  const int warp = threadIdx.x >> 5;
  if (p.trace && g < uint32_t(kTraceIters) && blockIdx.x < 2 && (threadIdx.x & 31) == 0 && warp < kTraceWarps)
    p.trace[((blockIdx.x * kTraceWarps + warp) * kTraceIters + g) * kTraceEv + ev] = clock64();
#endif
}

template <int D>
struct Cfg {
  static_assert(D == 128 || D == 64 || D == 72, "CTA-pair kernel: D in {64, 72, 128}");
  // Q / K rows (K-major): D/64 atoms of 64 columns with 128-byte swizzle; D = 72 adds one atom of
  // 16 columns with 32-byte swizzle whose last 8 columns the TMA zero-fills (QK^T K extent 80).
  static constexpr int kN128 = D / 64;
  static constexpr bool kTail = (D % 64) != 0;
  static constexpr int kDpK = kN128 * 64 + (kTail ? 16 : 0);
  static constexpr int kAtom = kRows * 128, kAtomT = kRows * 32;      // Q atoms (128 rows)
  static constexpr int kKHalfAtom = 64 * 128, kKHalfAtomT = 64 * 32;  // K-half atoms (64 keys)
  static constexpr int kQBytes = kN128 * kAtom + (kTail ? kAtomT : 0);
  static constexpr int kKBytes = kN128 * kKHalfAtom + (kTail ? kKHalfAtomT : 0);
  // V half (all 128 keys, MN-major): a main atom of kVCols columns per CTA (the pair's PV MMA has
  // N = 2 kVCols: 64 columns / 128B swizzle at D = 128, 32 columns / 64B swizzle at D = 64, 72)
  // and, at D = 72, a 16-column 32B-swizzled tail atom per CTA (columns [64 + 16 r, +16) of the
  // zero-padded 96: the second PV MMA has N = 32 into O columns 64-95).
  static constexpr int kVCols = D == 128 ? 64 : 32;
  static constexpr int kVRowBytes = 2 * kVCols;
  static constexpr uint32_t kVLayout = D == 128 ? ptx::kLayoutSW128 : ptx::kLayoutSW64;
  static constexpr int kVBytesA = 128 * kVRowBytes;
  static constexpr int kVBytes = kVBytesA + (kTail ? 128 * 32 : 0);
  static constexpr int kNPV = 2 * kVCols;                // N of the main PV MMA
  static constexpr int kOW = kNPV + (kTail ? 32 : 0);    // O columns in TMEM
  static constexpr int kStageBytes = ((kKBytes > kVBytes ? kKBytes : kVBytes) + 1023) / 1024 * 1024;
  // even: K in even stages, V in odd; D = 128 keeps 8 (4 key tiles) so the double-buffered Q fits
#ifdef XDIT_T_STAGES  // A/B builds: override the per-head-dim tuning below
  static constexpr int kStages = D == 128 ? 9 : XDIT_T_STAGES;
#else
  static constexpr int kStages = D == 128 ? 9 : (D == 64 ? 20 : 14);
#endif
  // Per-head-dim tuning (same-session A/Bs, profiles/r02_ab_tuning_d128.txt, r02_ab_tuning_d64_d72.txt):
  // at D = 128 one exp2 pair in 16 on the FMA pipe (1 in 8 at D = 64 / 72); softmax warps get 224
  // registers at D = 128, 208 at D = 64 (more for the TMA / MMA warps), 216 at D = 72 (setmaxnreg
  // split 256 x R + 128 x R' = 64512 of the 384 x 168 at launch).
#ifdef XDIT_T_EMUP
  static constexpr int kEmuPeriod = XDIT_T_EMUP;
#else
  static constexpr int kEmuPeriod = D == 128 ? 16 : 8;
#endif
#ifdef XDIT_T_REGS
  static constexpr uint32_t kRegsSoftmax = XDIT_T_REGS;
#else
  static constexpr uint32_t kRegsSoftmax = D == 128 ? 224 : (D == 64 ? 208 : 216);
#endif
  static constexpr uint32_t kRegsOther = (64512u - 256u * kRegsSoftmax) / 128u;
  static constexpr int kSmemBar = 1024;
  static constexpr int kQRegion = (kQBytes + 1023) / 1024 * 1024;
  static constexpr int kSmemBytes = 2 * kQRegion + kStages * kStageBytes + kSmemBar + 1024;
  // O columns per softmax warp in the epilogue: warp c of a lane quarter takes the 32-column chunks
  // c, c + 2, ... (D = 72: c = 0 also takes the 8 columns 64-71)
  static constexpr int kOChunks = ((D / 32) + 1) / 2;
  __host__ __device__ static constexpr uint32_t col_s(int b) { return uint32_t(b) * 128u; }
  __host__ __device__ static constexpr uint32_t col_p(int b) { return 256u + uint32_t(b) * 64u; }
  static constexpr uint32_t kColO = 384u;
  static_assert(kColO + kOW <= kTmemCols, "TMEM budget");
  // D = 64: QK^T as a TS MMA -- the unit's Q copied into TMEM (columns 448 + 32 qb, double-buffered
  // by unit parity; the only head dim where it fits beside S, P and O) by tcgen05.cp, so only K is
  // read from shared memory (same-session A/B: CogVideoX +0.8 %, SD3 ±0, profiles/r02_s3_ab_qtmem.txt)
  static constexpr bool kQT = D == 64;
  __host__ __device__ static constexpr uint32_t col_q(int qb) { return 448u + uint32_t(qb) * 32u; }
  static_assert(!kQT || col_q(1) + 32 <= kTmemCols, "TMEM budget (Q)");
  static_assert(kSmemBytes + 6 * 1024 <= 227 * 1024, "smem budget (dynamic + static)");
};

// One work unit: 256 query rows (this CTA: 128) of one (batch, head) against a key range.
struct Unit {
  int valid, b, h, m0, kv0, kv_len, piece, n_kv;
};

// Units [0, n_full) are whole items (query-tile pair, head, batch; query tile fastest) over all keys;
// each of the remaining n_tail items is split into n_split key ranges of kv_chunk keys (tail split).
__device__ __forceinline__ Unit decode_unit(const EpiParams& p, int u, uint32_t rank) {
  Unit U{};
  U.valid = u >= 0;
  if (!U.valid) return U;
  int item = u, kv0 = 0, kv_len = p.Skv, piece = -1;
  if (item >= p.n_full) {
    const int r = item - p.n_full;
    piece = r;
    item = p.n_full + r / p.n_split;
    kv0 = (r % p.n_split) * p.kv_chunk;
    kv_len = min(p.kv_chunk, p.Skv - kv0);
  }
  const int hb = item / p.n_qt;
  U.h = hb % p.H;
  U.b = hb / p.H;
  U.m0 = (item % p.n_qt) * kRowsPerItem + int(rank) * kRows;
  U.kv0 = kv0;
  U.kv_len = kv_len;
  U.piece = piece;
  U.n_kv = (kv_len + kKeys - 1) / kKeys;
  return U;
}

// The id of this pair's t-th unit from the broadcast ring (every role of both CTAs reads it): the
// leader's TMA lane stores it in the LEADER's smem and arrives on both CTAs' unit_full[slot]; leader
// roles read it locally, the peer's through distributed shared memory after a cluster-scope acquire.
__device__ __forceinline__ int ring_get(const int* ring, uint64_t* full, int t, uint32_t rank) {
  const int slot = t % kRing;
  if (rank == 0) {
    ptx::mbar_wait(&full[slot], (t / kRing) & 1);
    return *reinterpret_cast<const volatile int*>(&ring[slot]);
  }
  ptx::mbar_wait_acq_cluster(&full[slot], (t / kRing) & 1);
  return int(ptx::ld_cluster_u32(ptx::mapa(&ring[slot], 0)));
}

// Barrier waits of the single-purpose warps (TMA producer, MMA issuer): with a suspend-time hint,
// so the warp sleeps until the phase completes instead of re-polling (A/B: +0.5-2 %,
// profiles/r02_ab_softmax.txt; the softmax warps poll -- sleeping there cost 2-4 %).
__device__ __forceinline__ void role_wait(uint64_t* bar, uint32_t parity) { ptx::mbar_wait_sleep(bar, parity); }

// Scores of keys >= valid (columns col0.. of this 32-column block) -> -inf: exp2 gives exactly 0.
__device__ __forceinline__ void mask_tail(uint32_t (&a)[32], int col0, int valid) {
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (col0 + i >= valid) a[i] = f2u(-INFINITY);
}

// Row max of this warp's 64 raw scores (MASK: columns >= valid excluded).
template <bool MASK>
__device__ __forceinline__ float max64(const uint32_t (&a)[32], const uint32_t (&bq)[32], int valid) {
  float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
  for (int i = 0; i < 32; i += 4) {
    float x[4], y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      x[e] = u2f(a[i + e]);
      y[e] = u2f(bq[i + e]);
      if (MASK) {
        if (i + e >= valid) x[e] = -INFINITY;
        if (32 + i + e >= valid) y[e] = -INFINITY;
      }
    }
    m0 = fmax3(m0, x[0], x[1]);
    m1 = fmax3(m1, x[2], x[3]);
    m2 = fmax3(m2, y[0], y[1]);
    m3 = fmax3(m3, y[2], y[3]);
  }
  return fmax3(m0, m1, fmaxf(m2, m3));
}

// P = exp2(S * sl2 - m) for 32 of this warp's columns (col0: their first column within the warp's
// 64, for the ragged-tail mask) into 16 packed bf16x2 registers; returns the fp32 row sum of P.
// EMU of every PERIOD column pairs use the FMA-pipe polynomial (exp2_poly2) instead of MUFU.EX2.
template <bool MASK, int EMU, int PERIOD = 8>
__device__ __forceinline__ float exp_pack32(const uint32_t (&a)[32], int col0, int valid, float sl2,
                                            float neg_m, uint32_t* pk) {
  const uint64_t sc2 = pk2(sl2, sl2), nm2 = pk2(neg_m, neg_m);
  uint64_t acc0 = pk2(0.f, 0.f), acc1 = acc0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int col = col0 + 2 * i;
    const uint64_t x = fma2(pk2(u2f(a[2 * i]), u2f(a[2 * i + 1])), sc2, nm2);
    float p0, p1;
    if (!MASK && (i % PERIOD) < EMU) {
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
  float s0, s1, s2, s3;
  up2(acc0, s0, s1);
  up2(acc1, s2, s3);
  return (s0 + s1) + (s2 + s3);
}

// O (this lane's row, all D columns in TMEM) *= alpha -- the rare running-max move
template <int D>
__device__ __forceinline__ void scale_o(uint32_t tO, float alpha) {
#pragma unroll
  for (int cc = 0; cc < (D / 32) * 32; cc += 32) {
    uint32_t o[32];
    ptx::tmem_ld32(tO + cc, o);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 32; ++i) o[i] = f2u(u2f(o[i]) * alpha);
    ptx::tmem_st32(tO + cc, o);
  }
  if (D % 32) {  // D = 72: columns 64-71 (72-95 hold zeros)
    uint32_t o[8];
    ptx::tmem_ld8(tO + (D / 32) * 32, o);
    ptx::tmem_ld_wait();
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i] = f2u(u2f(o[i]) * alpha);
    ptx::tmem_st8(tO + (D / 32) * 32, o);
  }
  ptx::tmem_st_wait();
}

// 32 packed bf16 pairs *= s (s an exact power of two: exact unless the result leaves the range)
__device__ __forceinline__ void scale_bf16x2(uint32_t (&v)[32], float s) {
#pragma unroll
  for (int i = 0; i < 32; ++i)
    v[i] = ptx::pack_bf16x2(u2f(v[i] << 16) * s, u2f(v[i] & 0xffff0000u) * s);
}

// o[i] <- wbl * o[i] + wa * acc[i] for n consecutive fp32 columns (the fused ring merge, a7)
template <int N>
__device__ __forceinline__ void merge_cols(uint32_t* o, const float* acc, float wbl, float wa) {
  const float4* ap = reinterpret_cast<const float4*>(acc);
#pragma unroll
  for (int i = 0; i < N / 4; ++i) {
    const float4 y = ap[i];
    o[4 * i] = f2u(fmaf(wbl, u2f(o[4 * i]), wa * y.x));
    o[4 * i + 1] = f2u(fmaf(wbl, u2f(o[4 * i + 1]), wa * y.y));
    o[4 * i + 2] = f2u(fmaf(wbl, u2f(o[4 * i + 2]), wa * y.z));
    o[4 * i + 3] = f2u(fmaf(wbl, u2f(o[4 * i + 3]), wa * y.w));
  }
}

// store n fp32 columns scaled by sc, as fp32 or bf16
template <int N>
__device__ __forceinline__ void store_cols(const uint32_t* o, float sc, void* base, int64_t off, int of32) {
  if (of32) {
    float4* dp = reinterpret_cast<float4*>(static_cast<float*>(base) + off);
#pragma unroll
    for (int i = 0; i < N / 4; ++i)
      dp[i] = make_float4(u2f(o[4 * i]) * sc, u2f(o[4 * i + 1]) * sc, u2f(o[4 * i + 2]) * sc,
                          u2f(o[4 * i + 3]) * sc);
  } else {
    uint4* dp = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + off);
#pragma unroll
    for (int i = 0; i < N / 8; ++i)
      dp[i] = make_uint4(ptx::pack_bf16x2(u2f(o[8 * i]) * sc, u2f(o[8 * i + 1]) * sc),
                         ptx::pack_bf16x2(u2f(o[8 * i + 2]) * sc, u2f(o[8 * i + 3]) * sc),
                         ptx::pack_bf16x2(u2f(o[8 * i + 4]) * sc, u2f(o[8 * i + 5]) * sc),
                         ptx::pack_bf16x2(u2f(o[8 * i + 6]) * sc, u2f(o[8 * i + 7]) * sc));
  }
}

template <int D, int EMU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_fwd_2sm_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmQ16,
                        const __grid_constant__ CUtensorMap tmK16, const __grid_constant__ CUtensorMap tmV16,
                        const EpiParams p) {
  using C = Cfg<D>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;  // two Q buffers of kQRegion bytes (unit parity)
  uint8_t* sKV = smem + 2 * C::kQRegion;
  __shared__ float m_pub[2 * kRows];     // [step parity][row]: running max after that step
  __shared__ float xsum[2 * kRows];      // [warp pair half][row]: partial row sums for the epilogue
  __shared__ float xref[2 * kRows];      // [warp pair half][row]: the max those sums refer to
  __shared__ int unit_ring[kRing];       // leader: this pair's unit ids (written by its TMA warp)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + C::kStages * C::kStageBytes);
  uint64_t* q_full = bars;                    // leader [2]: both Q tiles of a unit landed
  uint64_t* q_empty = q_full + 2;             // each CTA [2]: the unit's last QK^T completed
  uint64_t* kv_full = q_empty + 2;            // leader: both halves of a K / V stage landed
  uint64_t* kv_empty = kv_full + C::kStages;  // each CTA: the pair's MMAs are done with a stage
  uint64_t* s_full = kv_empty + C::kStages;   // each CTA: S[b] written
  uint64_t* s_free = s_full + 2;              // leader: the pair's 8 softmax warps of S[b] loaded it
  uint64_t* p_full = s_free + 2;              // leader: the pair's 8 softmax warps of P[b] stored it
  uint64_t* pv_done = p_full + 2;             // each CTA: PV reading P[b] completed
  uint64_t* o_full = pv_done + 2;             // each CTA: a unit's last PV completed
  uint64_t* o_empty = o_full + 1;             // leader: the pair's 16 softmax warps read O out
  uint64_t* m_ready = o_empty + 1;            // [lane quarter][step parity]: m_pub written
  uint64_t* unit_full = m_ready + 8;          // each CTA [kRing]: unit_ring[slot] written
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(unit_full + kRing);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&q_full[i], 1);
      ptx::mbar_init(&q_empty[i], 1);
    }
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&kv_full[s], 1);
      ptx::mbar_init(&kv_empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(&s_full[t], 1);
      ptx::mbar_init(&s_free[t], 8);  // the 4 warps of step parity t in each CTA
      ptx::mbar_init(&p_full[t], 8);
      ptx::mbar_init(&pv_done[t], 1);
    }
    ptx::mbar_init(o_full, 1);
    ptx::mbar_init(o_empty, 16);
    for (int i = 0; i < 8; ++i) ptx::mbar_init(&m_ready[i], 32);
    for (int i = 0; i < kRing; ++i) ptx::mbar_init(&unit_full[i], 1);
    ptx::fence_mbar_init();
  }
  if (warp == kWarpMma) {
    ptx::tmem_alloc_pair(tmem_slot, kTmemCols);
    ptx::tmem_relinquish_pair();
  }
  if (warp == kWarpTma && lane == 0) {
    ptx::tma_prefetch_desc(&tmQ);
    ptx::tma_prefetch_desc(&tmK);
    ptx::tma_prefetch_desc(&tmV);
    if (C::kTail) {
      ptx::tma_prefetch_desc(&tmQ16);
      ptx::tma_prefetch_desc(&tmK16);
      ptx::tma_prefetch_desc(&tmV16);
    }
  }
  ptx::tc_fence_before();
  ptx::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated, before any remote use
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp >= 8) {
   ptx::setmaxnreg_dec<C::kRegsOther>();
   if (warp == kWarpTma) {
    // ===================================================== TMA producer (both CTAs)
    // The leader's lane 0 also hands out the units: the t-th unit of this pair is fetched when the
    // TMA warp starts it (after q_empty(t-2): every role has then read the ids of units <= t-4, so
    // a ring of 8 slots is never overwritten while still needed) and broadcast into both CTAs.
    const uint64_t pol_q = ptx::policy_evict_first();
    const uint64_t pol_kv = ptx::policy_evict_last();
    const int pid = blockIdx.x >> 1, npg = gridDim.x >> 1;
    uint32_t it = 0;  // K/V half loads issued so far (2 per key tile, across units)
    for (int t = 0;; ++t) {
      const int qb = t & 1;
      if (t >= 2) role_wait(&q_empty[qb], ((t - 2) >> 1) & 1);
      if (rank == 0 && lane == 0) {
        int u = p.unit_counter ? int(atomicAdd(p.unit_counter, 1u)) : pid + t * npg;
        if (u >= p.n_units) u = -1;
        *reinterpret_cast<volatile int*>(&unit_ring[t % kRing]) = u;
        ptx::mbar_arrive(&unit_full[t % kRing]);
        ptx::mbar_arrive_release_cluster(ptx::mapa(&unit_full[t % kRing], 1));
      }
      __syncwarp();
      const Unit U = decode_unit(p, ring_get(unit_ring, unit_full, t, rank), rank);
      if (!U.valid) break;
      uint8_t* q_dst = sQ + qb * C::kQRegion;
      const uint32_t qfull_cl = ptx::mapa(&q_full[qb], 0);
      if (ptx::elect_one()) {
        if (rank == 0) ptx::mbar_expect_tx(&q_full[qb], 2 * C::kQBytes);
        for (int a = 0; a < C::kN128; ++a)
          ptx::tma_load_4d_pair(q_dst + a * C::kAtom, &tmQ, qfull_cl, a * 64, U.h, U.m0, U.b, pol_q);
        if (C::kTail)
          ptx::tma_load_4d_pair(q_dst + C::kN128 * C::kAtom, &tmQ16, qfull_cl, C::kN128 * 64, U.h, U.m0, U.b,
                                pol_q);
      }
      __syncwarp();
      for (int i = 0; i < 2 * U.n_kv; ++i, ++it) {
        const int j = i >> 1, stage = it % C::kStages, round = it / C::kStages;
        if (round > 0) role_wait(&kv_empty[stage], (round - 1) & 1);
        stamp(p, it >> 1, (i & 1) ? 1 : 0);
        if (ptx::elect_one()) {
          if (rank == 0) ptx::mbar_expect_tx(&kv_full[stage], 2 * ((i & 1) ? C::kVBytes : C::kKBytes));
          const uint32_t full_cl = ptx::mapa(&kv_full[stage], 0);
          uint8_t* dst = sKV + stage * C::kStageBytes;
          const int key0 = U.kv0 + j * kKeys;
          if ((i & 1) == 0) {  // K half: keys [64 rank, 64 rank + 64) of the tile, all D columns
            for (int a = 0; a < C::kN128; ++a)
              ptx::tma_load_4d_pair(dst + a * C::kKHalfAtom, &tmK, full_cl, a * 64, U.h, key0 + int(rank) * 64,
                                    U.b, pol_kv);
            if (C::kTail)
              ptx::tma_load_4d_pair(dst + C::kN128 * C::kKHalfAtom, &tmK16, full_cl, C::kN128 * 64, U.h,
                                    key0 + int(rank) * 64, U.b, pol_kv);
          } else {  // V half: all 128 keys, head-dim columns [kVCols rank, kVCols rank + kVCols) (+ tail)
            ptx::tma_load_4d_pair(dst, &tmV, full_cl, int(rank) * C::kVCols, U.h, key0, U.b, pol_kv);
            if (C::kTail)
              ptx::tma_load_4d_pair(dst + C::kVBytesA, &tmV16, full_cl, 2 * C::kVCols + 16 * int(rank), U.h,
                                    key0, U.b, pol_kv);
          }
        }
        __syncwarp();
      }
    }
   } else if (warp == kWarpMma) {
    // ===================================================== MMA issuer (leader CTA, one lane)
    if (rank == 0) {
      constexpr uint32_t idesc_qk = ptx::idesc_bf16_f32(2 * kRows, kKeys, 0, 0);
      constexpr uint32_t idesc_pv = ptx::idesc_bf16_f32(2 * kRows, C::kNPV, 0, 1);
      constexpr uint32_t idesc_pv16 = ptx::idesc_bf16_f32(2 * kRows, 32, 0, 1);
      const uint32_t sQa = ptx::smem_u32(sQ), sKVa = ptx::smem_u32(sKV);
      auto kv_wait = [&](uint32_t idx) -> int {
        const int stage = idx % C::kStages;
        role_wait(&kv_full[stage], (idx / C::kStages) & 1);
        return stage;
      };
      // S[jb] = Q K_j^T: A = Q (K-major, 128B swizzle, atoms of 128 rows), B = the K halves
      // (K-major, atoms of 64 keys); 16-element K step k at atom k/4, byte 32 (k%4).
      // descriptors built once: a K step / stage / Q buffer adds its byte offset >> 4 to the start
      // address field (bits [0,14); smem offsets stay below 2^18, so no carry leaves the field)
      const uint64_t dq0 = ptx::sdesc_sw128(sQa, 16, 1024), dk0 = ptx::sdesc_sw128(sKVa, 16, 1024);
      const uint64_t dq16 = ptx::sdesc(sQa + C::kN128 * C::kAtom, 16, 8 * 32, ptx::kLayoutSW32);
      const uint64_t dk16 = ptx::sdesc(sKVa + C::kN128 * C::kKHalfAtom, 16, 8 * 32, ptx::kLayoutSW32);
      const uint64_t dv0 = ptx::sdesc(sKVa, C::kAtom, 8 * C::kVRowBytes, C::kVLayout);
      const uint64_t dv16 = ptx::sdesc(sKVa + C::kVBytesA, 16, 8 * 32, ptx::kLayoutSW32);
      auto qk = [&](int jb, int sK, int qb) {
        const uint64_t oq = uint64_t(uint32_t(qb * C::kQRegion) >> 4), ok = uint64_t(uint32_t(sK * C::kStageBytes) >> 4);
#pragma unroll
        for (int k = 0; k < C::kDpK / 16; ++k) {
          if constexpr (C::kQT)
            ptx::mma_ts_pair(tmem + C::col_s(jb), tmem + C::col_q(qb) + k * 8,
                             dk0 + ok + uint64_t(((k >> 2) * C::kKHalfAtom + (k & 3) * 32) >> 4), idesc_qk,
                             k > 0 ? 1u : 0u);
          else if (C::kTail && k == C::kN128 * 4)
            ptx::mma_ss_pair(tmem + C::col_s(jb), dq16 + oq, dk16 + ok, idesc_qk, 1u);
          else
            ptx::mma_ss_pair(tmem + C::col_s(jb), dq0 + oq + uint64_t(((k >> 2) * C::kAtom + (k & 3) * 32) >> 4),
                             dk0 + ok + uint64_t(((k >> 2) * C::kKHalfAtom + (k & 3) * 32) >> 4), idesc_qk,
                             k > 0 ? 1u : 0u);
        }
      };
      auto pv = [&](int jb, int sV, bool acc) {
        const uint64_t ov = uint64_t(uint32_t(sV * C::kStageBytes) >> 4);
#pragma unroll
        for (int k = 0; k < kKeys / 16; ++k) {
          ptx::mma_ts_pair(tmem + C::kColO, tmem + C::col_p(jb) + k * 8,
                           dv0 + ov + uint64_t((k * 16 * C::kVRowBytes) >> 4), idesc_pv, (acc || k > 0) ? 1u : 0u);
          if (C::kTail)
            ptx::mma_ts_pair(tmem + C::kColO + C::kNPV, tmem + C::col_p(jb) + k * 8,
                             dv16 + ov + uint64_t((k * 16 * 32) >> 4), idesc_pv16, (acc || k > 0) ? 1u : 0u);
        }
      };
      // Two cursors over this pair's stream of key tiles (global tile counter g across units): QK^T
      // runs two tiles ahead of PV, so S[g%2] is rewritten by QK^T(g+2) as soon as the softmax has
      // loaded S(g) -- across a unit boundary too (the next unit's Q is already in its buffer).
      struct Cur {
        int t, j, n_kv, valid;
        uint32_t g;
      };
      auto load = [&](Cur& c) {
        const Unit U = decode_unit(p, ring_get(unit_ring, unit_full, c.t, 0), 0);
        c.valid = U.valid;
        c.n_kv = U.valid ? U.n_kv : 0;
        c.j = 0;
      };
      auto advance = [&](Cur& c) {
        ++c.g;
        if (++c.j == c.n_kv) {
          ++c.t;
          load(c);
        }
      };
      auto issue_qk = [&](const Cur& c) {
        const int qb = c.t & 1;
        stamp(p, c.g, 0);
        if (c.j == 0) role_wait(&q_full[qb], (c.t >> 1) & 1);
        const int sK = kv_wait(2 * c.g);
        stamp(p, c.g, 1);
        if (c.g >= 2) role_wait(&s_free[c.g & 1], ((c.g - 2) >> 1) & 1);
        stamp(p, c.g, 2);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          if (C::kQT && c.j == 0) {  // the unit's Q into TMEM (in issue order before its QK^T)
#pragma unroll
            for (int k = 0; k < D / 16; ++k)
              ptx::tc_cp_pair_128x256b(tmem + C::col_q(qb) + k * 8,
                                       dq0 + uint64_t(uint32_t(qb * C::kQRegion) >> 4) + uint64_t((k * 32) >> 4));
          }
          qk(c.g & 1, sK, qb);
          ptx::tc_commit_pair(&s_full[c.g & 1]);
          ptx::tc_commit_pair(&kv_empty[sK]);
          if (c.j == c.n_kv - 1) ptx::tc_commit_pair(&q_empty[qb]);
        }
        __syncwarp();
        stamp(p, c.g, 3);
      };
      Cur qc{0, 0, 0, 0, 0u}, pc{0, 0, 0, 0, 0u};
      auto issue_pv = [&](const Cur& c) {
        stamp(p, c.g, 4);
        const int sV = kv_wait(2 * c.g + 1);
        stamp(p, c.g, 5);
        role_wait(&p_full[c.g & 1], (c.g >> 1) & 1);
        if (c.j == 0 && c.t > 0) role_wait(o_empty, (c.t - 1) & 1);  // O read out
        stamp(p, c.g, 6);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          pv(c.g & 1, sV, c.j > 0);
          ptx::tc_commit_pair(&pv_done[c.g & 1]);
          ptx::tc_commit_pair(&kv_empty[sV]);
          if (c.j == c.n_kv - 1) ptx::tc_commit_pair(o_full);
        }
        __syncwarp();
        stamp(p, c.g, 7);
      };
      {
        load(qc);
        load(pc);
        for (int w = 0; w < 2 && qc.valid; ++w) {
          issue_qk(qc);
          advance(qc);
        }
        while (pc.valid) {
          if (qc.valid) {
            issue_qk(qc);
            advance(qc);
          }
          issue_pv(pc);
          advance(pc);
        }
      }
    }
   }
  } else {
    ptx::setmaxnreg_inc<C::kRegsSoftmax>();
    // ===================================================== softmax (8 warps per CTA)
    // Warp w owns TMEM lanes / query rows 32 (w%4) .. +31 and the key tiles g = w/4 (mod 2) of the
    // pair's tile stream: the two warps of a lane quarter alternate steps, so one runs its exp2
    // stream while the other waits for S, loads it and stores P -- the MUFU pipe of the SM
    // sub-partition stays busy.  They share the rows' reference max (reading R1', below): the warp
    // of step g publishes the reference m(g) of its P in smem (mbarrier m_ready[w%4][g%2]) at the
    // END of its step, the warp of step g+1 of the same unit reconciles with it before releasing
    // P(g+1).  Each warp keeps its own partial row sum l_w relative to the reference it last used;
    // the unit's epilogue combines the two.
    const int g4 = warp & 3, c = warp >> 2;
    const int row_in_tile = g4 * 32 + lane;
    const uint32_t lane_off = uint32_t(g4 * 32) << 16;
    const float sl2 = p.scale_log2;
    const uint32_t s_free_cl = ptx::mapa(&s_free[c], 0);  // the leader's barriers for S[c] / P[c]
    const uint32_t p_full_cl = ptx::mapa(&p_full[c], 0);
    const uint32_t o_empty_cl = ptx::mapa(o_empty, 0);
    const uint32_t tO = tmem + lane_off + C::kColO;
    uint32_t gbase = 0;  // global index of the unit's first key tile
    for (int t = 0;; ++t) {
      const int uid = ring_get(unit_ring, unit_full, t, rank);
      if (uid < 0) break;
      int kv_len, n_kv;  // only these stay live through the tile loop; the rest is decoded after it
      {
        const Unit U = decode_unit(p, uid, rank);
        kv_len = U.kv_len;
        n_kv = U.n_kv;
      }
      float m_ref = -INFINITY, l = 0.f, m_used = 0.f, m_own = 0.f;
      for (int j = int((gbase ^ uint32_t(c)) & 1u); j < n_kv; j += 2) {
        const uint32_t g = gbase + uint32_t(j);
        ptx::mbar_wait_cluster(&s_full[c], (g >> 1) & 1);
        stamp(p, g, 0);
        ptx::tc_fence_after();
#ifdef XDIT_PROFILE
        if (p.diag) {  // profiling builds only: hand the barriers back without softmax work
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(s_free_cl);
          if (g >= 2) ptx::mbar_wait_cluster(&pv_done[c], ((g - 2) >> 1) & 1);
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_cluster(p_full_cl);
          if (j > 0) ptx::mbar_wait(&m_ready[g4 * 2 + ((g - 1) & 1)], ((g - 1) >> 1) & 1);
          m_pub[(g & 1) * kRows + row_in_tile] = 0.f;
          ptx::mbar_arrive(&m_ready[g4 * 2 + (g & 1)]);
          l = 1.f;
          m_ref = m_used = 0.f;
          continue;
        }
#endif
        uint32_t s0[32], s1[32], s2[32], s3[32];
        const uint32_t tS = tmem + lane_off + C::col_s(c);
        ptx::tmem_ld32(tS, s0);
        ptx::tmem_ld32(tS + 32, s1);
        ptx::tmem_ld32(tS + 64, s2);
        ptx::tmem_ld32(tS + 96, s3);
        ptx::tmem_ld_wait();
        stamp(p, g, 1);
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(s_free_cl);  // S[c] may be rewritten by QK^T(g+2)
        const int valid = kv_len - j * kKeys;  // keys of this tile that exist (C16)
        if (valid < kKeys) {  // ragged last tile: missing keys get score -inf (weight 0), once, here --
          // the max and exp code below then has no per-element mask (with the masked variants as
          // separate template instances the compiler if-converted them into every tile's exp loop)
          mask_tail(s0, 0, valid);
          mask_tail(s1, 32, valid);
          mask_tail(s2, 64, valid);
          mask_tail(s3, 96, valid);
        }
        // Reading R1': P(g) is computed straight against a candidate reference m_c
        // -- the tile's own max rounded up to an integer (log2 units) on the unit's first two tiles,
        // else this warp's reference of its previous tile -- so no max pass and no hand-over sits
        // before the exp2 stream.  The row sum flags the rare tile whose P could overflow (sum >
        // 2^64): it is redone against its own max.  Before releasing P(g) the warp reconciles with
        // the reference m(g-1) the other warp published at the END of step g-1 (normally long
        // done): P(g) and its sum are scaled by the exact power of two 2^(m_c - m(g-1)) and m(g) =
        // m(g-1); only a jump above 2^kMoveThresh moves the reference (O rescaled after PV(g-1)).
        float m_c;
        if (j <= 1) m_c = ceilf(fmaxf(max64<false>(s0, s1, 64), max64<false>(s2, s3, 64)) * sl2);
        else m_c = m_own;
        stamp(p, g, 2);
        // D = 128: the whole row of P stays in registers until the end of the step: one wait for
        // P[c] to be free (PV(g-2) done) right before both halves are stored, and the rare rescales
        // run in registers (same-session A/B: Flux +1.5-2 %; at D = 64 / 72 it costs 3-8 %, there the
        // first half goes out mid-step, profiles/r02_ab_p_late.txt)
        if constexpr (D == 128) {
        uint32_t pa[32], pb[32];
        const uint32_t tP = tmem + lane_off + C::col_p(c);
        float rs = exp_pack32<false, EMU, C::kEmuPeriod>(s0, 0, valid, sl2, -m_c, pa);
        rs += exp_pack32<false, EMU, C::kEmuPeriod>(s1, 32, valid, sl2, -m_c, pa + 16);
        stamp(p, g, 4);
        rs += exp_pack32<false, EMU, C::kEmuPeriod>(s2, 64, valid, sl2, -m_c, pb);
        rs += exp_pack32<false, EMU, C::kEmuPeriod>(s3, 96, valid, sl2, -m_c, pb + 16);
        if (__any_sync(0xffffffffu, !(rs <= 0x1p64f))) {  // rare (also catches inf / NaN): own max
          m_c = fmaxf(m_c, ceilf(fmaxf(max64<false>(s0, s1, 64), max64<false>(s2, s3, 64)) * sl2));
          rs = exp_pack32<false, EMU, C::kEmuPeriod>(s0, 0, valid, sl2, -m_c, pa);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s1, 32, valid, sl2, -m_c, pa + 16);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s2, 64, valid, sl2, -m_c, pb);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s3, 96, valid, sl2, -m_c, pb + 16);
        }
        float m_fin = m_c;
        if (j >= 1) {
          ptx::mbar_wait(&m_ready[g4 * 2 + ((g - 1) & 1)], ((g - 1) >> 1) & 1);
          stamp(p, g, 3);
          const float m_prev = m_pub[((g - 1) & 1) * kRows + row_in_tile];
          const float d = m_c - m_prev;
          const bool move = d > kMoveThresh;
          m_fin = move ? m_c : m_prev;
          if (__any_sync(0xffffffffu, d != 0.f)) {  // unit's second tile, or after a rare move
            if (__any_sync(0xffffffffu, move)) {  // O *= 2^(m_prev - m_c) once PV(g-1) is in
              const float alpha = move ? ldexpf(1.f, int(m_prev - m_c)) : 1.f;
              ptx::mbar_wait_cluster(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
              ptx::tc_fence_after();
              scale_o<D>(tO, alpha);
            }
            const float beta = move ? 1.f : ldexpf(1.f, int(d));  // exact (flushes below 2^-149)
            scale_bf16x2(pa, beta);
            scale_bf16x2(pb, beta);
            rs *= beta;
          }
        }
        m_pub[(g & 1) * kRows + row_in_tile] = m_fin;
        ptx::mbar_arrive(&m_ready[g4 * 2 + (g & 1)]);  // all 32 lanes (count 32)
        if (g >= 2) ptx::mbar_wait_cluster(&pv_done[c], ((g - 2) >> 1) & 1);  // P[c] free again
        stamp(p, g, 5);
        ptx::tc_fence_after();
        ptx::tmem_st32(tP, pa);       // keys 0..63
        ptx::tmem_st32(tP + 32, pb);  // keys 64..127
        if (m_fin != m_ref) {
          l *= ptx::ex2(m_ref - m_fin);  // 0 * 0 on this warp's first step of the unit
          m_ref = m_fin;
        }
        l += rs;
        m_own = m_fin;
        } else {
        uint32_t pk[32];
        const uint32_t tP = tmem + lane_off + C::col_p(c);
        auto exp2x = [&](const uint32_t (&a)[32], int col0, uint32_t* pko) -> float {
          return exp_pack32<false, EMU, C::kEmuPeriod>(a, col0, valid, sl2, -m_c, pko);
        };
        float rs = exp2x(s0, 0, pk);
        rs += exp2x(s1, 32, pk + 16);
        stamp(p, g, 4);
        if (g >= 2) ptx::mbar_wait_cluster(&pv_done[c], ((g - 2) >> 1) & 1);  // P[c] free again
        stamp(p, g, 5);
        ptx::tc_fence_after();
        ptx::tmem_st32(tP, pk);  // keys 0..63
        rs += exp2x(s2, 64, pk);
        rs += exp2x(s3, 96, pk + 16);
        if (__any_sync(0xffffffffu, !(rs <= 0x1p64f))) {  // rare (also catches inf / NaN): own max
          m_c = fmaxf(m_c, ceilf(fmaxf(max64<false>(s0, s1, 64), max64<false>(s2, s3, 64)) * sl2));
          rs = exp_pack32<false, EMU, C::kEmuPeriod>(s0, 0, valid, sl2, -m_c, pk);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s1, 32, valid, sl2, -m_c, pk + 16);
          ptx::tmem_st32(tP, pk);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s2, 64, valid, sl2, -m_c, pk);
          rs += exp_pack32<false, EMU, C::kEmuPeriod>(s3, 96, valid, sl2, -m_c, pk + 16);
        }
        float m_fin = m_c;
        if (j >= 1) {
          ptx::mbar_wait(&m_ready[g4 * 2 + ((g - 1) & 1)], ((g - 1) >> 1) & 1);
          stamp(p, g, 3);
          const float m_prev = m_pub[((g - 1) & 1) * kRows + row_in_tile];
          const float d = m_c - m_prev;
          const bool move = d > kMoveThresh;
          m_fin = move ? m_c : m_prev;
          if (__any_sync(0xffffffffu, d != 0.f)) {  // unit's second tile, or after a rare move
            if (__any_sync(0xffffffffu, move)) {  // O *= 2^(m_prev - m_c) once PV(g-1) is in
              const float alpha = move ? ldexpf(1.f, int(m_prev - m_c)) : 1.f;
              ptx::mbar_wait_cluster(&pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
              ptx::tc_fence_after();
              scale_o<D>(tO, alpha);
            }
            const float beta = move ? 1.f : ldexpf(1.f, int(d));  // exact (flushes below 2^-149)
            uint32_t q[32];
            ptx::tmem_st_wait();  // the first half's store has landed before it is read back
            ptx::tmem_ld32(tP, q);
            ptx::tmem_ld_wait();
            scale_bf16x2(q, beta);
            ptx::tmem_st32(tP, q);
            scale_bf16x2(pk, beta);
            rs *= beta;
          }
        }
        m_pub[(g & 1) * kRows + row_in_tile] = m_fin;
        ptx::mbar_arrive(&m_ready[g4 * 2 + (g & 1)]);  // all 32 lanes (count 32)
        ptx::tmem_st32(tP + 32, pk);  // keys 64..127
        if (m_fin != m_ref) {
          l *= ptx::ex2(m_ref - m_fin);  // 0 * 0 on this warp's first step of the unit
          m_ref = m_fin;
        }
        l += rs;
        m_own = m_fin;
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_cluster(p_full_cl);
        stamp(p, g, 6);
      }
      // ----------------------------------------------- the unit's epilogue: O / l, LSE
      // final m = m of the unit's last step; l = sum over both warps of l_w 2^(m_ref_w - m)
      const Unit U = decode_unit(p, uid, rank);
      const uint32_t glast = gbase + uint32_t(n_kv) - 1u;
      xsum[c * kRows + row_in_tile] = l;
      xref[c * kRows + row_in_tile] = m_ref;
      ptx::named_bar_sync(1 + g4, 64);
      m_used = m_pub[(glast & 1) * kRows + row_in_tile];
      l = xsum[row_in_tile] * ptx::ex2(xref[row_in_tile] - m_used) +
          xsum[kRows + row_in_tile] * ptx::ex2(xref[kRows + row_in_tile] - m_used);
      ptx::named_bar_sync(1 + g4, 64);  // xsum / xref / m_pub read: the next unit may rewrite them
      if (c != int(glast & 1u)) stamp(p, glast, 0);  // profiling: epilogue phases (warp not on the last tile)
      // O out of TMEM into registers, then hand TMEM's O to the next unit's first P.V
      ptx::mbar_wait_cluster(o_full, t & 1);
      if (c != int(glast & 1u)) stamp(p, glast, 1);  // profiling: epilogue phases (warp not on the last tile)
      ptx::tc_fence_after();
      uint32_t o[C::kOChunks][32];
      uint32_t o8[8];
#pragma unroll
      for (int k = 0; k < C::kOChunks; ++k)
        if (c * 32 + 64 * k < (D / 32) * 32) ptx::tmem_ld32(tO + c * 32 + 64 * k, o[k]);
      if (D % 32 && c == 0) ptx::tmem_ld8(tO + (D / 32) * 32, o8);
      ptx::tmem_ld_wait();
      if (c != int(glast & 1u)) stamp(p, glast, 2);  // profiling: epilogue phases (warp not on the last tile)
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_cluster(o_empty_cl);
      if (c != int(glast & 1u)) stamp(p, glast, 3);  // profiling: epilogue phases (warp not on the last tile)
      const int row = U.m0 + row_in_tile;
      const float inv_l = 1.f / l;
      RowDst dst = rowmap_dst(p.map, U.b, row, U.h);
      void* obase = p.o;
      float* lbase = p.lse;
      int of32 = p.out_f32;
      float lse_row = (m_used + log2f(l)) * 0.69314718055994530942f;
      // fused ring merge (a7): O = wa * O_acc + wb * O_s, LSE by log-sum-exp (lse_merge_kernel's
      // arithmetic); wb folds in 1/l.  Results go back to the accumulator or, at the last ring step,
      // to the final destination.
      const bool mrg = p.merge && U.piece < 0 && row < p.Sq;
      float wa = 0.f, wbl = inv_l;
      RowDst ad{0, 0};
      if (mrg) {
        ad = rowmap_dst(p.acc_map, U.b, row, U.h);
        const float la = p.acc_l_in[ad.l_off];
        const float M2 = fmaxf(la, lse_row);
        const float L2 = M2 + logf(expf(la - M2) + expf(lse_row - M2));
        wa = expf(la - L2);
        wbl = expf(lse_row - L2) * inv_l;
        lse_row = L2;
        if (!p.merge_final) {
          obase = p.acc_o;
          lbase = p.acc_l_out;
          of32 = 1;
          dst = ad;
        }
      }
      if (U.piece >= 0) {  // split tail unit: normalised fp32 partial for tail_merge_kernel
        const int64_t prow = int64_t(U.piece) * kRowsPerItem + int(rank) * kRows + row_in_tile;
        const int64_t n_pieces = int64_t(p.n_units) - p.n_full;
        obase = p.part;
        lbase = p.part + n_pieces * kRowsPerItem * D;
        of32 = 1;
        dst.o_off = prow * D;
        dst.l_off = prow;
      }
      const bool valid_row = row < p.Sq;
      const float sc = mrg ? 1.f : inv_l;
#pragma unroll
      for (int k = 0; k < C::kOChunks; ++k) {  // this warp's 32-column chunks of O
        const int col = c * 32 + 64 * k;
        if (col < (D / 32) * 32) {
          if (mrg) merge_cols<32>(o[k], p.acc_o + ad.o_off + col, wbl, wa);  // then stored with sc = 1
          if (valid_row) store_cols<32>(o[k], sc, obase, dst.o_off + col, of32);
        }
      }
      if (D % 32 && c == 0) {  // D = 72: columns 64-71
        constexpr int col = (D / 32) * 32;
        if (mrg) merge_cols<8>(o8, p.acc_o + ad.o_off + col, wbl, wa);
        if (valid_row) store_cols<8>(o8, sc, obase, dst.o_off + col, of32);
      }
      if (c == 0 && valid_row && lbase)
        lbase[dst.l_off] = U.piece >= 0 ? (m_used + log2f(l)) * 0.69314718055994530942f : lse_row;
      gbase += uint32_t(n_kv);
      if (c != int(glast & 1u)) stamp(p, glast, 5);  // profiling: epilogue phases (warp not on the last tile)
    }
  }
  __syncwarp();
  ptx::tc_fence_before();
  ptx::cluster_sync();  // the peer's TMEM / smem stay live until the leader's MMAs are all done
  ptx::tc_fence_after();
  if (warp == kWarpMma) ptx::tmem_dealloc_pair(tmem, kTmemCols);
}

template <int D, int EMU>
cudaError_t launch_kernel(dim3 grid, const CUtensorMap* m, const EpiParams& p, cudaStream_t st) {
  static DeviceFlags attr_set;  // cudaFuncSetAttribute done on device d
  if (!attr_set.test()) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_2sm_kernel<D, EMU>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<D>::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set.set();
  }
  attn_fwd_2sm_kernel<D, EMU><<<grid, kThreads, Cfg<D>::kSmemBytes, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p);
  note_launches(1);
  return cudaGetLastError();
}

template <int D>
cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
  using C = Cfg<D>;
  CUtensorMap m[6];
  if (!make_map(&m[0], a.q, a.B, a.Sq, a.H, D, a.q_b, a.q_s, a.q_h, 64, kRows) ||
      !make_map(&m[1], a.k, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, 64, 64) ||
      !make_map(&m[2], a.v, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, C::kVCols, kKeys))
    return cudaErrorInvalidValue;
  if (C::kTail) {
    if (!make_map(&m[3], a.q, a.B, a.Sq, a.H, D, a.q_b, a.q_s, a.q_h, 16, kRows) ||
        !make_map(&m[4], a.k, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, 16, 64) ||
        !make_map(&m[5], a.v, a.B, a.Skv, a.H, D, a.kv_b, a.kv_s, a.kv_h, 16, kKeys))
      return cudaErrorInvalidValue;
  } else {
    m[3] = m[0];
    m[4] = m[1];
    m[5] = m[2];
  }
  EpiParams p{};
  p.o = a.o;
  p.lse = a.lse;
  p.map = a.omap;
  p.H = a.H;
  p.Sq = a.Sq;
  p.Skv = a.Skv;
  p.out_f32 = a.out_f32;
  p.merge = a.merge;
  p.merge_final = a.merge_final;
  p.acc_o = a.acc_o;
  p.acc_l_in = a.acc_l_in;
  p.acc_l_out = a.acc_l_out;
  p.acc_map = a.acc_map;
  p.scale_log2 = float(1.4426950408889634 / std::sqrt(double(D)));
  // Work units (256 query rows of one (batch, head)); when the items leave a partial last round of
  // pairs, its items are split over key ranges written as normalised fp32 partials into the scratch
  // and merged by tail_merge_kernel (DESIGN.md §7.1 "tail split").
  p.n_qt = (a.Sq + kRowsPerItem - 1) / kRowsPerItem;
  const int items = p.n_qt * a.H * a.B;
  p.n_full = items;
  p.n_split = 1;
  p.kv_chunk = a.Skv;
  p.part = nullptr;
  int n_tail = 0;
  const int npairs = device_sm_count() / 2;
  // the last kCounterFloats floats of the scratch hold the unit counter (dynamic unit hand-out)
  const size_t part_floats = a.scratch_floats > kCounterFloats ? a.scratch_floats - kCounterFloats : 0;
  if (a.scratch && items > npairs && items % npairs) {
    const int rem = items % npairs, n_kv_tiles = (a.Skv + kKeys - 1) / kKeys;
    int ns = std::min(std::min(npairs / rem, 8), n_kv_tiles / 2);
    if (ns >= 2) {
      const int chunk = ((n_kv_tiles + ns - 1) / ns) * kKeys;
      ns = (a.Skv + chunk - 1) / chunk;
      const size_t need = size_t(rem) * ns * kRowsPerItem * (D + 1);
      if (ns >= 2 && need <= part_floats) {
        n_tail = rem;
        p.n_full = items - rem;
        p.n_split = ns;
        p.kv_chunk = chunk;
        p.part = a.scratch;
      }
    }
  }
  p.n_units = p.n_full + n_tail * p.n_split;
  p.unit_counter = nullptr;
  if (a.scratch && a.scratch_floats >= kCounterFloats) {
    p.unit_counter = reinterpret_cast<unsigned*>(a.scratch + a.scratch_floats - kCounterFloats);
    cudaError_t e = cudaMemsetAsync(p.unit_counter, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
  }
  const dim3 grid(2 * std::min(p.n_units, npairs));
#ifdef XDIT_PROFILE
  // profiling builds: XDIT_PROFILE_DIAG=1 in the environment runs the softmax-free skeleton,
  // XDIT_PROFILE_TRACE=<file> appends the first pair's clock64 stamps to <file> after the launch
  static const int diag = [] {
    const char* e = std::getenv("XDIT_PROFILE_DIAG");
    return e ? std::atoi(e) : 0;
  }();
  p.diag = diag;
  static const char* trace_file = std::getenv("XDIT_PROFILE_TRACE");
  constexpr size_t kTraceN = size_t(2) * kTraceWarps * kTraceIters * kTraceEv;
  static unsigned long long* trace = [] {
    unsigned long long* t = nullptr;
    if (trace_file) cudaMalloc(&t, sizeof(unsigned long long) * kTraceN);
    return t;
  }();
  p.trace = trace;
  if (trace) cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * kTraceN, st);
#endif
  cudaError_t err = launch_kernel<D, XDIT_EXP_EMU>(grid, m, p, st);
  if (err == cudaSuccess && n_tail) {
    const int rows = n_tail * kRowsPerItem;
    tail_merge_kernel<D><<<(rows + 7) / 8, 256, 0, st>>>(p.part, n_tail, p.n_split, p.n_full, p.n_qt, a.H,
                                                          a.Sq, p);
    note_launches(1);
    err = cudaGetLastError();
  }
#ifdef XDIT_PROFILE
  if (trace) {  // raw stamps [cta][warp][g][ev] of the first pair, appended to the trace file
    static unsigned long long h[kTraceN];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, trace, sizeof h, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(trace_file, "ab")) {
      std::fwrite(h, sizeof h, 1, f);
      std::fclose(f);
    }
  }
#endif
  return err;
}

}  // namespace pair2
}  // namespace

size_t attn_scratch_floats(int D) {
  return size_t(device_sm_count()) * kRowsPerItem * size_t(D + 1) + kCounterFloats;
}

bool attn_fused_merge_supported(int D) { return D == 128 || D == 64 || D == 72; }

cudaError_t launch_attn_fwd_bf16(const AttnArgs& a, cudaStream_t st) {
  if (a.Sq == 0 || a.B == 0) return cudaSuccess;
  switch (a.D) {
    case 128: return pair2::launch_d<128>(a, st);
    case 64: return pair2::launch_d<64>(a, st);
    case 72: return pair2::launch_d<72>(a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace xdit
