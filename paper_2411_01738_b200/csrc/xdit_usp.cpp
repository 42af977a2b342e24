// xdit_usp.cpp -- host side of libxdit_usp.so: argument validation, the in-context shard rule,
// workspace ownership, NCCL sub-communicators, and the stream/event orchestration of one USP
// attention call (include/xdit_usp.h).
//
// USP (§4.1.4) on a 2D mesh, rank g = i*u + j (reading C6):
//   Ulysses all-to-all within the row {i*u + j'} (§4.1.1) as grouped ncclSend/ncclRecv on the
//   Ulysses sub-communicator, on the caller's stream (not overlapped); Ring P2P within the
//   column {i'*u + j} (§4.1.1) as grouped ncclSend/ncclRecv on the Ring sub-communicator, on
//   an internal high-priority side stream that runs while the attention kernel of the current ring
//   step runs on the caller's stream (overlapped), joined back with events.  NCCL is the one
//   data plane; no host synchronisation anywhere in the call, which stays CUDA-graph
//   capturable.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "xdit_internal.h"

using xdit::AttnArgs;

namespace xdit {
static std::atomic<unsigned long long> g_launches{0};
void note_launches(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed); }
int device_sm_count() {
  static std::atomic<int> cache[128];  // 0 = not queried yet
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 127;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
}  // namespace xdit

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define XCUDA(call)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(XDIT_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)
#define XNCCL(call)                                                                           \
  do {                                                                                        \
    ncclResult_t r_ = (call);                                                                 \
    if (r_ != ncclSuccess)                                                                    \
      return fail(XDIT_ERR_NCCL, "%s failed: %s (%s:%d)", #call, ncclGetErrorString(r_), \
                  __FILE__, __LINE__);                                                        \
  } while (0)

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Balanced contiguous piece g of S tokens over n ranks (reading C5, np.array_split convention).
void piece(int S, int n, int g, int* off, int* len) {
  const int base = S / n, rem = S % n;
  *len = base + (g < rem ? 1 : 0);
  *off = g * base + (g < rem ? g : rem);
}

// Per-call geometry derived from the shard rule; identical on every rank of the SP group.
struct Plan {
  int N, u, r, g, i, j, Hh;
  std::vector<int> S_loc;  // per SP rank
  std::vector<int> S_blk;  // per ring index
  int Lmax, S_blk_max;
};

int make_plan(int B, int H, int S_txt, int S_img, int D, int u, int r, int g, Plan* P) {
  if (B <= 0 || H <= 0 || D <= 0 || S_txt < 0 || S_img < 0 || u <= 0 || r <= 0)
    return fail(XDIT_ERR_INVALID_ARG, "bad sizes B=%d H=%d D=%d S_txt=%d S_img=%d u=%d r=%d", B, H,
                D, S_txt, S_img, u, r);
  if (u > 8 || r > 8)
    return fail(XDIT_ERR_UNSUPPORTED, "ulysses and ring degrees are limited to 8 (got %d, %d)", u, r);
  if (g < 0 || g >= u * r) return fail(XDIT_ERR_INVALID_ARG, "rank %d out of range", g);
  if (H % u != 0)
    return fail(XDIT_ERR_DIVISIBILITY, "H=%d is not divisible by ulysses=%d (P:541)", H, u);
  P->N = u * r;
  P->u = u;
  P->r = r;
  P->g = g;
  P->i = g / u;
  P->j = g % u;
  P->Hh = H / u;
  P->S_loc.assign(P->N, 0);
  P->S_blk.assign(r, 0);
  P->Lmax = 0;
  for (int q = 0; q < P->N; ++q) {
    int to, tl, io, il;
    piece(S_txt, P->N, q, &to, &tl);
    piece(S_img, P->N, q, &io, &il);
    P->S_loc[q] = tl + il;
    if (P->S_loc[q] == 0)
      return fail(XDIT_ERR_EMPTY_SHARD, "rank %d of %d would hold no tokens (S=%d)", q, P->N,
                  S_txt + S_img);
    P->Lmax = std::max(P->Lmax, P->S_loc[q]);
    P->S_blk[q / u] += P->S_loc[q];
  }
  P->S_blk_max = *std::max_element(P->S_blk.begin(), P->S_blk.end());
  return XDIT_OK;
}

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Device buffers owned by a comm handle, sized by xdit_comm_reserve.
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

int ensure(Buf* b, size_t bytes) {
  if (bytes <= b->bytes) return XDIT_OK;
  if (b->p) cudaFree(b->p);
  b->p = nullptr;
  b->bytes = 0;
  if (bytes == 0) return XDIT_OK;
  XCUDA(cudaMalloc(&b->p, bytes));
  b->bytes = bytes;
  return XDIT_OK;
}

// Byte sizes of every workspace buffer for one problem (0 where the split does not need it).
struct Sizes {
  size_t uly3;     // Ulysses QKV exchange buffer (send and recv each)
  size_t qblk;     // unpacked Q block
  size_t kvslot;   // one K or V ring-block buffer
  size_t oacc;     // fp32 O accumulator / partial
  size_t lacc;     // fp32 LSE accumulator / partial
  size_t ochunk;   // reverse a2a chunk per peer (O + LSE)
  size_t ochunk_o; // O part of ochunk
};

Sizes sizes_for(const Plan& P, int B, int D, int eb) {
  Sizes s{};
  const size_t row = size_t(P.Hh) * D * eb;
  if (P.u > 1) {
    s.uly3 = size_t(P.u) * 3 * B * P.Lmax * row;
    s.qblk = size_t(B) * P.S_blk_max * row;
    s.ochunk_o = align16(size_t(B) * P.Lmax * row);
    s.ochunk = s.ochunk_o + align16(size_t(B) * P.Hh * P.Lmax * 4);
  }
  if (P.u > 1 || P.r > 1) s.kvslot = size_t(B) * P.S_blk_max * row;
  if (P.r > 1) {
    s.oacc = size_t(B) * P.S_blk_max * P.Hh * D * 4;
    s.lacc = size_t(B) * P.Hh * P.S_blk_max * 4;
  }
  return s;
}

xdit_rowmap plain_map(int B, int S, int H, int D) {
  // [B][S][H][D] tensor and lse [B][H][S]
  xdit_rowmap m{};
  m.nseg = 1;
  m.seg_off[0] = 0;
  m.seg_off[1] = S;
  m.o_seg = 0;
  m.o_b = int64_t(S) * H * D;
  m.o_s = int64_t(H) * D;
  m.o_h = D;
  m.l_seg = 0;
  m.l_b = int64_t(H) * S;
  m.l_h = S;
  return m;
}

int check_map(const xdit_rowmap* m, int rows) {
  if (!m) return fail(XDIT_ERR_INVALID_ARG, "row map is NULL");
  if (m->nseg < 1 || m->nseg > 8) return fail(XDIT_ERR_INVALID_ARG, "rowmap nseg=%d", m->nseg);
  if (m->seg_off[0] != 0 || m->seg_off[m->nseg] != rows)
    return fail(XDIT_ERR_INVALID_ARG, "rowmap segments must cover [0,%d)", rows);
  for (int s = 0; s < m->nseg; ++s)
    if (m->seg_off[s + 1] < m->seg_off[s]) return fail(XDIT_ERR_INVALID_ARG, "rowmap not monotone");
  return XDIT_OK;
}

int check_map_align(const xdit_rowmap* m, int vec_elems) {
  const int64_t v[4] = {m->o_seg, m->o_b, m->o_s, m->o_h};
  for (int64_t x : v)
    if (x % vec_elems != 0)
      return fail(XDIT_ERR_ALIGNMENT, "output strides must be multiples of %d elements", vec_elems);
  return XDIT_OK;
}

}  // namespace

namespace {

// CTAs NCCL may use for the ring's send/recv: they run while the attention grid holds every SM, so
// the ring only borrows the SMs its transfer needs -- Flux 1x8 moves 89 MB per step in ~0.84 ms of
// attention, 106 GB/s, a few channels of NVLink 5.  The Ulysses exchange is not
// overlapped and keeps NCCL's default (all channels).
constexpr int kRingMaxCTAs = 16;

struct Prof {  // per-phase timing events of the last call (xdit_comm_profile)
  bool on = false, made = false, recorded = false;
  cudaEvent_t t0 = nullptr, t_a2a = nullptr, t_end = nullptr, t_step[8] = {}, c0[8] = {}, c1[8] = {};
  xdit_phases ph{};
};

}  // namespace

struct xdit_comm_s {
  int nranks = 1, rank = 0, u = 1, r = 1, device = 0;
  ncclComm_t sp = nullptr;    // the SP group's communicator (the caller's, or ours: own_sp)
  ncclComm_t all = nullptr;   // private communicator over the whole group (p2p, all-gather)
  ncclComm_t uly = nullptr, ring = nullptr;  // Ulysses row / Ring column
  bool own_sp = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_recv[2] = {nullptr, nullptr};
  Buf uly_send, uly_recv, qblk, kv[2][2], oacc, lacc, otmp, ltmp, osend, orecv, tail;
  Prof prof;
};

namespace {

int comm_finish_init(xdit_comm_s* c) {
  XCUDA(cudaGetDevice(&c->device));
  int lo = 0, hi = 0;
  XCUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  XCUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  cudaEvent_t* evs[] = {&c->ev_fork, &c->ev_recv[0], &c->ev_recv[1]};
  for (cudaEvent_t* e : evs) XCUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  if (c->nranks > 1) {
    const int i = c->rank / c->u, j = c->rank % c->u;
    // ncclCommSplit is collective over the SP communicator; every rank takes the same branches.
    if (c->own_sp) {
      c->all = c->sp;
    } else {  // never issue work on the caller's communicator: a private copy for p2p / all-gather
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      XNCCL(ncclCommSplit(c->sp, 0, c->rank, &c->all, &cfg));
    }
    if (c->u > 1) {
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      XNCCL(ncclCommSplit(c->sp, i, j, &c->uly, &cfg));
    }
    if (c->r > 1) {
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      cfg.maxCTAs = kRingMaxCTAs;
      XNCCL(ncclCommSplit(c->sp, j, i, &c->ring, &cfg));
    }
  }
  return XDIT_OK;
}

int check_async(xdit_comm_s* c) {
  ncclComm_t cs[3] = {c->all, c->uly, c->ring};
  for (ncclComm_t x : cs) {
    if (!x) continue;
    ncclResult_t st = ncclSuccess;
    XNCCL(ncclCommGetAsyncError(x, &st));
    if (st != ncclSuccess && st != ncclInProgress)
      return fail(XDIT_ERR_NCCL, "pending NCCL async error: %s", ncclGetErrorString(st));
  }
  return XDIT_OK;
}

int attn_launch(const AttnArgs& a_in, int dtype, cudaStream_t st, const Buf* scratch = nullptr) {
  AttnArgs a = a_in;
  if (scratch && scratch->p) {
    a.scratch = static_cast<float*>(scratch->p);
    a.scratch_floats = scratch->bytes / sizeof(float);
  }
  cudaError_t e = dtype == 0 ? xdit::launch_attn_fwd_bf16(a, st) : xdit::launch_attn_fwd_f32(a, st);
  if (e != cudaSuccess)
    return fail(XDIT_ERR_CUDA, "attention launch failed: %s", cudaGetErrorString(e));
  return XDIT_OK;
}

#define XRET(x)            \
  do {                     \
    int rc_ = (x);         \
    if (rc_ != XDIT_OK) return rc_; \
  } while (0)

// Timing event of phase `e` on stream `s`, only while profiling and outside a graph capture.
struct Marks {
  Prof* p;
  bool on;
  int rec(cudaEvent_t e, cudaStream_t s) {
    if (on) XCUDA(cudaEventRecord(e, s));
    return XDIT_OK;
  }
};

// What a call does with the K,V it holds besides attending to them (NEXT 1 / NEXT 3).
struct KvOpts {
  void* keep = nullptr;  // xdit_usp_attention_kv: retain the SP group's K,V (reading R2)
  void* buf = nullptr;   // xdit_usp_attention_buf: write the fresh K,V into the persistent buffer at
  int S_buf = 0;         //   the tokens' rows (text token t -> txt_row + t, image token t -> img_row + t)
  int txt_row = 0;       //   and attend over all of it (reading R6)
  int img_row = 0;
};

// One USP attention call; eb = element bytes (2: bf16 / tcgen05 path, 4: fp32 / SIMT path).
int usp_call(const void* q, const void* k, const void* v, void* out, float* lse, int B, int H,
             int S_txt, int S_img, int D, int u, int r, cudaStream_t st, xdit_comm_s* c, int eb,
             const KvOpts& kvo = KvOpts{}) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (!q || !k || !v || !out) return fail(XDIT_ERR_INVALID_ARG, "q/k/v/out must not be NULL");
  if (u != c->u || r != c->r || u * r != c->nranks)
    return fail(XDIT_ERR_COMM_MISMATCH, "(ulysses=%d, ring=%d) does not match the handle (%d, %d, n=%d)",
                u, r, c->u, c->r, c->nranks);
  const int dtype = eb == 2 ? 0 : 1;
  if (dtype == 0 && D != 64 && D != 72 && D != 128)
    return fail(XDIT_ERR_UNSUPPORTED, "bf16 path supports D in {64,72,128}, got %d", D);
  if (dtype == 1 && (D < 1 || D > 256))
    return fail(XDIT_ERR_UNSUPPORTED, "fp32 path supports D in [1,256], got %d", D);
  if (dtype == 1 && (u * r > 1 || kvo.keep || kvo.buf) && (D % 4) != 0)
    return fail(XDIT_ERR_UNSUPPORTED, "fp32 multi-rank / KV-buffer path needs D %% 4 == 0, got %d", D);
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out) || !aligned16(lse) ||
      !aligned16(kvo.keep) || !aligned16(kvo.buf))
    return fail(XDIT_ERR_ALIGNMENT, "tensor pointers must be 16-byte aligned");
  if ((int64_t(H) * D * eb) % 16 != 0)
    return fail(XDIT_ERR_ALIGNMENT, "H*D*elem_bytes must be a multiple of 16");
  Plan P;
  XRET(make_plan(B, H, S_txt, S_img, D, u, r, c->rank, &P));
  const int S_sp = S_txt + S_img;
  if (kvo.buf && (kvo.txt_row < 0 || kvo.img_row < 0 || kvo.txt_row + S_txt > kvo.S_buf ||
                  kvo.img_row + S_img > kvo.S_buf))
    return fail(XDIT_ERR_INVALID_ARG, "KV buffer rows (text at %d, image at %d) exceed S_buf=%d", kvo.txt_row,
                kvo.img_row, kvo.S_buf);
  const Sizes need = sizes_for(P, B, D, eb);
  if (need.uly3 > c->uly_recv.bytes || need.qblk > c->qblk.bytes || need.kvslot > c->kv[1][0].bytes ||
      need.oacc > c->oacc.bytes || need.lacc > c->lacc.bytes || need.ochunk * P.u > c->osend.bytes * (P.u > 1))
    return fail(XDIT_ERR_WORKSPACE, "problem exceeds the reservation; call xdit_comm_reserve first");
  XRET(check_async(c));

  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  XCUDA(cudaStreamIsCapturing(st, &cap));
  Prof& pf = c->prof;
  Marks mk{&pf, pf.on && pf.made && cap == cudaStreamCaptureStatusNone};
  pf.recorded = mk.on;
  pf.ph = xdit_phases{};
  pf.ph.ulysses = u;
  pf.ph.ring = r;

  const int i = P.i, Hh = P.Hh, L = P.S_loc[c->rank], Sb = P.S_blk[i];
  const int64_t row = int64_t(Hh) * D;  // elements per (token) row of a head-block tensor
  auto blk_off = [&](int ib) {  // sequence offset of ring block ib in SP-shard order (R2 / R6)
    int o = 0;
    for (int x = 0; x < ib; ++x) o += P.S_blk[x];
    return o;
  };
  void* kvdst = kvo.keep ? kvo.keep : kvo.buf;       // where held K,V blocks are copied to
  const int kv_total = kvo.keep ? S_sp : kvo.S_buf;  // its sequence length
  // rows of ring block ib in it: kv_keep in SP-shard order (R2), kv_buf at the tokens' own rows (R6)
  auto segs_of = [&](int ib) {
    xdit::KvSegs sg{};
    if (kvo.keep) {
      sg.n = 1;
      sg.dst[0] = blk_off(ib);
      return sg;
    }
    int bo = 0;
    for (int p = 0; p < P.u; ++p) {
      int to, tl, io, il;
      piece(S_txt, P.N, ib * P.u + p, &to, &tl);
      piece(S_img, P.N, ib * P.u + p, &io, &il);
      if (tl) sg.src[sg.n] = bo, sg.dst[sg.n++] = kvo.txt_row + to;
      if (il) sg.src[sg.n] = bo + tl, sg.dst[sg.n++] = kvo.img_row + io;
      bo += tl + il;
    }
    return sg;
  };
  // the attention over the whole KV buffer (xdit_usp_attention_buf): Q block x kv_buf
  auto buf_attention = [&](AttnArgs a) {
    a.k = kvo.buf;
    a.v = static_cast<const char*>(kvo.buf) + size_t(B) * Hh * kvo.S_buf * D * eb;
    a.Skv = kvo.S_buf;
    a.kv_b = int64_t(Hh) * kvo.S_buf * D;
    a.kv_s = D;
    a.kv_h = int64_t(kvo.S_buf) * D;
    return attn_launch(a, dtype, st, &c->tail);
  };

  XRET(mk.rec(pf.t0, st));
  // ---- N == 1: one kernel straight from the caller's tensors into the caller's output
  if (P.N == 1) {
    AttnArgs a{};
    a.q = q; a.k = k; a.v = v; a.o = out; a.lse = lse;
    a.B = B; a.H = H; a.Sq = L; a.Skv = L; a.D = D;
    a.q_b = a.kv_b = int64_t(L) * H * D; a.q_s = a.kv_s = int64_t(H) * D; a.q_h = a.kv_h = D;
    a.omap = plain_map(B, L, H, D);
    a.out_f32 = dtype;
    if (kvdst)
      XCUDA(xdit::launch_kv_place(k, v, kvdst, B, H, L, kv_total, segs_of(0), D, a.kv_b, a.kv_s, a.kv_h, eb, st));
    XRET(mk.rec(pf.t_a2a, st));
    XRET(kvo.buf ? buf_attention(a) : attn_launch(a, dtype, st, &c->tail));
    XRET(mk.rec(pf.t_step[0], st));
    XRET(mk.rec(pf.t_end, st));
    return XDIT_OK;
  }

  // ---- a2-a4: Ulysses all-to-all of Q, K, V (scatter heads, gather sequence), caller's stream
  const void *Qp = q, *Kc = k, *Vc = v;
  int64_t q_b = int64_t(L) * H * D, q_s = int64_t(H) * D;
  if (P.u > 1) {
    const void* src[3] = {q, k, v};
    const size_t chunk = need.uly3 / P.u;  // [3][B][Lmax][Hh][D] per peer
    // pack: head block p of every local token into peer p's send chunk; this rank's own head
    // block (p = j) straight into its receive chunk (no self-message)
    xdit::ChunkDst cd{};
    for (int p = 0; p < P.u; ++p)
      cd.p[p] = static_cast<char*>(p == P.j ? c->uly_recv.p : c->uly_send.p) + size_t(p) * chunk;
    for (int t = 0; t < 3; ++t)
      XCUDA(xdit::launch_uly_pack_to(src[t], cd, B, L, P.Lmax, H, D, P.u, t, 3, eb, st));
    XNCCL(ncclGroupStart());
    for (int p = 0; p < P.u; ++p) {
      if (p == P.j) continue;
      XNCCL(ncclSend(static_cast<const char*>(c->uly_send.p) + p * chunk, chunk, ncclUint8, p, c->uly, st));
      XNCCL(ncclRecv(static_cast<char*>(c->uly_recv.p) + p * chunk, chunk, ncclUint8, p, c->uly, st));
    }
    XNCCL(ncclGroupEnd());
    pf.ph.a2a_in_bytes = int64_t(P.u - 1) * int64_t(chunk);
    int len[8] = {0};
    for (int p = 0; p < P.u; ++p) len[p] = P.S_loc[i * P.u + p];
    XCUDA(xdit::launch_uly_unpack(c->uly_recv.p, c->qblk.p, B, P.Lmax, Hh, D, P.u, len, 0, 3, eb, st));
    XCUDA(xdit::launch_uly_unpack(c->uly_recv.p, c->kv[0][0].p, B, P.Lmax, Hh, D, P.u, len, 1, 3, eb, st));
    XCUDA(xdit::launch_uly_unpack(c->uly_recv.p, c->kv[0][1].p, B, P.Lmax, Hh, D, P.u, len, 2, 3, eb, st));
    Qp = c->qblk.p;
    Kc = c->kv[0][0].p;
    Vc = c->kv[0][1].p;
    q_b = int64_t(Sb) * row;
    q_s = row;
  }
  if (kvdst)  // this rank's ring block, right after the all-to-all (or straight from the caller)
    XCUDA(xdit::launch_kv_place(Kc, Vc, kvdst, B, Hh, Sb, kv_total, segs_of(i), D, q_b, q_s, D, eb, st));
  XRET(mk.rec(pf.t_a2a, st));

  // ---- destination of the final O / LSE: the caller's tensors (u == 1) or the reverse-a2a
  //      send buffer, one segment per Ulysses peer (u > 1; reading C15) -- a8 fused into the
  //      epilogue that writes the final result
  void* dst = out;
  float* dst_lse = lse;
  xdit_rowmap fmap = plain_map(B, L, H, D);
  if (P.u > 1) {
    dst = c->osend.p;
    dst_lse = reinterpret_cast<float*>(static_cast<char*>(c->osend.p) + need.ochunk_o);
    fmap.nseg = P.u;
    fmap.seg_off[0] = 0;
    for (int p = 0; p < P.u; ++p) fmap.seg_off[p + 1] = fmap.seg_off[p] + P.S_loc[i * P.u + p];
    for (int p = P.u + 1; p < 9; ++p) fmap.seg_off[p] = fmap.seg_off[P.u];
    fmap.o_seg = int64_t(need.ochunk / eb);
    fmap.o_b = int64_t(P.Lmax) * row;
    fmap.o_s = row;
    fmap.o_h = D;
    fmap.l_seg = int64_t(need.ochunk / 4);
    fmap.l_b = int64_t(Hh) * P.Lmax;
    fmap.l_h = P.Lmax;
  }

  AttnArgs a{};
  a.q = Qp; a.B = B; a.H = Hh; a.Sq = Sb; a.D = D;
  a.q_b = q_b; a.q_s = q_s; a.q_h = D;
  if (P.r == 1) {
    // ---- a6 without ring: final bf16 (or fp32) output written straight to its destination
    a.k = Kc; a.v = Vc; a.Skv = Sb;
    a.kv_b = q_b; a.kv_s = q_s; a.kv_h = D;
    a.o = dst; a.lse = dst_lse; a.omap = fmap; a.out_f32 = dtype;
    XRET(kvo.buf ? buf_attention(a) : attn_launch(a, dtype, st, &c->tail));
    XRET(mk.rec(pf.t_step[0], st));
  } else {
    // ---- a5-a7: ring loop; step s attends to the KV block of ring index (i - s) mod r (C9) on the
    //      caller's stream while the side stream sends that block to i+1 and receives block
    //      (i - s - 1) mod r from i-1 into the other slot (Table 1: overlapped)
    const int nxt = (i + 1) % P.r, prv = (i - 1 + P.r) % P.r;
    const void* curK = Kc;
    const void* curV = Vc;
    xdit_rowmap accmap = plain_map(B, Sb, Hh, D);
    // a7 fused into the attention epilogue where the kernel supports it (bf16 CTA-pair kernel): step
    // s >= 1 merges its rows into O_acc in place (LSE_acc double-buffered: lacc <-> ltmp), the last
    // step writes the merged result straight to its final destination -- no fp32 partial round trip
    const bool fuse = dtype == 0 && xdit::attn_fused_merge_supported(D);
    float* l_in = static_cast<float*>(c->lacc.p);
    float* l_out = static_cast<float*>(c->ltmp.p);
    for (int s = 0; s < P.r; ++s) {
      const int src = ((i - s) % P.r + P.r) % P.r;
      const int Skv = P.S_blk[src];
      const int nsrc = ((src - 1) % P.r + P.r) % P.r;
      const int nslot = (s + 1) & 1;
      if (s < P.r - 1) {
        // side stream: the current block is complete and the other slot is free (its last reader,
        // step s-1's attention, precedes this point of the caller's stream)
        XCUDA(cudaEventRecord(c->ev_fork, st));
        XCUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        XRET(mk.rec(pf.c0[s], c->side));
        const size_t sbytes = size_t(B) * Skv * row * eb, rbytes = size_t(B) * P.S_blk[nsrc] * row * eb;
        XNCCL(ncclGroupStart());
        XNCCL(ncclSend(curK, sbytes, ncclUint8, nxt, c->ring, c->side));
        XNCCL(ncclSend(curV, sbytes, ncclUint8, nxt, c->ring, c->side));
        XNCCL(ncclRecv(c->kv[nslot][0].p, rbytes, ncclUint8, prv, c->ring, c->side));
        XNCCL(ncclRecv(c->kv[nslot][1].p, rbytes, ncclUint8, prv, c->ring, c->side));
        XNCCL(ncclGroupEnd());
        pf.ph.ring_bytes[s] = int64_t(2 * sbytes);
        XRET(mk.rec(pf.c1[s], c->side));
        XCUDA(cudaEventRecord(c->ev_recv[s & 1], c->side));
      }
      if (!kvo.buf) {
        a.k = curK; a.v = curV; a.Skv = Skv;
        a.kv_b = int64_t(Skv) * row; a.kv_s = row; a.kv_h = D;
        a.omap = accmap; a.out_f32 = 1;
        a.merge = 0;
        if (s == 0) {
          a.o = c->oacc.p; a.lse = static_cast<float*>(c->lacc.p);
        } else if (fuse) {
          const bool last = s == P.r - 1;
          a.merge = 1;
          a.merge_final = last ? 1 : 0;
          a.acc_o = static_cast<float*>(c->oacc.p);
          a.acc_l_in = l_in;
          a.acc_l_out = l_out;
          a.acc_map = accmap;
          if (last) {
            a.o = dst; a.lse = dst_lse; a.omap = fmap; a.out_f32 = dtype;
          }
        } else {
          a.o = c->otmp.p; a.lse = static_cast<float*>(c->ltmp.p);
        }
        XRET(attn_launch(a, dtype, st, &c->tail));
        if (fuse && s > 0) std::swap(l_in, l_out);
        if (s > 0 && !fuse) {
          const bool last = s == P.r - 1;
          XCUDA(xdit::launch_lse_merge(static_cast<float*>(c->oacc.p), static_cast<float*>(c->lacc.p),
                                       static_cast<const float*>(c->otmp.p),
                                       static_cast<const float*>(c->ltmp.p), B, Sb, Hh, D,
                                       last ? dst : nullptr, last ? dst_lse : nullptr, &fmap,
                                       dtype == 0 ? 0 : 1, st));
        }
      }
      XRET(mk.rec(pf.t_step[s], st));
      if (s < P.r - 1) {
        XCUDA(cudaStreamWaitEvent(st, c->ev_recv[s & 1], 0));  // block (i-s-1) arrived, my send is done
        curK = c->kv[nslot][0].p;
        curV = c->kv[nslot][1].p;
        if (kvdst)  // the incoming ring block joins the KV buffer
          XCUDA(xdit::launch_kv_place(curK, curV, kvdst, B, Hh, P.S_blk[nsrc], kv_total, segs_of(nsrc), D,
                                      int64_t(P.S_blk[nsrc]) * row, row, D, eb, st));
      }
    }
    if (kvo.buf) {  // every fresh block of the SP group is in the buffer: attend over all of it
      a.o = dst; a.lse = dst_lse; a.omap = fmap; a.out_f32 = dtype;
      XRET(buf_attention(a));
      XRET(mk.rec(pf.t_step[P.r - 1], st));
    }
  }

  // ---- a9-a10: reverse all-to-all of O (+ LSE) and unpack into the caller's layout
  if (P.u > 1) {
    const size_t oc = need.ochunk;
    XCUDA(cudaMemcpyAsync(static_cast<char*>(c->orecv.p) + P.j * oc, static_cast<const char*>(c->osend.p) + P.j * oc,
                          oc, cudaMemcpyDeviceToDevice, st));
    XNCCL(ncclGroupStart());
    for (int p = 0; p < P.u; ++p) {
      if (p == P.j) continue;
      XNCCL(ncclSend(static_cast<const char*>(c->osend.p) + p * oc, oc, ncclUint8, p, c->uly, st));
      XNCCL(ncclRecv(static_cast<char*>(c->orecv.p) + p * oc, oc, ncclUint8, p, c->uly, st));
    }
    XNCCL(ncclGroupEnd());
    pf.ph.a2a_out_bytes = int64_t(P.u - 1) * int64_t(oc);
    XCUDA(xdit::launch_uly_unpack_out(
        c->orecv.p,
        reinterpret_cast<const float*>(static_cast<const char*>(c->orecv.p) + need.ochunk_o),
        int64_t(oc), int64_t(oc), out, lse, B, L, P.Lmax, Hh, D, P.u, eb, st));
  }
  XRET(mk.rec(pf.t_end, st));
  return XDIT_OK;
}

int prof_make(Prof& p) {
  if (p.made) return XDIT_OK;
  cudaEvent_t* evs[3 + 3 * 8];
  int n = 0;
  evs[n++] = &p.t0;
  evs[n++] = &p.t_a2a;
  evs[n++] = &p.t_end;
  for (int s = 0; s < 8; ++s) {
    evs[n++] = &p.t_step[s];
    evs[n++] = &p.c0[s];
    evs[n++] = &p.c1[s];
  }
  for (int x = 0; x < n; ++x) XCUDA(cudaEventCreate(evs[x]));
  p.made = true;
  return XDIT_OK;
}

void prof_free(Prof& p) {
  if (!p.made) return;
  cudaEvent_t evs[] = {p.t0, p.t_a2a, p.t_end};
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  for (int s = 0; s < 8; ++s) {
    cudaEventDestroy(p.t_step[s]);
    cudaEventDestroy(p.c0[s]);
    cudaEventDestroy(p.c1[s]);
  }
  p.made = false;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* xdit_last_error(void) { return g_err.c_str(); }

int xdit_version(void) { return XDIT_ABI_VERSION; }

uint64_t xdit_launch_count(void) { return xdit::g_launches.load(std::memory_order_relaxed); }

int xdit_usp_shard(int S_txt, int S_img, int nranks, int g, int* txt_off, int* txt_len,
                   int* img_off, int* img_len) {
  if (S_txt < 0 || S_img < 0 || nranks < 1 || g < 0 || g >= nranks || !txt_off || !txt_len ||
      !img_off || !img_len)
    return fail(XDIT_ERR_INVALID_ARG, "xdit_usp_shard: bad arguments");
  piece(S_txt, nranks, g, txt_off, txt_len);
  piece(S_img, nranks, g, img_off, img_len);
  if (*txt_len + *img_len == 0)
    return fail(XDIT_ERR_EMPTY_SHARD, "rank %d of %d holds no tokens", g, nranks);
  return XDIT_OK;
}

int xdit_usp_plan(int B, int H, int S_txt, int S_img, int D, int ulysses, int ring, int rank,
                  xdit_plan* out) {
  if (!out) return fail(XDIT_ERR_INVALID_ARG, "out is NULL");
  Plan P;
  XRET(make_plan(B, H, S_txt, S_img, D, ulysses, ring, rank, &P));
  std::memset(out, 0, sizeof *out);
  out->nranks = P.N;
  out->rank = rank;
  out->ulysses = P.u;
  out->ring = P.r;
  out->i = P.i;
  out->j = P.j;
  out->Hh = P.Hh;
  out->S_loc = P.S_loc[rank];
  out->Lmax = P.Lmax;
  out->S_blk = P.S_blk[P.i];
  out->ring_next = (P.i + 1) % P.r;
  out->ring_prev = (P.i - 1 + P.r) % P.r;
  out->nseg = P.u;
  for (int p = 0; p < P.u; ++p) out->seg_off[p + 1] = out->seg_off[p] + P.S_loc[P.i * P.u + p];
  for (int p = P.u + 1; p < 9; ++p) out->seg_off[p] = out->seg_off[P.u];
  const Sizes sz = sizes_for(P, B, D, 2);
  out->a2a_bytes_per_peer = P.u > 1 ? int64_t(sz.uly3 / P.u) : 0;
  for (int s = 0; s < P.r; ++s) {
    const int src = ((P.i - s) % P.r + P.r) % P.r;
    out->ring_src[s] = src;
    out->ring_rows[s] = P.S_blk[src];
    out->ring_bytes[s] = s < P.r - 1 ? int64_t(2) * B * P.S_blk[src] * P.Hh * D * 2 : 0;
  }
  return XDIT_OK;
}

int xdit_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(XDIT_ERR_INVALID_ARG, "id_out is NULL");
  ncclUniqueId id;
  XNCCL(ncclGetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return XDIT_OK;
}

int xdit_comm_init(const void* unique_id, int nranks, int rank, int ulysses, int ring,
                   xdit_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || ulysses < 1 || ring < 1)
    return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_init: bad arguments");
  if (ulysses * ring != nranks)
    return fail(XDIT_ERR_COMM_MISMATCH, "ulysses*ring=%d != nranks=%d", ulysses * ring, nranks);
  if (nranks > 1 && !unique_id) return fail(XDIT_ERR_INVALID_ARG, "unique_id is NULL");
  auto* c = new xdit_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->u = ulysses;
  c->r = ring;
  if (nranks > 1) {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    ncclResult_t rr = ncclCommInitRank(&c->sp, nranks, id, rank);
    if (rr != ncclSuccess) {
      delete c;
      return fail(XDIT_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(rr));
    }
    c->own_sp = true;
  }
  int rc = comm_finish_init(c);
  if (rc != XDIT_OK) {
    xdit_comm_destroy(c);
    return rc;
  }
  *out = c;
  return XDIT_OK;
}

int xdit_comm_create(void* nccl_comm, int ulysses, int ring, xdit_comm_t* out) {
  if (!out || ulysses < 1 || ring < 1) return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_create: bad arguments");
  int n = 1, rank = 0;
  if (nccl_comm) {
    XNCCL(ncclCommCount(static_cast<ncclComm_t>(nccl_comm), &n));
    XNCCL(ncclCommUserRank(static_cast<ncclComm_t>(nccl_comm), &rank));
  } else if (ulysses * ring != 1) {
    return fail(XDIT_ERR_INVALID_ARG, "nccl_comm may be NULL only for ulysses*ring == 1");
  }
  if (ulysses * ring != n)
    return fail(XDIT_ERR_COMM_MISMATCH, "ulysses*ring=%d != communicator size %d", ulysses * ring, n);
  auto* c = new xdit_comm_s();
  c->nranks = n;
  c->rank = rank;
  c->u = ulysses;
  c->r = ring;
  c->sp = static_cast<ncclComm_t>(nccl_comm);
  c->own_sp = false;
  int rc = comm_finish_init(c);
  if (rc != XDIT_OK) {
    xdit_comm_destroy(c);
    return rc;
  }
  *out = c;
  return XDIT_OK;
}

int xdit_comm_reserve(xdit_comm_t c, int B, int H, int S_txt, int S_img, int D, int elem_bytes) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (elem_bytes != 2 && elem_bytes != 4) return fail(XDIT_ERR_UNSUPPORTED, "elem_bytes must be 2 or 4");
  Plan P;
  XRET(make_plan(B, H, S_txt, S_img, D, c->u, c->r, c->rank, &P));
  const Sizes s = sizes_for(P, B, D, elem_bytes);
  XCUDA(cudaStreamSynchronize(c->side));  // no ring transfer may still use a buffer being replaced
  XRET(ensure(&c->uly_send, s.uly3));
  XRET(ensure(&c->uly_recv, s.uly3));
  XRET(ensure(&c->qblk, s.qblk));
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) XRET(ensure(&c->kv[a][b], s.kvslot));
  XRET(ensure(&c->oacc, s.oacc));
  XRET(ensure(&c->lacc, s.lacc));
  XRET(ensure(&c->otmp, s.oacc));
  XRET(ensure(&c->ltmp, s.lacc));
  XRET(ensure(&c->osend, s.ochunk * P.u * (P.u > 1)));
  XRET(ensure(&c->orecv, s.ochunk * P.u * (P.u > 1)));
  if (elem_bytes == 2) XRET(ensure(&c->tail, xdit::attn_scratch_floats(D) * sizeof(float)));
  return XDIT_OK;
}

int xdit_comm_info(xdit_comm_t c, int* nranks, int* rank, int* ulysses, int* ring) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (nranks) *nranks = c->nranks;
  if (rank) *rank = c->rank;
  if (ulysses) *ulysses = c->u;
  if (ring) *ring = c->r;
  return XDIT_OK;
}

int xdit_comm_destroy(xdit_comm_t c) {
  if (!c) return XDIT_OK;
  if (c->side) cudaStreamSynchronize(c->side);
  cudaDeviceSynchronize();  // no kernel or NCCL operation of this handle still in flight
  Buf* bufs[] = {&c->uly_send, &c->uly_recv, &c->qblk, &c->kv[0][0], &c->kv[0][1], &c->kv[1][0],
                 &c->kv[1][1], &c->oacc, &c->lacc, &c->otmp, &c->ltmp, &c->osend, &c->orecv, &c->tail};
  for (Buf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->uly) ncclCommDestroy(c->uly);
  if (c->ring) ncclCommDestroy(c->ring);
  if (c->all && c->all != c->sp) ncclCommDestroy(c->all);
  if (c->sp && c->own_sp) ncclCommDestroy(c->sp);
  cudaEvent_t evs[] = {c->ev_fork, c->ev_recv[0], c->ev_recv[1]};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  prof_free(c->prof);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return XDIT_OK;
}

int xdit_p2p(xdit_comm_t c, const xdit_p2p_op* ops, int n, xdit_stream_t stream) {
  if (!c || n < 0 || (n > 0 && !ops)) return fail(XDIT_ERR_INVALID_ARG, "xdit_p2p: bad arguments");
  for (int x = 0; x < n; ++x) {
    if (ops[x].peer < 0 || ops[x].peer >= c->nranks || (ops[x].bytes && !ops[x].buf))
      return fail(XDIT_ERR_INVALID_ARG, "xdit_p2p: op %d (peer %d, %zu bytes) invalid for %d ranks", x, ops[x].peer,
                  ops[x].bytes, c->nranks);
    if (ops[x].peer == c->rank && ops[x].bytes)
      return fail(XDIT_ERR_INVALID_ARG, "xdit_p2p: op %d addresses this rank itself", x);
  }
  if (n == 0 || c->nranks == 1) return XDIT_OK;
  XRET(check_async(c));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  XNCCL(ncclGroupStart());
  for (int x = 0; x < n; ++x) {
    if (!ops[x].bytes) continue;
    if (ops[x].is_send)
      XNCCL(ncclSend(ops[x].buf, ops[x].bytes, ncclUint8, ops[x].peer, c->all, st));
    else
      XNCCL(ncclRecv(ops[x].buf, ops[x].bytes, ncclUint8, ops[x].peer, c->all, st));
  }
  XNCCL(ncclGroupEnd());
  return XDIT_OK;
}

int xdit_comm_profile(xdit_comm_t c, int enable) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (enable) XRET(prof_make(c->prof));
  c->prof.on = enable != 0;
  c->prof.recorded = false;
  return XDIT_OK;
}

int xdit_comm_phases(xdit_comm_t c, xdit_phases* out) {
  if (!c || !out) return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_phases: NULL argument");
  Prof& p = c->prof;
  *out = p.ph;
  out->valid = 0;
  if (!p.recorded) return XDIT_OK;
  XCUDA(cudaEventSynchronize(p.t_end));
  const int rs = c->r;
  for (int s = 0; s < rs - 1 && s < 8; ++s) XCUDA(cudaEventSynchronize(p.c1[s]));
  auto el = [](cudaEvent_t a, cudaEvent_t b, float* ms) -> int {
    XCUDA(cudaEventElapsedTime(ms, a, b));
    return XDIT_OK;
  };
  XRET(el(p.t0, p.t_end, &out->total_ms));
  XRET(el(p.t0, p.t_a2a, &out->a2a_in_ms));
  XRET(el(p.t_step[rs - 1], p.t_end, &out->a2a_out_ms));
  for (int s = 0; s < rs && s < 8; ++s) {
    XRET(el(s == 0 ? p.t_a2a : p.t_step[s - 1], p.t_step[s], &out->attn_ms[s]));
    if (s < rs - 1) XRET(el(p.c0[s], p.c1[s], &out->ring_comm_ms[s]));
  }
  out->valid = 1;
  return XDIT_OK;
}

int xdit_usp_attention(const void* q, const void* k, const void* v, void* out, float* lse, int B,
                       int H, int S_txt, int S_img, int D, int ulysses, int ring,
                       xdit_stream_t stream, xdit_comm_t comm) {
  return usp_call(q, k, v, out, lse, B, H, S_txt, S_img, D, ulysses, ring,
                  reinterpret_cast<cudaStream_t>(stream), comm, 2);
}

int xdit_usp_attention_f32(const float* q, const float* k, const float* v, float* out, float* lse,
                           int B, int H, int S_txt, int S_img, int D, int ulysses, int ring,
                           xdit_stream_t stream, xdit_comm_t comm) {
  return usp_call(q, k, v, out, lse, B, H, S_txt, S_img, D, ulysses, ring,
                  reinterpret_cast<cudaStream_t>(stream), comm, 4);
}

int xdit_usp_attention_kv(const void* q, const void* k, const void* v, void* out, float* lse, void* kv_keep,
                          int B, int H, int S_txt, int S_img, int D, int ulysses, int ring,
                          xdit_stream_t stream, xdit_comm_t comm) {
  if (!kv_keep) return fail(XDIT_ERR_INVALID_ARG, "kv_keep must not be NULL (use xdit_usp_attention)");
  KvOpts o;
  o.keep = kv_keep;
  return usp_call(q, k, v, out, lse, B, H, S_txt, S_img, D, ulysses, ring,
                  reinterpret_cast<cudaStream_t>(stream), comm, 2, o);
}

int xdit_usp_attention_buf(const void* q, const void* k, const void* v, void* out, float* lse, void* kv_buf, int B,
                           int H, int S_txt, int S_img, int D, int ulysses, int ring, int S_buf, int txt_row,
                           int img_row, int dtype, xdit_stream_t stream, xdit_comm_t comm) {
  if (!kv_buf) return fail(XDIT_ERR_INVALID_ARG, "kv_buf must not be NULL");
  if (dtype != 0 && dtype != 1) return fail(XDIT_ERR_UNSUPPORTED, "dtype must be 0 (bf16) or 1 (fp32)");
  KvOpts o;
  o.buf = kv_buf;
  o.S_buf = S_buf;
  o.txt_row = txt_row;
  o.img_row = img_row;
  return usp_call(q, k, v, out, lse, B, H, S_txt, S_img, D, ulysses, ring,
                  reinterpret_cast<cudaStream_t>(stream), comm, dtype == 0 ? 2 : 4, o);
}

int xdit_kv_retain(const void* k_blk, const void* v_blk, void* kv_keep, int B, int Hh, int S_blk, int S_total,
                   int seq_off, int D, int64_t src_b, int64_t src_s, int64_t src_h, int elem_bytes,
                   xdit_stream_t stream) {
  if (!k_blk || !v_blk || !kv_keep) return fail(XDIT_ERR_INVALID_ARG, "k_blk, v_blk, kv_keep must not be NULL");
  if (B < 0 || Hh < 1 || S_blk < 0 || D < 1 || seq_off < 0 || seq_off + S_blk > S_total ||
      (elem_bytes != 2 && elem_bytes != 4))
    return fail(XDIT_ERR_INVALID_ARG, "bad kv_retain shape (B=%d Hh=%d S_blk=%d S_total=%d off=%d D=%d eb=%d)", B,
                Hh, S_blk, S_total, seq_off, D, elem_bytes);
  const int vec_elems = 16 / elem_bytes;
  if (!aligned16(k_blk) || !aligned16(v_blk) || !aligned16(kv_keep) || D % vec_elems || src_b % vec_elems ||
      src_s % vec_elems || src_h % vec_elems)
    return fail(XDIT_ERR_ALIGNMENT, "kv_retain needs 16-byte aligned pointers, rows and strides");
  const cudaError_t e = xdit::launch_kv_retain(k_blk, v_blk, kv_keep, B, Hh, S_blk, S_total, seq_off, D, src_b,
                                               src_s, src_h, elem_bytes, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(XDIT_ERR_CUDA, "kv_retain launch failed: %s", cudaGetErrorString(e));
  return XDIT_OK;
}

int xdit_cfg_combine(const void* eps_cond, const void* eps_uncond, void* out, int64_t n, float g, int dtype,
                     xdit_stream_t stream) {
  if (!eps_cond || !eps_uncond || !out || n < 0 || (dtype != 0 && dtype != 1))
    return fail(XDIT_ERR_INVALID_ARG, "cfg_combine: NULL pointer, n < 0 or dtype not in {0,1}");
  if (!aligned16(eps_cond) || !aligned16(eps_uncond) || !aligned16(out) || n % (dtype == 0 ? 8 : 4))
    return fail(XDIT_ERR_ALIGNMENT, "cfg_combine needs 16-byte aligned buffers and n %% %d == 0",
                dtype == 0 ? 8 : 4);
  const cudaError_t e =
      xdit::launch_cfg_combine(eps_cond, eps_uncond, out, n, g, dtype, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(XDIT_ERR_CUDA, "cfg_combine launch failed: %s", cudaGetErrorString(e));
  return XDIT_OK;
}

int xdit_cfg_tail(const void* eps_local, void* eps_gather, void* eps_out, int64_t n, float g, int dtype,
                  xdit_stream_t stream, xdit_comm_t comm) {
  if (!comm) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (comm->nranks != 2)
    return fail(XDIT_ERR_COMM_MISMATCH, "cfg_tail needs a handle over exactly the 2 cfg ranks (got %d)",
                comm->nranks);
  if (!eps_local || !eps_gather || !eps_out || n < 0 || (dtype != 0 && dtype != 1))
    return fail(XDIT_ERR_INVALID_ARG, "cfg_tail: NULL pointer, n < 0 or dtype not in {0,1}");
  const int eb = dtype == 0 ? 2 : 4;
  if (!aligned16(eps_local) || !aligned16(eps_gather) || !aligned16(eps_out) || n % (dtype == 0 ? 8 : 4))
    return fail(XDIT_ERR_ALIGNMENT, "cfg_tail needs 16-byte aligned buffers and n %% %d == 0", dtype == 0 ? 8 : 4);
  XRET(check_async(comm));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // All-gather of the two branches' predictions over the cfg pair (rank 0 = conditional, rank 1 =
  // unconditional: reading R3) on the handle's private communicator, then the combine on every rank.
  XNCCL(ncclAllGather(eps_local, eps_gather, size_t(n) * eb, ncclUint8, comm->all, st));
  const char* gb = static_cast<const char*>(eps_gather);
  XCUDA(xdit::launch_cfg_combine(gb, gb + size_t(n) * eb, eps_out, n, g, dtype, st));
  return XDIT_OK;
}

size_t xdit_pf_block_workspace_bytes(int B, int n, int H, int D, int dtype) {
  if (B < 0 || n < 0 || H < 1 || D < 1 || (dtype != 0 && dtype != 1)) return 0;
  return xdit::pf_workspace_bytes(B, n, H, D, dtype);
}

int xdit_pf_block(void* h, void* kv_buf, const float* w, void* work, size_t work_bytes, int B, int H, int S, int off,
                  int n, int D, int dtype, xdit_stream_t stream) {
  if (!h || !kv_buf || !w || !work) return fail(XDIT_ERR_INVALID_ARG, "xdit_pf_block: NULL pointer");
  if (B < 0 || H < 1 || S < 1 || n < 0 || off < 0 || off + n > S || D < 1 || (dtype != 0 && dtype != 1))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_pf_block: bad sizes (B=%d H=%d S=%d off=%d n=%d D=%d dtype=%d)", B, H, S,
                off, n, D, dtype);
  if (dtype == 0 && D != 64 && D != 72 && D != 128)
    return fail(XDIT_ERR_UNSUPPORTED, "bf16 path supports D in {64,72,128}, got %d", D);
  if (dtype == 1 && (D > 256 || D % 8))
    return fail(XDIT_ERR_UNSUPPORTED, "fp32 path supports D %% 8 == 0 and D <= 256, got %d", D);
  if (!aligned16(h) || !aligned16(kv_buf) || !aligned16(w) || !aligned16(work))
    return fail(XDIT_ERR_ALIGNMENT, "xdit_pf_block: pointers must be 16-byte aligned");
  if (work_bytes < xdit::pf_workspace_bytes(B, n, H, D, dtype))
    return fail(XDIT_ERR_WORKSPACE, "xdit_pf_block: workspace of %zu bytes < %zu", work_bytes,
                xdit::pf_workspace_bytes(B, n, H, D, dtype));
  XCUDA(xdit::launch_pf_block(h, kv_buf, w, work, B, H, S, off, n, D, dtype, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_pf_sampler(void* x, const void* eps, int64_t n, float sigma, int dtype, xdit_stream_t stream) {
  if (!x || !eps || n < 0 || (dtype != 0 && dtype != 1)) return fail(XDIT_ERR_INVALID_ARG, "xdit_pf_sampler: bad arguments");
  if (!aligned16(x) || !aligned16(eps) || n % 8) return fail(XDIT_ERR_ALIGNMENT, "xdit_pf_sampler: 16-byte alignment, n %% 8 == 0");
  XCUDA(xdit::launch_pf_sampler(x, eps, n, sigma, dtype, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_pf_qkv(const void* h, const float* w, void* q, void* k, void* v, int B, int n, int H, int D, int dtype,
                xdit_stream_t stream) {
  if (!h || !w || !q || !k || !v || B < 0 || n < 0 || H < 1 || D < 1 || (dtype != 0 && dtype != 1))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_pf_qkv: bad arguments");
  if (D % 8 || !aligned16(h) || !aligned16(w) || !aligned16(q) || !aligned16(k) || !aligned16(v))
    return fail(XDIT_ERR_ALIGNMENT, "xdit_pf_qkv: D %% 8 == 0 and 16-byte aligned pointers required");
  XCUDA(xdit::launch_pf_qkv(h, w, q, k, v, B, n, H, D, dtype, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_pf_residual(void* h, const void* o, const float* w, int B, int n, int H, int D, int dtype,
                     xdit_stream_t stream) {
  if (!h || !o || !w || B < 0 || n < 0 || H < 1 || D < 1 || (dtype != 0 && dtype != 1))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_pf_residual: bad arguments");
  if (D % 8 || !aligned16(h) || !aligned16(o) || !aligned16(w))
    return fail(XDIT_ERR_ALIGNMENT, "xdit_pf_residual: D %% 8 == 0 and 16-byte aligned pointers required");
  XCUDA(xdit::launch_pf_residual(h, o, w, B, n, H, D, dtype, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_vae_conv3x3(const float* in, int H, int Ci, int W, const float* w, const float* b, float* out, int Co,
                     int act_up, xdit_stream_t stream) {
  if (!in || !w || !b || !out) return fail(XDIT_ERR_INVALID_ARG, "xdit_vae_conv3x3: NULL pointer");
  if (H < 0 || Ci < 1 || W < 0 || Co < 1 || (act_up != 0 && act_up != 1))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_vae_conv3x3: bad sizes (H=%d Ci=%d W=%d Co=%d act_up=%d)", H, Ci, W, Co,
                act_up);
  if (!aligned16(w)) return fail(XDIT_ERR_ALIGNMENT, "xdit_vae_conv3x3: weights must be 16-byte aligned");
  XCUDA(xdit::launch_vae_conv3x3(in, H, Ci, W, w, b, out, Co, act_up, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_vae_conv3x3_bf16(const void* in, int H, int Ci, int W, const void* wt, const float* b, void* out, int Co,
                          int act_up, xdit_stream_t stream) {
  if (!in || !wt || !b || !out) return fail(XDIT_ERR_INVALID_ARG, "xdit_vae_conv3x3_bf16: NULL pointer");
  if (H < 0 || Ci < 1 || W < 0 || Co < 1 || (act_up != 0 && act_up != 1))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_vae_conv3x3_bf16: bad sizes (H=%d Ci=%d W=%d Co=%d act_up=%d)", H, Ci, W,
                Co, act_up);
  if (Ci % 8 || !aligned16(in) || !aligned16(wt) || !aligned16(out))
    return fail(XDIT_ERR_ALIGNMENT, "xdit_vae_conv3x3_bf16: Ci %% 8 == 0 and 16-byte aligned pointers required");
  const cudaError_t e = xdit::launch_vae_conv_tc(in, H, Ci, W, wt, b, out, Co, act_up, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(XDIT_ERR_CUDA, "vae conv (tcgen05) launch failed: %s", cudaGetErrorString(e));
  return XDIT_OK;
}

int xdit_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H,
                  int Sq, int Skv, int D, int64_t q_b, int64_t q_s, int64_t q_h, int64_t kv_b,
                  int64_t kv_s, int64_t kv_h, const xdit_rowmap* omap, int dtype, int out_f32,
                  void* scratch, size_t scratch_bytes, xdit_stream_t stream) {
  if (!q || !k || !v || !o) return fail(XDIT_ERR_INVALID_ARG, "q/k/v/o must not be NULL");
  if (B < 0 || H <= 0 || Sq < 0 || Skv <= 0) return fail(XDIT_ERR_INVALID_ARG, "bad sizes");
  if (dtype != 0 && dtype != 1) return fail(XDIT_ERR_UNSUPPORTED, "dtype must be 0 (bf16) or 1 (fp32)");
  XRET(check_map(omap, Sq));
  if (dtype == 0) {
    if (D != 64 && D != 72 && D != 128) return fail(XDIT_ERR_UNSUPPORTED, "bf16 kernel supports D in {64,72,128}, got %d", D);
    if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o))
      return fail(XDIT_ERR_ALIGNMENT, "q/k/v/o must be 16-byte aligned");
    const int64_t st[6] = {q_b, q_s, q_h, kv_b, kv_s, kv_h};
    for (int64_t x : st)
      if (x % 8 != 0) return fail(XDIT_ERR_ALIGNMENT, "bf16 strides must be multiples of 8 elements");
    XRET(check_map_align(omap, out_f32 ? 4 : 8));
  } else {
    if (D < 1 || D > 256) return fail(XDIT_ERR_UNSUPPORTED, "fp32 kernel supports D in [1,256], got %d", D);
  }
  AttnArgs a{};
  a.q = q; a.k = k; a.v = v; a.o = o; a.lse = lse;
  a.B = B; a.H = H; a.Sq = Sq; a.Skv = Skv; a.D = D;
  a.q_b = q_b; a.q_s = q_s; a.q_h = q_h; a.kv_b = kv_b; a.kv_s = kv_s; a.kv_h = kv_h;
  a.omap = *omap;
  a.out_f32 = dtype == 1 ? 1 : out_f32;
  if (scratch) {
    if (!aligned16(scratch)) return fail(XDIT_ERR_ALIGNMENT, "scratch must be 16-byte aligned");
    a.scratch = static_cast<float*>(scratch);
    a.scratch_floats = scratch_bytes / sizeof(float);
  }
  return attn_launch(a, dtype, reinterpret_cast<cudaStream_t>(stream));
}

size_t xdit_attn_scratch_bytes(int D) {
  if (D <= 0) return 0;
  return xdit::attn_scratch_floats(D) * sizeof(float);
}

int xdit_lse_merge(float* o_acc, float* lse_acc, const float* o_s, const float* lse_s, int B, int S,
                   int Hh, int D, void* final, float* final_lse, const xdit_rowmap* final_map,
                   int final_dtype, xdit_stream_t stream) {
  if (!o_acc || !lse_acc || !o_s || !lse_s) return fail(XDIT_ERR_INVALID_ARG, "NULL merge operand");
  if (B < 0 || S < 0 || Hh <= 0 || D <= 0) return fail(XDIT_ERR_INVALID_ARG, "bad sizes");
  if (D % 4 != 0) return fail(XDIT_ERR_ALIGNMENT, "merge needs D %% 4 == 0");
  if (!aligned16(o_acc) || !aligned16(o_s)) return fail(XDIT_ERR_ALIGNMENT, "o_acc/o_s must be 16-byte aligned");
  if (final) {
    XRET(check_map(final_map, S));
    if (final_dtype != 0 && final_dtype != 1) return fail(XDIT_ERR_UNSUPPORTED, "final_dtype must be 0 or 1");
    XRET(check_map_align(final_map, 4));
  }
  XCUDA(xdit::launch_lse_merge(o_acc, lse_acc, o_s, lse_s, B, S, Hh, D, final, final_lse, final_map,
                               final_dtype, reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_uly_pack(const void* x, void* send, int B, int L, int Lmax, int H, int D, int u, int slot,
                  int nslots, int elem_bytes, xdit_stream_t stream) {
  if (!x || !send || B < 0 || L < 0 || Lmax < L || H <= 0 || D <= 0 || u < 1 || u > 8 || H % u != 0 ||
      slot < 0 || slot >= nslots || (elem_bytes != 2 && elem_bytes != 4))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_uly_pack: bad arguments");
  XCUDA(xdit::launch_uly_pack(x, send, B, L, Lmax, H, D, u, slot, nslots, elem_bytes,
                              reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_uly_unpack(const void* recv, void* y, int B, int Lmax, int Hh, int D, int u,
                    const int* len, int slot, int nslots, int elem_bytes, xdit_stream_t stream) {
  if (!recv || !y || !len || B < 0 || Hh <= 0 || D <= 0 || u < 1 || u > 8 || slot < 0 ||
      slot >= nslots || (elem_bytes != 2 && elem_bytes != 4))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_uly_unpack: bad arguments");
  for (int p = 0; p < u; ++p)
    if (len[p] < 0 || len[p] > Lmax) return fail(XDIT_ERR_INVALID_ARG, "xdit_uly_unpack: bad len");
  XCUDA(xdit::launch_uly_unpack(recv, y, B, Lmax, Hh, D, u, len, slot, nslots, elem_bytes,
                                reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

int xdit_uly_unpack_out(const void* orecv, const float* lrecv, int64_t peer_stride_bytes,
                        int64_t lse_peer_stride_bytes, void* out, float* lse, int B, int L,
                        int Lmax, int Hh, int D, int u, int elem_bytes, xdit_stream_t stream) {
  if (!orecv || !out || B < 0 || L < 0 || Lmax < L || Hh <= 0 || D <= 0 || u < 1 ||
      (elem_bytes != 2 && elem_bytes != 4))
    return fail(XDIT_ERR_INVALID_ARG, "xdit_uly_unpack_out: bad arguments");
  XCUDA(xdit::launch_uly_unpack_out(orecv, lrecv, peer_stride_bytes, lse_peer_stride_bytes, out, lse,
                                    B, L, Lmax, Hh, D, u, elem_bytes,
                                    reinterpret_cast<cudaStream_t>(stream)));
  return XDIT_OK;
}

}  // extern "C"
