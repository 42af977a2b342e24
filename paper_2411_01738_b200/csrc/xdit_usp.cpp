// xdit_usp.cpp -- host side of libxdit_usp.so: argument validation, the in-context shard rule,
// workspace ownership, NCCL sub-communicators, and the stream/event orchestration of one USP
// attention call (include/xdit_usp.h).
//
// USP (§4.1.4) on a 2D mesh, rank g = i*u + j (reading C6):
//   Ulysses a2a within the row {i*u + j'} (§4.1.1), Ring P2P within the column {i'*u + j}
//   (§4.1.1), every collective on an internal high-priority side stream joined back to the
//   caller's stream with events; no host synchronisation anywhere in the call.
//
// Two transports move the bytes:
//   * NCCL: grouped ncclSend/ncclRecv on the Ulysses / Ring sub-communicators;
//   * peer memory (xdit_comm_init_peer): every rank maps the receive buffers of the ranks it sends
//     to (CUDA IPC; over NVLink/NVSwitch between GPUs), the Ulysses pack kernel stores straight
//     into the peers' receive buffers, ring KV blocks and O chunks are copied peer-to-peer, and the
//     ranks order their streams with 32-bit flags in device memory -- cuStreamWriteValue32 into the
//     peer's flag (preceded by a system-wide fence) and cuStreamWaitValue32 (>=) on the local one.
//     No SM spins and no host thread waits, so the call stays stream-ordered and graph-capturable,
//     and several ranks may even share one GPU (how the multi-rank tests run on a 1-GPU box).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <unistd.h>

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
  if (m->seg_table)
    for (int s = 0; s < m->nseg && s < 8; ++s)
      if (m->o_seg_off[s] % vec_elems != 0)
        return fail(XDIT_ERR_ALIGNMENT, "segment offsets must be multiples of %d elements", vec_elems);
  return XDIT_OK;
}

}  // namespace

namespace {
// Peer-memory transport: exported buffers (blob handle index) and flag words.
enum { kHUly = 0, kHORecv = 1, kHKV = 2 /* kHKV + 2*slot + (0 K, 1 V) */, kHFlags = 6, kHMbox = 7, kNHandles = 8 };
// flag words: Ulysses data, O return, ring data / credit, mailbox data / ack (per source rank),
// CFG tail data / ack
enum { kFA2A = 0, kFO = 8, kFData = 16, kFCredit = 18, kFP2P = 32, kFAck = 40, kFCfg = 48, kFCfgAck = 50,
       kFlagWords = 64 };
constexpr uint32_t kBlobMagic = 0x31504458u;  // "XDP1"
struct PeerBlob {
  uint32_t magic;
  int32_t rank, nranks, u, r, device, pid;
  uint32_t valid;                    // bit k: handle k exported
  uint64_t bytes[kNHandles];         // allocation sizes
  cudaIpcMemHandle_t h[kNHandles];
};
static_assert(sizeof(PeerBlob) <= XDIT_PEER_BLOB_BYTES, "peer blob size");

struct MemOps {
  PFN_cuStreamWaitValue32_v11070 wait = nullptr;
  PFN_cuStreamWriteValue32_v11070 write = nullptr;
};
const MemOps* memops() {
  static MemOps m = [] {
    MemOps x;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      x.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(f);
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      x.write = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(f);
    return x;
  }();
  return (m.wait && m.write) ? &m : nullptr;
}
struct PeerMap {
  void* ptr[kNHandles] = {};
  uint64_t bytes[kNHandles] = {};
  bool opened[kNHandles] = {};  // true: an IPC mapping this handle must close
};
}  // namespace

struct xdit_comm_s {
  int nranks = 1, rank = 0, u = 1, r = 1, device = 0;
  int transport = XDIT_TRANSPORT_NCCL;
  uint32_t* flags = nullptr;  // peer transport: kFlagWords words written by the peers
  bool connected = false;
  std::vector<PeerMap> peer;  // peer transport: per SP rank (self = local pointers)
  size_t mbox_region = 0;     // peer transport: mailbox bytes per source rank
  uint32_t cfg_epoch = 0;     // peer transport: xdit_cfg_tail calls issued
  ncclComm_t sp = nullptr, uly = nullptr, ring = nullptr;
  bool own_sp = false;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_a2a = nullptr, ev_o = nullptr, ev_o_a2a = nullptr;
  cudaEvent_t ev_kdone[2] = {nullptr, nullptr}, ev_recv[2] = {nullptr, nullptr};
  Buf uly_send, uly_recv, qblk, kv[2][2], oacc, lacc, otmp, ltmp, osend, orecv, tail, mbox;
};

namespace {

int comm_finish_init(xdit_comm_s* c) {
  XCUDA(cudaGetDevice(&c->device));
  int lo = 0, hi = 0;
  XCUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  XCUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  cudaEvent_t* evs[] = {&c->ev_start, &c->ev_a2a, &c->ev_o, &c->ev_o_a2a,
                        &c->ev_kdone[0], &c->ev_kdone[1], &c->ev_recv[0], &c->ev_recv[1]};
  for (cudaEvent_t* e : evs) XCUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  if (c->transport == XDIT_TRANSPORT_PEER) {
    if (!memops()) return fail(XDIT_ERR_UNSUPPORTED, "stream memory operations (cuStreamWaitValue32) unavailable");
    XCUDA(cudaMalloc(&c->flags, kFlagWords * sizeof(uint32_t)));
    XCUDA(cudaMemset(c->flags, 0, kFlagWords * sizeof(uint32_t)));
    const uint32_t one = 1;  // my ring successor's slot 1 is free before the first call
    XCUDA(cudaMemcpy(c->flags + kFCredit + 1, &one, sizeof one, cudaMemcpyHostToDevice));
    XCUDA(cudaDeviceSynchronize());  // zeroed before any peer can map and write them
  } else if (c->nranks > 1) {
    const int i = c->rank / c->u, j = c->rank % c->u;
    // ncclCommSplit is collective over the SP communicator; every rank takes the same branches.
    if (c->u > 1) XNCCL(ncclCommSplit(c->sp, i, j, &c->uly, nullptr));
    if (c->r > 1) XNCCL(ncclCommSplit(c->sp, j, i, &c->ring, nullptr));
  }
  return XDIT_OK;
}

int check_async(xdit_comm_s* c) {
  ncclComm_t cs[3] = {c->sp, c->uly, c->ring};
  for (ncclComm_t x : cs) {
    if (!x) continue;
    ncclResult_t st = ncclSuccess;
    XNCCL(ncclCommGetAsyncError(x, &st));
    if (st != ncclSuccess && st != ncclInProgress)
      return fail(XDIT_ERR_NCCL, "pending NCCL async error: %s", ncclGetErrorString(st));
  }
  return XDIT_OK;
}

// ---- peer-memory transport helpers
void close_peers(xdit_comm_s* c) {
  for (PeerMap& m : c->peer)
    for (int k = 0; k < kNHandles; ++k)
      if (m.opened[k] && m.ptr[k]) cudaIpcCloseMemHandle(m.ptr[k]);
  c->peer.clear();
  c->connected = false;
}

// Local exported buffers by handle index.
Buf* exported(xdit_comm_s* c, int k) {
  switch (k) {
    case kHUly: return &c->uly_recv;
    case kHORecv: return &c->orecv;
    case kHKV + 0: return &c->kv[0][0];
    case kHKV + 1: return &c->kv[0][1];
    case kHKV + 2: return &c->kv[1][0];
    case kHKV + 3: return &c->kv[1][1];
    case kHMbox: return &c->mbox;
    default: return nullptr;
  }
}

// Stream-ordered signal: *peer_flag = v after all prior work of `st` (system-wide fence first).
int post_flag(cudaStream_t st, uint32_t* peer_flag, uint32_t v) {
  const CUresult r = memops()->write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(peer_flag), v,
                                     CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(XDIT_ERR_CUDA, "cuStreamWriteValue32 failed (%d)", int(r));
  return XDIT_OK;
}
// Stream-ordered wait: later work of `st` starts once (int32)(*flag - v) >= 0.
int wait_flag(cudaStream_t st, const uint32_t* flag, uint32_t v) {
  const CUresult r = memops()->wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), v,
                                    CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(XDIT_ERR_CUDA, "cuStreamWaitValue32 failed (%d)", int(r));
  return XDIT_OK;
}

// Byte-exact all-to-all of `chunk` bytes per peer on `comm` (send[p] -> peer p -> recv[p]).
int a2a(ncclComm_t comm, int n, const void* send, void* recv, size_t chunk, cudaStream_t st) {
  XNCCL(ncclGroupStart());
  for (int p = 0; p < n; ++p) {
    XNCCL(ncclSend(static_cast<const char*>(send) + p * chunk, chunk, ncclUint8, p, comm, st));
    XNCCL(ncclRecv(static_cast<char*>(recv) + p * chunk, chunk, ncclUint8, p, comm, st));
  }
  XNCCL(ncclGroupEnd());
  return XDIT_OK;
}

int attn_launch(const AttnArgs& a_in, int dtype, cudaStream_t st, const Buf* scratch = nullptr) {
  AttnArgs a = a_in;
  if (scratch && scratch->p) {
    a.scratch = static_cast<float*>(scratch->p);
    a.scratch_floats = scratch->bytes / sizeof(float);
  }
  cudaError_t e = dtype == 0 ? xdit::launch_attn_fwd_sm100(a, st) : xdit::launch_attn_fwd_f32(a, st);
  if (e != cudaSuccess)
    return fail(XDIT_ERR_CUDA, "attention launch failed: %s", cudaGetErrorString(e));
  return XDIT_OK;
}

#define XRET(x)            \
  do {                     \
    int rc_ = (x);         \
    if (rc_ != XDIT_OK) return rc_; \
  } while (0)

// One USP attention call; eb = element bytes (2: bf16 / tcgen05 path, 4: fp32 / SIMT path).
int usp_call(const void* q, const void* k, const void* v, void* out, float* lse, int B, int H,
             int S_txt, int S_img, int D, int u, int r, cudaStream_t st, xdit_comm_s* c, int eb,
             void* kv_keep = nullptr) {
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
  if (dtype == 1 && u * r > 1 && (D % 4) != 0)
    return fail(XDIT_ERR_UNSUPPORTED, "fp32 multi-rank path needs D %% 4 == 0, got %d", D);
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(out) || !aligned16(lse) ||
      !aligned16(kv_keep))
    return fail(XDIT_ERR_ALIGNMENT, "tensor pointers must be 16-byte aligned");
  if ((int64_t(H) * D * eb) % 16 != 0)
    return fail(XDIT_ERR_ALIGNMENT, "H*D*elem_bytes must be a multiple of 16");
  Plan P;
  XRET(make_plan(B, H, S_txt, S_img, D, u, r, c->rank, &P));
  const Sizes need = sizes_for(P, B, D, eb);
  if (need.uly3 > c->uly_recv.bytes || need.qblk > c->qblk.bytes || need.kvslot > c->kv[1][0].bytes ||
      need.oacc > c->oacc.bytes || need.lacc > c->lacc.bytes || need.ochunk * P.u > c->osend.bytes * (P.u > 1))
    return fail(XDIT_ERR_WORKSPACE, "problem exceeds the reservation; call xdit_comm_reserve first");
  XRET(check_async(c));
  const bool peer = c->transport == XDIT_TRANSPORT_PEER && P.N > 1;
  if (peer) {
    if (!c->connected)
      return fail(XDIT_ERR_NOT_CONNECTED, "peer transport: call xdit_comm_peer_connect after xdit_comm_reserve");
    for (int q = 0; q < P.N; ++q) {  // buffers this rank writes into on peer q
      const PeerMap& m = c->peer[q];
      const bool uly_peer = q / P.u == P.i && P.u > 1, ring_next = q == ((P.i + 1) % P.r) * P.u + P.j && P.r > 1;
      bool ok = !(uly_peer || ring_next) || m.ptr[kHFlags];
      if (uly_peer) ok = ok && m.bytes[kHUly] >= need.uly3 && m.bytes[kHORecv] >= need.ochunk * P.u;
      if (ring_next)
        for (int k = 0; k < 4; ++k) ok = ok && m.bytes[kHKV + k] >= need.kvslot;
      if (!ok)
        return fail(XDIT_ERR_WORKSPACE,
                    "peer %d's mapped workspace is smaller than this problem (flags %p, uly %llu/%zu, orecv %llu/%zu, "
                    "kv %llu/%zu)", q, m.ptr[kHFlags], (unsigned long long)m.bytes[kHUly], need.uly3,
                    (unsigned long long)m.bytes[kHORecv], need.ochunk * P.u, (unsigned long long)m.bytes[kHKV],
                    need.kvslot);
    }
  }
  // Peer transport flags are binary: the writer sets 1 (after its data), the owner waits for 1 and
  // resets 0 before anything that lets the writer set it again -- so every stream operation carries
  // constant values and the call replays correctly from a captured CUDA graph.

  const int i = P.i, Hh = P.Hh, L = P.S_loc[c->rank], Sb = P.S_blk[i];
  const int64_t row = int64_t(Hh) * D;  // elements per (token) row of a head-block tensor
  // NEXT 1 (reading R2): the KV buffer holds every ring block at its offset in SP-shard order
  const int S_sp = S_txt + S_img;
  auto blk_off = [&](int ib) {
    int o = 0;
    for (int x = 0; x < ib; ++x) o += P.S_blk[x];
    return o;
  };

  // ---- N == 1: one kernel straight from the caller's tensors into the caller's output
  if (P.N == 1) {
    AttnArgs a{};
    a.q = q; a.k = k; a.v = v; a.o = out; a.lse = lse;
    a.B = B; a.H = H; a.Sq = L; a.Skv = L; a.D = D;
    a.q_b = a.kv_b = int64_t(L) * H * D; a.q_s = a.kv_s = int64_t(H) * D; a.q_h = a.kv_h = D;
    a.omap = plain_map(B, L, H, D);
    a.out_f32 = dtype;
    if (kv_keep)
      XCUDA(xdit::launch_kv_retain(k, v, kv_keep, B, H, L, S_sp, 0, D, a.kv_b, a.kv_s, a.kv_h, eb, st));
    return attn_launch(a, dtype, st, &c->tail);
  }

  XCUDA(cudaEventRecord(c->ev_start, st));
  XCUDA(cudaStreamWaitEvent(c->side, c->ev_start, 0));

  // ---- a2-a4: Ulysses all-to-all of Q, K, V (scatter heads, gather sequence)
  const void *Qp = q, *Kc = k, *Vc = v;
  int64_t q_b = int64_t(L) * H * D, q_s = int64_t(H) * D;
  if (P.u > 1) {
    const void* src[3] = {q, k, v};
    if (peer) {
      // pack = all-to-all: head block p of every local token is stored straight into Ulysses peer
      // p's receive buffer at this rank's chunk (P.j); then flag each peer and wait for theirs.
      xdit::PeerDst pd{};
      for (int p = 0; p < P.u; ++p)
        pd.p[p] = static_cast<char*>(c->peer[i * P.u + p].ptr[kHUly]) + size_t(P.j) * (need.uly3 / P.u);
      for (int t = 0; t < 3; ++t)
        XCUDA(xdit::launch_uly_pack_to(src[t], pd, B, L, P.Lmax, H, D, P.u, t, 3, eb, st));
      for (int p = 0; p < P.u; ++p)
        if (p != P.j) XRET(post_flag(st, static_cast<uint32_t*>(c->peer[i * P.u + p].ptr[kHFlags]) + kFA2A + P.j, 1));
      for (int p = 0; p < P.u; ++p)
        if (p != P.j) {  // peer p sets it again only after my O return of this call (after this reset)
          XRET(wait_flag(st, c->flags + kFA2A + p, 1));
          XRET(post_flag(st, c->flags + kFA2A + p, 0));
        }
    } else {
      for (int t = 0; t < 3; ++t)
        XCUDA(xdit::launch_uly_pack(src[t], c->uly_send.p, B, L, P.Lmax, H, D, P.u, t, 3, eb, st));
      XCUDA(cudaEventRecord(c->ev_a2a, st));
      XCUDA(cudaStreamWaitEvent(c->side, c->ev_a2a, 0));
      XRET(a2a(c->uly, P.u, c->uly_send.p, c->uly_recv.p, need.uly3 / P.u, c->side));
      XCUDA(cudaEventRecord(c->ev_a2a, c->side));
      XCUDA(cudaStreamWaitEvent(st, c->ev_a2a, 0));
    }
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
  if (kv_keep)  // this rank's ring block, right after the all-to-all (or straight from the caller)
    XCUDA(xdit::launch_kv_retain(Kc, Vc, kv_keep, B, Hh, Sb, S_sp, blk_off(i), D, q_b, q_s, D, eb, st));

  // ---- destination of the final O / LSE: the caller's tensors (u == 1) or the reverse-a2a
  //      send buffer, one segment per Ulysses peer (u > 1; reading C15)
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
    if (peer) {  // a9 fused into the epilogue: segment p is stored straight into peer p's O receive
                 // buffer at this rank's chunk (P.j); the final kernel's stores are the all-to-all
      fmap.seg_table = 1;
      const char* ob = static_cast<const char*>(dst);
      const char* lb = reinterpret_cast<const char*>(dst_lse);
      for (int p = 0; p < P.u; ++p) {
        const char* chunk = static_cast<const char*>(c->peer[i * P.u + p].ptr[kHORecv]) + size_t(P.j) * need.ochunk;
        fmap.o_seg_off[p] = (chunk - ob) / eb;
        fmap.l_seg_off[p] = (chunk + need.ochunk_o - lb) / 4;
      }
    }
  }

  AttnArgs a{};
  a.q = Qp; a.B = B; a.H = Hh; a.Sq = Sb; a.D = D;
  a.q_b = q_b; a.q_s = q_s; a.q_h = D;
  if (P.r == 1) {
    // ---- a6 without ring: final bf16 (or fp32) output written straight to its destination
    a.k = Kc; a.v = Vc; a.Skv = Sb;
    a.kv_b = q_b; a.kv_s = q_s; a.kv_h = D;
    a.o = dst; a.lse = dst_lse; a.omap = fmap; a.out_f32 = dtype;
    XRET(attn_launch(a, dtype, st, &c->tail));
  } else {
    // ---- a5-a7: ring loop; step s attends to the KV block of ring index (i - s) mod r (C9)
    const int nxt_peer = (i + 1) % P.r, prv_peer = (i - 1 + P.r) % P.r;
    // peer transport: slot credits.  Rank i pushes its current block into next's slot (s+1)&1 at
    // step s <= r-2 once next's credit for that slot is set (it waits, resets, pushes, sets next's
    // data flag).  A rank posts credit[s&1] to prev exactly once per push prev will make into that
    // slot: after step 0 (slot 0, pushed at prev's step 1, if r >= 3), after steps 1..r-3 (pushed at
    // prev's step s+1), and after its last odd step (slot 1, pushed at prev's step 0 of the NEXT
    // call; credit[1] starts set).  Each post follows the reader's last use of the slot and its own
    // push out of it, and every wait is matched by one post, so the flags end each call in the
    // state they started it (credit[1] = 1, the rest 0).
    const PeerMap* pnext = peer ? &c->peer[nxt_peer * P.u + P.j] : nullptr;
    const PeerMap* pprev = peer ? &c->peer[prv_peer * P.u + P.j] : nullptr;
    const int last_odd = ((P.r - 1) & 1) ? P.r - 1 : P.r - 2;  // r >= 2
    auto credit_after = [&](int st_) { return (st_ == 0 && P.r >= 3) || (st_ >= 1 && st_ <= P.r - 3) || st_ == last_odd; };
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
      const int nslot = (s + 1) & 1;
      if (s < P.r - 1) {
        // side stream: current block must be complete (recorded on st), next slot must be free
        XCUDA(cudaEventRecord(c->ev_start, st));
        XCUDA(cudaStreamWaitEvent(c->side, c->ev_start, 0));
        const int nsrc = ((src - 1) % P.r + P.r) % P.r;
        const size_t sbytes = size_t(B) * Skv * row * eb, rbytes = size_t(B) * P.S_blk[nsrc] * row * eb;
        if (peer) {
          XRET(wait_flag(c->side, c->flags + kFCredit + nslot, 1));
          XRET(post_flag(c->side, c->flags + kFCredit + nslot, 0));
          XCUDA(cudaMemcpyAsync(pnext->ptr[kHKV + 2 * nslot], curK, sbytes, cudaMemcpyDefault, c->side));
          XCUDA(cudaMemcpyAsync(pnext->ptr[kHKV + 2 * nslot + 1], curV, sbytes, cudaMemcpyDefault, c->side));
          XRET(post_flag(c->side, static_cast<uint32_t*>(pnext->ptr[kHFlags]) + kFData + nslot, 1));
          (void)rbytes;
        } else {
          XNCCL(ncclGroupStart());
          XNCCL(ncclSend(curK, sbytes, ncclUint8, nxt_peer, c->ring, c->side));
          XNCCL(ncclSend(curV, sbytes, ncclUint8, nxt_peer, c->ring, c->side));
          XNCCL(ncclRecv(c->kv[nslot][0].p, rbytes, ncclUint8, prv_peer, c->ring, c->side));
          XNCCL(ncclRecv(c->kv[nslot][1].p, rbytes, ncclUint8, prv_peer, c->ring, c->side));
          XNCCL(ncclGroupEnd());
        }
        XCUDA(cudaEventRecord(c->ev_recv[s & 1], c->side));
      }
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
      if (s < P.r - 1) {
        XCUDA(cudaStreamWaitEvent(st, c->ev_recv[s & 1], 0));  // (peer: my push out of this block is done)
        if (peer) {
          if (credit_after(s)) XRET(post_flag(st, static_cast<uint32_t*>(pprev->ptr[kHFlags]) + kFCredit + (s & 1), 1));
          XRET(wait_flag(st, c->flags + kFData + nslot, 1));
          XRET(post_flag(st, c->flags + kFData + nslot, 0));
        }
        curK = c->kv[nslot][0].p;
        curV = c->kv[nslot][1].p;
        if (kv_keep) {  // the incoming ring block (index (i - s - 1) mod r) joins the KV buffer
          const int nsrc = ((src - 1) % P.r + P.r) % P.r;
          XCUDA(xdit::launch_kv_retain(curK, curV, kv_keep, B, Hh, P.S_blk[nsrc], S_sp, blk_off(nsrc), D,
                                       int64_t(P.S_blk[nsrc]) * row, row, D, eb, st));
        }
      } else if (peer && credit_after(s)) {  // last step odd: slot 1's credit for prev's next call
        XRET(post_flag(st, static_cast<uint32_t*>(pprev->ptr[kHFlags]) + kFCredit + (s & 1), 1));
      }
    }
  }

  // ---- a9-a10: reverse all-to-all of O (+ LSE) and unpack into the caller's layout
  if (P.u > 1) {
    if (peer) {  // the final epilogue already stored chunk p in peer p's receive buffer: flag, wait
      for (int p = 0; p < P.u; ++p)
        if (p != P.j) XRET(post_flag(st, static_cast<uint32_t*>(c->peer[i * P.u + p].ptr[kHFlags]) + kFO + P.j, 1));
      for (int p = 0; p < P.u; ++p)
        if (p != P.j) {  // peer p sets it again only after my next call's pack (after this reset)
          XRET(wait_flag(st, c->flags + kFO + p, 1));
          XRET(post_flag(st, c->flags + kFO + p, 0));
        }
    } else {
      XCUDA(cudaEventRecord(c->ev_o, st));
      XCUDA(cudaStreamWaitEvent(c->side, c->ev_o, 0));
      XRET(a2a(c->uly, P.u, c->osend.p, c->orecv.p, need.ochunk, c->side));
      XCUDA(cudaEventRecord(c->ev_o_a2a, c->side));
      XCUDA(cudaStreamWaitEvent(st, c->ev_o_a2a, 0));
    }
    XCUDA(xdit::launch_uly_unpack_out(
        c->orecv.p,
        reinterpret_cast<const float*>(static_cast<const char*>(c->orecv.p) + need.ochunk_o),
        int64_t(need.ochunk), int64_t(need.ochunk), out, lse, B, L, P.Lmax, Hh, D, P.u, eb, st));
  }
  return XDIT_OK;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char* xdit_last_error(void) { return g_err.c_str(); }

int xdit_version(void) { return 20000; }  // 2.0.0: xdit_rowmap gained the segment table (ABI break)

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

int xdit_comm_init_peer(int nranks, int rank, int ulysses, int ring, xdit_comm_t* out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks || ulysses < 1 || ring < 1)
    return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_init_peer: bad arguments");
  if (ulysses * ring != nranks)
    return fail(XDIT_ERR_COMM_MISMATCH, "ulysses*ring=%d != nranks=%d", ulysses * ring, nranks);
  auto* c = new xdit_comm_s();
  c->nranks = nranks;
  c->rank = rank;
  c->u = ulysses;
  c->r = ring;
  c->transport = XDIT_TRANSPORT_PEER;
  int rc = comm_finish_init(c);
  if (rc != XDIT_OK) {
    xdit_comm_destroy(c);
    return rc;
  }
  *out = c;
  return XDIT_OK;
}

int xdit_comm_transport(xdit_comm_t c) { return c ? c->transport : -1; }

int xdit_comm_peer_export(xdit_comm_t c, void* blob) {
  if (!c || !blob) return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_peer_export: NULL argument");
  if (c->transport != XDIT_TRANSPORT_PEER) return fail(XDIT_ERR_INVALID_ARG, "handle does not use the peer transport");
  PeerBlob b{};
  b.magic = kBlobMagic;
  b.rank = c->rank;
  b.nranks = c->nranks;
  b.u = c->u;
  b.r = c->r;
  b.device = c->device;
  b.pid = int32_t(getpid());
  for (int k = 0; k < kNHandles; ++k) {
    void* p = k == kHFlags ? static_cast<void*>(c->flags) : exported(c, k)->p;
    if (!p) continue;
    XCUDA(cudaIpcGetMemHandle(&b.h[k], p));
    b.bytes[k] = k == kHFlags ? kFlagWords * sizeof(uint32_t) : exported(c, k)->bytes;
    b.valid |= 1u << k;
  }
  std::memset(blob, 0, XDIT_PEER_BLOB_BYTES);
  std::memcpy(blob, &b, sizeof b);
  return XDIT_OK;
}

int xdit_comm_peer_connect(xdit_comm_t c, const void* blobs) {
  if (!c || !blobs) return fail(XDIT_ERR_INVALID_ARG, "xdit_comm_peer_connect: NULL argument");
  if (c->transport != XDIT_TRANSPORT_PEER) return fail(XDIT_ERR_INVALID_ARG, "handle does not use the peer transport");
  std::vector<PeerBlob> bl(c->nranks);
  for (int q = 0; q < c->nranks; ++q) {
    std::memcpy(&bl[q], static_cast<const char*>(blobs) + size_t(q) * XDIT_PEER_BLOB_BYTES, sizeof(PeerBlob));
    const PeerBlob& b = bl[q];
    if (b.magic != kBlobMagic || b.rank != q || b.nranks != c->nranks || b.u != c->u || b.r != c->r)
      return fail(XDIT_ERR_COMM_MISMATCH, "peer blob %d is not rank %d of this (%d x %d) mesh", q, q, c->u, c->r);
    if (q != c->rank && b.pid == int32_t(getpid()))
      return fail(XDIT_ERR_UNSUPPORTED, "ranks %d and %d live in one process (one process per rank)", q, c->rank);
  }
  XCUDA(cudaDeviceSynchronize());
  close_peers(c);
  c->peer.assign(c->nranks, PeerMap{});
  const int i = c->rank / c->u, j = c->rank % c->u;
  const int nxt = ((i + 1) % c->r) * c->u + j;
  for (int q = 0; q < c->nranks; ++q) {
    PeerMap& m = c->peer[q];
    const bool uly_peer = q / c->u == i && c->u > 1;
    for (int k = 0; k < kNHandles; ++k) {
      const bool want = (k == kHFlags || k == kHMbox) ? true  // any rank may message any rank
                                     : (k < kHKV ? uly_peer : (c->r > 1 && q == nxt));
      if (!want || !(bl[q].valid & (1u << k))) continue;
      m.bytes[k] = bl[q].bytes[k];
      if (q == c->rank) {
        m.ptr[k] = k == kHFlags ? static_cast<void*>(c->flags) : exported(c, k)->p;
        continue;
      }
      cudaError_t e = cudaIpcOpenMemHandle(&m.ptr[k], bl[q].h[k], cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        m.ptr[k] = nullptr;
        close_peers(c);
        return fail(XDIT_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d, buffer %d): %s", q, k, cudaGetErrorString(e));
      }
      m.opened[k] = true;
    }
  }
  c->connected = true;
  return XDIT_OK;
}

int xdit_comm_mailbox_reserve(xdit_comm_t c, size_t bytes_per_src) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (c->transport != XDIT_TRANSPORT_PEER) return fail(XDIT_ERR_INVALID_ARG, "handle does not use the peer transport");
  const size_t region = (bytes_per_src + 255) & ~size_t(255);
  if (region <= c->mbox_region) return XDIT_OK;
  XCUDA(cudaDeviceSynchronize());  // peers' writes into the old mailbox drained (caller: after a barrier)
  XRET(ensure(&c->mbox, region * c->nranks));
  c->mbox_region = region;
  c->connected = false;  // peers must map the new mailbox
  return XDIT_OK;
}

int xdit_p2p_mailbox(xdit_comm_t c, int src, void** ptr, size_t* bytes) {
  if (!c || !ptr || src < 0 || src >= c->nranks) return fail(XDIT_ERR_INVALID_ARG, "xdit_p2p_mailbox: bad arguments");
  if (!c->mbox.p) return fail(XDIT_ERR_WORKSPACE, "no mailbox reserved (xdit_comm_mailbox_reserve)");
  *ptr = static_cast<char*>(c->mbox.p) + size_t(src) * c->mbox_region;
  if (bytes) *bytes = c->mbox_region;
  return XDIT_OK;
}

namespace {
int p2p_check(xdit_comm_s* c, int peer_rank) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (c->transport != XDIT_TRANSPORT_PEER) return fail(XDIT_ERR_INVALID_ARG, "handle does not use the peer transport");
  if (!c->connected) return fail(XDIT_ERR_NOT_CONNECTED, "peer transport: connect after (re)reserving");
  if (peer_rank < 0 || peer_rank >= c->nranks) return fail(XDIT_ERR_INVALID_ARG, "rank %d out of range", peer_rank);
  return XDIT_OK;
}
}  // namespace

int xdit_p2p_put(xdit_comm_t c, int dst, const void* src, size_t bytes, size_t dst_off, uint32_t tag,
                 xdit_stream_t stream) {
  XRET(p2p_check(c, dst));
  if (!src && bytes) return fail(XDIT_ERR_INVALID_ARG, "xdit_p2p_put: src is NULL");
  if (dst_off + bytes > c->mbox_region)
    return fail(XDIT_ERR_WORKSPACE, "xdit_p2p_put: %zu bytes at offset %zu exceed the %zu-byte mailbox region", bytes,
                dst_off, c->mbox_region);
  const PeerMap& m = c->peer[dst];
  if (!m.ptr[kHMbox] || !m.ptr[kHFlags]) return fail(XDIT_ERR_WORKSPACE, "rank %d has no mapped mailbox", dst);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (bytes)
    XCUDA(cudaMemcpyAsync(static_cast<char*>(m.ptr[kHMbox]) + size_t(c->rank) * c->mbox_region + dst_off, src, bytes,
                          cudaMemcpyDefault, st));
  return post_flag(st, static_cast<uint32_t*>(m.ptr[kHFlags]) + kFP2P + c->rank, tag);
}

int xdit_p2p_wait(xdit_comm_t c, int src, uint32_t tag, xdit_stream_t stream) {
  XRET(p2p_check(c, src));
  return wait_flag(reinterpret_cast<cudaStream_t>(stream), c->flags + kFP2P + src, tag);
}

int xdit_p2p_ack(xdit_comm_t c, int sender, uint32_t tag, xdit_stream_t stream) {
  XRET(p2p_check(c, sender));
  const PeerMap& m = c->peer[sender];
  if (!m.ptr[kHFlags]) return fail(XDIT_ERR_WORKSPACE, "rank %d's flags are not mapped", sender);
  return post_flag(reinterpret_cast<cudaStream_t>(stream), static_cast<uint32_t*>(m.ptr[kHFlags]) + kFAck + c->rank,
                   tag);
}

int xdit_p2p_wait_ack(xdit_comm_t c, int receiver, uint32_t tag, xdit_stream_t stream) {
  XRET(p2p_check(c, receiver));
  return wait_flag(reinterpret_cast<cudaStream_t>(stream), c->flags + kFAck + receiver, tag);
}

int xdit_comm_reserve(xdit_comm_t c, int B, int H, int S_txt, int S_img, int D, int elem_bytes) {
  if (!c) return fail(XDIT_ERR_INVALID_ARG, "comm handle is NULL");
  if (elem_bytes != 2 && elem_bytes != 4) return fail(XDIT_ERR_UNSUPPORTED, "elem_bytes must be 2 or 4");
  Plan P;
  XRET(make_plan(B, H, S_txt, S_img, D, c->u, c->r, c->rank, &P));
  const Sizes s = sizes_for(P, B, D, elem_bytes);
  void* before[kNHandles] = {};
  for (int k = 0; k < kHFlags; ++k) before[k] = exported(c, k)->p;  // (the mailbox is not reallocated here)
  if (c->transport == XDIT_TRANSPORT_PEER) XCUDA(cudaDeviceSynchronize());  // peers' writes drained
  XRET(ensure(&c->uly_send, s.uly3 * (c->transport == XDIT_TRANSPORT_NCCL)));
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
  for (int k = 0; k < kHFlags; ++k)
    if (exported(c, k)->p != before[k]) c->connected = false;  // peers must map the new buffers
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
  if (c->transport == XDIT_TRANSPORT_PEER) cudaDeviceSynchronize();
  close_peers(c);
  if (c->flags) cudaFree(c->flags);
  Buf* bufs[] = {&c->uly_send, &c->uly_recv, &c->qblk, &c->kv[0][0], &c->kv[0][1], &c->kv[1][0],
                 &c->kv[1][1], &c->oacc, &c->lacc, &c->otmp, &c->ltmp, &c->osend, &c->orecv, &c->tail,
                 &c->mbox};
  for (Buf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->uly) ncclCommDestroy(c->uly);
  if (c->ring) ncclCommDestroy(c->ring);
  if (c->sp && c->own_sp) ncclCommDestroy(c->sp);
  cudaEvent_t evs[] = {c->ev_start, c->ev_a2a, c->ev_o, c->ev_o_a2a,
                       c->ev_kdone[0], c->ev_kdone[1], c->ev_recv[0], c->ev_recv[1]};
  for (cudaEvent_t e : evs)
    if (e) cudaEventDestroy(e);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
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
  return usp_call(q, k, v, out, lse, B, H, S_txt, S_img, D, ulysses, ring,
                  reinterpret_cast<cudaStream_t>(stream), comm, 2, kv_keep);
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
  // unconditional: reading R3), then the combine on every rank.
  const size_t bytes = size_t(n) * eb;
  if (comm->transport == XDIT_TRANSPORT_PEER) {
    // peer transport: eps_local -> the peer's mailbox (after the peer acknowledged the previous
    // call's), flag; own copy into eps_gather[rank]; wait for the peer's flag, copy its prediction out
    // of the mailbox into eps_gather[1 - rank], acknowledge.
    if (!comm->connected) return fail(XDIT_ERR_NOT_CONNECTED, "peer transport: connect after (re)reserving");
    if (bytes > comm->mbox_region)
      return fail(XDIT_ERR_WORKSPACE, "cfg_tail: %zu bytes exceed the %zu-byte mailbox region "
                  "(xdit_comm_mailbox_reserve)", bytes, comm->mbox_region);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    XCUDA(cudaStreamIsCapturing(st, &cs));
    if (cs != cudaStreamCaptureStatusNone)  // its flags carry per-call epochs (immediates)
      return fail(XDIT_ERR_UNSUPPORTED, "cfg_tail over the peer transport cannot be captured in a CUDA graph");
    const int me = comm->rank, other = 1 - me;
    const uint32_t e = ++comm->cfg_epoch;
    const PeerMap& m = comm->peer[other];
    char* gb = static_cast<char*>(eps_gather);
    XRET(wait_flag(st, comm->flags + kFCfgAck + other, e - 1));
    XCUDA(cudaMemcpyAsync(static_cast<char*>(m.ptr[kHMbox]) + size_t(me) * comm->mbox_region, eps_local, bytes,
                          cudaMemcpyDefault, st));
    XRET(post_flag(st, static_cast<uint32_t*>(m.ptr[kHFlags]) + kFCfg + me, e));
    XCUDA(cudaMemcpyAsync(gb + size_t(me) * bytes, eps_local, bytes, cudaMemcpyDeviceToDevice, st));
    XRET(wait_flag(st, comm->flags + kFCfg + other, e));
    XCUDA(cudaMemcpyAsync(gb + size_t(other) * bytes, static_cast<char*>(comm->mbox.p) + size_t(other) * comm->mbox_region,
                          bytes, cudaMemcpyDeviceToDevice, st));
    XRET(post_flag(st, static_cast<uint32_t*>(m.ptr[kHFlags]) + kFCfgAck + me, e));
    XCUDA(xdit::launch_cfg_combine(gb, gb + bytes, eps_out, n, g, dtype, st));
    return XDIT_OK;
  }
  XNCCL(ncclAllGather(eps_local, eps_gather, size_t(n) * eb, ncclUint8, comm->sp, st));
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
  if (!x || !send || B < 0 || L < 0 || Lmax < L || H <= 0 || D <= 0 || u < 1 || H % u != 0 ||
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
