/*
 * xdit_usp.h -- C ABI of libxdit_usp.so, the B200 (sm_100a) USP attention hot path of xDiT
 * (arXiv 2411.01738).  PAPER.md = /root/reference/PAPER.md (cited as P:<line> §<section>).
 *
 * The operation: full (non-causal) multi-head attention softmax(Q K^T / sqrt(D)) V over the joint
 * [text; image] token sequence of a DiT block ("full attention" P:257 §4.1.2; joint sequence
 * P:185-187 §3, §4.1.1), sharded by Unified Sequence Parallelism: a 2D mesh "where the
 * columns are SP-Ring groups and rows are SP-Ulysses groups" (§4.1.4).  Ulysses
 * "employs All2All communications to transform the partitioning along the sequence dimension into
 * partitioning along the head dimension" (§4.1.1); Ring is "a parallel version of Flash
 * Attention ... utilizing peer-to-peer (P2P) transmission of K and V subblock" (§4.1.1),
 * whose per-block partial results are merged by log-sum-exp.  CFG parallelism (§4.2) is
 * an outer batch split: the caller builds one communicator per CFG group and passes that group's
 * batch; nothing in this ABI sees it.
 *
 * Conventions (every function):
 *   - Return value: XDIT_OK (0) or an xdit_status code; the library never aborts.  The message of
 *     the last non-OK return on the calling thread is xdit_last_error().
 *   - Tensor pointers are DEVICE pointers owned by the caller (e.g. torch tensors) unless stated.
 *     The library never frees, retains or allocates caller memory; it allocates only inside
 *     xdit_comm_reserve (workspace owned by the comm handle).
 *   - All enqueueing functions are stream-ordered on the caller's `stream` and return without a
 *     host synchronisation; results are valid when `stream` reaches the enqueue point.
 *   - Scale is fixed to 1/sqrt(D) with the true head dim D (reading C1).  LSE is the
 *     natural log of sum_j exp(scaled logit_j), fp32 (reading C2).
 *   - bf16 = IEEE bfloat16 stored as uint16; fp32 = IEEE binary32.
 *   - Global joint sequence order is [text; image] (reading C4); S = S_txt + S_img.
 */
#ifndef XDIT_USP_H
#define XDIT_USP_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define XDIT_API __attribute__((visibility("default")))
#else
#define XDIT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct xdit_comm_s* xdit_comm_t; /* opaque: mesh, NCCL sub-communicators, workspace */
typedef struct CUstream_st* xdit_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum xdit_status {
  XDIT_OK = 0,
  XDIT_ERR_INVALID_ARG = 1,   /* null pointer, non-positive size, mismatched scalars */
  XDIT_ERR_UNSUPPORTED = 2,   /* head dim or dtype not supported by this entry point */
  XDIT_ERR_DIVISIBILITY = 3,  /* H % ulysses != 0 -- P:541 "16 does not divide evenly into 24" */
  XDIT_ERR_COMM_MISMATCH = 4, /* ulysses*ring != comm size, or (u,r) differs from the handle's */
  XDIT_ERR_EMPTY_SHARD = 5,   /* some rank would hold zero tokens (reading C5) */
  XDIT_ERR_ALIGNMENT = 6,     /* pointer not 16-byte aligned or row bytes not a multiple of 16 */
  XDIT_ERR_CUDA = 7,          /* a CUDA runtime/driver call failed (message has the name) */
  XDIT_ERR_NCCL = 8,          /* an NCCL call failed, or an async NCCL error was pending */
  XDIT_ERR_WORKSPACE = 9      /* problem exceeds the reservation made by xdit_comm_reserve */
} xdit_status;

/* Thread-local, NUL-terminated message for the last non-OK return ("" if none).  Valid until the
 * next call on the same thread.  Never NULL. */
XDIT_API const char* xdit_last_error(void);

/* Library ABI version (major*10000 + minor*100 + patch).  A caller compiled against this header
 * must check xdit_version() == XDIT_ABI_VERSION before passing any struct (xdit_rowmap, xdit_plan,
 * xdit_p2p_op, xdit_phases) across the boundary: the layouts are fixed per ABI version.
 * 3.0.0: NCCL is the only data plane (the round-1 peer-memory transport and its mailbox are gone,
 * xdit_rowmap lost its segment table); xdit_p2p, per-phase timing, the KV-buffer call. */
#define XDIT_ABI_VERSION 30000
XDIT_API int xdit_version(void);

/* Number of CUDA kernels this library has launched in this process (all devices, monotonic).
 * Read before and after a region to count the library's own launches in it. */
XDIT_API uint64_t xdit_launch_count(void);

/* ------------------------------------------------------------------------------------------ */
/* Shard rule (§4.1.1; reading C5).  In-context conditioning: "splits both the        */
/* Condition Tensor and Image Tensor along the sequence dimension. Then, it concatenates        */
/* corresponding shards of condition and image input to form a local sequence."                 */
/* Text and image are split separately into nranks balanced contiguous pieces: piece g has      */
/* floor(S/n) + (g < S mod n) tokens (np.array_split convention).  Rank g's local sequence is   */
/* concat(text piece g, image piece g), S_loc = *txt_len + *img_len.  Pure host function.       */
/* Errors: INVALID_ARG (negative sizes, nranks<1, g out of range); EMPTY_SHARD if S_loc == 0.    */
/* Outputs are written even for EMPTY_SHARD.                                                    */
/* ------------------------------------------------------------------------------------------ */
XDIT_API int xdit_usp_shard(int S_txt, int S_img, int nranks, int g, int* txt_off, int* txt_len,
                   int* img_off, int* img_len);

/* ------------------------------------------------------------------------------------------ */
/* Communicators.  One handle per SP group (= one CFG group).  Mesh (reading C6): SP rank  */
/* g = i*ulysses + j, i = ring index (SP-Ring column), j = Ulysses index (SP-Ulysses row).  Every  */
/* byte between ranks moves over NCCL (NVLink / NVSwitch between the GPUs of one node): the handle */
/* splits the SP communicator into the Ulysses row (color i, key j), the Ring column (color j,     */
/* key i) and a private copy of the whole group (point-to-point messages, all-gathers), and owns   */
/* all workspace.  Collectives and sends/receives run on an internal high-priority side stream     */
/* joined to the caller's stream with events, or on the caller's stream itself; no call of the hot */
/* path synchronises the host.                                                                     */
/* ------------------------------------------------------------------------------------------ */

/* Writes a fresh NCCL unique id (an opaque 128-byte blob) to id_out (HOST memory, >=128 bytes).
 * Rank 0 of the SP group calls it and broadcasts the bytes to the other ranks (e.g. with
 * torch.distributed), which then call xdit_comm_init.  Errors: INVALID_ARG, NCCL. */
XDIT_API int xdit_nccl_unique_id(void* id_out);

/* Collective over the nranks = ulysses*ring ranks of one SP group: builds the SP communicator
 * from `unique_id` (HOST, 128 bytes) on the current CUDA device, then splits the sub-communicators.
 * With nranks == 1, unique_id may be NULL and no NCCL object is made.
 * Errors: INVALID_ARG, COMM_MISMATCH (ulysses*ring != nranks), NCCL, CUDA. */
XDIT_API int xdit_comm_init(const void* unique_id, int nranks, int rank, int ulysses, int ring,
                   xdit_comm_t* out);

/* Same as xdit_comm_init but splits an existing ncclComm_t of the SP group -- the communicator a
 * framework already owns, e.g. torch ProcessGroupNCCL's `_comm_ptr()` (torch bundles NCCL 2.28.x,
 * the version this library links).  Collective over that communicator.  The handle never issues
 * work on nccl_comm itself (only on the communicators split from it) and does not take ownership.
 * nccl_comm may be NULL only when ulysses*ring == 1.  Errors: INVALID_ARG, COMM_MISMATCH, NCCL, CUDA. */
XDIT_API int xdit_comm_create(void* nccl_comm, int ulysses, int ring, xdit_comm_t* out);

/* ---- Point-to-point messages between ranks of a handle, for the patch activations PipeFusion
 * passes between stages "via asynchronous P2P" (NEXT 3) and the boundary rows of the
 * patch-parallel VAE (NEXT 4).  One call = one NCCL group of sends and receives on the
 * handle's private communicator, enqueued on `stream` (no host synchronisation); every message is
 * matched by the peer's op of the same size in ITS call, so any pattern in which each call's peers
 * issue matching calls is deadlock-free.  buf: DEVICE memory, `bytes` long (0 allowed: no-op). */
typedef struct xdit_p2p_op {
  int32_t peer;     /* rank of the handle's group */
  int32_t is_send;  /* 1 send buf to peer, 0 receive into buf from peer */
  void* buf;
  size_t bytes;
} xdit_p2p_op;
/* Errors: INVALID_ARG (NULL / peer out of range / n < 0), NCCL. */
XDIT_API int xdit_p2p(xdit_comm_t comm, const xdit_p2p_op* ops, int n, xdit_stream_t stream);

/* ---- Per-phase timing of xdit_usp_attention (SURVEY §5 "CUDA events per phase").  While
 * profiling is enabled, each call records timing events at its phase boundaries (not inside a
 * CUDA-graph capture, where they would be illegal: captured calls record nothing).  After the
 * call, xdit_comm_phases waits for its last event (HOST-synchronising) and reports:
 *   total_ms          : first to last event of the call (caller's stream)
 *   a2a_in_ms         : Ulysses pack + all-to-all of Q,K,V + unpack (u > 1)
 *   attn_ms[s]        : ring step s on the caller's stream: waiting for KV block s, attention
 *                       (with the merge fused into its epilogue) -- s < ring
 *   ring_comm_ms[s]   : the side stream's send/recv of the next KV block during step s (s < ring-1)
 *   a2a_out_ms        : reverse all-to-all of O (+LSE) + unpack (u > 1)
 *   *_bytes           : the bytes this rank SENT in that phase (Table 1 algorithmic bytes)
 * valid = 0 if the last call recorded nothing. */
typedef struct xdit_phases {
  int32_t valid, ulysses, ring, pad_;
  float total_ms, a2a_in_ms, a2a_out_ms, pad2_;
  float attn_ms[8];
  float ring_comm_ms[8];
  int64_t a2a_in_bytes, a2a_out_bytes;
  int64_t ring_bytes[8];
} xdit_phases;
XDIT_API int xdit_comm_profile(xdit_comm_t comm, int enable);
XDIT_API int xdit_comm_phases(xdit_comm_t comm, xdit_phases* out);

/* Allocates (or grows) the device workspace for a problem: Ulysses send/recv buffers, the
 * unpacked Q block, two ring KV slots, fp32 ring accumulators.  Call once per shape before the
 * hot loop (all ranks, same scalars); xdit_usp_attention never allocates, so the call path is
 * CUDA-graph capturable.  elem_bytes = 2 (bf16 path) or 4 (fp32 path).  S_txt/S_img are
 * GLOBAL token counts.  Errors: INVALID_ARG, DIVISIBILITY, EMPTY_SHARD, UNSUPPORTED, CUDA. */
XDIT_API int xdit_comm_reserve(xdit_comm_t comm, int B, int H, int S_txt, int S_img, int D, int elem_bytes);

/* Reports the handle's mesh.  Any output pointer may be NULL. */
XDIT_API int xdit_comm_info(xdit_comm_t comm, int* nranks, int* rank, int* ulysses, int* ring);

/* Frees the workspace and the NCCL objects the handle created (device-synchronising).
 * NULL is accepted and ignored. */
XDIT_API int xdit_comm_destroy(xdit_comm_t comm);

/* Per-rank geometry of one USP call, as the library will execute it (pure host function; all
 * ranks compute identical plans from identical scalars).  Exposed so host logic can be checked
 * without a GPU (e.g. multi-process gloo tests).  Ring step s uses the KV block of ring index
 * ring_src[s] = (i - s) mod ring (reading C9) with ring_rows[s] keys; the Ulysses exchange pads
 * every shard to Lmax rows; seg_off[] are this rank's ring-block row offsets of its Ulysses peers'
 * shards (one segment per peer, reading C6/C7). */
typedef struct xdit_plan {
  int32_t nranks, rank, ulysses, ring;
  int32_t i, j;        /* ring index (column) and Ulysses index (row) of `rank` */
  int32_t Hh;          /* heads per Ulysses rank = H / ulysses */
  int32_t S_loc;       /* tokens held by `rank` (= txt_len + img_len) */
  int32_t Lmax;        /* max S_loc over the SP group (a2a padding) */
  int32_t S_blk;       /* rows of this rank's ring block (queries after the Ulysses a2a) */
  int32_t ring_next, ring_prev;      /* ring-communicator ranks this rank sends to / receives from */
  int32_t nseg, seg_off[9];          /* ring-block rows contributed by Ulysses peer p: [off[p], off[p+1]) */
  int32_t ring_src[8], ring_rows[8]; /* per ring step s < ring */
  int64_t a2a_bytes_per_peer;        /* Q,K,V exchange chunk (bf16 elements x 2 bytes) */
  int64_t ring_bytes[8];             /* K+V bytes sent at step s (0 on the last step) */
} xdit_plan;
XDIT_API int xdit_usp_plan(int B, int H, int S_txt, int S_img, int D, int ulysses, int ring,
                           int rank, xdit_plan* out);

/* ------------------------------------------------------------------------------------------ */
/* The hot path: one USP attention call.                                 */
/*                                                                                              */
/* q, k, v, out : this rank's local tokens, [B][S_loc][H][D] contiguous, bf16; S_loc from        */
/*                xdit_usp_shard(S_txt, S_img, ulysses*ring, rank).  16-byte aligned.            */
/* lse          : fp32 [B][H][S_loc] (natural log) or NULL to skip (reading C15).               */
/* B, H, D      : batch of this SP (CFG) group, heads, head dim.  D in {64, 72, 128} (UNSUPPORTED*/
/*                otherwise; the fp32 entry point takes any D in [1, 256]).                     */
/* S_txt, S_img : GLOBAL text / image token counts of the joint sequence.                       */
/* ulysses,ring : degrees; must equal the handle's; H % ulysses == 0 (DIVISIBILITY).             */
/* stream       : caller's CUDA stream; the ring's NCCL send/recv run on an internal side stream */
/*                (joined back with events), the Ulysses exchanges on `stream`.                 */
/* comm         : handle from xdit_comm_init/create, reserved for this shape (WORKSPACE).        */
/*                                                                                              */
/* Steps: pack Q,K,V by head block -> Ulysses all-to-all -> unpack to the ring    */
/* block -> r ring steps {attention on the current KV block (tcgen05 kernel) || send/recv of the */
/* next KV block; LSE merge} -> bf16 cast + pack by destination -> reverse all-to-all of O and   */
/* LSE -> unpack into out/lse.  Invalid arguments are rejected before anything is enqueued, so a */
/* failing rank never leaves a peer hanging inside a collective (all ranks must pass identical  */
/* scalars).  Not re-entrant per handle.  Deterministic run to run for a fixed (ulysses, ring). */
/* ------------------------------------------------------------------------------------------ */
XDIT_API int xdit_usp_attention(const void* q, const void* k, const void* v, void* out, float* lse, int B,
                       int H, int S_txt, int S_img, int D, int ulysses, int ring,
                       xdit_stream_t stream, xdit_comm_t comm);

/* fp32-input mode: identical contract with fp32 q, k, v, out; SIMT fp32 arithmetic throughout
 * (no tensor cores), any D in [1, 256] with D*4 a multiple of 16 bytes when ulysses*ring > 1. */
XDIT_API int xdit_usp_attention_f32(const float* q, const float* k, const float* v, float* out, float* lse,
                           int B, int H, int S_txt, int S_img, int D, int ulysses, int ring,
                           xdit_stream_t stream, xdit_comm_t comm);

/* USP attention that also RETAINS the K,V the rank receives (
 * DESIGN.md reading R2) -- the KV buffer of hybrid SP + PipeFusion, which "standard SP
 * implementations ... discard after the Attention computation".  Same contract and result as
 * xdit_usp_attention (bf16 only), plus:
 *   kv_keep : DEVICE bf16 [2][B][H/ulysses][S_txt+S_img][D] (K then V), 16-byte aligned, caller
 *             owned, not NULL (INVALID_ARG).  Filled with the K,V of EVERY token of the SP group for
 *             this rank's Ulysses head block j = rank % ulysses (heads [j H/u, (j+1) H/u)), the
 *             sequence in SP-shard order: rank 0's local rows (text shard, then image shard), then
 *             rank 1's, ...  Ranks sharing a head block end with identical buffers.
 * Costs one extra HBM copy of each K,V block the rank holds (2 x B x H/u x S x D x 2 bytes). */
XDIT_API int xdit_usp_attention_kv(const void* q, const void* k, const void* v, void* out, float* lse,
                                   void* kv_keep, int B, int H, int S_txt, int S_img, int D, int ulysses,
                                   int ring, xdit_stream_t stream, xdit_comm_t comm);

/* USP attention of one PipeFusion patch over a persistent KV buffer -- the attention of hybrid
 * PipeFusion x SP (§4.1.4: "the KV involved in Attention
 * computation on different devices within the SP group should be consistent"; R6).
 * q, k, v, out, lse: this rank's local rows of the PATCH, exactly as in xdit_usp_attention with
 *          S_txt / S_img the patch's joint token counts (text rides with patch 0).
 * kv_buf : DEVICE [2][B][H/ulysses][S_buf][D] (K then V, head-major), this rank's Ulysses head block
 *          j = rank % ulysses, the block's KV over the WHOLE sequence; caller-owned and persistent
 *          across diffusion steps, rows in the tokens' global order.  The SP group's fresh K,V of
 *          the patch -- received through the Ulysses all-to-all (its ring block) and the ring
 *          rotation (the other r-1 ring blocks), "the intermediate results ... stored in each
 *          device's KV Buffer" -- are written to their tokens' rows: the patch's text token
 *          t to row txt_row + t, its image token t to row img_row + t; the other rows keep what
 *          they hold (stale K,V of the previous step); then the local queries attend
 *          over all S_buf rows.  Ranks of one head block therefore hold identical buffers, and the
 *          buffer is the one-device PipeFusion buffer restricted to the head block.
 * dtype  : 0 bf16 (tcgen05 kernel, D in {64,72,128}), 1 fp32 (SIMT kernel).
 * Errors: as xdit_usp_attention, plus INVALID_ARG (kv_buf NULL, rows beyond S_buf). */
XDIT_API int xdit_usp_attention_buf(const void* q, const void* k, const void* v, void* out, float* lse,
                                    void* kv_buf, int B, int H, int S_txt, int S_img, int D, int ulysses,
                                    int ring, int S_buf, int txt_row, int img_row, int dtype,
                                    xdit_stream_t stream, xdit_comm_t comm);

/* CFG-parallel step tail ("performs an Allgather operation on
 * the latent space results"; reading R3).
 * xdit_cfg_combine: out = eps_uncond + g * (eps_cond - eps_uncond) elementwise over n elements,
 *   computed in fp32 and rounded once (RNE) to dtype (0 bf16, 1 fp32).  All DEVICE buffers, 16-byte
 *   aligned, n a multiple of 8 (bf16) / 4 (fp32) (ALIGNMENT).  out may alias either input.
 * xdit_cfg_tail: the same after an NCCL all-gather of each rank's eps_local (n elements) over the
 *   handle's ranks, which must be exactly the 2 ranks of a cfg pair (COMM_MISMATCH otherwise;
 *   CUDA-graph capturable):
 *   rank 0 contributes the conditional, rank 1 the unconditional prediction.  eps_gather: DEVICE
 *   scratch of 2*n elements (receives [eps_cond; eps_uncond]); eps_out receives the combination on
 *   both ranks.  Stream-ordered on `stream`; errors: INVALID_ARG, ALIGNMENT, NCCL, CUDA. */
XDIT_API int xdit_cfg_combine(const void* eps_cond, const void* eps_uncond, void* out, int64_t n, float g,
                              int dtype, xdit_stream_t stream);
XDIT_API int xdit_cfg_tail(const void* eps_local, void* eps_gather, void* eps_out, int64_t n, float g,
                           int dtype, xdit_stream_t stream, xdit_comm_t comm);

/* ------------------------------------------------------------------------------------------ */
/* Stage entry points (single device).  xdit_usp_attention is composed of exactly these          */
/* launches plus NCCL; they are exported so a single GPU can drive every (ulysses, ring) split   */
/* as virtual ranks in tests.  All strides are in ELEMENTS; the innermost (d) stride is 1.       */
/* ------------------------------------------------------------------------------------------ */

/* Destination map of an output row block (used where a kernel writes O and LSE).  Block row t
 * belongs to segment s with seg_off[s] <= t < seg_off[s+1] (nseg in [1,8], seg_off[0] = 0,
 * seg_off[nseg] = number of rows); its element (b, t, h, d) goes to
 *   o + s*o_seg + b*o_b + (t - seg_off[s])*o_s + h*o_h + d
 * and its LSE (b, h, t) to  lse + s*l_seg + b*l_b + h*l_h + (t - seg_off[s]).
 * A single segment with o_seg = l_seg = 0 is a plain strided tensor.  This lets the final
 * epilogue write straight into the reverse all-to-all send buffer (one segment per Ulysses peer),
 * so the bf16 cast and the reverse pack (a8) cost no pass of their own. */
typedef struct xdit_rowmap {
  int32_t nseg;
  int32_t seg_off[9];
  int64_t o_seg, o_b, o_s, o_h;
  int64_t l_seg, l_b, l_h;
} xdit_rowmap;

/* Flash attention forward of one (Q block, KV block) pair -- SURVEY §8(a) step a6.
 * q: [B][Sq][H][D] with strides (q_b, q_s, q_h); k, v: [B][Skv][H][D] with strides
 * (kv_b, kv_s, kv_h) shared by k and v.  dtype: 0 = bf16 inputs on the tcgen05/TMEM/TMA kernel
 * (D in {64,72,128}; q,k,v 16-byte aligned, strides multiples of 8 elements), 1 = fp32 inputs on the
 * SIMT kernel (D in [1,256]).  out_f32: 0 writes O as bf16 through `omap` (final output);
 * 1 writes O as fp32 through `omap` (ring partial).  lse may be NULL (skipped).
 * The bf16 kernel is persistent: one CTA pair per TPC loops over work units (256 query rows of one
 * (b, h) against a key range).  scratch: optional 16-byte aligned DEVICE buffer of scratch_bytes
 * (>= xdit_attn_scratch_bytes(D) to be used), owned by the caller and not shared with a concurrent
 * launch; with it the kernel hands the units out through an atomic counter at the buffer's end
 * (reset by a 4-byte memset on `stream` before the launch) and splits the last, partial round of
 * units over key ranges (merged by an LSE-weighted tail kernel); NULL hands the units out
 * round-robin and runs every unit over all keys.  Results are the same within rounding either way
 * (bitwise the same when no tail split applies).
 * Errors: INVALID_ARG, UNSUPPORTED, ALIGNMENT, CUDA. */
XDIT_API int xdit_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse, int B, int H,
                  int Sq, int Skv, int D, int64_t q_b, int64_t q_s, int64_t q_h, int64_t kv_b,
                  int64_t kv_s, int64_t kv_h, const xdit_rowmap* omap, int dtype, int out_f32,
                  void* scratch, size_t scratch_bytes, xdit_stream_t stream);

/* Scratch bytes xdit_attn_fwd can use for head dim D on the current device (0 for D <= 0). */
XDIT_API size_t xdit_attn_scratch_bytes(int D);

/* Ring partial-output merge ("parallel version of Flash Attention").
 * o_acc, o_s: fp32 [B][S][Hh][D] contiguous; lse_acc, lse_s: fp32 [B][Hh][S].
 *   L = M + log(exp(lse_acc - M) + exp(lse_s - M)), M = max(lse_acc, lse_s)
 *   O = exp(lse_acc - L) * o_acc + exp(lse_s - L) * o_s
 * If final == NULL: O, L overwrite o_acc, lse_acc.  Else the merged O is cast (RNE) to
 * final_dtype (0 bf16, 1 fp32) and written with L through *final_map into `final` / `final_lse`
 * (final_lse may be NULL).  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_lse_merge(float* o_acc, float* lse_acc, const float* o_s, const float* lse_s, int B, int S,
                   int Hh, int D, void* final, float* final_lse, const xdit_rowmap* final_map,
                   int final_dtype, xdit_stream_t stream);

/* Ulysses pack: x [B][L][H][D] (contiguous, elem_bytes each) ->
 * send[p][t][B][Lmax][H/u][D] for p in [0,u) with t = `slot` of `nslots`, i.e. head block p of
 * every local token into peer p's contiguous chunk (u in [1, 8]).  Rows L..Lmax-1 are left untouched.
 * Errors: INVALID_ARG (also u > 8), ALIGNMENT, CUDA. */
XDIT_API int xdit_uly_pack(const void* x, void* send, int B, int L, int Lmax, int H, int D, int u, int slot,
                  int nslots, int elem_bytes, xdit_stream_t stream);

/* Ulysses unpack: recv[p][t][B][Lmax][Hh][D] (slot t of nslots) ->
 * y[B][S_blk][Hh][D] with y rows = concat over p of the first len[p] rows of peer p's chunk
 * (S_blk = sum len[p], u <= 8).  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_uly_unpack(const void* recv, void* y, int B, int Lmax, int Hh, int D, int u,
                    const int* len, int slot, int nslots, int elem_bytes, xdit_stream_t stream);

/* Reverse unpack: orecv[p][B][Lmax][Hh][D] (+ lrecv[p][B][Hh][Lmax]
 * fp32, may be NULL) -> out[B][L][H][D] with h = p*Hh + hh (+ lse[B][H][L] if non-NULL).
 * Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_uly_unpack_out(const void* orecv, const float* lrecv, int64_t peer_stride_bytes,
                        int64_t lse_peer_stride_bytes, void* out, float* lse, int B, int L,
                        int Lmax, int Hh, int D, int u, int elem_bytes, xdit_stream_t stream);

/* KV retention stage: copy a K and a V block [B][S_blk][Hh][D] (element
 * (b, t, h, d) at base + b*src_b + t*src_s + h*src_h + d) into kv_keep [2][B][Hh][S_total][D]
 * (K half, then V half) at sequence rows [seq_off, seq_off + S_blk).  xdit_usp_attention_kv calls it
 * for its ring block after the all-to-all and for every incoming ring block.  16-byte aligned
 * pointers; D and the strides multiples of 16 bytes / elem_bytes (2 or 4).
 * Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_kv_retain(const void* k_blk, const void* v_blk, void* kv_keep, int B, int Hh, int S_blk,
                            int S_total, int seq_off, int D, int64_t src_b, int64_t src_s, int64_t src_h,
                            int elem_bytes, xdit_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* PipeFusion (§4.1.2; reading R4).  The stage-  */
/* local work of one PipeFusion micro-step on a synthetic DiT stack: one block applied to one     */
/* patch, attending over the block's KV buffer in which the patch's own K,V are fresh and the     */
/* other patches' are whatever the buffer holds -- this step's for patches already processed at   */
/* this block, the previous step's for the rest ("uses stale activations from the previous        */
/* timestep to provide context").  The pipeline schedule (which patch on which stage   */
/* when, P2P of patch activations) is the caller's (paper_2411_01738_b200/pipefusion.py).          */
/* ------------------------------------------------------------------------------------------ */

/* Device workspace xdit_pf_block needs for a patch of n rows (0 for invalid arguments). */
XDIT_API size_t xdit_pf_block_workspace_bytes(int B, int n, int H, int D, int dtype);

/* Synthetic DiT block on one patch (reading R4):
 *   K,V buffer rows [off, off+n) <- h*wk, h*wv;   h <- h + g * softmax((h*wq) Kbuf^T / sqrt(D)) Vbuf
 * h      : DEVICE [B][n][H][D], the patch's hidden rows (updated in place)
 * kv_buf : DEVICE [2][B][H][S][D] (K then V, head-major) -- the block's buffer over the whole sequence
 * w      : DEVICE fp32 [4][H][D] = (wq, wk, wv, g)
 * work   : DEVICE scratch of >= xdit_pf_block_workspace_bytes(B, n, H, D, dtype) bytes
 * dtype  : 0 = bf16 h / kv_buf (tcgen05 attention, D in {64,72,128}), 1 = fp32 (SIMT, D % 8 == 0, <= 256)
 * Products are formed in fp32 and rounded once; the attention output stays fp32 until the residual.
 * Stream-ordered on `stream`, no allocation, no host sync.
 * Errors: INVALID_ARG, UNSUPPORTED, ALIGNMENT (16-byte pointers), WORKSPACE, CUDA. */
XDIT_API int xdit_pf_block(void* h, void* kv_buf, const float* w, void* work, size_t work_bytes, int B, int H, int S,
                           int off, int n, int D, int dtype, xdit_stream_t stream);

/* The two halves of xdit_pf_block around the attention, for hybrid PipeFusion x SP, where the
 * patch's attention is the USP call xdit_usp_attention_buf (NEXT 3; reading R6):
 * xdit_pf_qkv     : q, k, v [B][n][H][D] <- h * wq, h * wk, h * wv (fp32 products, one rounding).
 * xdit_pf_residual: h <- h + g * o, o [B][n][H][D] of h's dtype (the USP call's output).
 * w: DEVICE fp32 [4][H][D] = (wq, wk, wv, g).  dtype 0 bf16 / 1 fp32; 16-byte aligned, D % 8 == 0.
 * Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_pf_qkv(const void* h, const float* w, void* q, void* k, void* v, int B, int n, int H, int D,
                         int dtype, xdit_stream_t stream);
XDIT_API int xdit_pf_residual(void* h, const void* o, const float* w, int B, int n, int H, int D, int dtype,
                              xdit_stream_t stream);

/* Synthetic sampler step (reading R4): x <- x - sigma * eps over n elements (n % 8 == 0), DEVICE
 * buffers of dtype 0 (bf16) or 1 (fp32); fp32 math, one rounding.  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_pf_sampler(void* x, const void* eps, int64_t n, float sigma, int dtype, xdit_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* patch-parallel VAE decode (§4.3; reading R5). */
/* Devices hold row bands of the feature maps; before every conv a band receives one boundary row  */
/* from each neighbour ("the exchange of the boundary data for convolutional operators";    */
/* paper_2411_01738_b200/vae.py moves them with xdit_p2p over NCCL), so activation memory per      */
/* device falls to ~1/N and the decode stays exact.                                         */
/* ------------------------------------------------------------------------------------------ */

/* One decoder conv on a row band: out = conv3x3(in) + b, zero padding in x only.
 * in   : DEVICE fp32 [H+2][Ci][W] -- the band's H rows with its top and bottom halo rows (zeros at
 *        the image edges, which is the serial conv's zero padding)
 * w, b : DEVICE fp32 [Co][Ci][3][3] (16-byte aligned), [Co]
 * out  : DEVICE fp32 [H][Co][W], or with act_up = 1 (a decoder stage) SiLU then nearest x2 upsample,
 *        [2H][Co][2W]
 * Each output pixel is summed in one fixed order, so a band produces exactly the pixels of the
 * whole-image call.  Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_vae_conv3x3(const float* in, int H, int Ci, int W, const float* w, const float* b, float* out,
                              int Co, int act_up, xdit_stream_t stream);

/* The same conv on the tensor cores (tcgen05 implicit GEMM, bf16 in / fp32 accumulate / bf16 out;
 * DESIGN.md §7.7).  Channels-innermost layouts:
 * in   : DEVICE bf16 [H+2][W][Ci] (band + halo rows), Ci % 8 == 0
 * wt   : DEVICE bf16 [9][Co][Ci] (tap-major: wt[3*dy+dx][co][ci] = w[co][ci][dy][dx]);  b: fp32 [Co]
 * out  : DEVICE bf16 [H][W][Co8], or with act_up = 1 SiLU + nearest x2 upsample, [2H][2W][Co8];
 *        Co8 = Co rounded up to a multiple of 8 (16-byte rows for the TMA stores), channels >= Co are 0
 * Each pixel's accumulation is the same MMA sequence in any band (bit-exact patch parallelism).
 * Errors: INVALID_ARG, ALIGNMENT, CUDA. */
XDIT_API int xdit_vae_conv3x3_bf16(const void* in, int H, int Ci, int W, const void* wt, const float* b, void* out,
                                   int Co, int act_up, xdit_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* XDIT_USP_H */
