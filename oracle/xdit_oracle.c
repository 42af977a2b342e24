/*
 * xdit_oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the USP attention hot path
 * of xDiT (arXiv 2411.01738).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2411_01738_b200/) never
 * links, loads or calls it, and this file shares no code, header, table or constant with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   - xo_attention: full, non-causal multi-head softmax attention, softmax(Q K^T / sqrt(D)) V, with
 *     the log-sum-exp of every row.  "full attention" P:257 §4.1.2; "mutual computation between
 *     tokens" P:69 §1; scale 1/sqrt(D) per DESIGN.md reading C1; LSE definition reading C2.  It is
 *     the plain definition written out in fp64, ascending summation order, no blocking.
 *   - xo_attention_rows: the same definition for a caller-chosen subset of query rows (rows are
 *     independent, so this is an exact subset of xo_attention, used at full bench sizes).
 *   - xo_shard: the in-context sequence-parallel shard rule, "splits both the Condition Tensor and
 *     Image Tensor along the sequence dimension. Then, it concatenates corresponding shards"
 *     P:240 §4.1.1; balanced contiguous split for non-divisible lengths (reading C5).
 *   - xo_usp_emulate: the USP split of P:382-384 §4.1.4 (Ulysses rows x Ring columns, reading C6/C7),
 *     emulated step by step in fp64: per rank, the Ulysses all-to-all (§4.1.1) is an index
 *     gather (scatter heads, gather sequence), the ring loop (§4.1.1, "parallel version of
 *     Flash Attention ... P2P transmission of K and V subblock") visits KV blocks in the order of
 *     reading C9 and merges block results by log-sum-exp, then the reverse all-to-all returns the
 *     rows to their owner.  The method claims it "yields the same results as the serial version"
 *     (P:240), so this must equal xo_attention up to fp64 rounding.
 *
 * Layouts (all row-major, fp64):
 *   q, out: [B][Sq][H][D];  k, v: [B][Skv][H][D];  lse: [B][H][Sq]  (natural log, scaled logits).
 *
 * Threads: plain pthreads over (b, h, query-row chunks); each output element is computed by exactly
 * one thread in a fixed order, so results are bitwise deterministic for any thread count.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define XO_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------------ */
/* One query row of the plain definition (PAPER, reading C1/C2/C3):                       */
/*   s_j = (sum_d q_d k_jd) * scale ;  m = max_j s_j ; e_j = exp(s_j - m) ; l = sum_j e_j      */
/*   out_d = (sum_j e_j v_jd) / l ;   lse = m + log(l)                                          */
/* k_row(j) = k + j*k_stride, v_row(j) = v + j*v_stride (element strides).                      */
/* scratch must hold Skv doubles.                                                               */
/* ------------------------------------------------------------------------------------------ */
static void attention_row(const double* q, const double* k, const double* v, long k_stride,
                          long v_stride, int Skv, int D, double scale, double* out, double* lse,
                          double* scratch) {
  double m = -INFINITY;
  for (int j = 0; j < Skv; ++j) {
    const double* kj = k + (long)j * k_stride;
    double dot = 0.0;
    for (int d = 0; d < D; ++d) dot += q[d] * kj[d];
    scratch[j] = dot * scale;
    if (scratch[j] > m) m = scratch[j];
  }
  double l = 0.0;
  for (int j = 0; j < Skv; ++j) {
    scratch[j] = exp(scratch[j] - m);
    l += scratch[j];
  }
  for (int d = 0; d < D; ++d) {
    double acc = 0.0;
    for (int j = 0; j < Skv; ++j) acc += scratch[j] * v[(long)j * v_stride + d];
    out[d] = acc / l;
  }
  *lse = m + log(l);
}

/* ------------------------------------------------------------------------------------------ */
/* Threaded driver over (b, h, row) work items.                                                  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
  const double *q, *k, *v;
  double *out, *lse;
  int B, Sq, Skv, H, D;
  double scale;
  const int64_t* rows; /* NULL: all rows; else nrows query-row indices */
  int nrows;
  long n_items; /* B*H*nrows */
  int nthreads, tid;
} job_t;

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(J->Skv > 0 ? J->Skv : 1));
  if (!scratch) return (void*)1;
  const long HD = (long)J->H * J->D;
  /* static block partition of the item range: deterministic assignment */
  long per = (J->n_items + J->nthreads - 1) / J->nthreads;
  long lo = per * J->tid, hi = lo + per;
  if (hi > J->n_items) hi = J->n_items;
  for (long it = lo; it < hi; ++it) {
    int r = (int)(it % J->nrows);
    long bh = it / J->nrows;
    int h = (int)(bh % J->H), b = (int)(bh / J->H);
    long i = J->rows ? (long)J->rows[r] : (long)r; /* global query row */
    const double* qrow = J->q + ((long)b * J->Sq + i) * HD + (long)h * J->D;
    const double* kb = J->k + (long)b * J->Skv * HD + (long)h * J->D;
    const double* vb = J->v + (long)b * J->Skv * HD + (long)h * J->D;
    double* orow;
    double* l;
    if (J->rows) { /* compact outputs: out [B][nrows][H][D], lse [B][H][nrows] */
      orow = J->out + ((long)b * J->nrows + r) * HD + (long)h * J->D;
      l = J->lse + ((long)b * J->H + h) * J->nrows + r;
    } else {
      orow = J->out + ((long)b * J->Sq + i) * HD + (long)h * J->D;
      l = J->lse + ((long)b * J->H + h) * J->Sq + i;
    }
    attention_row(qrow, kb, vb, HD, HD, J->Skv, J->D, J->scale, orow, l, scratch);
  }
  free(scratch);
  return NULL;
}

static int run_jobs(job_t base, int nthreads) {
  if (nthreads <= 0) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    nthreads = n > 0 ? (int)n : 1;
  }
  if (nthreads > 256) nthreads = 256;
  if (base.n_items < nthreads) nthreads = base.n_items > 0 ? (int)base.n_items : 1;
  pthread_t th[256];
  job_t jobs[256];
  int rc = 0;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = base;
    jobs[t].nthreads = nthreads;
    jobs[t].tid = t;
    if (pthread_create(&th[t], NULL, worker, &jobs[t]) != 0) {
      nthreads = t;
      rc = -2;
      break;
    }
  }
  for (int t = 0; t < nthreads; ++t) {
    void* ret = NULL;
    pthread_join(th[t], &ret);
    if (ret) rc = -3;
  }
  return rc;
}

/* Returns the thread count the oracle would use for nthreads<=0 (for reporting). */
XO_EXPORT int xo_default_threads(void) {
  long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)(n > 256 ? 256 : n) : 1;
}

/* Full attention on global tensors.  scale <= 0 selects 1/sqrt(D) (reading C1). */
XO_EXPORT int xo_attention(const double* q, const double* k, const double* v, double* out,
                           double* lse, int B, int Sq, int Skv, int H, int D, double scale,
                           int nthreads) {
  if (!q || !k || !v || !out || !lse || B < 0 || Sq < 0 || Skv <= 0 || H <= 0 || D <= 0) return -1;
  job_t J;
  memset(&J, 0, sizeof J);
  J.q = q; J.k = k; J.v = v; J.out = out; J.lse = lse;
  J.B = B; J.Sq = Sq; J.Skv = Skv; J.H = H; J.D = D;
  J.scale = scale > 0 ? scale : 1.0 / sqrt((double)D);
  J.rows = NULL;
  J.nrows = Sq;
  J.n_items = (long)B * H * Sq;
  if (J.n_items == 0) return 0;
  return run_jobs(J, nthreads);
}

/* Attention for a subset of query rows; out [B][nrows][H][D], lse [B][H][nrows]. */
XO_EXPORT int xo_attention_rows(const double* q, const double* k, const double* v,
                                const int64_t* rows, int nrows, double* out, double* lse, int B,
                                int Sq, int Skv, int H, int D, double scale, int nthreads) {
  if (!q || !k || !v || !rows || !out || !lse || nrows <= 0 || B <= 0 || Skv <= 0 || H <= 0 ||
      D <= 0)
    return -1;
  for (int r = 0; r < nrows; ++r)
    if (rows[r] < 0 || rows[r] >= Sq) return -1;
  job_t J;
  memset(&J, 0, sizeof J);
  J.q = q; J.k = k; J.v = v; J.out = out; J.lse = lse;
  J.B = B; J.Sq = Sq; J.Skv = Skv; J.H = H; J.D = D;
  J.scale = scale > 0 ? scale : 1.0 / sqrt((double)D);
  J.rows = rows;
  J.nrows = nrows;
  J.n_items = (long)B * H * nrows;
  return run_jobs(J, nthreads);
}

/* ------------------------------------------------------------------------------------------ */
/* Shard rule (§4.1.1, reading C5): text and image are split separately; rank g gets the  */
/* g-th balanced contiguous piece of each, floor(S/N) + (g < S mod N) tokens (np.array_split).  */
/* Its local sequence is concat(text piece, image piece).                                       */
/* ------------------------------------------------------------------------------------------ */
static void balanced_piece(int S, int N, int g, int* off, int* len) {
  int base = S / N, rem = S % N;
  *len = base + (g < rem ? 1 : 0);
  *off = g * base + (g < rem ? g : rem);
}

XO_EXPORT int xo_shard(int S_txt, int S_img, int N, int g, int* txt_off, int* txt_len,
                       int* img_off, int* img_len) {
  if (S_txt < 0 || S_img < 0 || N <= 0 || g < 0 || g >= N) return -1;
  balanced_piece(S_txt, N, g, txt_off, txt_len);
  balanced_piece(S_img, N, g, img_off, img_len);
  if (*txt_len + *img_len == 0) return -5; /* empty shard: reading C5 */
  return 0;
}

/* Global joint-sequence row of local row t on rank g: [text; image] order (reading C4). */
static long local_to_global(int S_txt, int S_img, int N, int g, int t) {
  int to, tl, io, il;
  balanced_piece(S_txt, N, g, &to, &tl);
  balanced_piece(S_img, N, g, &io, &il);
  if (t < tl) return to + t;
  return (long)S_txt + io + (t - tl);
}

/* ------------------------------------------------------------------------------------------ */
/* USP split emulator (§4.1.4; §4.1.1; readings C5-C9, C15).                */
/*                                                                                              */
/* Mesh: N = u*r ranks, rank g = i*u + j; i = ring index (column of the 2D mesh: SP-Ring group), */
/* j = Ulysses index (row: SP-Ulysses group) -- reading C6.                                      */
/* Step 1 (Ulysses all-to-all): rank (i,j) gathers, from every rank (i,j') of its Ulysses */
/*   group, that rank's local tokens restricted to head block j (contiguous heads, reading C7).  */
/*   Its "ring block" is therefore the rows of shards i*u .. i*u+u-1, in that order.             */
/* Step 2 (Ring): for s = 0..r-1 the rank attends its ring-block queries to the KV block  */
/*   of ring index (i - s) mod r (reading C9), getting (O_s, LSE_s), and merges sequentially:    */
/*     LSE = M + log(exp(LSE_acc - M) + exp(LSE_s - M)),  M = max(LSE_acc, LSE_s)               */
/*     O   = exp(LSE_acc - LSE) O_acc + exp(LSE_s - LSE) O_s                                     */
/* Step 3 (reverse all-to-all): each query row's result returns to the rank owning that token.  */
/* Everything is fp64; the "communication" is index bookkeeping on global arrays.                */
/* ------------------------------------------------------------------------------------------ */
XO_EXPORT int xo_usp_emulate(const double* q, const double* k, const double* v, double* out,
                             double* lse, int B, int H, int S_txt, int S_img, int D, int u, int r) {
  if (!q || !k || !v || !out || !lse || B <= 0 || H <= 0 || D <= 0 || u <= 0 || r <= 0) return -1;
  if (H % u != 0) return -3; /* reading C8: "16 does not divide evenly into 24" */
  const int N = u * r, S = S_txt + S_img, Hu = H / u;
  const long HD = (long)H * D;
  const double scale = 1.0 / sqrt((double)D);
  for (int g = 0; g < N; ++g) {
    int a, b_, c, d;
    if (xo_shard(S_txt, S_img, N, g, &a, &b_, &c, &d) != 0) return -5;
  }
  /* ring block row lists: blk_rows[i] = global rows of shards i*u..i*u+u-1 in order */
  long** blk_rows = (long**)calloc((size_t)r, sizeof(long*));
  int* blk_len = (int*)calloc((size_t)r, sizeof(int));
  int max_blk = 0;
  for (int i = 0; i < r; ++i) {
    int n = 0;
    for (int jj = 0; jj < u; ++jj) {
      int to, tl, io, il;
      xo_shard(S_txt, S_img, N, i * u + jj, &to, &tl, &io, &il);
      n += tl + il;
    }
    blk_len[i] = n;
    if (n > max_blk) max_blk = n;
    blk_rows[i] = (long*)malloc(sizeof(long) * (size_t)n);
    int p = 0;
    for (int jj = 0; jj < u; ++jj) {
      int to, tl, io, il, g = i * u + jj;
      xo_shard(S_txt, S_img, N, g, &to, &tl, &io, &il);
      for (int t = 0; t < tl + il; ++t) blk_rows[i][p++] = local_to_global(S_txt, S_img, N, g, t);
    }
  }
  /* gathered KV block (one head) and scratch */
  double* kblk = (double*)malloc(sizeof(double) * (size_t)max_blk * D);
  double* vblk = (double*)malloc(sizeof(double) * (size_t)max_blk * D);
  double* scratch = (double*)malloc(sizeof(double) * (size_t)max_blk);
  double* o_acc = (double*)malloc(sizeof(double) * (size_t)D);
  double* o_s = (double*)malloc(sizeof(double) * (size_t)D);
  int seen_rows = 0;
  for (int g = 0; g < N; ++g) {
    const int i = g / u, j = g % u;
    /* Step 1: this rank's queries = ring block i, heads [j*Hu, (j+1)*Hu) */
    for (int bb = 0; bb < B; ++bb) {
      for (int hh = 0; hh < Hu; ++hh) {
        const int h = j * Hu + hh;
        for (int t = 0; t < blk_len[i]; ++t) {
          const long gi = blk_rows[i][t];
          const double* qrow = q + ((long)bb * S + gi) * HD + (long)h * D;
          double lse_acc = 0.0;
          /* Step 2: ring loop, KV block of ring index (i - s) mod r */
          for (int s = 0; s < r; ++s) {
            const int src = ((i - s) % r + r) % r;
            for (int t2 = 0; t2 < blk_len[src]; ++t2) {
              const long gk = blk_rows[src][t2];
              memcpy(kblk + (long)t2 * D, k + ((long)bb * S + gk) * HD + (long)h * D,
                     sizeof(double) * D);
              memcpy(vblk + (long)t2 * D, v + ((long)bb * S + gk) * HD + (long)h * D,
                     sizeof(double) * D);
            }
            double lse_s;
            attention_row(qrow, kblk, vblk, D, D, blk_len[src], D, scale, s == 0 ? o_acc : o_s,
                          s == 0 ? &lse_acc : &lse_s, scratch);
            if (s > 0) {
              const double M = lse_acc > lse_s ? lse_acc : lse_s;
              const double L = M + log(exp(lse_acc - M) + exp(lse_s - M));
              const double wa = exp(lse_acc - L), ws = exp(lse_s - L);
              for (int d = 0; d < D; ++d) o_acc[d] = wa * o_acc[d] + ws * o_s[d];
              lse_acc = L;
            }
          }
          /* Step 3: reverse all-to-all -- the row goes back to its owner's slot.  In global
           * coordinates that is simply row gi, head h. */
          memcpy(out + ((long)bb * S + gi) * HD + (long)h * D, o_acc, sizeof(double) * D);
          lse[((long)bb * H + h) * S + gi] = lse_acc;
          ++seen_rows;
        }
      }
    }
  }
  for (int i = 0; i < r; ++i) free(blk_rows[i]);
  free(blk_rows); free(blk_len); free(kblk); free(vblk); free(scratch); free(o_acc); free(o_s);
  /* every (b, row, head) must have been produced exactly once */
  return seen_rows == B * S * H ? 0 : -4;
}
