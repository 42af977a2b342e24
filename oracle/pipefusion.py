"""fp64 oracle for PipeFusion on a synthetic DiT stack -- TEST INFRASTRUCTURE.

Only ``tests/`` and ``bench``-side tools may import this module; the product package never does
and shares no code with it.  numpy fp64; the one library primitive is ``oracle.attention`` (the
plain softmax(QK^T/sqrt(D))V definition).

What it follows (§4.1.2):
  * "partitions the input latent image into patches and the DiTs transformer model into layers ...
    assigning each partition of consecutive layers to a GPU": stage d of N owns blocks
    [d L/N, (d+1) L/N);
  * "divided into M non-overlapping patches, allowing each GPU to process one patch with its
    assigned layers in parallel": micro-step tau, stage d works on patch tau - d;
  * "a device can start its computation without waiting for full spatial activations at timestep
    T. Instead, it uses stale activations from the previous timestep to provide context":
    block l's attention for patch m reads a per-block KV buffer holding the K,V of every patch as
    last computed -- this step for patches already processed at block l, the previous step for the
    others (SPEC S:330-335 KVBuffer);
  * "we usually conduct several diffusion iterations synchronously, called warmup steps":
    the first `warmup` steps run every block over the whole sequence (no staleness);
  * "text vectors are concatenated with Patch0": text tokens ride with patch 0.

Readings (R4): the synthetic DiT block l maps the hidden state h [B,S,H,D] as
    q = h * wq_l,  k = h * wk_l,  v = h * wv_l      (per-channel weights, [H,D])
    h <- h + g_l * softmax(q k^T / sqrt(D)) v        (per head)
the model output is eps = h after the L blocks, and the sampler step is x <- x - sigma * eps.
Patches: image tokens split into M balanced contiguous pieces (np.array_split), patch 0 = text +
image piece 0, patch m > 0 = image piece m ([text; image] order, reading C4).

Functions:
  patch_bounds(S_txt, S_img, M)               -> [(off, len)] in the joint sequence
  replay_stamps(N, M, L, T, warmup)           -> {(s, m, l): stamps of all M patches' KV visible}
  serial_eps(x, W)                            -> eps of one full-sequence (synchronous) step
  pipefusion(x, W, T, M, warmup, sigma, S_txt, N=1, order="patch") -> x after T steps, per-step xs
  hybrid(x, W, T, M, warmup, sigma, S_txt, u, r, naive=False) -> x, per-rank KV buffers
"""
from __future__ import annotations

import numpy as np

from . import attention, local_rows


def patch_bounds(S_txt: int, S_img: int, M: int):
    """[(offset, length)] of the M patches in the joint [text; image] sequence (R4)."""
    if M < 1 or S_img < M:
        raise ValueError("need 1 <= M <= S_img")
    base, rem = divmod(S_img, M)
    out, off = [], S_txt
    for m in range(M):
        n = base + (1 if m < rem else 0)
        if m == 0:
            out.append((0, S_txt + n))
        else:
            out.append((off, n))
        off += n
    return out


def stages(N: int, L: int):
    """Blocks of stage d: [d L/N, (d+1) L/N) (SPEC S:390 'L % N == 0')."""
    if N < 1 or L % N:
        raise ValueError("L must be a multiple of N")
    return [list(range(d * L // N, (d + 1) * L // N)) for d in range(N)]


def replay_stamps(N: int, M: int, L: int, T: int, warmup: int):
    """Brute-force discrete-event replay of the PipeFusion schedule (no numerics).

    Step s = 0..T-1 in execution order.  Warmup steps refresh every patch of every block before any
    attention reads it (synchronous).  Pipelined steps run micro-steps tau = 0..M+N-2; in micro-step
    tau stage d processes patch m = tau - d through its blocks: it first writes patch m's fresh K,V
    (stamp s) into block l's buffer, then attends over the buffer.  Returns, for every (s, m, l),
    the tuple of stamps (the step whose K,V each patch contributes) that attention reads."""
    st = stages(N, L)
    stamp = [[None] * M for _ in range(L)]
    seen = {}
    for s in range(T):
        if s < warmup:
            for l in range(L):
                for m in range(M):
                    stamp[l][m] = s
                for m in range(M):
                    seen[(s, m, l)] = tuple(stamp[l])
            continue
        for tau in range(M + N - 1):
            for d in range(N):
                m = tau - d
                if 0 <= m < M:
                    for l in st[d]:
                        stamp[l][m] = s
                        seen[(s, m, l)] = tuple(stamp[l])
    return seen


def _block(h, kbuf, vbuf, wq, wg):
    """h + g * attention(h * wq, Kbuf, Vbuf) -- one synthetic DiT block for the rows of h (R4)."""
    q = h * wq
    o, _ = attention(q, kbuf, vbuf)
    return h + wg * o


def serial_eps(x, W):
    """One synchronous step: every block over the whole sequence (the serial DiT forward)."""
    h = np.asarray(x, np.float64)
    for (wq, wk, wv, wg) in W:
        h = _block(h, h * wk, h * wv, wq, wg)
    return h


def pipefusion(x, W, T: int, M: int, warmup: int, sigma: float, S_txt: int, N: int = 1, order: str = "patch"):
    """x after T sampler steps of PipeFusion (reading R4), plus the x after each step.

    x: [B, S, H, D]; W: list of L tuples (wq, wk, wv, g), each [H, D].  order="patch" evaluates
    patch-major (for m: for l), the sequential definition; order="pipeline" evaluates the same step
    in the micro-step order of an N-stage pipeline (for tau: for d: m = tau - d: for l in stage d).
    Both must give identical numbers: a patch's attention at block l reads the same buffer in
    either order (the N-independence of the staleness pattern)."""
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    x = np.array(x, np.float64)
    B, S, H, D = x.shape
    L = len(W)
    P = patch_bounds(S_txt, S - S_txt, M)
    kbuf = [np.zeros_like(x) for _ in range(L)]
    vbuf = [np.zeros_like(x) for _ in range(L)]
    xs = []
    for s in range(T):
        if s < warmup:
            h = x.copy()
            for l, (wq, wk, wv, wg) in enumerate(W):
                kbuf[l][:], vbuf[l][:] = h * wk, h * wv
                h = _block(h, kbuf[l], vbuf[l], wq, wg)
            eps = h
        else:
            eps = np.empty_like(x)
            hp = [x[:, o:o + n].copy() for (o, n) in P]  # per-patch hidden state
            if order == "patch":
                work = [(m, l) for m in range(M) for l in range(L)]
            else:
                st = stages(N, L)
                work = [(tau - d, l) for tau in range(M + N - 1) for d in range(N)
                        if 0 <= tau - d < M for l in st[d]]
            for (m, l) in work:
                wq, wk, wv, wg = W[l]
                o, n = P[m]
                h = hp[m]
                kbuf[l][:, o:o + n], vbuf[l][:, o:o + n] = h * wk, h * wv  # fresh K,V of patch m
                hp[m] = _block(h, kbuf[l], vbuf[l], wq, wg)
            for m, (o, n) in enumerate(P):
                eps[:, o:o + n] = hp[m]
        x = x - sigma * eps
        xs.append(x.copy())
    return x, xs


def hybrid(x, W, T: int, M: int, warmup: int, sigma: float, S_txt: int, u: int, r: int, naive: bool = False):
    """Hybrid PipeFusion x SP (§4.1.4; R6), fp64, emulating
    the SP group's u*r ranks and their per-rank KV buffers step by step.

      * "The entire hidden state is first split into M patches along the sequence dimension, and each
        patch is further split into sp_degree patches": rank g of the SP group holds, of every
        item (a patch, or the whole sequence in a synchronous warmup step), the rows the in-context
        shard rule gives it on the item's own [text; image] tokens (reading C5);
      * USP: rank g = (i, j) = (g // u, g % u) computes the attention output of the query
        rows of its ring block i (the rows of ranks i*u .. i*u+u-1) for its Ulysses head block j
        (reading C7), against ITS OWN KV buffer of block l -- heads of block j, every sequence row;
      * the buffers: before the attention of an item at block l, rank g writes the item's fresh K,V
        into its buffer.  naive=False: "after communication of K and V in SP-Ulysses and SP-Ring, the
        intermediate results ... are stored in each device's KV Buffer" -- the rank keeps the
        K,V of every row of the item it received (all-to-all: its ring block; ring: the others), i.e.
        all the item's rows, heads of block j.  naive=True: "standard SP", which discards
        them -- the rank writes only the rows it holds itself, so the buffers of an SP group diverge.

    The item order is the sequential (patch-major) definition of `pipefusion`; the pipeline order of
    the stages does not change a patch's buffer contents (pinned for `pipefusion`).  Returns the
    latent after T steps and the final buffers kv[g][l] = (K [B,S,H/u,D], V [B,S,H/u,D])."""
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    x = np.array(x, np.float64)
    B, S, H, D = x.shape
    N, Hh, L = u * r, H // u, len(W)
    if H % u:
        raise ValueError("H % ulysses != 0 (P:541)")
    P = patch_bounds(S_txt, S - S_txt, M)
    kb = [[np.zeros((B, S, Hh, D)) for _ in range(L)] for _ in range(N)]
    vb = [[np.zeros((B, S, Hh, D)) for _ in range(L)] for _ in range(N)]
    for s in range(T):
        items = [None] if s < warmup else list(range(M))
        eps = np.empty_like(x)
        for m in items:
            if m is None:
                base, it_txt, it_img, img_base = 0, S_txt, S - S_txt, S_txt
            else:
                o, n = P[m]
                base, it_txt = o, (S_txt if m == 0 else 0)
                it_img, img_base = n - it_txt, (S_txt if m == 0 else o)
            # global rows of every rank's shard of the item (text shard, then image shard)
            own = []
            for g in range(N):
                lr = local_rows(it_txt, it_img, N, g)
                own.append(np.where(lr < it_txt, lr, lr - it_txt + img_base))
            rows = np.concatenate(own)
            h = x[:, rows].copy()                       # the item's hidden rows, in SP-shard order
            pos = {int(t): k for k, t in enumerate(rows)}
            for l, (wq, wk, wv, wg) in enumerate(W):
                q, k, v = h * wq, h * wk, h * wv
                for g in range(N):  # fresh K,V into each rank's buffer (its head block j)
                    j = g % u
                    keep = rows if not naive else own[g]
                    kk = [pos[int(t)] for t in keep]
                    kb[g][l][:, keep] = k[:, kk][:, :, j * Hh:(j + 1) * Hh]
                    vb[g][l][:, keep] = v[:, kk][:, :, j * Hh:(j + 1) * Hh]
                o_att = np.empty_like(h)
                for g in range(N):  # rank (i, j): ring block i's queries x head block j
                    i, j = g // u, g % u
                    blk = np.concatenate([own[i * u + p] for p in range(u)])
                    qq = [pos[int(t)] for t in blk]
                    oo, _ = attention(q[:, qq][:, :, j * Hh:(j + 1) * Hh], kb[g][l], vb[g][l])
                    o_att[:, qq, j * Hh:(j + 1) * Hh] = oo
                h = h + wg * o_att
            eps[:, rows] = h
        x = x - sigma * eps
    return x, [[(kb[g][l], vb[g][l]) for l in range(L)] for g in range(N)]
