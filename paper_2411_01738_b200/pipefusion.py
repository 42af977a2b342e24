"""PipeFusion on a synthetic DiT stack -- SURVEY §8(f) NEXT 3 (§4.1.2
§4.1.4; readings R4, R6).

Host orchestration only (argument marshalling and the schedule): every block of every patch runs in
the library -- `xdit_pf_block` (fresh-K,V scatter into the block's KV buffer, tcgen05 attention of the
patch over the whole buffer, residual) on one device, or `xdit_pf_qkv` + the USP call over the KV
buffer `xdit_usp_attention_buf` + `xdit_pf_residual` inside an SP group -- and the sampler step in
`xdit_pf_sampler`; patch activations move between stages with `xdit_p2p` (NCCL).

Schedule: stage d of N owns blocks [d L/N, (d+1) L/N) and their KV buffers; patch m
enters stage d once stage d-1 has finished it, so stages work on different patches concurrently
(micro-step tau: stage d on patch tau - d).  The first `warmup` steps run every block over the whole
sequence.  Text tokens ride with patch 0.

Hybrid PipeFusion x SP: the devices form a pipefusion_degree x sp_degree mesh; each
stage is an SP group (ulysses x ring) that splits every patch once more along the sequence (the
in-context shard rule) and runs USP attention over the block's KV buffer, into which the SP
call writes the fresh K,V of the WHOLE patch it received through the all-to-all and the ring ("the
intermediate results ... are stored in each device's KV Buffer") -- so every rank of a head
block holds the same buffer, and the result equals pure PipeFusion with the same (N, M).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from . import usp


def patch_bounds(S_txt: int, S_img: int, M: int) -> List[Tuple[int, int]]:
    """(offset, length) of the M patches of the joint [text; image] sequence: the image tokens in M
    pieces by the library's balanced split (xdit_usp_shard), the text with patch 0 (R4)."""
    if M < 1 or S_img < M:
        raise ValueError("need 1 <= M <= S_img")
    out = []
    for m in range(M):
        _, _, io, il = usp.shard(0, S_img, M, m)
        out.append((0, S_txt + il) if m == 0 else (S_txt + io, il))
    return out


def workspace_bytes(B: int, n: int, H: int, D: int, dtype: int) -> int:
    return int(usp.lib().xdit_pf_block_workspace_bytes(B, n, H, D, dtype))


def _dt(t) -> int:
    import torch
    return 1 if t.dtype == torch.float32 else 0


def block(h, kv_buf, w, work, *, S: int, off: int, stream=None):
    """One synthetic DiT block on one patch (xdit_pf_block): h [B, n, H, D] in place."""
    B, n, H, D = h.shape
    rc = usp.lib().xdit_pf_block(usp._ptr(h), usp._ptr(kv_buf), usp._ptr(w), usp._ptr(work),
                                 work.numel() * work.element_size(), B, H, S, off, n, D, _dt(h), usp._stream(stream))
    usp._check(rc, "xdit_pf_block")


def qkv(h, w, q, k, v, stream=None):
    """q, k, v <- h * wq, h * wk, h * wv (xdit_pf_qkv)."""
    B, n, H, D = h.shape
    usp._check(usp.lib().xdit_pf_qkv(usp._ptr(h), usp._ptr(w), usp._ptr(q), usp._ptr(k), usp._ptr(v), B, n, H, D,
                                     _dt(h), usp._stream(stream)), "xdit_pf_qkv")


def residual(h, o, w, stream=None):
    """h <- h + g * o (xdit_pf_residual)."""
    B, n, H, D = h.shape
    usp._check(usp.lib().xdit_pf_residual(usp._ptr(h), usp._ptr(o), usp._ptr(w), B, n, H, D, _dt(h),
                                          usp._stream(stream)), "xdit_pf_residual")


def sampler(x, eps, sigma: float, stream=None):
    """x <- x - sigma * eps (xdit_pf_sampler); contiguous tensors of the same shape."""
    rc = usp.lib().xdit_pf_sampler(usp._ptr(x), usp._ptr(eps), x.numel(), float(sigma), _dt(x), usp._stream(stream))
    usp._check(rc, "xdit_pf_sampler")


class SyntheticDiT:
    """L synthetic DiT blocks (reading R4): weights[l] = (wq, wk, wv, g), each [H, D]."""

    def __init__(self, weights: Sequence[Sequence], device="cuda"):
        import torch
        self.w = [torch.stack([torch.as_tensor(x, dtype=torch.float32) for x in wl]).contiguous().to(device)
                  for wl in weights]
        self.L = len(self.w)


def run(x0, dit: SyntheticDiT, *, T: int, M: int, warmup: int, sigma: float, S_txt: int, stages: int = 1):
    """T sampler steps of PipeFusion from latent x0 [B, S, H, D] (bf16 or fp32, CUDA) on ONE device,
    the N stages as concurrent CUDA streams (patch m enters stage d after an event of stage d-1);
    returns x."""
    import torch
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    N, L = stages, dit.L
    if N < 1 or L % N:
        raise ValueError("the number of blocks must be a multiple of the number of stages")
    B, S, H, D = x0.shape
    dtype = _dt(x0)
    P = patch_bounds(S_txt, S - S_txt, M)
    dev = x0.device
    x = x0.clone()
    kv = [torch.zeros((2, B, H, S, D), dtype=x0.dtype, device=dev) for _ in range(L)]
    n_max = max(n for _, n in P)
    u8 = torch.uint8
    work_full = torch.empty(workspace_bytes(B, S, H, D, dtype), dtype=u8, device=dev)
    work = [torch.empty(workspace_bytes(B, n_max, H, D, dtype), dtype=u8, device=dev) for _ in range(N)]
    hp = [torch.empty((B, n, H, D), dtype=x0.dtype, device=dev) for _, n in P]
    h_full = torch.empty_like(x)
    main = torch.cuda.current_stream(dev)
    streams = [torch.cuda.Stream(device=dev) for _ in range(N)]
    done = [[torch.cuda.Event() for _ in range(N)] for _ in range(M)]
    stage_blocks = [list(range(d * L // N, (d + 1) * L // N)) for d in range(N)]
    for s in range(T):
        if s < warmup:  # synchronous step over the whole sequence
            h_full.copy_(x)
            for l in range(L):
                block(h_full, kv[l], dit.w[l], work_full, S=S, off=0, stream=main)
            sampler(x, h_full, sigma, stream=main)
            continue
        for st in streams:
            st.wait_stream(main)
        for m, (o, n) in enumerate(P):
            for d in range(N):
                st = streams[d]
                with torch.cuda.stream(st):
                    if d == 0:
                        hp[m].copy_(x[:, o:o + n])
                    else:
                        st.wait_event(done[m][d - 1])
                    for l in stage_blocks[d]:
                        block(hp[m], kv[l], dit.w[l], work[d], S=S, off=o, stream=st)
                    if d == N - 1:  # this patch's eps is final: its sampler step (x rows of patch m)
                        for b in range(B):
                            sampler(x[b, o:o + n], hp[m][b], sigma, stream=st)
                    done[m][d].record(st)
        for st in streams:
            main.wait_stream(st)
    return x


# --------------------------------------------------------------------------- multi-device schedule
def work_items(T: int, M: int, warmup: int):
    """The items every stage processes, in order: (step, None) = a synchronous full-sequence pass
    (warmup), (step, m) = patch m of a pipelined step."""
    return [(s, None) for s in range(min(warmup, T))] + [(s, m) for s in range(warmup, T) for m in range(M)]


def micro_schedule(N: int, T: int, M: int, warmup: int):
    """Lock-step micro-step schedule of an N-stage pipeline (pure host logic, identical on every rank).

    Every micro-step each stage processes at most one item -- the next in its order, once its input
    is there: stage d > 0 needs stage d-1 to have processed the item in an EARLIER micro-step (the
    activation travels in the send/receive group that closes that micro-step, "devices send
    micro-step patch activations to subsequent devices via asynchronous P2P"); stage 0 needs
    the eps of every item of the previous step that covers the same rows (sent back by the last
    stage).  Returns a list of micro-steps, each a list of N item indices (or None)."""
    items = work_items(T, M, warmup)
    K = len(items)
    done_at = [[None] * K for _ in range(N)]  # micro-step at which stage d processed item k
    nxt = [0] * N
    steps = []
    tau = 0

    def eps_ready(k, t):  # stage 0 may start item k at micro-step t
        s, m = items[k]
        if s == 0:
            return True
        need = [j for j, (s2, m2) in enumerate(items) if s2 == s - 1 and (m is None or m2 is None or m2 == m)]
        return all(done_at[N - 1][j] is not None and done_at[N - 1][j] < t for j in need)

    while min(nxt) < K:
        row = [None] * N
        for d in range(N):
            k = nxt[d]
            if k >= K:
                continue
            ready = eps_ready(k, tau) if d == 0 else (done_at[d - 1][k] is not None and done_at[d - 1][k] < tau)
            if ready:
                row[d] = k
        for d, k in enumerate(row):
            if k is not None:
                done_at[d][k] = tau
                nxt[d] += 1
        steps.append(row)
        tau += 1
        if tau > 4 * (K + N) * max(1, N):
            raise RuntimeError("PipeFusion schedule did not converge")
    return steps


def _rows_of(S_txt_g: int, item, P, sp: int, g: int):
    """Global sequence rows of SP rank g's local shard of `item`, and the item's joint (S_txt, S_img)
    and buffer rows of its first text / image token (txt_row, img_row) -- the in-context shard rule
     applied to the item's tokens."""
    import torch
    s, m = item
    if m is None:  # the whole sequence
        it_txt, it_img, img_base = S_txt_g, P[-1][0] + P[-1][1] - S_txt_g, S_txt_g
    else:
        o, n = P[m]
        it_txt = S_txt_g if m == 0 else 0
        it_img = n - it_txt
        img_base = S_txt_g if m == 0 else o
    to, tl, io, il = usp.shard(it_txt, it_img, sp, g)
    rows = torch.cat([torch.arange(to, to + tl), img_base + torch.arange(io, io + il)])
    return rows, it_txt, it_img, 0, img_base


def run_mesh(x0, weights, *, stage: int, stages: int, chain: "usp.Comm", sp_comm: "usp.Comm", T: int, M: int,
             warmup: int, sigma: float, S_txt: int, kv_out=None):
    """PipeFusion over a stages x sp mesh, one PROCESS per device (pure PipeFusion when the SP group
    is one rank).  This rank is stage `stage` of `stages` and SP rank sp_comm.rank of its stage's SP
    group (ulysses x ring); `chain` links the ranks of the same SP position across the stages (rank
    of `chain` = stage index).  Patch activations (this rank's shard of each item) move stage to stage,
    the last stage's eps back to stage 0, in one xdit_p2p group per micro-step (deadlock-free: every
    rank of a chain runs the same micro_schedule).

    x0: the initial latent [B, S, H, D] on this rank's GPU (stage 0 uses it); weights: all L blocks'
    (wq, wk, wv, g).  Returns the latent after T steps on stage 0 (every stage-0 rank holds all of
    it), None elsewhere.  kv_out: a list that receives this rank's KV buffers (its blocks; heads of
    its Ulysses block), for consistency checks."""
    import torch
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    N, d = stages, stage
    L = len(weights)
    if L % N:
        raise ValueError("the number of blocks must be a multiple of the number of stages")
    B, S, H, D = x0.shape
    u, r = sp_comm.ulysses, sp_comm.ring
    sp, g = u * r, sp_comm.rank
    Hh = H // u
    dt, dev = x0.dtype, x0.device
    P = patch_bounds(S_txt, S - S_txt, M)
    items = work_items(T, M, warmup)
    sched = micro_schedule(N, T, M, warmup)
    geo = [_rows_of(S_txt, it, P, sp, g) for it in items]
    mine = list(range(d * L // N, (d + 1) * L // N))
    dit = SyntheticDiT([weights[l] for l in mine], device=dev)
    kv = [torch.zeros((2, B, Hh, S, D), dtype=dt, device=dev) for _ in mine]  # head block j = g % u, all rows
    n_max = max(len(gm[0]) for gm in geo)
    flat = B * n_max * H * D
    act = [torch.empty(flat, dtype=dt, device=dev) for _ in range(2)]  # item k lives in act[k % 2]
    eps_in, tq, tk, tv, to_ = (torch.empty(flat, dtype=dt, device=dev) for _ in range(5))
    st = torch.cuda.current_stream(dev)
    x = x0.clone() if d == 0 else None

    def view(buf, k):  # contiguous [B, n_k, H, D] view of a flat buffer for item k
        return buf[:B * len(geo[k][0]) * H * D].view(B, -1, H, D)

    work = None
    if sp == 1:  # pure PipeFusion: the one-device block kernel on the item's contiguous rows
        work = torch.empty(workspace_bytes(B, n_max, H, D, _dt(x0)), dtype=torch.uint8, device=dev)

    def stage_blocks(k):
        rows, it_txt, it_img, txt_row, img_row = geo[k]
        h = view(act[k % 2], k)
        if sp == 1:
            for i in range(len(mine)):
                block(h, kv[i], dit.w[i], work, S=S, off=int(rows[0]), stream=st)
            return h
        q, kk, v, o = (view(t, k) for t in (tq, tk, tv, to_))
        for i in range(len(mine)):
            qkv(h, dit.w[i], q, kk, v, stream=st)
            usp.attention_buf(q, kk, v, kv[i], S_txt=it_txt, S_img=it_img, txt_row=txt_row, img_row=img_row,
                              comm=sp_comm, ulysses=u, ring=r, out=o, stream=st)
            residual(h, o, dit.w[i], stream=st)
        return h

    def gather_x(step_items):  # stage-0 ranks of the SP group exchange the rows each one updated
        if sp == 1:
            return
        rows = [torch.cat([_rows_of(S_txt, it, P, sp, q)[0] for it in step_items]) for q in range(sp)]
        mine_rows = x[:, rows[g].to(dev)].contiguous()
        bufs = {q: torch.empty((B, len(rows[q]), H, D), dtype=dt, device=dev) for q in range(sp) if q != g}
        ops = [(q, "send", mine_rows) for q in range(sp) if q != g] + [(q, "recv", bufs[q]) for q in bufs]
        sp_comm.p2p(ops, stream=st)
        for q, b in bufs.items():
            x[:, rows[q].to(dev)] = b

    last_full = max(k for k, (s, m) in enumerate(items) if m is None)
    for row in sched:
        k = row[d]
        if k is not None:
            rows = geo[k][0]
            if d == 0:
                if k == last_full + 1:  # warmup -> pipelined: the shards change from sequence to patches
                    gather_x([items[last_full]])
                view(act[k % 2], k).copy_(x[:, rows.to(dev)])
            stage_blocks(k)
            if N == 1:  # eps is final here: the sampler step of the item's rows
                _apply_eps(x, view(act[k % 2], k), rows, sigma, st)
        # the micro-step's send / receive group along the chain
        if N > 1:
            ops = []
            if k is not None:
                ops.append(((d + 1) % N, "send", view(act[k % 2], k)))
            src = (d - 1) % N
            ks = row[src]
            if ks is not None:
                ops.append((src, "recv", view(eps_in if d == 0 else act[ks % 2], ks)))
            if ops:
                chain.p2p(ops, stream=st)
            if d == 0 and ks is not None:  # eps of item ks arrived from the last stage
                _apply_eps(x, view(eps_in, ks), geo[ks][0], sigma, st)
    if kv_out is not None:
        kv_out.extend(kv)
    if d == 0:
        s_last = items[-1][0]
        gather_x([it for it in items if it[0] == s_last])
        return x
    return None


def _apply_eps(x, eps, rows, sigma, st):
    """x[:, rows] <- x[:, rows] - sigma * eps (the rows of one item; xdit_pf_sampler on a gathered copy)."""
    import torch
    idx = rows.to(x.device)
    with torch.cuda.stream(st):
        xr = x[:, idx].contiguous()
        sampler(xr, eps, sigma, stream=st)
        x[:, idx] = xr
