"""PipeFusion on a synthetic DiT stack -- SURVEY §8(f) NEXT 3 (§4.1.2; R4).

Host orchestration only (argument marshalling and the schedule): every block of every patch runs in
the library's `xdit_pf_block` (fresh-K,V scatter into the block's KV buffer, tcgen05 attention of the
patch over the whole buffer, residual), the sampler step in `xdit_pf_sampler`.

Schedule: stage d of N owns blocks [d L/N, (d+1) L/N) and their KV buffers and runs on
its own CUDA stream; patch m enters stage d once stage d-1 has finished it (an event -- the in-process
form of PipeFusion's asynchronous patch P2P), so stages work on different patches
concurrently (micro-step tau: stage d on patch tau - d).  The first `warmup` steps run every block
over the whole sequence.  Text tokens ride with patch 0.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from . import usp


def patch_bounds(S_txt: int, S_img: int, M: int) -> List[Tuple[int, int]]:
    """(offset, length) of the M patches of the joint [text; image] sequence: image tokens in M
    balanced contiguous pieces, text with patch 0 (reading R4)."""
    if M < 1 or S_img < M:
        raise ValueError("need 1 <= M <= S_img")
    base, rem = divmod(S_img, M)
    out, off = [], S_txt
    for m in range(M):
        n = base + (1 if m < rem else 0)
        out.append((0, S_txt + n) if m == 0 else (off, n))
        off += n
    return out


def workspace_bytes(B: int, n: int, H: int, D: int, dtype: int) -> int:
    return int(usp.lib().xdit_pf_block_workspace_bytes(B, n, H, D, dtype))


def block(h, kv_buf, w, work, *, S: int, off: int, stream=None):
    """One synthetic DiT block on one patch (xdit_pf_block): h [B, n, H, D] in place."""
    import torch
    B, n, H, D = h.shape
    dtype = 1 if h.dtype == torch.float32 else 0
    rc = usp.lib().xdit_pf_block(usp._ptr(h), usp._ptr(kv_buf), usp._ptr(w), usp._ptr(work),
                                 work.numel() * work.element_size(), B, H, S, off, n, D, dtype, usp._stream(stream))
    usp._check(rc, "xdit_pf_block")


def sampler(x, eps, sigma: float, stream=None):
    """x <- x - sigma * eps (xdit_pf_sampler); contiguous tensors of the same shape."""
    import torch
    dtype = 1 if x.dtype == torch.float32 else 0
    rc = usp.lib().xdit_pf_sampler(usp._ptr(x), usp._ptr(eps), x.numel(), float(sigma), dtype, usp._stream(stream))
    usp._check(rc, "xdit_pf_sampler")


class SyntheticDiT:
    """L synthetic DiT blocks (reading R4): weights[l] = (wq, wk, wv, g), each [H, D]."""

    def __init__(self, weights: Sequence[Sequence], device="cuda"):
        import torch
        self.w = [torch.stack([torch.as_tensor(x, dtype=torch.float32) for x in wl]).contiguous().to(device)
                  for wl in weights]
        self.L = len(self.w)


def run(x0, dit: SyntheticDiT, *, T: int, M: int, warmup: int, sigma: float, S_txt: int, stages: int = 1):
    """T sampler steps of PipeFusion from latent x0 [B, S, H, D] (bf16 or fp32, CUDA); returns x."""
    import torch
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    N, L = stages, dit.L
    if N < 1 or L % N:
        raise ValueError("the number of blocks must be a multiple of the number of stages")
    B, S, H, D = x0.shape
    dtype = 1 if x0.dtype == torch.float32 else 0
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


def run_stage(x0, weights, comm, *, T: int, M: int, warmup: int, sigma: float, S_txt: int):
    """PipeFusion with one PROCESS per stage: this rank is stage d = comm.rank of N = comm size,
    owning blocks [d L/N, (d+1) L/N) and their KV buffers; patch activations move stage to stage, and
    the last stage's eps back to stage 0, through the library's peer-transport mailbox ("devices send
    micro-step patch activations to subsequent devices via asynchronous P2P").

    x0: the initial latent [B, S, H, D] on this rank's GPU (only stage 0 uses it); weights: all L
    blocks' (wq, wk, wv, g).  Collective over the comm's ranks.  Returns x after T steps on stage 0,
    None elsewhere.

    Messages on each (sender -> receiver) channel carry increasing tags; the message of step s for
    patch m lands in the receiver's region at (s % 2) * slot + the patch rows' offset, the sender
    first waits for the ack of the previous message in that space (step s - 2), and the receiver acks
    once it has consumed it.  A stage runs its blocks IN the mailbox (in place) and forwards from
    there, so an activation crosses each stage boundary once.  Stage 0 applies patch m's sampler step when patch m's eps arrives, just before it starts
    patch m of the next step (the pipeline runs across step boundaries)."""
    import torch
    if warmup < 1:
        raise ValueError("PipeFusion needs >= 1 warmup step to fill the KV buffers (P:282)")
    N, d = comm.ulysses * comm.ring, comm.rank
    L = len(weights)
    if L % N:
        raise ValueError("the number of blocks must be a multiple of the number of stages")
    B, S, H, D = x0.shape
    dt = x0.dtype
    dev = x0.device
    eb = x0.element_size()
    dtype = 1 if dt == torch.float32 else 0
    P = patch_bounds(S_txt, S - S_txt, M)
    full = B * S * H * D * eb
    slot_bytes = (full + 255) // 256 * 256
    comm.mailbox(2 * slot_bytes)
    mine = list(range(d * L // N, (d + 1) * L // N))
    dit = SyntheticDiT([weights[l] for l in mine], device=dev)
    kv = [torch.zeros((2, B, H, S, D), dtype=dt, device=dev) for _ in mine]
    work_full = torch.empty(workspace_bytes(B, S, H, D, dtype), dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream(dev)
    prev, nxt = (d - 1) % N, (d + 1) % N
    # Message counters of the channels prev -> d and d -> nxt (stage 0 receives from the last stage)
    # and, per mailbox space, the tag of the last message written there -- kept on the handle: the
    # device flags keep their values across calls.  A message of step s for patch m lives at
    # (s % 2) * slot + its rows' byte offset (patches never overlap; a synchronous step's full latent
    # covers them all), so a sender only waits for the receiver to have consumed the message of step
    # s - 2 in that space -- never one of the current step, which would close a cycle with stage 0
    # consuming the eps of step s only while it runs step s + 1.
    tags = comm.p2p_tags.setdefault("pipefusion", {"in": 0, "out": 0, "last": {}})
    tag_in, tag_out, last = tags["in"], tags["out"], tags["last"]
    row_bytes = H * D * eb
    if tag_out:  # a new call (shapes may differ): everything sent before has been consumed
        comm.wait_ack(nxt, tag_out, stream=st)
    last.clear()
    x = x0.clone() if d == 0 else None
    hloc = torch.empty_like(x0) if d == 0 else None
    pending = []  # stage 0: (step, patch) whose eps is still to come (deferred sampler steps)

    def space(s, m):
        return (s % 2) * slot_bytes + (0 if m is None else B * P[m][0] * row_bytes)

    def recv(shape, s, m):
        nonlocal tag_in
        tag_in += 1
        comm.wait(prev, tag_in, stream=st)
        return comm.mailbox_view(prev, shape, dt, offset=space(s, m)), tag_in

    def send(h, s, m):
        nonlocal tag_out
        par = s % 2
        keys = [k for k in last if k[0] == par] if m is None else [(par, m), (par, None)]
        need = max([last.get(k, 0) for k in keys] + [0])
        if need:
            comm.wait_ack(nxt, need, stream=st)
        tag_out += 1
        last[(par, m)] = tag_out
        comm.put(nxt, h, tag_out, offset=space(s, m), stream=st)

    def blocks(h, off, work):
        for i in range(len(mine)):
            block(h, kv[i], dit.w[i], work, S=S, off=off, stream=st)

    def finish_patch(s, m):  # stage 0: eps of patch m (step s) arrives from the last stage -> sampler
        o, n = P[m]
        eps, t = recv((B, n, H, D), s, m)
        for b in range(B):
            sampler(x[b, o:o + n], eps[b], sigma, stream=st)
        comm.ack(prev, t, stream=st)

    n_max = max(n for _, n in P)
    work = torch.empty(workspace_bytes(B, n_max, H, D, dtype), dtype=torch.uint8, device=dev)
    for s in range(T):
        if s < warmup:  # synchronous over the whole sequence
            if d == 0:
                h = hloc
                h.copy_(x)
            else:
                h, t = recv((B, S, H, D), s, None)
            blocks(h, 0, work_full)
            if N == 1:
                sampler(x, h, sigma, stream=st)
                continue
            send(h, s, None)
            if d > 0:
                comm.ack(prev, t, stream=st)
            else:
                eps, t = recv((B, S, H, D), s, None)
                sampler(x, eps, sigma, stream=st)
                comm.ack(prev, t, stream=st)
            continue
        for m, (o, n) in enumerate(P):
            if d == 0:
                if pending:
                    finish_patch(*pending.pop(0))
                h = hloc[:, :n]
                h = torch.empty((B, n, H, D), dtype=dt, device=dev) if not h.is_contiguous() else h
                h.copy_(x[:, o:o + n])
            else:
                h, t = recv((B, n, H, D), s, m)
            blocks(h, o, work)
            if N == 1:
                for b in range(B):
                    sampler(x[b, o:o + n], h[b], sigma, stream=st)
                continue
            send(h, s, m)
            if d > 0:
                comm.ack(prev, t, stream=st)
        if d == 0 and N > 1:
            pending = [(s, m) for m in range(M)]
    if d == 0:
        while pending:
            finish_patch(*pending.pop(0))
    tags["in"], tags["out"] = tag_in, tag_out
    return x if d == 0 else None
