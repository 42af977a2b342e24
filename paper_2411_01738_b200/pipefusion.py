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
