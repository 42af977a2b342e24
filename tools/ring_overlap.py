"""Ring overlap timeline ("overlapped"): a 1 x r ring split run as r processes through the
public call, rank 0 under torch.profiler (CUPTI): per ring step, the interval of the attention
kernel on the caller's stream and of the NCCL send/recv kernel on the library's side stream, and
how much of the transfer kernel runs under attention.  On the 1-GPU box the ranks share the GPU and
NCCL moves bytes over its socket transport, so the transfer kernels are long -- the timeline shows
the streams' concurrency, not NVLink bandwidth.

    python tools/ring_overlap.py [--ring 2] [--S 16896] [--H 8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world, port, a):
    from tests._mp import setup
    setup(rank, world, port)
    import torch
    import torch.distributed as dist
    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv
    dev = torch.device("cuda", torch.cuda.current_device())
    S_txt, S_img = 512, a.S - 512
    to, tl, io, il = usp.shard(S_txt, S_img, world, rank)
    gq, gk, gv = qkv(1, a.S, a.H, a.D, seed=7, device=dev)
    idx = torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)]).to(dev)
    q, k, v = (t.index_select(1, idx).contiguous() for t in (gq, gk, gv))
    comm = usp.Comm(1, world, group=dist.group.WORLD)
    comm.reserve(1, a.H, S_txt, S_img, a.D, 2)
    out = torch.empty_like(q)
    lse = torch.empty(1, a.H, q.shape[1], device=dev)

    def call():
        usp.attention(q, k, v, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=1, ring=world, out=out, lse=lse)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    dist.barrier()
    if rank != 0:  # every rank takes part in the ring; rank 0 records the timeline
        for _ in range(a.calls):
            call()
        torch.cuda.synchronize()
    if rank == 0:
      try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(a.calls):
                call()
            torch.cuda.synchronize()
        ker = []
        for e in prof.events():
            name = e.name
            if "attn_fwd_2sm" in name or "nccl" in name.lower():
                ker.append((e.time_range.start, e.time_range.end, "attn" if "attn_fwd_2sm" in name else "nccl", name[:60]))
        ker.sort()
        attn = [(s, t) for s, t, kind, _ in ker if kind == "attn"]
        nccl = [(s, t) for s, t, kind, _ in ker if kind == "nccl"]
        rows = []
        for s, t in nccl:
            cover = sum(max(0.0, min(t, t2) - max(s, s2)) for s2, t2 in attn)
            rows.append({"nccl_us": t - s, "under_attention_us": cover, "frac": cover / max(t - s, 1e-9)})
        summary = {"world": world, "S": a.S, "H": a.H, "D": a.D, "calls": a.calls,
                   "attention_kernels": len(attn), "nccl_kernels": len(nccl),
                   "attention_us": [t - s for s, t in attn], "nccl": rows,
                   "note": "ranks share one GPU; NCCL over its socket transport (functional timeline)"}
        with open(a.out, "a") as f:
            f.write(json.dumps(summary) + "\n")
        if a.trace:
            prof.export_chrome_trace(a.trace)
      except Exception:
        import traceback
        with open(a.out, "a") as f:
            f.write(json.dumps({"error": traceback.format_exc()}) + "\n")
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()
    os._exit(0)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--ring", type=int, default=2)
    ap.add_argument("--S", type=int, default=16896)
    ap.add_argument("--H", type=int, default=8)
    ap.add_argument("--D", type=int, default=128)
    ap.add_argument("--calls", type=int, default=2)
    ap.add_argument("--trace", default="")
    ap.add_argument("--out", default="gpurun_out/ring_overlap.jsonl")
    a = ap.parse_args()
    import multiprocessing as mp
    from tests._mp import _port
    ctx = mp.get_context("spawn")
    port = _port()
    ps = [ctx.Process(target=worker, args=(g, a.ring, port, a)) for g in range(a.ring)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(600)
    sys.exit(max(p.exitcode or 0 for p in ps))
