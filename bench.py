#!/usr/bin/env python
"""bench.py -- USP attention throughput on B200 (xDiT arXiv 2411.01738 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config flux] [--ulysses u --ring r]
    python bench.py --impl reference ...      # the fp64 CPU oracle on the host cores (baseline arm)

A "step" is one USP attention call (pack -> all-to-all -> ring of tcgen05
attention + LSE merge -> reverse all-to-all) over one batch of synthetic Q/K/V of the workload.
N=1 default workload: Flux.1 4096px (B=1, H=24, D=128, 512 text + 65536 image tokens), the shape
BASELINE.json's north_star targets.  Multi-GPU: one process per GPU under
torchrun (torch.distributed/NCCL for the barrier and the max over ranks); the library moves the USP
bytes itself (peer-memory transport, or NCCL with --transport nccl); the same global problem is
split over N ranks (strong scaling), CFG groups when the workload has them.  Rank 0 prints ONE JSON
line.  XDIT_SHARE_GPU=1 puts every rank on cuda:0 with a gloo process group -- a functional check of
the N > 1 path on a 1-GPU box (its timings are not scaling numbers).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "USP attention TFLOP/s & ms/layer at 1/2/4/8 B200; % of bf16 tensor peak"
UNIT = "TFLOP/s"
DATASHEET_BF16_TFLOPS = 2250.0
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="flux")
    ap.add_argument("--ulysses", type=int, default=0)
    ap.add_argument("--ring", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--transport", default="peer", choices=["peer", "nccl"],
                    help="multi-rank byte movement: the library's peer-memory transport or NCCL")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="N > 1: time eager calls instead of replaying the step captured in a CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    return ap.parse_args()


def attn_kernel_name(D: int) -> str:
    """The bf16 attention kernel the library dispatches for head dim D (attn_fwd_sm100.cu)."""
    if D in (64, 72, 128) and os.environ.get("XDIT_ATTN_KERNEL") != "1sm":
        return "attn_fwd_2sm_kernel"
    return "attn_fwd_sm100_kernel"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", p["bf16_tflops"])), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


def default_split(N: int, H: int, cfg: int):
    """cfg first ("when using CFG, CFG parallelism must be used"), then Ulysses-heavy on
    NVLink, the remainder on the ring."""
    c = cfg if N % cfg == 0 and N >= cfg else 1
    sp = N // c
    u = max(d for d in range(1, sp + 1) if sp % d == 0 and H % d == 0)
    return c, u, sp // u


# ------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """Samples SM clock and throttle reasons via NVML while the timed region runs."""

    def __init__(self, dev_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self._ok = True
        except Exception:
            pass
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": getattr(nv, "nvmlClocksEventReasonGpuIdle", 0x1),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self._ok:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------ CPU oracle
def oracle_sample(w, seconds: float, rank_seed: int = 0):
    """Time the fp64 oracle (as it stands) on a bounded row sample of workload `w` on the host cores.
    Returns (flops_per_second, cores, description)."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(rank_seed)
    S, D = w.S, w.D
    # one (b, h) slice of the global problem: K, V of all S keys, a strided sample of query rows
    k = rng.standard_normal((1, S, 1, D))
    v = rng.standard_normal((1, S, 1, D))
    q = rng.standard_normal((1, S, 1, D))
    cores = oracle.default_threads()
    per_row = 4.0 * S * D
    n = max(cores, 8)
    while True:  # calibrate: grow the sample until it costs >= 1/4 of the target
        rows = np.linspace(0, S - 1, n).astype(np.int64)
        t0 = time.perf_counter()
        oracle.attention_rows(q, k, v, rows)
        dt = time.perf_counter() - t0
        if dt >= seconds / 4 or n >= S:
            break
        n = min(S, int(n * max(2.0, (seconds / 4) / max(dt, 1e-3))))
    # final timed run at the target size
    n = min(S, max(n, int(n * seconds / max(dt, 1e-3))))
    rows = np.linspace(0, S - 1, n).astype(np.int64)
    t0 = time.perf_counter()
    oracle.attention_rows(q, k, v, rows)
    dt = time.perf_counter() - t0
    desc = (f"{n} query rows x 1 (batch, head) of {w.name} (S={S}, D={D}) in fp64, "
            f"{dt:.1f}s; rate scaled to the full 4*B*H*S^2*D workload")
    return n * per_row / dt, cores, desc, dt


def ours_config(args, w):
    """The `config` object our arm prints for the same launch (so both lines name one workload)."""
    N = args.gpus
    cfg, u, r = default_split(N, w.H, w.cfg)
    if args.ulysses or args.ring:
        u = args.ulysses or max(1, N // cfg // max(1, args.ring))
        r = args.ring or max(1, N // cfg // u)
    sp = u * r
    B = w.B * w.cfg // cfg
    L = w.S // sp + (1 if w.S % sp else 0)
    flush = 4 * B * L * w.H * w.D * 2 < 2 * L2_BYTES
    return {"workload": w.name, "B": w.B * w.cfg, "H": w.H, "D": w.D, "S_txt": w.S_txt, "S_img": w.S_img,
            "cfg": cfg, "ulysses": u, "ring": r, "transport": args.transport if sp > 1 else None,
            "l2": "flushed between steps" if flush else "inputs larger than L2"}


def comm_summary(pl, B: int, w, u: int, r: int, ms: float):
    """Algorithmic bytes this rank sends per call (Table 1): the Ulysses
    Q,K,V exchange and the O (+LSE) return to the u-1 peers, and r-1 ring steps of K,V; and the time
    they take at NVLink 5's 900 GB/s per direction -- the share of the call a perfectly overlapped
    transport would need (the Ulysses part is not overlapped)."""
    if u * r == 1:
        return None
    a2a = (u - 1) * pl.a2a_bytes_per_peer  # Q, K, V to the u-1 peers
    o_ret = (u - 1) * (B * pl.Lmax * pl.Hh * w.D * 2 + B * pl.Hh * pl.Lmax * 4) if u > 1 else 0
    ring = sum(pl.ring_bytes[s] for s in range(r))
    tot = a2a + o_ret + ring
    return {"bytes_per_rank": int(tot), "ulysses_bytes": int(a2a + o_ret), "ring_bytes": int(ring),
            "ms_at_900GBps": tot / 900e9 * 1e3, "share_of_call_at_900GBps": tot / 900e9 * 1e3 / ms}


def run_reference(args, w, rank: int):
    if rank != 0:
        return 0
    flops_step = w.flops()
    rates = []
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps))
    for it in range(args.warmup + args.steps):
        rate, cores, desc, dt = oracle_sample(w, per_step if it >= args.warmup else 1.0, rank_seed=it)
        if it >= args.warmup:
            rates.append(rate)
    rate = statistics.median(rates)
    tflops = rate / 1e12
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": flops_step / rate * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": ours_config(args, w),
        "cpu_baseline": {"value": tflops, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": tflops, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    from paper_2411_01738_b200.inputs import WORKLOADS
    w = WORKLOADS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import torch
    import torch.distributed as dist
    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv, seed_for

    N = world
    share = os.environ.get("XDIT_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg, u, r = default_split(N, w.H, w.cfg)
    if args.ulysses or args.ring:
        u = args.ulysses or max(1, N // cfg // max(1, args.ring))
        r = args.ring or max(1, N // cfg // u)
    assert cfg * u * r == N, f"cfg*u*r = {cfg}*{u}*{r} != N={N}"
    sp = u * r
    cfg_group, sp_rank = rank // sp, rank % sp
    group = None
    if N > 1:
        groups = [dist.new_group(list(range(c * sp, (c + 1) * sp))) for c in range(cfg)]
        group = groups[cfg_group]
    # batch handled by this CFG group: CFG splits the 2-latent batch
    B = w.B * w.cfg // cfg
    comm = usp.Comm(u, r, group=group if sp > 1 else None, transport=args.transport)
    comm.reserve(B, w.H, w.S_txt, w.S_img, w.D, 2)
    to, tl, io, il = usp.shard(w.S_txt, w.S_img, sp, sp_rank)
    L = tl + il
    # global Q,K,V of this CFG group, seeded, generated on the device; keep this rank's shard
    gq, gk, gv = qkv(B, w.S, w.H, w.D, seed=seed_for(w, cfg_group), device=dev)
    idx = torch.cat([torch.arange(to, to + tl), w.S_txt + torch.arange(io, io + il)]).to(dev)
    q, k, v = (t.index_select(1, idx).contiguous() for t in (gq, gk, gv))
    del gq, gk, gv
    out = torch.empty_like(q)
    lse = torch.empty((B, w.H, L), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        usp.attention(q, k, v, S_txt=w.S_txt, S_img=w.S_img, comm=comm, ulysses=u, ring=r, out=out, lse=lse)

    def barrier():
        if N > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if N == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    working_set = 4 * q.numel() * q.element_size()
    flush = working_set < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    for _ in range(args.warmup):
        step()
    barrier()
    # N > 1: the step (a dozen kernels and stream flag operations per call) is captured once in a
    # CUDA graph and replayed -- the peer transport's binary flags make replays valid -- so host
    # enqueue cost does not pace the short multi-rank calls.  Falls back to eager calls if capture fails.
    graph, graph_note = None, None
    n_pre = usp.launch_count()
    if N > 1 and not args.no_graph:
        try:
            cs = torch.cuda.Stream(device=dev)
            cs.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(cs):
                with torch.cuda.graph(g, stream=cs):
                    step()
            torch.cuda.synchronize()
            g.replay()  # one untimed replay
            barrier()
            graph = g
        except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
            graph_note = f"capture failed, eager: {type(ex).__name__}: {ex}"[:200]
            torch.cuda.synchronize()
            barrier()
    n_captured = usp.launch_count()
    timed_step = graph.replay if graph is not None else step
    n0 = usp.launch_count()
    with ClockSampler(local) as clocks:
        if not flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(args.steps):
                timed_step()
            e1.record(stream)
            barrier()
            ms = e0.elapsed_time(e1) / args.steps
        else:  # small working set: flush L2 between steps, time each step on its own
            tot = 0.0
            for _ in range(args.steps):
                scratch.fill_(1.0)
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                timed_step()
                e1.record(stream)
                barrier()
                tot += e0.elapsed_time(e1)
            ms = tot / args.steps
    launches = (usp.launch_count() - n0) // args.steps
    if graph is not None:  # replays launch the captured kernels without passing through the library:
        launches = n_captured - n_pre  # the library's launches recorded into the graph (one call)

    ms = max_over_ranks(ms)
    flops = w.flops()  # whole job (all CFG groups)
    tflops = flops / (ms * 1e-3) / 1e12

    # ---- dominant kernel alone: the tcgen05 attention kernel on this rank's ring-block shapes,
    #      timed with events on the launching stream over K launches (roofline numerator)
    pl = usp.plan(B, w.H, w.S_txt, w.S_img, w.D, u, r, sp_rank)
    Hh, Sb = pl.Hh, pl.S_blk
    kq = torch.empty((B, Sb, Hh, w.D), dtype=torch.bfloat16, device=dev).normal_()
    kk, kv_ = torch.empty_like(kq).normal_(), torch.empty_like(kq).normal_()
    ko = torch.empty_like(kq)
    kl = torch.empty((B, Hh, Sb), dtype=torch.float32, device=dev)
    kmap = usp.RowMap.plain(B, Sb, Hh, w.D)
    kscr = torch.empty(usp.attn_scratch_bytes(w.D) // 4, dtype=torch.float32, device=dev)

    def kern():  # same launch configuration as inside the USP call (tail split enabled)
        usp.attn_fwd(kq, kk, kv_, ko, kl, B=B, H=Hh, Sq=Sb, Skv=Sb, D=w.D,
                     q_strides=(Sb * Hh * w.D, Hh * w.D, w.D), kv_strides=(Sb * Hh * w.D, Hh * w.D, w.D),
                     omap=kmap, scratch=kscr)
    for _ in range(2):
        kern()
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(stream)
    for _ in range(args.steps):
        kern()
    k1.record(stream)
    torch.cuda.synchronize()
    kern_ms = max_over_ranks(k0.elapsed_time(k1) / args.steps)
    kern_flops = 4.0 * B * Hh * Sb * Sb * w.D
    del kq, kk, kv_, ko, kl

    # ---- end to end through the public API with host buffers (pinned), copies inside the region
    hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
    hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()
    hlse = torch.empty(lse.shape, dtype=lse.dtype).pin_memory()

    def e2e_step():
        dq, dk, dv = (t.to(dev, non_blocking=True) for t in (hq, hk, hv))
        o2, l2 = usp.attention(dq, dk, dv, S_txt=w.S_txt, S_img=w.S_img, comm=comm, ulysses=u, ring=r)
        hout.copy_(o2, non_blocking=True)
        hlse.copy_(l2, non_blocking=True)
    e2e_steps = max(1, min(args.steps, 5))
    e2e_step()
    barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    f1.record(stream)
    barrier()
    e2e_serial_ms = max_over_ranks(f0.elapsed_time(f1) / e2e_steps)

    # Streamed: the same per-step work (H2D of the step's Q,K,V, the USP call, D2H of O and LSE) with
    # the H2D of step i+1 and the D2H of step i-1 on copy streams overlapping step i's attention
    # (double-buffered device inputs / outputs) -- how a caller feeding a sequence of layers or
    # requests from host memory would drive the API.  Every copy is inside the timed region.
    cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    din = [[torch.empty_like(t, device=dev) for t in (hq, hk, hv)] for _ in range(2)]
    dout = [(torch.empty_like(out), torch.empty_like(lse)) for _ in range(2)]
    ev = {key: [torch.cuda.Event() for _ in range(2)] for key in ("in", "comp", "out")}

    def e2e_streamed(n, start_ev):
        cin.wait_event(start_ev)
        with torch.cuda.stream(cin):
            for dst, src in zip(din[0], (hq, hk, hv)):
                dst.copy_(src, non_blocking=True)
            ev["in"][0].record(cin)
        for i in range(n):
            b = i & 1
            if i + 1 < n:  # prefetch the next step's inputs into the other buffer (free after step i-1)
                if i >= 1:
                    cin.wait_event(ev["comp"][1 - b])
                with torch.cuda.stream(cin):
                    for dst, src in zip(din[1 - b], (hq, hk, hv)):
                        dst.copy_(src, non_blocking=True)
                    ev["in"][1 - b].record(cin)
            stream.wait_event(ev["in"][b])
            if i >= 2:
                stream.wait_event(ev["out"][b])  # output buffer b drained to host by step i-2's copy
            usp.attention(*din[b], S_txt=w.S_txt, S_img=w.S_img, comm=comm, ulysses=u, ring=r,
                          out=dout[b][0], lse=dout[b][1])
            ev["comp"][b].record(stream)
            cout.wait_event(ev["comp"][b])
            with torch.cuda.stream(cout):
                hout.copy_(dout[b][0], non_blocking=True)
                hlse.copy_(dout[b][1], non_blocking=True)
                ev["out"][b].record(cout)
        stream.wait_event(ev["out"][(n - 1) & 1])

    g0 = torch.cuda.Event()
    g0.record(stream)
    e2e_streamed(2, g0)  # warm-up
    torch.cuda.synchronize()
    barrier()
    # steady state of the copy/compute pipeline: the first step's H2D and the last D2H are not
    # hidden, so they are amortised over 16 steps (all copies stay inside the timed region)
    n_stream = 16
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    e2e_streamed(n_stream, f0)
    f1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(f0.elapsed_time(f1) / n_stream)
    del din, dout
    h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv))
    d2h = hout.numel() * hout.element_size() + hlse.numel() * hlse.element_size()

    peak, peak_sus, peak_src = peaks()
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and N == 1:
            rate, cores, desc, _ = oracle_sample(w, args.cpu_seconds)
            cpu = {"value": rate / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc}
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tj = json.load(f)
            key = f"{w.name}:{B}x{Hh}x{Sb}x{w.D}"
            traffic = tj.get(key)
        except Exception:
            pass
        kern_tflops = kern_flops / (kern_ms * 1e-3) / 1e12
        line = {
            "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": w.name, "B": w.B * w.cfg, "H": w.H, "D": w.D, "S_txt": w.S_txt,
                       "S_img": w.S_img, "cfg": cfg, "ulysses": u, "ring": r,
                       "transport": comm.transport if sp > 1 else None,
                       "cuda_graph": graph is not None,
                       **({"cuda_graph_note": graph_note} if graph_note else {}),
                       **({"shared_gpu": True} if share and N > 1 else {}),
                       "l2": "flushed between steps" if flush else "inputs larger than L2"},
            "ms_per_layer": ms,
            "tflops_per_gpu": tflops / N,
            "pct_of_bf16_peak_measured": 100.0 * tflops / N / peak,
            "pct_of_bf16_peak_datasheet": 100.0 * tflops / N / DATASHEET_BF16_TFLOPS,
            "e2e": {"value": flops / (e2e_ms * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "api": "paper_2411_01738_b200.attention (pinned host -> device, result -> host)",
                    "mode": "streamed: H2D of step i+1 and D2H of step i-1 on copy streams overlap step i",
                    "steps": n_stream,
                    "serial": {"value": flops / (e2e_serial_ms * 1e-3) / 1e12, "ms_per_step": e2e_serial_ms,
                               "mode": "H2D, call, D2H back to back on one stream"}},
            "gpu_launches": int(launches),
            "comm": comm_summary(pl, B, w, u, r, ms),
            "roofline": {"bound": "tensor", "kernel": attn_kernel_name(w.D), "achieved": kern_tflops,
                         "peak": peak, "unit": "TFLOP/s", "frac": kern_tflops / peak, "traffic": traffic,
                         "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                         "frac_of_sustained": kern_tflops / peak_sus,
                         "kernel_ms": kern_ms, "kernel_flops": kern_flops,
                         "shape": f"B={B} H={Hh} Sq=Skv={Sb} D={w.D}"},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    torch.cuda.synchronize()
    if N > 1:  # peers may still map this rank's buffers: everyone drained before anyone frees
        dist.barrier()
    comm.destroy()
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
