#!/usr/bin/env python
"""bench.py -- USP attention throughput on B200 (xDiT arXiv 2411.01738 hot path).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config flux] [--ulysses u --ring r]
    python bench.py --impl reference ...      # the fp64 CPU oracle on the host cores (baseline arm)

A "step" is one USP attention call (pack -> all-to-all -> ring of tcgen05
attention + LSE merge -> reverse all-to-all) over one batch of synthetic Q/K/V of the workload.
N=1 default workload: Flux.1 4096px (B=1, H=24, D=128, 512 text + 65536 image tokens), the shape
BASELINE.json's north_star targets.

Multi-GPU: one process per GPU.  `--gpus N` with N > 1 started without torchrun re-launches itself
under torch.distributed.run (N local ranks, 127.0.0.1); under torchrun WORLD_SIZE must equal
--gpus.  The ranks form an NCCL process group; the library splits its communicator (Ulysses rows,
Ring columns) and moves every USP byte over NCCL.  The same global problem is split over the N ranks
(strong scaling), CFG groups first when the workload has them.  T(1) -- the same whole-job problem
on one GPU -- is measured in the same job by rank 0, so the line carries the parallel efficiency
T(1) / (N T(N)).  Rank 0 prints ONE JSON line.  `--share-gpu` runs N ranks on cuda:0 (each rank a
distinct NCCL host id, socket transport): a functional check of the N > 1 path on a 1-GPU box whose
timings are not scaling numbers.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "USP attention TFLOP/s & ms/layer at 1/2/4/8 B200; % of bf16 tensor peak"
UNIT = "TFLOP/s"
DATASHEET_BF16_TFLOPS = 2250.0
NVLINK_GBPS_PER_DIR = 900.0
L2_BYTES = 126 * 1024 * 1024


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="flux")
    ap.add_argument("--ulysses", type=int, default=0)
    ap.add_argument("--ring", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--share-gpu", action="store_true",
                    help="N > 1 ranks on cuda:0 (functional check on a 1-GPU box; not a scaling number)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-t1", action="store_true", help="N > 1: skip the same-job T(1) measurement")
    ap.add_argument("--no-graph", action="store_true",
                    help="N > 1: time eager calls instead of replaying the step captured in a CUDA graph")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU time of the oracle sample")
    return ap.parse_args(argv)


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


def split_for(args, w):
    cfg, u, r = default_split(args.gpus, w.H, w.cfg)
    if args.ulysses or args.ring:
        u = args.ulysses or max(1, args.gpus // cfg // max(1, args.ring))
        r = args.ring or max(1, args.gpus // cfg // u)
    return cfg, u, r


def ours_config(args, w):
    """The `config` object both arms print for the same launch (the reference arm prints it too, so
    the two lines name one workload)."""
    cfg, u, r = split_for(args, w)
    sp = u * r
    B = w.B * w.cfg // cfg
    L = w.S // sp + (1 if w.S % sp else 0)
    flush = 4 * B * L * w.H * w.D * 2 < 2 * L2_BYTES
    return {"workload": w.name, "B": w.B * w.cfg, "H": w.H, "D": w.D, "S_txt": w.S_txt, "S_img": w.S_img,
            "cfg": cfg, "ulysses": u, "ring": r, "data_plane": "nccl" if args.gpus > 1 else None,
            "l2": "flushed between steps" if flush else "inputs larger than L2"}


def comm_summary(pl, B: int, w, u: int, r: int, ms: float):
    """Algorithmic bytes this rank sends per call (Table 1): the Ulysses
    Q,K,V exchange and the O (+LSE) return to the u-1 peers, and r-1 ring steps of K,V; and the time
    they take at NVLink 5's 900 GB/s per direction -- the share of the call a perfectly overlapped
    data plane would need (the Ulysses part is not overlapped)."""
    if u * r == 1:
        return None
    a2a = (u - 1) * pl.a2a_bytes_per_peer  # Q, K, V to the u-1 peers
    o_ret = (u - 1) * (B * pl.Lmax * pl.Hh * w.D * 2 + B * pl.Hh * pl.Lmax * 4) if u > 1 else 0
    ring = sum(pl.ring_bytes[s] for s in range(r))
    tot = a2a + o_ret + ring
    return {"bytes_per_rank": int(tot), "ulysses_bytes": int(a2a + o_ret), "ring_bytes": int(ring),
            "ms_at_900GBps": tot / (NVLINK_GBPS_PER_DIR * 1e9) * 1e3,
            "share_of_call_at_900GBps": tot / (NVLINK_GBPS_PER_DIR * 1e9) * 1e3 / ms}


def phase_summary(phs):
    """Per-phase times (max over ranks) and the achieved NVLink-direction bandwidth of each exchange:
    the bytes a rank sends in the phase / the phase's time, against 900 GB/s per direction."""
    if not phs or any(p is None for p in phs):
        return None
    r = len(phs[0]["attn_ms"])
    mx = lambda key: max(p[key] for p in phs)  # noqa: E731
    out = {"ranks": len(phs), "total_ms": mx("total_ms"), "a2a_in_ms": mx("a2a_in_ms"),
           "a2a_out_ms": mx("a2a_out_ms"),
           "attn_ms": [max(p["attn_ms"][s] for p in phs) for s in range(r)],
           "ring_comm_ms": [max(p["ring_comm_ms"][s] for p in phs) for s in range(r - 1)]}

    def gbps(b, ms):
        return b / (ms * 1e-3) / 1e9 if ms > 0 else None
    p0 = phs[0]
    bw = {}
    if p0["a2a_in_bytes"]:
        g = gbps(p0["a2a_in_bytes"], out["a2a_in_ms"])
        bw["a2a_in"] = {"bytes_per_rank": p0["a2a_in_bytes"], "GBps": g, "frac_of_900": g / NVLINK_GBPS_PER_DIR,
                        "note": "phase time includes the pack and unpack kernels"}
    if p0["a2a_out_bytes"]:
        g = gbps(p0["a2a_out_bytes"], out["a2a_out_ms"])
        bw["a2a_out"] = {"bytes_per_rank": p0["a2a_out_bytes"], "GBps": g, "frac_of_900": g / NVLINK_GBPS_PER_DIR,
                         "note": "phase time includes the unpack kernels"}
    if r > 1:
        rb, rt = sum(p0["ring_bytes"]), sum(out["ring_comm_ms"])
        g = gbps(rb, rt)
        bw["ring"] = {"bytes_per_rank": rb, "GBps": g, "frac_of_900": g / NVLINK_GBPS_PER_DIR,
                      "hidden_under_attention": rt <= sum(out["attn_ms"]),
                      "note": "side-stream send/recv time, overlapped with the attention kernel (P:356)"}
    out["bandwidth"] = bw
    return out


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


def clock_ceilings(D: int, sm_mhz, n_sm: int, achieved: float):
    """The kernel's two unit ceilings at the clock the run actually held ("report the
    exp-limited ceiling beside the achieved fraction"): the tensor pipe (8192 dense bf16 FLOP per clock
    per SM) and the MUFU (16 ex2 per clock per SM; one exp2 per 4D FLOPs, the FMA-pipe offload of
    attn_fwd_2sm.cu -- 1 pair in 16 at D = 128, 1 in 8 below -- taken off it).  DESIGN.md 7.1b."""
    if not sm_mhz:
        return None
    hz = float(sm_mhz) * 1e6
    f_fma = 1.0 / 16 if D == 128 else 1.0 / 8
    tensor = 8192.0 * n_sm * hz / 1e12
    mufu = 16.0 * n_sm * hz * 4 * D / (1.0 - f_fma) / 1e12
    binding = "mufu" if mufu < tensor else "tensor"
    return {"sm_mhz": sm_mhz, "tensor_tflops_at_clock": tensor, "mufu_exp2_tflops_at_clock": mufu,
            "exp2_on_fma_pipe": f_fma, "binding": binding,
            "frac_of_binding": achieved / min(tensor, mufu)}


# ------------------------------------------------------------------------------------ CPU oracle
def cpu_baseline_leg(w, seconds: float, q_rows, k_heads, v_heads, rows_desc: str, got=None):
    """The cpu_baseline leg: the fp64 oracle, as it stands, on the host cores, on a bounded sample of
    the workload -- query rows x heads of the benched inputs (q_rows [B, n, h, D], k/v_heads
    [B, S, h, D], host tensors) -- sized to ~`seconds` of CPU time.  Timed on the sample and scaled to
    TFLOP/s.  When `got` = (O [B, n, h, D], LSE [B, h, n]) of the benched GPU call on the same rows x
    heads is given, the same oracle rows are the parity check of the benched run (§8(d) result
    record).  Returns (cpu_baseline dict, parity dict or None)."""
    import numpy as np
    import oracle
    f = lambda t: t.to("cpu").double().numpy()  # noqa: E731
    K, V = f(k_heads), f(v_heads)
    Qall = f(q_rows)
    B, n_all, h, D = Qall.shape
    S = K.shape[1]
    cores = oracle.default_threads()
    per_row = 4.0 * S * D * h * B
    n = min(n_all, max(cores, 8))
    while True:  # calibrate: grow the sample until it costs >= 1/4 of the target
        t0 = time.perf_counter()
        oracle.attention(Qall[:, :n], K, V)
        dt = time.perf_counter() - t0
        if dt >= seconds / 4 or n >= n_all:
            break
        n = min(n_all, int(n * max(2.0, (seconds / 4) / max(dt, 1e-3))))
    n = min(n_all, max(n, int(n * seconds / max(dt, 1e-3))))
    t0 = time.perf_counter()
    ref_o, ref_l = oracle.attention(Qall[:, :n], K, V)
    dt = time.perf_counter() - t0
    cpu = {"value": n * per_row / dt / 1e12, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{n} query rows x {h} heads x B={B} of {w.name} (S={S}, D={D}; {rows_desc}) in fp64, "
                     f"{dt:.1f}s on the host cores; rate scaled to TFLOP/s"}
    par = None
    if got is not None:
        go, gl = f(got[0])[:, :n], f(got[1])[:, :, :n]
        d = go - ref_o
        par = {"err_O_maxabs": float(np.abs(d).max()),
               "err_O_relL2": float(np.linalg.norm(d) / np.linalg.norm(ref_o)),
               "err_LSE_maxabs": float(np.abs(gl - ref_l).max()),
               "oracle_rows_checked": int(n * h * B),
               "gates": {"O_maxabs": 2e-2, "LSE_maxabs": 1e-3, "O_relL2_internal": 1e-2, "LSE_internal": 1e-4}}
        par["pass"] = bool(par["err_O_maxabs"] <= 2e-2 and par["err_LSE_maxabs"] <= 1e-3 and
                           par["err_O_relL2"] <= 1e-2)
    return cpu, par


def run_reference(args, w, rank: int):
    """The baseline arm for this tier: the fp64 oracle as it stands, on the host cores (rank 0 only),
    each step a bounded row sample of the workload; ms_per_step is extrapolated from the sample."""
    if rank != 0:
        return 0
    import torch
    from paper_2411_01738_b200.inputs import qkv, seed_for
    flops_step = w.flops()
    rates, desc = [], None
    per_step = max(2.0, args.cpu_seconds / max(1, args.steps))
    gen_S = w.S
    gq, gk, gv = qkv(1, gen_S, 1, w.D, seed=seed_for(w, 0))  # one (batch, head) of the global problem
    rows = torch.linspace(0, gen_S - 1, min(gen_S, 4096)).long()
    for it in range(args.warmup + args.steps):
        cpu, _ = cpu_baseline_leg(w, per_step if it >= args.warmup else 1.0, gq[:, rows], gk, gv,
                                  "one (b, h) slice, strided rows")
        if it >= args.warmup:
            rates.append(cpu["value"])
            desc = cpu
    tflops = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": flops_step / (tflops * 1e12) * 1e3,
        "extrapolated": True, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": ours_config(args, w),
        "cpu_baseline": {**desc, "value": tflops},
        "e2e": {"value": tflops, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------ launch
def relaunch_under_torchrun(args, argv):
    """`--gpus N` (N > 1) without torchrun: one process per GPU via torch.distributed.run."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    from paper_2411_01738_b200.inputs import WORKLOADS
    w = WORKLOADS[args.config]
    env_world = os.environ.get("WORLD_SIZE")
    if args.gpus > 1 and env_world is None:
        return relaunch_under_torchrun(args, argv)
    world = int(env_world or "1")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch one process per GPU")
    if args.impl == "reference":
        return run_reference(args, w, rank)

    import torch
    import torch.distributed as dist

    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv, seed_for

    N = world
    if N > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # NCCL init lines on stderr: ranks, devices,
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")   # bus ids, transports (the driver can check N)
        if args.share_gpu:
            os.environ["NCCL_HOSTID"] = f"xdit-bench-rank-{rank}"
            os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
            local = 0
        elif torch.cuda.device_count() < N:
            raise SystemExit(f"bench.py: --gpus {N} needs {N} GPUs, this node has {torch.cuda.device_count()} "
                             "(--share-gpu runs a functional check on one)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if N > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg, u, r = split_for(args, w)
    assert cfg * u * r == N, f"cfg*u*r = {cfg}*{u}*{r} != N={N}"
    sp = u * r
    cfg_group, sp_rank = rank // sp, rank % sp
    group = None
    if N > 1:
        groups = [dist.new_group(list(range(c * sp, (c + 1) * sp))) for c in range(cfg)]
        group = groups[cfg_group]
    # batch handled by this CFG group: CFG splits the 2-latent batch
    B = w.B * w.cfg // cfg
    comm = usp.Comm(u, r, group=group if sp > 1 else None)
    comm.reserve(B, w.H, w.S_txt, w.S_img, w.D, 2)
    to, tl, io, il = usp.shard(w.S_txt, w.S_img, sp, sp_rank)
    L = tl + il
    # global Q,K,V of this CFG group, seeded, generated on the device; keep this rank's shard
    gq, gk, gv = qkv(B, w.S, w.H, w.D, seed=seed_for(w, cfg_group), device=dev)
    idx = torch.cat([torch.arange(to, to + tl), w.S_txt + torch.arange(io, io + il)]).to(dev)
    q, k, v = (t.index_select(1, idx).contiguous() for t in (gq, gk, gv))
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
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather_obj(o):
        if N == 1:
            return [o]
        allo = [None] * N
        dist.all_gather_object(allo, o)
        return allo

    working_set = 4 * q.numel() * q.element_size()
    flush = working_set < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def timed(fn, steps):
        """Mean ms of `steps` calls of fn on the device (CUDA events on the caller's stream, max over
        ranks): back to back when the inputs exceed L2, else one call at a time after an L2 flush."""
        if not flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            barrier()
            e0.record(stream)
            for _ in range(steps):
                fn()
            e1.record(stream)
            barrier()
            return e0.elapsed_time(e1) / steps
        tot = 0.0
        for _ in range(steps):
            scratch.fill_(1.0)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            barrier()
            tot += e0.elapsed_time(e1)
        return tot / steps

    for _ in range(args.warmup):
        step()
    barrier()
    # N > 1: the step (a dozen kernels and NCCL operations per call) is captured once in a CUDA graph
    # and replayed, so host enqueue cost does not pace the short multi-rank calls.  Falls back to
    # eager calls if capture fails.
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
    g = None  # only `graph` references the captured graph (teardown order, below)
    n_captured = usp.launch_count()
    timed_step = graph.replay if graph is not None else step
    n0 = usp.launch_count()
    with ClockSampler(local) as clocks:
        ms = timed(timed_step, args.steps)
    launches = (usp.launch_count() - n0) // args.steps
    if graph is not None:  # replays launch the captured kernels without passing through the library:
        launches = n_captured - n_pre  # the library's launches recorded into the graph (one call)
    ms = max_over_ranks(ms)
    flops = w.flops()  # whole job (all CFG groups)
    tflops = flops / (ms * 1e-3) / 1e12

    # ---- per-phase events of the same calls (eager, profiled): the dominant kernel's time (the
    #      attention launches of each ring step on the caller's stream) and the exchanges' bandwidth
    comm.profile(True)
    prof = []
    for _ in range(max(3, min(args.steps, 10))):
        if flush:
            scratch.fill_(1.0)
        barrier()
        step()
        prof.append(comm.phases())
    comm.profile(False)
    attn_ms = statistics.mean(sum(p["attn_ms"]) for p in prof)
    phs = gather_obj(prof[-1])
    phases = phase_summary(phs) if N > 1 else None
    pl = usp.plan(B, w.H, w.S_txt, w.S_img, w.D, u, r, sp_rank)
    kern_flops = sum(4.0 * B * pl.Hh * pl.S_blk * pl.ring_rows[s] * w.D for s in range(r))
    kern_ms = prof_kern_ms = max_over_ranks(attn_ms)
    kern_timing = ("per-phase CUDA events of profiled calls after the timed region (xdit_comm_profile): the "
                   "attention launches of every ring step on the caller's stream, mean over the calls")
    if N == 1:
        # at N = 1 a step is the attention kernel itself (plus the 4-byte reset of its unit counter):
        # the dominant kernel's duration is the timed region's own per-step device time
        kern_ms = ms
        kern_timing = ("CUDA events on the launching stream around the timed steps; at N = 1 a step is one "
                       "attention launch (+ a 4-byte cudaMemsetAsync of its unit counter)")

    # ---- parity of the benched run + the cpu_baseline leg (rank 0: a sample of ITS rows / heads)
    cpu, parity = None, None
    if rank == 0 and not args.no_cpu_baseline:
        rows_loc = torch.linspace(0, L - 1, min(L, 2048)).long()
        hs = sorted({0, w.H // 2, w.H - 1})
        hsel = torch.tensor(hs, device=dev)
        q_rows = q[:, rows_loc.to(dev)].index_select(2, hsel)
        got = (out[:, rows_loc.to(dev)].index_select(2, hsel), lse[:, :, rows_loc.to(dev)].index_select(1, hsel))
        cpu, parity = cpu_baseline_leg(w, args.cpu_seconds if N == 1 else min(args.cpu_seconds, 5.0), q_rows,
                                       gk.index_select(2, hsel), gv.index_select(2, hsel),
                                       f"rank 0's rows, heads {hs}", got=got)
        if N > 1:
            cpu = None  # the CPU baseline is reported at N = 1 only; the parity check stays
    del gq, gk, gv

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

    # ---- T(1): the same whole-job problem (every CFG group's batch) on ONE GPU, in this job (rank 0)
    t1 = None
    if N > 1 and not args.no_t1:
        barrier()
        if rank == 0:
            Bt = w.B * w.cfg
            parts = [qkv(w.B * w.cfg // cfg, w.S, w.H, w.D, seed=seed_for(w, c), device=dev) for c in range(cfg)]
            q1, k1, v1 = (torch.cat([p[t] for p in parts], dim=0) for t in range(3))
            del parts
            o1 = torch.empty_like(q1)
            l1 = torch.empty((Bt, w.H, w.S), dtype=torch.float32, device=dev)
            big = 4 * q1.numel() * q1.element_size() >= 2 * L2_BYTES
            with usp.Comm(1, 1) as c1:
                def step1():
                    usp.attention(q1, k1, v1, S_txt=w.S_txt, S_img=w.S_img, comm=c1, out=o1, lse=l1)
                for _ in range(args.warmup):
                    step1()
                n1 = max(2, min(args.steps, 5))
                tot = 0.0
                for _ in range(1 if big else n1):  # inputs > L2: back to back; else flush + one call
                    if not big:
                        scratch.fill_(1.0)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                    for _ in range(n1 if big else 1):
                        step1()
                    e1.record(stream)
                    torch.cuda.synchronize()
                    tot += e0.elapsed_time(e1)
                t1 = tot / n1
            del q1, k1, v1, o1, l1
        barrier()

    peak, peak_sus, peak_src = peaks()
    ranks = gather_obj({"rank": rank, "device": local, "pci_bus_id": torch.cuda.get_device_properties(dev).pci_bus_id
                        if hasattr(torch.cuda.get_device_properties(dev), "pci_bus_id") else None,
                        "name": torch.cuda.get_device_name(dev), "comm": comm.source})
    if rank == 0:
        kern_tflops = kern_flops / (kern_ms * 1e-3) / 1e12
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                traffic = json.load(f).get(f"{w.name}:{B}x{pl.Hh}x{pl.S_blk}x{w.D}")
        except Exception:
            pass
        share = args.share_gpu and N > 1
        line = {
            "metric": METRIC, "value": tflops, "unit": UNIT, "n_gpus": N, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {**ours_config(args, w), **({"shared_gpu": True} if share else {})},
            "cuda_graph": graph is not None,
            **({"cuda_graph_note": graph_note} if graph_note else {}),
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
            "parity": parity,
            "roofline": {"bound": "tensor", "kernel": "attn_fwd_2sm_kernel", "achieved": kern_tflops,
                         "peak": peak, "unit": "TFLOP/s", "frac": kern_tflops / peak, "traffic": traffic,
                         "peak_source": f"{peak_src} bf16 burst (MEASURED_PEAKS.json bf16_tflops)",
                         "frac_of_sustained": kern_tflops / peak_sus,
                         "frac_of_datasheet": kern_tflops / DATASHEET_BF16_TFLOPS,
                         "kernel_ms": kern_ms, "kernel_flops": kern_flops,
                         "timing": kern_timing, "profiled_kernel_ms": prof_kern_ms,
                         "shape": f"B={B} H={pl.Hh} Sq={pl.S_blk} Skv={[pl.ring_rows[s] for s in range(r)]} D={w.D}"},
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        line["roofline"]["ceilings"] = clock_ceilings(w.D, line["clocks"].get("sm_mhz"),
                                                      torch.cuda.get_device_properties(dev).multi_processor_count,
                                                      kern_tflops)
        if N > 1:
            line["comm"] = comm_summary(pl, B, w, u, r, ms)
            line["phases"] = phases
            line["t1_ms"] = t1
            line["parallel_efficiency"] = (t1 / (N * ms)) if t1 else None
            line["ranks"] = ranks
            line["nccl_version"] = ".".join(str(x) for x in torch.cuda.nccl.version())
        print(json.dumps(line), flush=True)
    # teardown: the captured graph holds NCCL operations of the library's communicators, so it goes
    # before them (destroying a communicator a live graph still references can block), then the
    # library's communicators, then torch's process group
    del graph, timed_step
    torch.cuda.synchronize()
    if N > 1:
        dist.barrier()
    comm.destroy()
    if N > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
