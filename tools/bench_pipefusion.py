"""Measure the PipeFusion patch step on a BASELINE-shaped latent.

    python tools/bench_pipefusion.py [--config flux] [--M 4] [--L 4] [--stages 1] [--steps 3]

Times (CUDA events on the launching streams, after warm-up):
  * one xdit_pf_block on one patch (n = S/M query rows against the whole S-row KV buffer) --
    attention FLOPs 4*B*H*n*S*D per call, the step's dominant kernel, reported against the measured
    bf16 peak like bench.py's roofline;
  * a full pipelined diffusion step of an L-block synthetic DiT (paper_2411_01738_b200.pipefusion.run
    with warmup=1, T=2, minus the warm-up step) -- attention FLOPs L*4*B*H*S^2*D per step.
Prints one JSON line.  Synthetic seeded inputs (inputs.qkv recipe), random per-channel weights.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2411_01738_b200 import pipefusion as pf  # noqa: E402
from paper_2411_01738_b200.inputs import WORKLOADS, qkv, seed_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="flux")
ap.add_argument("--M", type=int, default=4)
ap.add_argument("--L", type=int, default=4)
ap.add_argument("--stages", type=int, default=1)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
w = WORKLOADS[a.config]
B, S, H, D = w.B, w.S, w.H, w.D
x0 = qkv(B, S, H, D, seed=seed_for(w), device="cuda")[0]
gen = torch.Generator(device="cuda").manual_seed(7)
W = [[torch.empty(H, D, device="cuda").uniform_(0.2, 0.4, generator=gen) for _ in range(2)] +
     [torch.empty(H, D, device="cuda").uniform_(0.5, 1.5, generator=gen),
      torch.empty(H, D, device="cuda").uniform_(0.4, 0.8, generator=gen)] for _ in range(a.L)]
dit = pf.SyntheticDiT(W)
P = pf.patch_bounds(w.S_txt, w.S_img, a.M)

# ---- one block on one patch (the largest, patch 0 with the text)
o, n = P[0]
kv = torch.empty((2, B, H, S, D), dtype=torch.bfloat16, device="cuda").normal_()
h = x0[:, o:o + n].contiguous()
work = torch.empty(pf.workspace_bytes(B, n, H, D, 0), dtype=torch.uint8, device="cuda")
for _ in range(3):
    pf.block(h, kv, dit.w[0], work, S=S, off=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    pf.block(h, kv, dit.w[0], work, S=S, off=o)
e1.record()
torch.cuda.synchronize()
blk_ms = e0.elapsed_time(e1) / a.iters
blk_flops = 4.0 * B * H * n * S * D
del kv, h, work

# ---- whole pipelined steps: run(T=2) - run(T=1) isolates one pipelined step (same warm-up step)
def timed(T):
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    pf.run(x0, dit, T=T, M=a.M, warmup=1, sigma=0.3, S_txt=w.S_txt, stages=a.stages)
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1)

timed(2)
t1 = min(timed(1) for _ in range(2))
t2 = min(timed(2) for _ in range(2))
step_ms = t2 - t1
step_flops = a.L * 4.0 * B * H * S * S * D
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
    peak = float(json.load(f)["bf16_tflops"])
line = {
    "what": "PipeFusion patch step (SURVEY 8(f) NEXT 3) on a synthetic DiT stack",
    "config": {"workload": w.name, "B": B, "H": H, "D": D, "S": S, "M": a.M, "L": a.L, "stages": a.stages,
               "patch0_rows": n},
    "block": {"ms": blk_ms, "tflops": blk_flops / blk_ms / 1e9, "frac_of_measured_bf16_peak": blk_flops / blk_ms / 1e9 / peak,
              "flops": blk_flops, "shape": f"Sq={n} Skv={S} (KV buffer head-major)"},
    "pipelined_step": {"ms": step_ms, "tflops": step_flops / step_ms / 1e9,
                       "frac_of_measured_bf16_peak": step_flops / step_ms / 1e9 / peak},
    "peak_tflops": peak,
}
print(json.dumps(line), flush=True)
