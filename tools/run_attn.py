"""Drive the attention stage kernel alone (for ncu / compute-sanitizer / quick timing).

    python tools/run_attn.py --B 1 --H 24 --S 66048 --D 128 --iters 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01738_b200 import usp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--H", type=int, default=24)
ap.add_argument("--S", type=int, default=66048)
ap.add_argument("--Skv", type=int, default=0)
ap.add_argument("--D", type=int, default=128)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--out-f32", type=int, default=0)
ap.add_argument("--scratch", type=int, default=1, help="pass the scratch (tail split + dynamic unit hand-out)")
a = ap.parse_args()
Skv = a.Skv or a.S
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(a.B, a.S, a.H, a.D, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(a.B, Skv, a.H, a.D, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(a.B, Skv, a.H, a.D, device="cuda", generator=g).to(torch.bfloat16)
o = torch.empty(q.shape, dtype=torch.float32 if a.out_f32 else torch.bfloat16, device="cuda")
lse = torch.empty(a.B, a.H, a.S, device="cuda")
scratch = torch.empty(usp.attn_scratch_bytes(a.D) // 4, device="cuda") if a.scratch else None
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for it in range(a.iters):
    e0.record()
    usp.attn_fwd(q, k, v, o, lse, B=a.B, H=a.H, Sq=a.S, Skv=Skv, D=a.D,
                 q_strides=(a.S * a.H * a.D, a.H * a.D, a.D), kv_strides=(Skv * a.H * a.D, a.H * a.D, a.D),
                 omap=usp.RowMap.plain(a.B, a.S, a.H, a.D), out_f32=a.out_f32, scratch=scratch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"iter {it}: {ms:.3f} ms  {4*a.B*a.H*a.S*Skv*a.D/ms/1e9:.1f} TFLOP/s", flush=True)
