"""A/B: K/V in the caller's token-major layout [B][S][H][D] vs head-major [B][H][S][D] for the attention
kernel at one shape (CUDA events, interleaved repetitions)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01738_b200 import usp
ap = argparse.ArgumentParser(); ap.add_argument("--S", type=int, default=66048); ap.add_argument("--H", type=int, default=24)
ap.add_argument("--D", type=int, default=128); ap.add_argument("--iters", type=int, default=10); ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args(); B, S, H, D = 1, a.S, a.H, a.D
q = torch.randn(B, S, H, D, device="cuda").bfloat16()
k = torch.randn(B, S, H, D, device="cuda").bfloat16(); v = torch.randn(B, S, H, D, device="cuda").bfloat16()
kh, vh = k.transpose(1, 2).contiguous(), v.transpose(1, 2).contiguous()
o = torch.empty_like(q); lse = torch.empty(B, H, S, device="cuda")
scr = torch.empty(usp.attn_scratch_bytes(D) // 4, device="cuda")
m = usp.RowMap.plain(B, S, H, D)
def go(head_major):
    kk, vv = (kh, vh) if head_major else (k, v)
    kvs = (H * S * D, D, S * D) if head_major else (S * H * D, H * D, D)
    usp.attn_fwd(q, kk, vv, o, lse, B=B, H=H, Sq=S, Skv=S, D=D, q_strides=(S * H * D, H * D, D), kv_strides=kvs, omap=m, scratch=scr)
ref = None
for hm in (0, 1):
    go(hm); torch.cuda.synchronize()
    if ref is None: ref = o.clone()
    else: print("max diff between layouts:", (o.float() - ref.float()).abs().max().item())
for rep in range(a.reps):
    for hm in (0, 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters): go(hm)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        print(f"{'head-major ' if hm else 'token-major'} S={S} D={D}: {ms:.3f} ms  {4*B*H*S*S*D/ms/1e9:.1f} TFLOP/s", flush=True)
