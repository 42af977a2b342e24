"""Quick numerical probe of the attention stage kernel against the fp64 oracle (debug helper)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2411_01738_b200 import usp
from paper_2411_01738_b200.inputs import qkv

def run(B, H, Sq, Skv, D, seed=1):
    q, _, _ = qkv(B, Sq, H, D, seed=seed)
    _, k, v = qkv(B, Skv, H, D, seed=seed + 1)
    ro, rl = oracle.attention(q.double().numpy(), k.double().numpy(), v.double().numpy())
    o = torch.empty(B, Sq, H, D, dtype=torch.float32, device="cuda")
    l = torch.empty(B, H, Sq, device="cuda")
    usp.attn_fwd(q.cuda(), k.cuda(), v.cuda(), o, l, B=B, H=H, Sq=Sq, Skv=Skv, D=D,
                 q_strides=(Sq*H*D, H*D, D), kv_strides=(Skv*H*D, H*D, D), omap=usp.RowMap.plain(B, Sq, H, D), out_f32=1)
    torch.cuda.synchronize()
    e = np.abs(o.double().cpu().numpy() - ro)
    el = np.abs(l.double().cpu().numpy() - rl)
    print(f"B{B} H{H} Sq{Sq} Skv{Skv} D{D}: O maxerr {e.max():.3e}  LSE maxerr {el.max():.3e}")
    if e.max() > 1e-2:
        per_row = e.max(axis=(0, 2, 3)); per_col = e.max(axis=(0, 1, 2))
        bad_rows = np.nonzero(per_row > 1e-2)[0]
        print("   bad rows:", bad_rows[:10], "...", len(bad_rows), " bad cols:", np.nonzero(per_col > 1e-2)[0][:40])
        print("   lse bad rows:", np.nonzero(el.max(axis=(0,1)) > 1e-3)[0][:10])

for args in [(1,1,256,192,128), (1,1,256,1024,128), (1,4,512,777,128), (2,3,300,333,72)]:
    for _ in range(3): run(*args)
