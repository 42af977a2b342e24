"""Per-item overhead of the attention kernel: the same total work (B*H*n_qt = 2368 items = 32 waves
of 74 CTA pairs, equal bytes) at S = 1024 ... 16384, so time = waves * (tiles_per_item * t + c);
a least-squares fit gives the per-tile time t and the per-item overhead c (prologue, pipeline fill,
epilogue, CTA launch).

    python tools/sweep_items.py [--D 72] [--iters 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01738_b200 import usp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--D", type=int, nargs="+", default=[64, 72, 128])
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--items", type=int, default=2368)
a = ap.parse_args()
for D in a.D:
    pts = []
    for S in (1024, 2048, 4096, 8192, 16384):
        n_qt = S // 256
        H = a.items // n_qt
        g = torch.Generator(device="cuda").manual_seed(0)
        q, k, v = (torch.randn(1, S, H, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
        o = torch.empty_like(q)
        lse = torch.empty(1, H, S, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def call():
            usp.attn_fwd(q, k, v, o, lse, B=1, H=H, Sq=S, Skv=S, D=D, q_strides=(S * H * D, H * D, D),
                         kv_strides=(S * H * D, H * D, D), omap=usp.RowMap.plain(1, S, H, D), out_f32=0)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        tf = 4.0 * H * S * S * D / ms / 1e9
        waves = a.items / 74.0
        us_item = ms * 1e3 / waves
        pts.append((S // 128, us_item))
        print(f"D={D} S={S:6d} H={H:5d}: {ms:.3f} ms  {tf:7.1f} TFLOP/s  {us_item:8.2f} us/item "
              f"({S // 128} tiles)", flush=True)
        del q, k, v, o, lse
    n = len(pts)
    sx = sum(x for x, _ in pts); sy = sum(y for _, y in pts)
    sxx = sum(x * x for x, _ in pts); sxy = sum(x * y for x, y in pts)
    t = (n * sxy - sx * sy) / (n * sxx - sx * sx)
    c = (sy - t * sx) / n
    print(f"D={D}: fit per-tile {t:.3f} us, per-item overhead {c:.2f} us (= {c / t:.1f} tiles)", flush=True)
