"""Unit-boundary timeline of the persistent pair kernel (profiling build, -DXDIT_PROFILE).

    XDIT_LIB=paper_2411_01738_b200/libxdit_usp_prof.so python tools/trace_boundary.py --S 4429 --H 24 --D 64

Prints, per global key tile g of the first CTA pair, when S(g) landed and P(g) was released (the
slowest lane quarter, leader clock), and the MMA issuer's QK^T / P.V issue stamps, so the cycles a
unit boundary costs (epilogue, first tiles' max pass) can be read off around g = n_kv, 2 n_kv, ...
"""
import argparse
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--H", type=int, default=24)
ap.add_argument("--S", type=int, default=4429)
ap.add_argument("--D", type=int, default=64)
a = ap.parse_args()
W, IT, EV = 10, 96, 8
path = tempfile.mktemp(suffix=".trace")
os.environ["XDIT_PROFILE_TRACE"] = path
import torch  # noqa: E402

from paper_2411_01738_b200 import usp  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(a.B, a.S, a.H, a.D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
o = torch.empty_like(q)
lse = torch.empty(a.B, a.H, a.S, device="cuda")
for _ in range(2):
    usp.attn_fwd(q, k, v, o, lse, B=a.B, H=a.H, Sq=a.S, Skv=a.S, D=a.D, q_strides=(a.S * a.H * a.D, a.H * a.D, a.D),
                 kv_strides=(a.S * a.H * a.D, a.H * a.D, a.D), omap=usp.RowMap.plain(a.B, a.S, a.H, a.D))
torch.cuda.synchronize()
raw = np.fromfile(path, dtype=np.uint64).reshape(-1, 2, W, IT, EV)[-1].astype(np.int64)
os.unlink(path)
n_kv = (a.S + 127) // 128
t0 = raw[0, 0, 0, 0]
print(f"n_kv = {n_kv} tiles per unit; times in leader cycles from S(0) landed")
print("   g  S_land(max q)  P_rel(max q)  dP   step(max)  QKiss  PVwait_done  PViss")
prev = None
for gg in range(min(IT, 3 * n_kv + 4)):
    c = gg & 1
    s_land = max(raw[cta, qq + 4 * c, gg, 0] for cta in (0,) for qq in range(4)) - t0
    p_rel = max(raw[0, qq + 4 * c, gg, 6] for qq in range(4)) - t0
    step = max(raw[0, qq + 4 * c, gg, 6] - raw[0, qq + 4 * c, gg, 0] for qq in range(4))
    qk = raw[0, 9, gg, 3] - t0
    pvw = raw[0, 9, gg, 6] - t0
    pv = raw[0, 9, gg, 7] - t0
    d = p_rel - prev if prev is not None else 0
    mark = "  <- unit start" if gg % n_kv == 0 else ""
    print(f"{gg:4d} {s_land:12d} {p_rel:12d} {d:6d} {step:9d} {qk:8d} {pvw:10d} {pv:8d}{mark}")
    prev = p_rel
print("\nepilogue of each unit (the warp that did not run the unit's last tile; max over lane quarters, leader clock):")
print("  unit  P_rel(last)  barriers  o_full  O_ld  o_empty  stores_done  next S_land")
for u in range(1, 3):
    gl = u * n_kv - 1
    if gl + 1 >= IT:
        break
    cp = 1 - (gl & 1)
    ev = lambda e: max(raw[0, qq + 4 * cp, gl, e] for qq in range(4)) - t0  # noqa: E731
    p_rel = max(raw[0, qq + 4 * (gl & 1), gl, 6] for qq in range(4)) - t0
    nxt = max(raw[0, qq + 4 * ((gl + 1) & 1), gl + 1, 0] for qq in range(4)) - t0
    print(f"  {u - 1:4d} {p_rel:11d} {ev(0):9d} {ev(1):7d} {ev(2):5d} {ev(3):8d} {ev(5):12d} {nxt:12d}")
