"""Softmax step phases of the pair kernel, in execution order (profiling build, -DXDIT_PROFILE).

    XDIT_LIB=paper_2411_01738_b200/libxdit_usp_prof.so python tools/trace_steps.py --S 17776 --H 48 --D 64

Per lane quarter of both CTAs, medians over the first unit's steady-state tiles:
  idle   previous step's P release -> S(g) landed (the warp starved for S)
  ld     S landed -> S in registers (tcgen05.ld x4)
  pre    -> candidate reference ready (s_free arrive, ragged mask, m_c)
  exp1   -> first half of the exp2 stream done
  pvw    -> P buffer free (pv_done of g-2)          [D < 128]
  exp2   -> second half done, overflow check, m_ready(g-1) wait passed
  post   -> P(g) released (reconcile, m publish, P store, p_full arrive)
(D = 128 stores all of P at the end: pvw comes after exp2 there, and is folded into post.)
"""
import argparse
import os
import statistics
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=1)
ap.add_argument("--H", type=int, default=48)
ap.add_argument("--S", type=int, default=17776)
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
G = range(8, min(88, a.S // 128 - 2))
med = lambda xs: statistics.median(xs)  # noqa: E731
if a.D == 128:
    seq = [("ld", 0, 1), ("pre", 1, 2), ("exp1", 2, 4), ("exp2", 4, 3), ("post", 3, 6)]
else:
    seq = [("ld", 0, 1), ("pre", 1, 2), ("exp1", 2, 4), ("pvw", 4, 5), ("exp2", 5, 3), ("post", 3, 6)]
print(f"B={a.B} H={a.H} S={a.S} D={a.D}; cycles, medians over tiles {G.start}..{G.stop - 1}")
print("cta q    idle " + " ".join(f"{n:>6s}" for n, _, _ in seq) + "   step  period")
for cta in (0, 1):
    for qq in range(4):
        w = lambda gg: qq + 4 * (gg & 1)  # noqa: E731
        idle = med([raw[cta, w(gg), gg, 0] - raw[cta, w(gg), gg - 2, 6] for gg in G])
        ph = [med([raw[cta, w(gg), gg, e1] - raw[cta, w(gg), gg, e0] for gg in G]) for _, e0, e1 in seq]
        step = med([raw[cta, w(gg), gg, 6] - raw[cta, w(gg), gg, 0] for gg in G])
        per = med([raw[cta, w(gg), gg, 6] - raw[cta, w(gg - 1), gg - 1, 6] for gg in G])
        print(f"{cta:3d} {qq}  {idle:6.0f} " + " ".join(f"{x:6.0f}" for x in ph) + f" {step:6.0f} {per:6.0f}")
