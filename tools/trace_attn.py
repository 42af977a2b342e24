"""Per-role timeline of the CTA-pair attention kernel (profiling build, -DXDIT_PROFILE).

    python -m paper_2411_01738_b200.build --tag=prof -DXDIT_PROFILE
    XDIT_LIB=paper_2411_01738_b200/libxdit_usp_prof.so python tools/trace_attn.py --S 17776 --H 48 --D 64

One launch; the first CTA pair's clock64 stamps per global key tile g (kernel attn_fwd_2sm.cu,
stamp()) are dumped to a file and summarised: the tile period, each softmax warp's step phases, the
lag of every lane quarter (both CTAs) behind the fastest when it releases P, and the MMA issuer's
waits.  Medians over tiles 8..88 (steady state of the first unit).
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
ap.add_argument("--diag", type=int, default=0)
a = ap.parse_args()
W, IT, EV = 10, 96, 8
path = tempfile.mktemp(suffix=".trace")
os.environ["XDIT_PROFILE_TRACE"] = path
os.environ["XDIT_PROFILE_DIAG"] = str(a.diag)
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
med = lambda xs: statistics.median(xs) if xs else float("nan")  # noqa: E731


def sm(cta, g, ev):  # softmax warp of lane quarter qq handling tile g
    return [raw[cta, qq + 4 * (g & 1), g, ev] for qq in range(4)]


print(f"shape B={a.B} H={a.H} S={a.S} D={a.D} diag={a.diag}")
for cta in (0, 1):
    per = [raw[cta, 0 + 4 * (g & 1), g, 0] - raw[cta, 0 + 4 * ((g - 1) & 1), g - 1, 0] for g in G]
    print(f"cta {cta}: tile period (S ready, quarter 0) median {med(per):.0f} cycles")
    names = ["S wait->ld", "ld->max", "max->m handed", "m->exp half", "exp half->P free", "P free->P released"]
    for qq in range(4):
        ph = []
        for e in range(6):
            xs = []
            for g in G:
                wq = qq + 4 * (g & 1)
                t0, t1 = raw[cta, wq, g, e], raw[cta, wq, g, e + 1]
                if e == 2 and t1 == 0:  # j == 0 (no hand-over wait) never happens in G
                    continue
                xs.append(t1 - t0)
            ph.append(med(xs))
        step = med([raw[cta, qq + 4 * (g & 1), g, 6] - raw[cta, qq + 4 * (g & 1), g, 0] for g in G])
        gap = med([raw[cta, qq + 4 * (g & 1), g, 0] - raw[cta, qq + 4 * (g & 1), g - 2, 6] for g in G])
        print(f"  quarter {qq}: step {step:.0f} (" + ", ".join(f"{n} {x:.0f}" for n, x in zip(names, ph)) +
              f"); idle before S(g) {gap:.0f}")
# lane-quarter lag when releasing P(g), aligned per CTA on the multicast s_full of quarter 0
lag = {}
for cta in (0, 1):
    for qq in range(4):
        lag[(cta, qq)] = med([(raw[cta, qq + 4 * (g & 1), g, 6] - raw[cta, 4 * (g & 1), g, 0]) for g in G])
base = min(lag.values())
print("P(g) released, cycles after S(g) landed (per CTA clock): " +
      "  ".join(f"c{c}q{qq} {lag[(c, qq)]:.0f}" for (c, qq) in sorted(lag)))
# MMA issuer (leader, warp 9)
m = raw[0, 9]
rows = {"K wait": (0, 1), "s_free wait": (1, 2), "QK issue": (2, 3), "->PV": (3, 4), "V wait": (4, 5),
        "p_full wait": (5, 6), "PV issue": (6, 7)}
print("MMA warp per tile: " + ", ".join(f"{n} {med([m[g, b] - m[g, a_] for g in G]):.0f}"
                                        for n, (a_, b) in rows.items()))
print(f"MMA warp loop period {med([m[g, 7] - m[g - 1, 7] for g in G]):.0f}")
# TMA producer: how far ahead of the MMA's K wait it issues
t = raw[0, 8]
print(f"TMA K issued, cycles before the MMA needs it: {med([m[g, 1] - t[g, 0] for g in G]):.0f}")
