"""Single-GPU model of one rank of an N-GPU USP call (no NVLink here): rank 0's device work for
each (ulysses, ring) split of a workload -- Q/K/V pack + unpack around the all-to-all, the attention
of every ring step (stage kernel xdit_attn_fwd on the rank's real block shapes), the ring LSE merges
(UNFUSED stage kernel: an upper bound, the product fuses them into the epilogue) and the output
unpack -- timed with CUDA events, plus T(1) of the whole problem on this GPU.  Projection:
T(N) = compute + Ulysses bytes / BW (not overlapped) + ring steps' excess over their
attention (overlapped); efficiency = T(1) / (N T(N)) at BW = 900 GB/s (NVLink 5 per
direction) and a derated 600 GB/s.

    python tools/rank_model.py [--config flux] [--N 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2411_01738_b200 import usp  # noqa: E402
from paper_2411_01738_b200.inputs import WORKLOADS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="flux")
ap.add_argument("--N", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
w = WORKLOADS[a.config]
B, H, D = w.B * w.cfg, w.H, w.D
dev = torch.device("cuda")
scratch = torch.empty(usp.attn_scratch_bytes(D) // 4, dtype=torch.float32, device=dev)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def attn(q, k, v, o, l, Hh, Sq, Skv, out_f32=0):
    usp.attn_fwd(q, k, v, o, l, B=B, H=Hh, Sq=Sq, Skv=Skv, D=D, q_strides=(Sq * Hh * D, Hh * D, D),
                 kv_strides=(Skv * Hh * D, Hh * D, D), omap=usp.RowMap.plain(B, Sq, Hh, D), out_f32=out_f32,
                 scratch=scratch)


# T(1): the whole problem on one GPU
S = w.S
q1, k1, v1 = (torch.randn(B, S, H, D, device=dev).to(torch.bfloat16) for _ in range(3))
o1, l1 = torch.empty_like(q1), torch.empty(B, H, S, device=dev)
t1 = timed(lambda: attn(q1, k1, v1, o1, l1, H, S, S), a.reps)
del q1, k1, v1, o1, l1
flops = 4.0 * B * H * S * S * D
print(json.dumps({"config": w.name, "N": 1, "t_ms": t1, "tflops": flops / t1 / 1e9}), flush=True)
for N in a.N:
    for u in [d for d in range(1, N + 1) if N % d == 0 and H % d == 0]:
        r = N // u
        P = usp.plan(B, H, w.S_txt, w.S_img, D, u, r, 0)
        Hh, Sb, L, Lmax = P.Hh, P.S_blk, P.S_loc, P.Lmax
        x = [torch.randn(B, L, H, D, device=dev).to(torch.bfloat16) for _ in range(3)]
        send = torch.empty((u, 3, B, Lmax, Hh, D), dtype=torch.bfloat16, device=dev)
        blk = [torch.randn(B, Sb, Hh, D, device=dev).to(torch.bfloat16) for _ in range(3)]
        kvs = [(torch.randn(B, P.ring_rows[s], Hh, D, device=dev).to(torch.bfloat16),
                torch.randn(B, P.ring_rows[s], Hh, D, device=dev).to(torch.bfloat16)) for s in range(r)]
        acc_o = torch.empty(B, Sb, Hh, D, device=dev)
        acc_l = torch.empty(B, Hh, Sb, device=dev)
        tmp_o, tmp_l = torch.empty_like(acc_o), torch.empty_like(acc_l)
        o_bf = torch.empty(B, Sb, Hh, D, dtype=torch.bfloat16, device=dev)
        out = torch.empty(B, L, H, D, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(B, H, L, device=dev)
        lens = [sum(usp.shard(w.S_txt, w.S_img, N, p)[1::2]) for p in range(u)]  # ring block 0's ranks

        def pack():
            if u > 1:
                for t in range(3):
                    usp.uly_pack(x[t], send, B=B, L=L, Lmax=Lmax, H=H, D=D, u=u, slot=t, nslots=3, elem_bytes=2)
                for t in range(3):
                    usp.uly_unpack(send, blk[t], B=B, Lmax=Lmax, Hh=Hh, D=D, u=u, lens=lens, slot=t, nslots=3,
                                   elem_bytes=2)

        def ring():
            for s in range(r):
                k, v = (blk[1], blk[2]) if s == 0 else kvs[s]
                if r == 1:
                    attn(blk[0], k, v, o_bf, acc_l, Hh, Sb, P.ring_rows[s])
                elif s == 0:
                    attn(blk[0], k, v, acc_o, acc_l, Hh, Sb, P.ring_rows[s], out_f32=1)
                else:
                    attn(blk[0], k, v, tmp_o, tmp_l, Hh, Sb, P.ring_rows[s], out_f32=1)
                    usp.lse_merge(acc_o, acc_l, tmp_o, tmp_l, B=B, S=Sb, Hh=Hh, D=D)

        def unpack_out():
            if u > 1:
                oc = send.numel() * 2 // (3 * u)
                usp.uly_unpack_out(send.data_ptr(), send.data_ptr(), oc, oc, out, lse, B=B, L=L, Lmax=Lmax, Hh=Hh,
                                   D=D, u=u, elem_bytes=2)

        t_pack = timed(pack, a.reps) if u > 1 else 0.0
        t_ring = timed(ring, a.reps)
        t_attn_steps = [timed(lambda s=s: attn(blk[0], *((blk[1], blk[2]) if s == 0 else kvs[s]),
                                               tmp_o, tmp_l, Hh, Sb, P.ring_rows[s], out_f32=1), a.reps)
                        for s in range(r)]
        t_unp = timed(unpack_out, a.reps) if u > 1 else 0.0
        X = B * L * H * D * 2
        uly_bytes = (4 * (u - 1) / u) * X + ((u - 1) / u) * B * L * H * 4
        ring_step_bytes = [2 * B * P.ring_rows[s] * Hh * D * 2 for s in range(r)]
        comp = t_pack + t_ring + t_unp
        res = {"config": w.name, "N": N, "u": u, "r": r, "Hh": Hh, "S_blk": Sb, "compute_ms": comp,
               "pack_unpack_ms": t_pack + t_unp, "ring_ms": t_ring, "attn_step_ms": t_attn_steps,
               "uly_bytes": int(uly_bytes), "ring_bytes_per_step": ring_step_bytes[0]}
        for bw in (900.0, 600.0):
            exposed = uly_bytes / (bw * 1e9) * 1e3
            ring_excess = sum(max(0.0, ring_step_bytes[s] / (bw * 1e9) * 1e3 - t_attn_steps[s]) for s in range(r - 1))
            tN = comp + exposed + ring_excess
            res[f"proj_eff_{int(bw)}GBps"] = t1 / (N * tN)
        res["compute_only_eff"] = t1 / (N * comp)
        print(json.dumps(res), flush=True)
        del x, send, blk, kvs, acc_o, acc_l, tmp_o, tmp_l, o_bf, out, lse
        torch.cuda.empty_cache()
