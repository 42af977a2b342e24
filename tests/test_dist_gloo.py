"""Multi-process (gloo, CPU) tests of the N>1 host logic.

Each process is one SP rank.  It asks libxdit_usp.so for its plan (xdit_usp_plan -- the same
geometry xdit_usp_attention executes), checks the plans of all ranks agree with each other, and then
runs the USP data flow for real across processes: Ulysses all-to-all over the row group (gloo
all_to_all_single), r-1 ring send/recv steps to the plan's ring neighbours, the LSE merge in the
plan's order, the reverse all-to-all -- with the fp64 oracle as the per-block attention.  The result
on every rank must equal the serial oracle on that rank's tokens ("the computation yields the same
results as the serial version", §4.1.1).  No GPU is needed: this exercises the mesh, shard,
ring-order and merge logic of the multi-GPU path.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


PLAN_FIELDS = ["i", "j", "Hh", "S_loc", "Lmax", "S_blk", "ring_next", "ring_prev", "nseg"]


def worker(rank, world, port, u, r, B, H, S_txt, S_img, D, q, k, v, ref_o, ref_l, errq):
    try:
        import sys
        sys.path.insert(0, ROOT)
        import oracle
        from paper_2411_01738_b200 import usp
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        N = u * r
        P = usp.plan(B, H, S_txt, S_img, D, u, r, rank)
        i, j, Hh = P.i, P.j, P.Hh
        assert (i, j) == (rank // u, rank % u)  # reading C6: g = i*u + j
        # ---- all plans agree with each other
        mine = torch.tensor([getattr(P, f) for f in PLAN_FIELDS] + list(P.seg_off) + list(P.ring_src) +
                            list(P.ring_rows), dtype=torch.int64)
        allp = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(allp, mine)
        nf = len(PLAN_FIELDS)
        S_loc = [int(x[3]) for x in allp]
        seg = allp[rank][nf:nf + 9].tolist()
        assert seg[:u + 1] == [sum(S_loc[i * u:i * u + p]) for p in range(u + 1)]
        assert P.Lmax == max(S_loc) and P.S_blk == sum(S_loc[i * u:(i + 1) * u])
        for s in range(r - 1):  # what ring index i sends at step s is what i+1 uses at step s+1
            nxt = allp[((i + 1) % r) * u + j]
            assert int(nxt[nf + 9 + s + 1]) == P.ring_src[s] and int(nxt[nf + 17 + s + 1]) == P.ring_rows[s]
        # ---- the data flow, across processes
        to, tl, io, il = usp.shard(S_txt, S_img, N, rank)
        loc = np.concatenate([np.arange(to, to + tl), S_txt + np.arange(io, io + il)])
        L, Lmax = P.S_loc, P.Lmax
        row_groups = [dist.new_group([ii * u + p for p in range(u)]) for ii in range(r)]
        # a2-a4: Ulysses all-to-all of Q, K, V: send head block p (padded to Lmax rows) to peer p
        x = np.zeros((u, 3, B, Lmax, Hh, D))
        for t, src in enumerate((q, k, v)):
            for p in range(u):
                x[p, t, :, :L] = src[:, loc][:, :, p * Hh:(p + 1) * Hh]
        y = torch.empty(x.shape, dtype=torch.float64)
        if u > 1:
            dist.all_to_all_single(y, torch.from_numpy(x), group=row_groups[i])
        else:
            y = torch.from_numpy(x)
        y = y.numpy()
        lens = [S_loc[i * u + p] for p in range(u)]
        blk = [np.concatenate([y[p, t, :, :lens[p]] for p in range(u)], axis=1) for t in range(3)]
        # a5-a7: ring; KV travels to ring_next, arrives from ring_prev; merge in step order (C9)
        qb, kb, vb = blk
        acc_o = acc_l = None
        for s in range(r):
            assert kb.shape[1] == P.ring_rows[s]
            o_s, l_s = oracle.attention(qb, kb, vb)
            if s == 0:
                acc_o, acc_l = o_s, l_s
            else:
                M = np.maximum(acc_l, l_s)
                Lse = M + np.log(np.exp(acc_l - M) + np.exp(l_s - M))
                wa = np.exp(acc_l - Lse).transpose(0, 2, 1)[..., None]
                ws = np.exp(l_s - Lse).transpose(0, 2, 1)[..., None]
                acc_o, acc_l = wa * acc_o + ws * o_s, Lse
            if s < r - 1:
                nxt_rank, prv_rank = P.ring_next * u + j, P.ring_prev * u + j
                send = torch.from_numpy(np.ascontiguousarray(np.stack([kb, vb])))
                rows_next = P.ring_rows[s + 1]
                recv = torch.empty((2, B, rows_next, Hh, D), dtype=torch.float64)
                reqs = [dist.isend(send, nxt_rank), dist.irecv(recv, prv_rank)]
                for rq in reqs:
                    rq.wait()
                kb, vb = recv[0].numpy(), recv[1].numpy()
        # a8-a10: reverse all-to-all: rows of Ulysses peer p's shard go back to peer p
        ob = np.zeros((u, B, Lmax, Hh, D))
        lb = np.zeros((u, B, Hh, Lmax))
        for p in range(u):
            ob[p, :, :lens[p]] = acc_o[:, seg[p]:seg[p + 1]]
            lb[p, :, :, :lens[p]] = acc_l[:, :, seg[p]:seg[p + 1]]
        packed = torch.from_numpy(np.concatenate([ob.reshape(u, -1), lb.reshape(u, -1)], axis=1).copy())
        got = torch.empty_like(packed)
        if u > 1:
            dist.all_to_all_single(got, packed, group=row_groups[i])
        else:
            got = packed
        got = got.numpy()
        no = B * Lmax * Hh * D
        out = np.concatenate([got[p, :no].reshape(B, Lmax, Hh, D)[:, :L] for p in range(u)], axis=2)
        lse = np.concatenate([got[p, no:].reshape(B, Hh, Lmax)[:, :, :L] for p in range(u)], axis=1)
        np.testing.assert_allclose(out, ref_o[:, loc], rtol=0, atol=1e-12)
        np.testing.assert_allclose(lse, ref_l[:, :, loc], rtol=0, atol=1e-12)
        dist.barrier()
        dist.destroy_process_group()
    except BaseException as e:  # report to the parent
        import traceback
        errq.put(f"rank {rank}: {e!r}\n{traceback.format_exc()}")
        raise


@pytest.mark.parametrize("u,r", [(2, 1), (1, 2), (2, 2), (4, 1), (1, 4)])
def test_gloo_usp_dataflow(u, r):
    import oracle
    B, H, S_txt, S_img, D = 2, 4, 7, 61, 8
    rng = np.random.default_rng(u * 10 + r)
    q, k, v = (rng.standard_normal((B, S_txt + S_img, H, D)) for _ in range(3))
    ref_o, ref_l = oracle.attention(q, k, v)
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    world = u * r
    port = free_port()
    procs = [ctx.Process(target=worker, args=(rk, world, port, u, r, B, H, S_txt, S_img, D, q, k, v, ref_o, ref_l,
                                               errq)) for rk in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    assert not errs, "\n".join(errs)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
