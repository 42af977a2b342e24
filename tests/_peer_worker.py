"""Worker of tests/test_gpu_peer.py: one process = one SP rank, all ranks on cuda:0.

Each rank joins a gloo process group (host plumbing only: the one-time exchange of the peer
transport's buffer descriptors), builds its local joint shard of seeded global Q, K, V (reading
C4/C5), runs `xdit_usp_attention` through the public binding with the peer-memory transport for
every (ulysses, ring) split of the world, and checks ITS OWN output rows against the fp64 oracle
("the computation yields the same results as the serial version").  Results go to a JSON file
per rank; the test process asserts on them.
"""
import json
import os
import traceback


def _local_index(usp, torch, S_txt, S_img, N, g):
    to, tl, io, il = usp.shard(S_txt, S_img, N, g)
    return torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)])


def run(rank: int, world: int, port: int, splits, cases, out_dir: str):
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        import oracle
        from paper_2411_01738_b200 import usp
        from paper_2411_01738_b200.inputs import qkv
        from tests._util import assert_bf16, assert_f32, errors, f64

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        for (u, r) in splits:
            comm = usp.Comm(u, r, transport="peer")
            assert comm.transport == "peer" and usp.lib().xdit_comm_transport(comm.handle) == 1
            for ci, (B, H, S_txt, S_img, D, dt, keep) in enumerate(cases):
                dtype = torch.float32 if dt == "f32" else torch.bfloat16
                S = S_txt + S_img
                q, k, v = qkv(B, S, H, D, seed=500 + ci, dtype=dtype)
                idx = _local_index(usp, torch, S_txt, S_img, world, rank)
                ql, kl, vl = (t[:, idx].contiguous().cuda() for t in (q, k, v))
                kv_keep = None
                if keep:
                    kv_keep = torch.zeros(2, B, H // u, S, D, dtype=dtype, device="cuda")
                o1, l1 = usp.attention(ql, kl, vl, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r,
                                       kv_keep=kv_keep)
                o2, l2 = usp.attention(ql, kl, vl, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r)
                torch.cuda.synchronize()
                ref_o, ref_l = oracle.attention_rows(f64(q), f64(k), f64(v), idx.numpy())
                e = errors(o1, l1, ref_o, ref_l)
                (assert_f32 if dt == "f32" else assert_bf16)(e)
                # fixed split => bitwise run-to-run determinism (reading C12), also across epochs
                assert torch.equal(o1, o2) and torch.equal(l1, l2), "second call differs"
                if keep:  # SURVEY §8(f) NEXT 1, reading R2: bit-exact vs the oracle's KV buffer
                    ref_kv = oracle.kv_keep(f64(k), f64(v), S_txt, u, r, rank)
                    assert (f64(kv_keep) == ref_kv).all(), "kv_keep differs from oracle.kv_keep"
                res["checks"].append({"u": u, "r": r, "case": ci, **e})
            torch.cuda.synchronize()
            dist.barrier()
            comm.destroy()
            dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
