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


def run_pipefusion(rank: int, world: int, port: int, cases, out_dir: str):
    """One PipeFusion stage per process (paper_2411_01738_b200.pipefusion.run_stage) over the peer
    transport's mailbox; stage 0 checks the final latent against the fp64 staleness oracle and,
    bitwise, against the in-process N-stage schedule (pipefusion.run)."""
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import numpy as np
        import torch
        import torch.distributed as dist

        from oracle import pipefusion as opf
        from paper_2411_01738_b200 import pipefusion as pf
        from paper_2411_01738_b200 import usp
        from paper_2411_01738_b200.inputs import qkv

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        comm = usp.Comm(world, 1, transport="peer")
        for ci, (B, S_txt, S_img, H, D, L, T, M, warmup, dt) in enumerate(cases):
            dtype = torch.float32 if dt == "f32" else torch.bfloat16
            x0 = qkv(B, S_txt + S_img, H, D, seed=40 + ci, dtype=dtype)[0]
            rng = np.random.default_rng(40 + ci)
            W = [tuple(rng.uniform(0.2, 0.4, (H, D)).astype(np.float32) for _ in range(2)) +
                 (rng.uniform(0.5, 1.5, (H, D)).astype(np.float32), rng.uniform(0.4, 0.8, (H, D)).astype(np.float32))
                 for _ in range(L)]
            kw = dict(T=T, M=M, warmup=warmup, sigma=0.5, S_txt=S_txt)
            x = pf.run_stage(x0.cuda(), W, comm, **kw)
            torch.cuda.synchronize()
            if rank == 0:
                same = pf.run(x0.cuda(), pf.SyntheticDiT(W), stages=world, **kw)
                torch.cuda.synchronize()
                assert torch.equal(x, same), "multi-process stages differ from the in-process schedule"
                W64 = [tuple(w.astype(np.float64) for w in wl) for wl in W]
                want, _ = opf.pipefusion(x0.double().numpy(), W64, **kw)
                got = x.double().cpu().numpy()
                if dt == "f32":
                    err = float(np.abs(got - want).max() / np.abs(want).max())
                    assert err <= 1e-3, err
                else:
                    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
                    assert err <= 2e-2, err
                res["checks"].append({"case": ci, "err": err})
            dist.barrier()
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


def run_cfg_tail(rank: int, world: int, port: int, cases, out_dir: str):
    """CFG step tail over the peer transport (NEXT 2): rank 0 = conditional, rank 1 = unconditional
    branch; every rank's combined eps against oracle.cfg_combine (exact at g = 0, 1)."""
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import numpy as np
        import torch
        import torch.distributed as dist

        import oracle
        from paper_2411_01738_b200 import usp

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        comm = usp.Comm(2, 1, transport="peer")
        comm.mailbox(max(n for n, _, _ in cases) * 4)
        for ci, (n, dt, g) in enumerate(cases):
            dtype = torch.float32 if dt == "f32" else torch.bfloat16
            gen = torch.Generator().manual_seed(70 + ci)
            both = torch.randn(2, n, generator=gen).to(dtype)
            out = usp.cfg_tail(both[rank].cuda(), g, comm=comm)
            out2 = usp.cfg_tail(both[rank].cuda(), g, comm=comm)  # second call: the ack protocol
            torch.cuda.synchronize()
            c, u = both[0].double().numpy(), both[1].double().numpy()
            ref = oracle.cfg_combine(c, u, g)
            got = out.double().cpu().numpy()
            # same bound as tests/test_gpu_cfg.py: fp32 cancellation (+ one bf16 RNE rounding)
            bound = (abs(g) * np.abs(c) + abs(1 - g) * np.abs(u)) * 2.0 ** -22 + (np.abs(ref) * 2.0 ** -8 if dt == "bf16" else 0)
            assert np.all(np.abs(got - ref) <= bound + 1e-30)
            assert torch.equal(out, out2)
            if g in (0.0, 1.0):
                assert torch.equal(out.cpu(), both[1 if g == 0.0 else 0]), "combine not exact at g in {0, 1}"
            res["checks"].append({"case": ci})
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


def run_vae(rank: int, world: int, port: int, cases, out_dir: str):
    """Patch-parallel VAE decode, one process per row band (paper_2411_01738_b200.vae.decode_band):
    each band equals the same rows of the one-device GPU decode bit for bit and of the fp64 oracle."""
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import numpy as np
        import torch
        import torch.distributed as dist

        from oracle import vae as ovae
        from paper_2411_01738_b200 import usp, vae

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        comm = usp.Comm(world, 1, transport="peer")
        for ci, (h, c, w, widths, tc) in enumerate(cases):
            rng = np.random.default_rng(80 + ci)
            lat = rng.standard_normal((h, c, w)).astype(np.float32)
            L, cin = [], c
            for co in list(widths) + [3]:
                L.append(((rng.standard_normal((co, cin, 3, 3)) / np.sqrt(9 * cin)).astype(np.float32),
                          (rng.standard_normal(co) * 0.1).astype(np.float32)))
                cin = co
            dec = vae.Decoder(L, tc=tc)
            o, n = vae.bands(h, world)[rank]
            x0 = dec.prepare(torch.from_numpy(lat).cuda())
            mine = vae.decode_band(x0[o:o + n].contiguous(), dec, comm)
            whole = vae.decode(x0, dec)
            torch.cuda.synchronize()
            up = 2 ** len(widths)
            assert torch.equal(mine, whole[o * up:(o + n) * up]), "band differs from the one-device decode"
            want = ovae.serial_decode(lat, [(a.astype(np.float64), b.astype(np.float64)) for a, b in L])
            want = want[o * up:(o + n) * up]
            if tc:  # bf16 [H][W][C'] -> [H][C][W]
                got = mine[:, :, :3].permute(0, 2, 1).double().cpu().numpy()
                err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
                assert err <= 2e-2, err
            else:
                err = float(np.abs(mine.cpu().double().numpy() - want).max() / np.abs(want).max())
                assert err <= 1e-5, err
            res["checks"].append({"case": ci, "err": err, "band_rows": int(mine.shape[0])})
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


def run_graph(rank: int, world: int, port: int, cases, out_dir: str):
    """The peer-transport USP call captured in a CUDA graph and replayed, interleaved with eager
    calls: every replay equals the eager result bit for bit (binary set/reset flags carry constant
    values, so the captured stream operations stay valid; include/xdit_usp.h)."""
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist

        from paper_2411_01738_b200 import usp
        from paper_2411_01738_b200.inputs import qkv

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        for (u, r) in cases:
            comm = usp.Comm(u, r, transport="peer")
            S_txt, S_img, H, D = 7, 300, 8, 64
            q, k, v = qkv(1, S_txt + S_img, H, D, seed=11 + u)
            to, tl, io, il = usp.shard(S_txt, S_img, world, rank)
            idx = torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)])
            ql, kl, vl = (t[:, idx].contiguous().cuda() for t in (q, k, v))
            kw = dict(S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r)
            ref_o, ref_l = usp.attention(ql, kl, vl, **kw)  # eager (reserve + connect happen here)
            torch.cuda.synchronize()
            out = torch.empty_like(ref_o)
            lse = torch.empty_like(ref_l)
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    usp.attention(ql, kl, vl, out=out, lse=lse, **kw)
            torch.cuda.synchronize()
            for rep in range(4):
                out.zero_()
                lse.zero_()
                g.replay()
                if rep == 1:  # an eager call between replays keeps the flag states in step
                    o2, l2 = usp.attention(ql, kl, vl, **kw)
                    torch.cuda.synchronize()
                    assert torch.equal(o2, ref_o) and torch.equal(l2, ref_l), "eager call after a replay differs"
                torch.cuda.synchronize()
                assert torch.equal(out, ref_o) and torch.equal(lse, ref_l), f"replay {rep} differs (u={u}, r={r})"
            res["checks"].append({"u": u, "r": r})
            torch.cuda.synchronize()
            dist.barrier()
            del g
            comm.destroy()
            dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


def run_errors(rank: int, world: int, port: int, cases, out_dir: str):
    """Peer-transport error paths (include/xdit_usp.h): a call after a reallocating reserve without
    re-connecting -> NOT_CONNECTED; a mailbox message larger than the region -> WORKSPACE; the mesh
    of the blobs must match the handle -> COMM_MISMATCH; nothing is enqueued on failure."""
    res = {"rank": rank, "checks": [], "error": None}
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import ctypes

        import torch
        import torch.distributed as dist

        from paper_2411_01738_b200 import usp

        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        L = usp.lib()
        comm = usp.Comm(world, 1, transport="peer")
        comm.reserve(1, 2 * world, 0, 64 * world, 64, 2)
        # grow the workspace behind the binding's back: the peers' mappings are stale now
        torch.cuda.synchronize()
        dist.barrier()
        usp._check(L.xdit_comm_reserve(comm.handle, 1, 2 * world, 0, 4096 * world, 64, 2), "xdit_comm_reserve")
        q = torch.zeros(1, 4096, 2 * world, 64, dtype=torch.bfloat16, device="cuda")
        rc = L.xdit_usp_attention(usp._ptr(q), usp._ptr(q), usp._ptr(q), usp._ptr(q), None, 1, 2 * world, 0,
                                  4096 * world, 64, world, 1, usp._stream(None), comm.handle)
        assert usp.XDIT_STATUS[rc] == "NOT_CONNECTED", (rc, usp.last_error())
        res["checks"].append("not_connected")
        comm.mailbox(1024)
        src = torch.zeros(4096, dtype=torch.uint8, device="cuda")
        try:
            comm.put((rank + 1) % world, src, 1)
            raise AssertionError("oversized put was accepted")
        except usp.XditError as e:
            assert e.status == "WORKSPACE", e
        res["checks"].append("workspace")
        blob = (ctypes.c_uint8 * (usp.PEER_BLOB_BYTES * world))()
        rc = L.xdit_comm_peer_connect(comm.handle, ctypes.cast(blob, ctypes.c_void_p))  # all-zero blobs
        assert usp.XDIT_STATUS[rc] == "COMM_MISMATCH", (rc, usp.last_error())
        res["checks"].append("mismatch")
        torch.cuda.synchronize()
        dist.barrier()
        comm.destroy()
        dist.barrier()
        dist.destroy_process_group()
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)
