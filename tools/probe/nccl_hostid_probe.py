"""Probe: can NCCL run several ranks on ONE GPU when each rank claims its own host (NCCL_HOSTID)?
Rank g runs with NCCL_HOSTID=xdit-rank-g, so NCCL's duplicate-GPU check (same host hash + bus id)
does not fire and the ranks talk over the socket transport on the loopback interface."""
import os, sys, time, multiprocessing as mp, socket, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

def worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), NCCL_HOSTID=f"xdit-rank-{rank}",
                          NCCL_SOCKET_IFNAME="lo", NCCL_DEBUG="WARN")
        import torch, torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        t = torch.full((1 << 20,), float(rank + 1), device="cuda")
        dist.all_reduce(t)
        ok1 = float(t[0]) == world * (world + 1) / 2
        x = torch.full((1 << 20,), float(rank), device="cuda"); y = torch.empty_like(x)
        ops = [dist.P2POp(dist.isend, x, (rank + 1) % world), dist.P2POp(dist.irecv, y, (rank - 1) % world)]
        for w in dist.batch_isend_irecv(ops): w.wait()
        torch.cuda.synchronize()
        ok2 = float(y[0]) == (rank - 1) % world
        pg = dist.distributed_c10d._get_default_group()
        comm_ptr = pg._get_backend(torch.device("cuda"))._comm_ptr()
        # our library over NCCL: (world,1) and (1,world)
        from paper_2411_01738_b200 import usp
        import oracle
        from paper_2411_01738_b200.inputs import qkv
        from tests._util import errors, f64
        res = {}
        for (u, r) in [(world, 1), (1, world)]:
            comm = usp.Comm(u, r, transport="nccl")
            B, H, S_txt, S_img, D = 1, 8, 17, 600, 128
            qq, kk, vv = qkv(B, S_txt + S_img, H, D, seed=7)
            to, tl, io, il = usp.shard(S_txt, S_img, world, rank)
            idx = torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)])
            ql, kl, vl = (z[:, idx].contiguous().cuda() for z in (qq, kk, vv))
            t0 = time.time()
            o, l = usp.attention(ql, kl, vl, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r)
            torch.cuda.synchronize()
            ro, rl = oracle.attention_rows(f64(qq), f64(kk), f64(vv), idx.numpy())
            res[f"{u}x{r}"] = (errors(o, l, ro, rl), time.time() - t0)
            comm.destroy()
        dist.barrier()
        q.put((rank, ok1, ok2, comm_ptr != 0, res, None))
        dist.destroy_process_group()
    except Exception:
        q.put((rank, None, None, None, None, traceback.format_exc()))

if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(g, world, port, q)) for g in range(world)]
    [p.start() for p in ps]
    for _ in ps:
        print(q.get(timeout=600), flush=True)
    [p.join(60) for p in ps]
