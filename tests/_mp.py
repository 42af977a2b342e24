"""Multi-process harness for the -m gpu tests: one process per rank, NCCL between them.

On a box with >= world GPUs rank g runs on cuda:g (NVLink / NVSwitch between the ranks).  On a
smaller box (the 1-GPU test box) every rank runs on cuda:0 and claims its own host id
(NCCL_HOSTID=xdit-test-rank-<g>): NCCL refuses two ranks of one communicator on the same GPU of the
same host, and with distinct host ids it connects them through its socket transport on the loopback
interface instead -- the library's NCCL code path, unchanged, only slower bytes.  Each rank writes a
JSON result; the test process asserts on them.
"""
import json
import multiprocessing as mp
import os
import socket
import tempfile
import traceback


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def setup(rank: int, world: int, port: int, backend: str = "nccl"):
    """Device + env + torch.distributed for one rank; returns the device index."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    share = torch.cuda.device_count() < world
    dev = 0 if share else rank
    if share:
        os.environ["NCCL_HOSTID"] = f"xdit-test-rank-{rank}"
        os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return dev


def teardown():
    import torch
    import torch.distributed as dist
    torch.cuda.synchronize()
    dist.barrier()
    dist.destroy_process_group()


def _entry(fn_name, rank, world, port, args, out_dir):
    res = {"rank": rank, "checks": [], "error": None}
    try:
        from tests import _mp_worker
        getattr(_mp_worker, fn_name)(rank, world, port, res, *args)
    except Exception:
        res["error"] = traceback.format_exc()
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
        json.dump(res, f)


def run_world(world: int, fn_name: str, *args, timeout: float = 1200):
    """Run tests._mp_worker.<fn_name>(rank, world, port, res, *args) in `world` processes; return
    the per-rank result dicts after asserting that every rank finished without an error."""
    ctx = mp.get_context("spawn")
    port = _port()
    with tempfile.TemporaryDirectory() as d:
        procs = [ctx.Process(target=_entry, args=(fn_name, g, world, port, args, d)) for g in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout)
        hung = [g for g, p in enumerate(procs) if p.is_alive()]
        for p in procs:
            if p.is_alive():
                p.kill()
        assert not hung, f"ranks {hung} did not finish within {timeout}s"
        out = []
        for g in range(world):
            path = os.path.join(d, f"rank{g}.json")
            assert os.path.exists(path), f"rank {g} wrote no result (exit code {procs[g].exitcode})"
            with open(path) as f:
                out.append(json.load(f))
    for r in out:
        assert r["error"] is None, f"rank {r['rank']}:\n{r['error']}"
    return out
