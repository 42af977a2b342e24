"""Multi-process USP through the peer-memory transport.

The real multi-rank call path -- one process per SP rank, the library's peer transport moving the
Ulysses all-to-all (pack kernel storing into the peers' receive buffers), the ring K/V
rotation (peer copies into the successor's free slot while attention runs) and the O/LSE
return, with cross-rank stream ordering through device flags -- run with all ranks on the one GPU
of the test box (CUDA IPC works between processes on one device exactly as between NVLink peers).
Every rank checks its own rows against the fp64 oracle for every (ulysses, ring) factorisation of
the world size, bitwise determinism of a repeated call, and the retained KV
buffer (NEXT 1, reading R2).  Shapes change between cases, so re-reservation + re-connection is
exercised too.
"""
import json
import multiprocessing as mp
import os
import socket
import tempfile

import pytest

pytestmark = pytest.mark.gpu

# (B, H, S_txt, S_img, D, dtype, check kv_keep): ragged text + image shards, every bf16 head dim,
# the fp32 mode; H = 8 divides every Ulysses degree up to 8.
CASES = [(2, 8, 33, 400, 64, "bf16", True), (1, 8, 0, 700, 72, "bf16", False),
         (1, 8, 17, 300, 128, "bf16", True), (1, 8, 9, 150, 64, "f32", False)]
SPLITS = {2: [(2, 1), (1, 2)], 4: [(2, 2), (4, 1), (1, 4)], 8: [(2, 4), (4, 2), (8, 1), (1, 8)]}


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run_world(world: int, splits, cases, timeout: float = 900, fn: str = "run"):
    from tests import _peer_worker
    ctx = mp.get_context("spawn")
    port = _port()
    target = getattr(_peer_worker, fn)
    args = (lambda g, d: (g, world, port, splits, cases, d)) if fn == "run" else (lambda g, d: (g, world, port, cases, d))
    with tempfile.TemporaryDirectory() as d:
        procs = [ctx.Process(target=target, args=args(g, d)) for g in range(world)]
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
        if fn == "run":
            assert len(r["checks"]) == len(splits) * len(cases)
    return out


@pytest.mark.parametrize("world", [2, 4, 8])
def test_peer_transport_usp_all_splits(world):
    _run_world(world, SPLITS[world], CASES)


def test_peer_transport_toy_2x2_config0():
    """BASELINE.json configs[0]: toy DiT attention, B=1, H=4, D=64, 1024 tokens, Ulysses=2 x Ring=2,
    four real processes, against the unsplit fp64 oracle."""
    _run_world(4, [(2, 2)], [(1, 4, 0, 1024, 64, "bf16", True)])


# (B, S_txt, S_img, H, D, L, T, M, warmup, dtype): PipeFusion stages as processes (NEXT 3)
PF_CASES = [(1, 9, 300, 2, 64, 4, 3, 4, 1, "f32"), (2, 0, 256, 2, 128, 4, 4, 4, 2, "bf16"),
            (1, 16, 400, 2, 72, 8, 3, 8, 1, "bf16")]


@pytest.mark.parametrize("world", [2, 4])
def test_pipefusion_stage_processes(world):
    """One PipeFusion stage per process, patch activations and eps moved by the peer transport's
    mailbox ("asynchronous P2P"): stage 0's latent equals the in-process schedule bit for bit
    and the fp64 staleness oracle within the NEXT 3 gates."""
    out = _run_world(world, None, PF_CASES, fn="run_pipefusion")
    assert len(out[0]["checks"]) == len(PF_CASES)


def test_cfg_tail_peer_transport():
    """NEXT 2 over the peer transport: the two CFG branches gathered through the mailbox and
    combined on both ranks, twice (the ack protocol), against oracle.cfg_combine."""
    cases = [(4096, "bf16", 4.5), (4096, "f32", 7.5), (64, "bf16", 0.0), (64, "f32", 1.0)]
    out = _run_world(2, None, cases, fn="run_cfg_tail")
    assert all(len(r["checks"]) == len(cases) for r in out)


@pytest.mark.parametrize("world", [2, 4])
def test_vae_band_processes(world):
    """NEXT 4: one process per latent row band, halo rows exchanged through the mailbox before
    every conv: each band is bit-identical to the one-device decode and matches the oracle."""
    cases = [(16, 4, 24, (32, 16), False), (13, 16, 9, (64,), False), (12, 4, 140, (64, 32), True)]
    out = _run_world(world, None, cases, fn="run_vae")
    assert all(len(r["checks"]) == len(cases) for r in out)


@pytest.mark.parametrize("world,splits", [(2, [(2, 1), (1, 2)]), (4, [(2, 2), (1, 4)])])
def test_peer_transport_graph_replay(world, splits):
    """The peer-transport USP call captured in a CUDA graph replays bit-identically (4 replays with
    an eager call in between) for Ulysses, Ring and hybrid splits."""
    out = _run_world(world, None, splits, fn="run_graph")
    assert all(len(r["checks"]) == len(splits) for r in out)


def test_peer_transport_error_paths():
    out = _run_world(2, None, None, fn="run_errors")
    assert all(r["checks"] == ["not_connected", "workspace", "mismatch"] for r in out)


@pytest.mark.parametrize("world,splits", [(2, [(1, 2)]), (4, [(1, 4), (2, 2)])])
def test_peer_ring_fused_merge_with_tail_split(world, splits):
    """Ring splits on a ring block large enough that the attention grid's last partial wave is split
    over key ranges (tail_merge_kernel), so the ring merge fused into the epilogue AND into the tail
    merge both run (a7), against the fp64 oracle; D = 64 and 128."""
    cases = [(2, 8, 40, 2600 * world // 2, 64, "bf16", False), (1, 8, 17, 5200 * world // 2, 128, "bf16", False)]
    _run_world(world, splits, cases)
