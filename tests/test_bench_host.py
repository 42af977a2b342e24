"""Host logic of bench.py (no GPU): the default mesh choice (CFG first, then the largest Ulysses degree
dividing H -- P:414), the config object both arms print, and the algorithmic
communication bytes per rank (Table 1)."""
import pytest

import bench
from paper_2411_01738_b200 import usp
from paper_2411_01738_b200.inputs import WORKLOADS


def test_default_split():
    assert bench.default_split(1, 24, 1) == (1, 1, 1)
    assert bench.default_split(8, 24, 1) == (1, 8, 1)       # Flux: Ulysses 8 (24 % 8 == 0)
    assert bench.default_split(8, 16, 1) == (1, 8, 1)       # PixArt
    assert bench.default_split(8, 48, 2) == (2, 4, 1)       # CogVideoX: CFG 2 x USP 4
    assert bench.default_split(1, 48, 2) == (1, 1, 1)       # one GPU: both CFG branches on it
    assert bench.default_split(6, 24, 1) == (1, 6, 1)
    c, u, r = bench.default_split(8, 12, 1)                 # 12 % 8 != 0: Ulysses 4, ring 2
    assert (c, u, r) == (1, 4, 2)


def test_reference_arm_prints_our_config():
    for name in ("flux", "pixart", "cogvideox"):
        a = bench.parse(["--gpus", "8", "--config", name])
        cfg = bench.ours_config(a, WORKLOADS[name])
        assert cfg["workload"] == name and cfg["cfg"] * cfg["ulysses"] * cfg["ring"] == 8
        assert cfg["data_plane"] == "nccl"
    a = bench.parse([])
    cfg = bench.ours_config(a, WORKLOADS["flux"])
    assert cfg["data_plane"] is None and cfg["l2"] == "inputs larger than L2"
    assert a.gpus == 1 and a.config == "flux" and a.warmup >= 3


def test_world_size_must_match_gpus(monkeypatch):
    """Under torchrun, WORLD_SIZE != --gpus fails loudly instead of benchmarking another N."""
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "0")
    with pytest.raises(SystemExit) as e:
        bench.main(["--gpus", "8", "--impl", "reference"])
    assert "WORLD_SIZE=2" in str(e.value)


def test_gpus_without_torchrun_relaunches(monkeypatch):
    """--gpus N (N > 1) without WORLD_SIZE re-launches under torch.distributed.run with N local ranks."""
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def test_phase_summary_bandwidth():
    ph = {"total_ms": 2.0, "a2a_in_ms": 0.2, "a2a_out_ms": 0.1, "attn_ms": [0.8, 0.8], "ring_comm_ms": [0.5],
          "a2a_in_bytes": 90_000_000, "a2a_out_bytes": 30_000_000, "ring_bytes": [180_000_000]}
    s = bench.phase_summary([ph, dict(ph, a2a_in_ms=0.3)])
    assert s["a2a_in_ms"] == 0.3 and abs(s["bandwidth"]["a2a_in"]["GBps"] - 300.0) < 1e-9
    assert abs(s["bandwidth"]["ring"]["GBps"] - 360.0) < 1e-9 and s["bandwidth"]["ring"]["hidden_under_attention"]


def test_comm_bytes_match_table1():
    """Flux N = 8: 177.5 MB (8x1), 253.6 MB (4x2), 405.8 MB (2x4), 710.2 MB (1x8)."""
    w = WORKLOADS["flux"]
    want = {(8, 1): 177.5e6, (4, 2): 253.6e6, (2, 4): 405.8e6, (1, 8): 710.2e6}
    for (u, r), mb in want.items():
        pl = usp.plan(w.B, w.H, w.S_txt, w.S_img, w.D, u, r, 0)
        got = bench.comm_summary(pl, w.B, w, u, r, 1.0)["bytes_per_rank"]
        assert abs(got - mb) / mb < 0.01, (u, r, got, mb)
    assert bench.comm_summary(usp.plan(1, 24, 512, 65536, 128, 1, 1, 0), 1, w, 1, 1, 1.0) is None


def test_clock_ceilings():
    """The unit ceilings the bench prints beside the achieved fraction: at D = 64 the
    MUFU binds (16 ex2/clk/SM, one exp2 per 4D FLOPs, 1/8 of them on the FMA pipe), at D = 128 the
    tensor pipe (8192 FLOP/clk/SM) -- both scale with the clock the run held."""
    import bench
    c = bench.clock_ceilings(64, 1000, 100, 100.0)
    assert c["binding"] == "mufu"
    assert abs(c["mufu_exp2_tflops_at_clock"] - 16 * 100 * 1e9 * 256 / (7 / 8) / 1e12) < 1e-9
    assert abs(c["tensor_tflops_at_clock"] - 8192 * 100 * 1e9 / 1e12) < 1e-9
    assert abs(c["frac_of_binding"] - 100.0 / c["mufu_exp2_tflops_at_clock"]) < 1e-12
    c = bench.clock_ceilings(128, 1000, 100, 100.0)
    assert c["binding"] == "tensor" and c["exp2_on_fma_pipe"] == 1 / 16
    assert bench.clock_ceilings(64, None, 100, 1.0) is None
