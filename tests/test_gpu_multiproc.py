"""Multi-process USP through NCCL: one process per rank, the library's
NCCL data plane moving the Ulysses all-to-all, the ring K/V rotation overlapped with
attention and the O/LSE return.  On the 1-GPU test box all ranks share cuda:0 and
NCCL connects them through its socket transport (tests/_mp.py); on an 8-GPU box the same tests run
one rank per GPU over NVLink.  Every rank checks its own rows against the fp64 oracle.
"""
import pytest

from tests._mp import run_world

pytestmark = pytest.mark.gpu

# (B, H, S_txt, S_img, D, dtype, check kv_keep): ragged text + image shards, every bf16 head dim,
# the fp32 mode; H = 8 divides every Ulysses degree up to 8.
CASES = [(2, 8, 33, 400, 64, "bf16", True), (1, 8, 0, 700, 72, "bf16", False),
         (1, 8, 17, 300, 128, "bf16", True), (1, 8, 9, 150, 64, "f32", False)]
SPLITS = {2: [(2, 1), (1, 2)], 4: [(2, 2), (4, 1), (1, 4)], 8: [(2, 4), (4, 2), (8, 1), (1, 8)]}


@pytest.mark.parametrize("world", [2, 4, 8])
def test_usp_all_splits(world):
    out = run_world(world, "usp_splits", SPLITS[world], CASES)
    assert all(len(r["checks"]) == len(SPLITS[world]) * len(CASES) for r in out)


def test_usp_gloo_bootstrap():
    """A gloo process group (host plumbing only): the library builds its own NCCL communicator from
    a unique id broadcast over it (xdit_comm_init) instead of splitting torch's (xdit_comm_create)."""
    run_world(2, "usp_splits", [(2, 1), (1, 2)], CASES[:1], "gloo")


def test_toy_2x2_config0():
    """BASELINE.json configs[0]: toy DiT attention, B=1, H=4, D=64, 1024 tokens, Ulysses=2 x Ring=2,
    four processes, against the unsplit fp64 oracle (all rows)."""
    run_world(4, "usp_splits", [(2, 2)], [(1, 4, 0, 1024, 64, "bf16", True)])


def test_ring_fused_merge_with_tail_split():
    """Ring splits on blocks large enough that the attention grid's last partial wave is split over
    key ranges (tail_merge_kernel), so the ring merge fused into the epilogue AND into the tail
    merge both run (a7), D = 64, 72 and 128."""
    cases = [(2, 8, 40, 5200, 64, "bf16", False), (2, 16, 0, 4096, 72, "bf16", False),
             (1, 8, 17, 10400, 128, "bf16", False)]
    run_world(2, "usp_splits", [(1, 2)], cases)


# ---- BASELINE.json workloads at full size through the product call (sampled rows x heads)
def test_baseline_world2():
    """PixArt-Sigma SP 2 (Ulysses-only and Ring-only; 1x2 reaches the D = 72 fused merge with the
    tail split) and Flux.1 4096px at 2 x 1."""
    run_world(2, "baseline_configs", [("pixart", 1, 1, 2), ("pixart", 1, 2, 1), ("flux", 1, 2, 1)])


def test_baseline_world4():
    """SD3-medium Ulysses-only / Ring-only / hybrid (4x1, 1x4, 2x2), PixArt 2x2, and the CFG outer
    split: CogVideoX cfg 2 x (2 x 1) -- each CFG group an independent SP group on its own latent
    (P:409-414), both groups' rows against the oracle."""
    run_world(4, "baseline_configs", [("sd3", 1, 4, 1), ("sd3", 1, 1, 4), ("sd3", 1, 2, 2), ("pixart", 1, 2, 2),
                                      ("cogvideox", 2, 2, 1)])


def test_baseline_world8():
    """The 8-GPU configurations: Flux.1 8x1, 2x4, 4x2, 1x8; SD3 8x1, 4x2, 1x8; PixArt 1x8, 2x4;
    CogVideoX CFG 2 x USP 4 (4x1, 2x2, 1x4) -- BASELINE configs 2-5."""
    cases = [("flux", 1, 8, 1), ("flux", 1, 2, 4), ("flux", 1, 4, 2), ("flux", 1, 1, 8),
             ("sd3", 1, 8, 1), ("sd3", 1, 4, 2), ("sd3", 1, 1, 8), ("pixart", 1, 1, 8), ("pixart", 1, 2, 4),
             ("cogvideox", 2, 4, 1), ("cogvideox", 2, 2, 2), ("cogvideox", 2, 1, 4)]
    out = run_world(8, "baseline_configs", cases, timeout=2400)
    assert all(len(r["checks"]) == len(cases) for r in out)


@pytest.mark.parametrize("world,splits", [(2, [(2, 1), (1, 2)]), (4, [(2, 2), (1, 4)])])
def test_graph_replay(world, splits):
    """The NCCL USP call captured in a CUDA graph replays bit-identically (4 replays with an eager
    call in between) for Ulysses, Ring and hybrid splits."""
    out = run_world(world, "graph_replay", splits)
    assert all(len(r["checks"]) == len(splits) for r in out)


def test_error_paths():
    out = run_world(2, "error_paths")
    assert all(r["checks"] == ["workspace", "mismatch", "p2p_peer", "buf_rows", "valid_after"] for r in out)


def test_cfg_tail():
    """NEXT 2 over NCCL: the two CFG branches all-gathered and combined on both ranks, twice."""
    cases = [(4096, "bf16", 4.5), (4096, "f32", 7.5), (64, "bf16", 0.0), (64, "f32", 1.0)]
    out = run_world(2, "cfg_tail", cases)
    assert all(len(r["checks"]) == len(cases) for r in out)


@pytest.mark.parametrize("world", [2, 4])
def test_vae_band_processes(world):
    """NEXT 4: one process per latent row band, halo rows exchanged before every conv."""
    cases = [(16, 4, 24, (32, 16), False), (13, 16, 9, (64,), False), (12, 4, 140, (64, 32), True)]
    out = run_world(world, "vae_bands", cases)
    assert all(len(r["checks"]) == len(cases) for r in out)


# (B, S_txt, S_img, H, D, L, T, M, warmup, dtype)
PF_CASES = [(1, 9, 300, 2, 64, 4, 3, 4, 1, "f32"), (2, 0, 256, 2, 128, 4, 4, 4, 2, "bf16"),
            (1, 16, 400, 2, 72, 8, 3, 8, 1, "bf16")]
PF_HYBRID_CASES = [(1, 9, 300, 4, 64, 4, 3, 4, 1, "f32"), (1, 16, 512, 4, 128, 4, 4, 4, 1, "bf16"),
                   (2, 0, 384, 4, 72, 4, 3, 3, 2, "bf16")]


@pytest.mark.parametrize("world", [2, 4])
def test_pipefusion_stage_processes(world):
    """Pure PipeFusion, one stage per process ("asynchronous P2P"): stage 0's latent equals the
    one-device schedule bit for bit and the fp64 staleness oracle within the NEXT 3 gates."""
    run_world(world, "pipefusion_mesh", [(world, 1, 1)], PF_CASES)


@pytest.mark.parametrize("world,meshes", [(2, [(1, 2, 1), (1, 1, 2)]), (4, [(2, 2, 1), (2, 1, 2)]),
                                          (8, [(2, 2, 2), (4, 2, 1)])])
def test_pipefusion_x_usp_hybrid(world, meshes):
    """Hybrid PipeFusion x USP (NEXT 3 as scoped): pipefusion_degree x (ulysses x ring)
    meshes; the SP call keeps the fresh K,V it receives in the KV buffer, so the latents equal the
    pure-PipeFusion oracle with the same (pp, M) within the gates and the ranks of one head block hold
    bitwise-identical buffers."""
    out = run_world(world, "pipefusion_mesh", meshes, PF_HYBRID_CASES)
    assert all(len(r["checks"]) == len(meshes) * len(PF_HYBRID_CASES) for r in out)
