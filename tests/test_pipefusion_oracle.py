"""Pins of the PipeFusion oracle (oracle/pipefusion.py).

Each pin checks the oracle against something other than itself: the paper's fresh-area description
(Fig. 5: within a timestep the fresh patch set grows by one per micro-step), the
synchronous limits (warmup = T, M = 1 -> the serial DiT), the N-independence of
the staleness pattern (a micro-step-ordered replay gives the same numbers), a closed form (g = 0:
x_T = (1 - sigma)^T x_0), and a hand derivation of the stale context a patch sees (written with the
attention primitive directly).
"""
import itertools

import numpy as np
import pytest

import oracle
from oracle import pipefusion as pf


def weights(L, H, D, seed, gscale=0.5):
    rng = np.random.default_rng(seed)
    return [tuple(rng.uniform(0.5, 1.5, (H, D)) for _ in range(3)) + (gscale * rng.uniform(0.5, 1.5, (H, D)),)
            for _ in range(L)]


def inputs(B=1, S_txt=5, S_img=40, H=2, D=8, seed=0):
    return np.random.default_rng(seed).standard_normal((B, S_txt + S_img, H, D))


def test_patch_bounds_partition_and_text_with_patch0():
    for S_txt, S_img, M in [(0, 10, 1), (0, 10, 3), (7, 64, 4), (77, 4096, 8), (5, 9, 9)]:
        P = pf.patch_bounds(S_txt, S_img, M)
        assert P[0][0] == 0 and len(P) == M
        assert sum(n for _, n in P) == S_txt + S_img
        for (o0, n0), (o1, _) in zip(P, P[1:]):
            assert o0 + n0 == o1
        img = [n for _, n in P]
        img[0] -= S_txt
        assert img == [len(a) for a in np.array_split(np.arange(S_img), M)]  # balanced (R4)
    with pytest.raises(ValueError):
        pf.patch_bounds(0, 3, 4)


@pytest.mark.parametrize("N,M", [(1, 1), (1, 4), (2, 2), (2, 4), (4, 4), (4, 8), (8, 8)])
def test_replay_fresh_area_grows_by_one_patch_per_micro_step(N, M):
    """Fig. 5 / P:277-279: at a pipelined step s, patch m at any block sees this step's K,V for
    patches 0..m (already processed at that block) and the previous step's for m+1..M-1."""
    L, T, warmup = 8, 4, 1
    seen = pf.replay_stamps(N, M, L, T, warmup)
    assert len(seen) == T * M * L
    for (s, m, l), st in seen.items():
        if s < warmup:
            assert st == (s,) * M
        else:
            assert st == tuple(s if j <= m else s - 1 for j in range(M)), (s, m, l, st)
    # the staleness pattern does not depend on the number of stages (SPEC S:431 hybrid == pure)
    assert seen == pf.replay_stamps(1, M, L, T, warmup)


def test_replay_warmup_saturation():
    seen = pf.replay_stamps(4, 4, 8, 3, 3)
    assert all(st == (s,) * 4 for (s, _, _), st in seen.items())  # SPEC S:401 warmup >= T: all fresh


def test_replay_monotone_fresh_set():
    seen = pf.replay_stamps(4, 6, 8, 3, 1)
    for s, l in itertools.product(range(1, 3), range(8)):
        fresh = [sum(1 for x in seen[(s, m, l)] if x == s) for m in range(6)]
        assert fresh == sorted(fresh) and fresh[-1] == 6  # non-shrinking


def serial_run(x, W, T, sigma):
    xs = []
    for _ in range(T):
        x = x - sigma * pf.serial_eps(x, W)
        xs.append(x)
    return x, xs


def test_warmup_all_steps_is_serial():
    x, W = inputs(), weights(3, 2, 8, 1)
    got, _ = pf.pipefusion(x, W, T=3, M=4, warmup=3, sigma=0.3, S_txt=5)
    want, _ = serial_run(x, W, 3, 0.3)
    assert np.array_equal(got, want)


def test_one_patch_is_serial():
    """M = 1: the pipelined branch's only patch is the whole sequence, so its KV is always fresh."""
    x, W = inputs(seed=2), weights(4, 2, 8, 2)
    got, _ = pf.pipefusion(x, W, T=3, M=1, warmup=1, sigma=0.25, S_txt=5)
    want, _ = serial_run(x, W, 3, 0.25)
    assert np.allclose(got, want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("N,M", [(2, 2), (2, 4), (4, 4)])
def test_pipeline_order_equals_patch_order(N, M):
    x, W = inputs(seed=3), weights(4, 2, 8, 3)
    a, _ = pf.pipefusion(x, W, T=3, M=M, warmup=1, sigma=0.3, S_txt=5, N=N, order="pipeline")
    b, _ = pf.pipefusion(x, W, T=3, M=M, warmup=1, sigma=0.3, S_txt=5)
    assert np.array_equal(a, b)


def test_no_attention_closed_form():
    x, W = inputs(seed=4), weights(2, 2, 8, 4, gscale=0.0)
    got, xs = pf.pipefusion(x, W, T=4, M=3, warmup=1, sigma=0.2, S_txt=5)
    assert np.allclose(got, 0.8 ** 4 * x, rtol=1e-14, atol=0)
    assert np.allclose(xs[0], 0.8 * x, rtol=1e-14, atol=0)


def test_stale_context_hand_derivation():
    """L = 1, M = 2, warmup = 1, T = 2.  Step 0 is synchronous: x1 = x0 - sigma eps(x0).  At step 1,
    patch 0 attends to its own fresh K,V (from x1) and patch 1's STALE K,V (from x0); patch 1 then
    sees both fresh (patch 0's block-0 K,V come from x1 too), i.e. the serial rows."""
    S_txt, S_img, H, D, sigma = 3, 20, 2, 8, 0.4
    x0, W = inputs(S_txt=S_txt, S_img=S_img, seed=5), weights(1, H, D, 5)
    wq, wk, wv, g = W[0]
    (o0, n0), (o1, n1) = pf.patch_bounds(S_txt, S_img, 2)
    x1 = x0 - sigma * (x0 + g * oracle.attention(x0 * wq, x0 * wk, x0 * wv)[0])
    ctx = np.concatenate([x1[:, o0:o0 + n0], x0[:, o1:o1 + n1]], axis=1)
    eps0 = x1[:, o0:o0 + n0] + g * oracle.attention(x1[:, o0:o0 + n0] * wq, ctx * wk, ctx * wv)[0]
    eps1 = x1[:, o1:o1 + n1] + g * oracle.attention(x1[:, o1:o1 + n1] * wq, x1 * wk, x1 * wv)[0]
    x2 = x1 - sigma * np.concatenate([eps0, eps1], axis=1)
    got, xs = pf.pipefusion(x0, W, T=2, M=2, warmup=1, sigma=sigma, S_txt=S_txt)
    assert np.allclose(xs[0], x1, rtol=0, atol=1e-13)
    assert np.allclose(got, x2, rtol=0, atol=1e-13)
    # and it is NOT the serial result: staleness is visible
    ser, _ = serial_run(x0, W, 2, sigma)
    assert np.abs(got - ser).max() > 1e-3


# ---- hybrid PipeFusion x SP (NEXT 3 as scoped)
HYBRID_SPLITS = [(1, 1), (2, 1), (1, 2), (2, 2), (4, 1), (1, 4), (2, 4), (4, 2)]


@pytest.mark.parametrize("u,r", HYBRID_SPLITS)
def test_hybrid_equals_pure_pipefusion(u, r):
    """SPEC S:431 "Hybrid = pure PipeFusion: for any sp_degree, hybrid latents equal pure PipeFusion
    latents with identical (pipefusion_degree, M) within 1e-10" -- SP is exact once the SP group
    keeps the K,V it receives, ragged shards and text with patch 0 included."""
    x = inputs(B=2, S_txt=5, S_img=43, H=4, D=8, seed=3)
    W = weights(3, 4, 8, 4)
    kw = dict(T=4, M=3, warmup=1, sigma=0.3, S_txt=5)
    want, _ = pf.pipefusion(x, W, **kw)
    got, kv = pf.hybrid(x, W, u=u, r=r, **kw)
    assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()
    # "the KV involved in Attention computation on different devices within the SP group should be
    # consistent": ranks of one head block hold identical buffers
    for g in range(u * r):
        for g2 in range(g % u, u * r, u):
            for l in range(3):
                assert np.array_equal(kv[g][l][0], kv[g2][l][0]) and np.array_equal(kv[g][l][1], kv[g2][l][1])


@pytest.mark.parametrize("u,r", [(2, 1), (1, 2), (2, 2)])
def test_hybrid_naive_sp_diverges(u, r):
    """The "standard SP" ablation ("device 0 only updates K, V belonging to the even-numbered
    patches"): discarding the received K,V leaves buffers inconsistent and the latent wrong."""
    x = inputs(B=1, S_txt=3, S_img=40, H=2, D=8, seed=5)
    W = weights(2, 2, 8, 6)
    kw = dict(T=3, M=4, warmup=1, sigma=0.3, S_txt=3)
    want, _ = pf.pipefusion(x, W, **kw)
    bad, kv = pf.hybrid(x, W, u=u, r=r, naive=True, **kw)
    assert np.abs(bad - want).max() > 1e-3 * np.abs(want).max()
    assert any(not np.array_equal(kv[0][0][0], kv[g][0][0]) for g in range(u, u * r, u)) or r == 1


def test_hybrid_all_synchronous_is_serial():
    """warmup = T: every step synchronous, so hybrid = the serial DiT forward."""
    x = inputs(B=1, S_txt=4, S_img=24, H=2, D=8, seed=7)
    W = weights(2, 2, 8, 8)
    got, _ = pf.hybrid(x, W, T=2, M=3, warmup=2, sigma=0.4, S_txt=4, u=2, r=2)
    want = x.copy()
    for _ in range(2):
        want = want - 0.4 * pf.serial_eps(want, W)
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
