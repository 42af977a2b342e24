"""SURVEY §8(f) NEXT 1-2 oracles pinned against what the paper and the mathematics fix (no GPU)."""
import numpy as np
import pytest

import oracle

SPLITS = [(1, 1), (2, 1), (1, 2), (2, 2), (4, 2), (2, 4), (8, 1), (1, 8)]


def _kv(B=2, S=37, H=8, D=4, seed=0):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((B, S, H, D)), rng.standard_normal((B, S, H, D))


@pytest.mark.parametrize("u,r", SPLITS)
def test_kv_keep_holds_every_token_once(u, r):
    """the rank ends with the KV of the whole SP-group sequence for its heads: every
    global row appears exactly once and carries the global K/V of that row."""
    k, v = _kv()
    S_txt = 5
    B, S, H, D = k.shape
    for g in range(u * r):
        buf = oracle.kv_keep(k, v, S_txt, u, r, g)
        assert buf.shape == (2, B, H // u, S, D)
        j, Hh = g % u, H // u
        # recover each buffer row's global index by matching against the global K (distinct rows)
        kk = k[:, :, j * Hh:(j + 1) * Hh].transpose(0, 2, 1, 3)  # [B, Hh, S, D]
        idx = [int(np.argmin(np.abs(kk[0, 0] - buf[0, 0, 0, t]).sum(-1))) for t in range(S)]
        assert sorted(idx) == list(range(S))
        np.testing.assert_array_equal(buf[0], kk[:, :, idx])
        vv = v[:, :, j * Hh:(j + 1) * Hh].transpose(0, 2, 1, 3)
        np.testing.assert_array_equal(buf[1], vv[:, :, idx])


@pytest.mark.parametrize("u,r", SPLITS)
def test_kv_keep_consistent_within_head_block(u, r):
    """SPEC S:430 hybrid-KV consistency: ranks that share a Ulysses head block (same g mod u) hold
    elementwise-identical buffers; pure Ring (u=1) gives every rank all heads."""
    k, v = _kv(seed=1)
    bufs = [oracle.kv_keep(k, v, 3, u, r, g) for g in range(u * r)]
    for g in range(u * r):
        np.testing.assert_array_equal(bufs[g], bufs[g % u])
    if u == 1:
        assert bufs[0].shape[2] == k.shape[2]


def test_kv_keep_single_rank_is_head_major_k_v():
    k, v = _kv(S=9)
    buf = oracle.kv_keep(k, v, 4, 1, 1, 0)
    np.testing.assert_array_equal(buf[0], k.transpose(0, 2, 1, 3))
    np.testing.assert_array_equal(buf[1], v.transpose(0, 2, 1, 3))


def test_kv_keep_shard_order():
    """Rows follow SP-shard order: rank p's local rows (text shard, then image shard) before p+1's."""
    S_txt, S_img, N = 3, 10, 4
    k = np.arange(S_txt + S_img, dtype=np.float64).reshape(1, -1, 1, 1) * np.ones((1, 1, 2, 1))
    buf = oracle.kv_keep(k, k, S_txt, 2, 2, 1)
    got = buf[0, 0, 0, :, 0].astype(int).tolist()
    want = []
    for p in range(N):
        to, tl, io, il = oracle.shard(S_txt, S_img, N, p)
        want += list(range(to, to + tl)) + [S_txt + x for x in range(io, io + il)]
    assert got == want


def test_cfg_combine_special_cases():
    """g = 0 gives eps_uncond, g = 1 gives eps_cond; linear in g (closed form)."""
    rng = np.random.default_rng(3)
    c, u = rng.standard_normal(1000), rng.standard_normal(1000)
    np.testing.assert_array_equal(oracle.cfg_combine(c, u, 0.0), u)
    np.testing.assert_allclose(oracle.cfg_combine(c, u, 1.0), c, rtol=0, atol=1e-15)
    a, b = oracle.cfg_combine(c, u, 2.0), oracle.cfg_combine(c, u, 5.0)
    np.testing.assert_allclose(oracle.cfg_combine(c, u, 7.5), a + (b - a) * (7.5 - 2.0) / 3.0, atol=1e-12)
    assert abs(oracle.cfg_combine([3.0], [1.0], 7.5)[0] - 16.0) == 0.0  # 1 + 7.5 * 2
