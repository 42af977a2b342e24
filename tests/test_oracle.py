"""Pins for the fp64 CPU oracle (oracle/xdit_oracle.c) against things other than itself.

Each test pins the oracle to the paper, the mathematics, or an independent computation:
  * a hand-worked 2-token example (tests/golden/two_token.json),
  * SPEC closed forms and the q=0 special case,
  * a 40-digit Decimal evaluation of the definition on tiny inputs (different arithmetic, exact
    to ~1e-38, so the oracle must agree to fp64 rounding),
  * invariants of softmax attention (key-permutation invariance, query-permutation equivariance,
    key-offset invariance with the exact LSE shift, V-affine equivariance, LSE bounds, rows of P
    summing to one, identity-attention canary),
  * the paper's exactness claim "the computation yields the same results as the serial version"
    (§4.1.1) for the USP split emulator over every (ulysses, ring) factorisation.
A plausible mistake (dropped key, wrong sign, transposed q/k, head mix-up, wrong scale, wrong
shard order or merge weight) fails at least one of these.
"""
import decimal
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rnd(shape, seed, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


# ---------------------------------------------------------------- hand-worked example
def test_two_token_golden():
    g = json.load(open(os.path.join(GOLD, "two_token.json")))
    q, k, v = (np.array(g[n], dtype=np.float64) for n in ("q", "k", "v"))
    out, lse = oracle.attention(q, k, v)
    tol = g["tolerance"]
    np.testing.assert_allclose(out[0, :, 0, 0], g["expected"]["out"], rtol=0, atol=tol)
    np.testing.assert_allclose(lse[0, 0, :], g["expected"]["lse"], rtol=0, atol=tol)
    # the softmax weights themselves: recover P from O with v = [1, 0] / [0, 1]
    for col, vv in enumerate(([1.0, 0.0], [0.0, 1.0])):
        o2, _ = oracle.attention(q, k, np.array(vv).reshape(1, 2, 1, 1))
        np.testing.assert_allclose(o2[0, 0, 0, 0], g["expected"]["P_row0"][col], atol=tol)
        np.testing.assert_allclose(o2[0, 1, 0, 0], g["expected"]["P_row1"][col], atol=tol)


def test_two_token_at_D64():
    # q0 = 8 ln3 e0, k0 = e0, k1 = 0 -> scaled score ln3 at D=64 (scale 1/8)
    D = 64
    q = np.zeros((1, 2, 1, D)); q[0, 0, 0, 0] = 8 * math.log(3)
    k = np.zeros((1, 2, 1, D)); k[0, 0, 0, 0] = 1.0
    v = np.zeros((1, 2, 1, D)); v[0, 0, 0, :] = 1.0; v[0, 1, 0, :] = 5.0
    out, lse = oracle.attention(q, k, v)
    np.testing.assert_allclose(out[0, 0, 0], 2.0, atol=1e-14)
    np.testing.assert_allclose(out[0, 1, 0], 3.0, atol=1e-14)
    assert abs(lse[0, 0, 0] - math.log(4)) < 1e-14
    assert abs(lse[0, 0, 1] - math.log(2)) < 1e-14


# ---------------------------------------------------------------- SPEC closed forms
def test_single_key_gives_v0():
    q = rnd((2, 7, 3, 16), 1); k = rnd((2, 1, 3, 16), 2); v = rnd((2, 1, 3, 16), 3)
    out, lse = oracle.attention(q, k, v)
    np.testing.assert_array_equal(out, np.broadcast_to(v, out.shape))
    np.testing.assert_allclose(lse, np.einsum("bshd,bhd->bhs", q, k[:, 0]) / 4.0, atol=1e-13)


def test_equal_logits_give_mean():  # SPEC S:73 and q=0
    S, D = 37, 8
    q = np.zeros((1, 5, 2, D)); k = rnd((1, S, 2, D), 4); v = rnd((1, S, 2, D), 5)
    out, lse = oracle.attention(q, k, v)
    np.testing.assert_allclose(out, np.broadcast_to(v.mean(axis=1, keepdims=True), out.shape), atol=1e-14)
    np.testing.assert_allclose(lse, math.log(S), atol=1e-14)


# ---------------------------------------------------------------- independent high-precision evaluation
def decimal_attention(q, k, v):
    """The definition evaluated in 40-digit decimal arithmetic (no max subtraction, no fp64)."""
    decimal.getcontext().prec = 40
    Dd = decimal.Decimal
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    scale = Dd(1) / Dd(D).sqrt()
    out = np.zeros(q.shape); lse = np.zeros((B, H, Sq))
    for b in range(B):
        for h in range(H):
            for i in range(Sq):
                s = [sum(Dd(float(q[b, i, h, d])) * Dd(float(k[b, j, h, d])) for d in range(D)) * scale
                     for j in range(Skv)]
                e = [x.exp() for x in s]
                z = sum(e)
                for d in range(D):
                    out[b, i, h, d] = float(sum(e[j] * Dd(float(v[b, j, h, d])) for j in range(Skv)) / z)
                lse[b, h, i] = float(z.ln())
    return out, lse


@pytest.mark.parametrize("shape", [(1, 3, 1, 2, 4), (2, 5, 2, 7, 3), (1, 4, 3, 9, 5)])
def test_matches_decimal_brute_force(shape):
    B, Sq, H, Skv, D = shape
    q = rnd((B, Sq, H, D), 10, 1.5); k = rnd((B, Skv, H, D), 11, 1.5); v = rnd((B, Skv, H, D), 12)
    out, lse = oracle.attention(q, k, v)
    ro, rl = decimal_attention(q, k, v)
    np.testing.assert_allclose(out, ro, rtol=0, atol=1e-13)
    np.testing.assert_allclose(lse, rl, rtol=0, atol=1e-13)


def test_rows_subset_is_exact():
    q = rnd((2, 40, 3, 8), 20); k = rnd((2, 33, 3, 8), 21); v = rnd((2, 33, 3, 8), 22)
    out, lse = oracle.attention(q, k, v)
    rows = np.array([0, 5, 39, 17])
    o2, l2 = oracle.attention_rows(q, k, v, rows)
    np.testing.assert_array_equal(o2, out[:, rows])
    np.testing.assert_array_equal(l2, lse[:, :, rows])


def test_thread_count_determinism():
    q = rnd((1, 50, 2, 8), 23); k = rnd((1, 50, 2, 8), 24); v = rnd((1, 50, 2, 8), 25)
    a = oracle.attention(q, k, v, nthreads=1)
    b = oracle.attention(q, k, v, nthreads=7)
    np.testing.assert_array_equal(a[0], b[0]); np.testing.assert_array_equal(a[1], b[1])


# ---------------------------------------------------------------- invariants
@pytest.fixture(scope="module")
def qkv():
    return rnd((2, 48, 3, 16), 30), rnd((2, 64, 3, 16), 31), rnd((2, 64, 3, 16), 32)


def test_rows_of_P_sum_to_one(qkv):
    q, k, _ = qkv
    out, _ = oracle.attention(q, k, np.ones_like(k))
    np.testing.assert_allclose(out, 1.0, atol=1e-14)


def test_key_permutation_invariance(qkv):
    q, k, v = qkv
    perm = np.random.default_rng(0).permutation(k.shape[1])
    a = oracle.attention(q, k, v); b = oracle.attention(q, k[:, perm], v[:, perm])
    np.testing.assert_allclose(a[0], b[0], atol=1e-14); np.testing.assert_allclose(a[1], b[1], atol=1e-13)


def test_query_permutation_equivariance(qkv):
    q, k, v = qkv
    perm = np.random.default_rng(1).permutation(q.shape[1])
    a = oracle.attention(q, k, v); b = oracle.attention(q[:, perm], k, v)
    np.testing.assert_array_equal(a[0][:, perm], b[0]); np.testing.assert_array_equal(a[1][:, :, perm], b[1])


def test_key_offset(qkv):
    q, k, v = qkv
    c = rnd((1, 1, 1, 16), 33)
    a = oracle.attention(q, k, v); b = oracle.attention(q, k + c, v)
    np.testing.assert_allclose(a[0], b[0], atol=1e-13)
    shift = np.einsum("bshd,d->bhs", q, c[0, 0, 0]) / 4.0
    np.testing.assert_allclose(b[1], a[1] + shift, atol=1e-12)


def test_v_affine(qkv):
    q, k, v = qkv
    a = oracle.attention(q, k, v); b = oracle.attention(q, k, 2.5 * v - 0.75)
    np.testing.assert_allclose(b[0], 2.5 * a[0] - 0.75, atol=1e-13)
    np.testing.assert_array_equal(a[1], b[1])


def test_lse_bounds(qkv):
    q, k, v = qkv
    _, lse = oracle.attention(q, k, v)
    s = np.einsum("bihd,bjhd->bhij", q, k) / 4.0
    smax = s.max(axis=-1)
    assert np.all(lse >= smax - 1e-12) and np.all(lse <= smax + math.log(k.shape[1]) + 1e-12)


def test_identity_attention_canary():
    S, D, alpha = 256, 64, 200.0
    k = rnd((1, S, 1, D), 40); k /= np.linalg.norm(k, axis=-1, keepdims=True)
    v = rnd((1, S, 1, D), 41)
    out, _ = oracle.attention(alpha * k, k, v)
    np.testing.assert_allclose(out, v, atol=2e-3)


# ---------------------------------------------------------------- shard rule (reading C5)
@pytest.mark.parametrize("S_txt,S_img,N", [(0, 4096, 8), (333, 4096, 8), (226, 17550, 4), (512, 65536, 8),
                                           (5, 27, 3), (7, 9, 8)])
def test_shard_partitions(S_txt, S_img, N):
    txt = [oracle.shard(S_txt, S_img, N, g)[:2] for g in range(N)]
    img = [oracle.shard(S_txt, S_img, N, g)[2:] for g in range(N)]
    for parts, S in ((txt, S_txt), (img, S_img)):
        ref = np.array_split(np.arange(S), N)
        for (off, ln), r in zip(parts, ref):
            assert ln == len(r) and (ln == 0 or off == r[0])
    allrows = np.concatenate([oracle.local_rows(S_txt, S_img, N, g) for g in range(N)])
    assert sorted(allrows.tolist()) == list(range(S_txt + S_img))


def test_shard_empty_is_error():
    with pytest.raises(ValueError):
        oracle.shard(0, 3, 4, 3)


# ---------------------------------------------------------------- USP split emulator
SPLITS = [(1, 1), (2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2), (2, 4), (1, 8)]


@pytest.mark.parametrize("u,r", SPLITS)
@pytest.mark.parametrize("S_txt,S_img", [(0, 64), (5, 43)])
def test_usp_emulator_equals_serial(u, r, S_txt, S_img):
    B, H, D = 2, 8, 8
    S = S_txt + S_img
    q = rnd((B, S, H, D), 50); k = rnd((B, S, H, D), 51); v = rnd((B, S, H, D), 52)
    ref_o, ref_l = oracle.attention(q, k, v)
    o, l = oracle.usp_emulate(q, k, v, S_txt, u, r)
    np.testing.assert_allclose(o, ref_o, rtol=0, atol=1e-12)
    np.testing.assert_allclose(l, ref_l, rtol=0, atol=1e-12)
    if u == 1 and r == 1:  # degree 1 is bit-identical to serial
        np.testing.assert_array_equal(o, ref_o); np.testing.assert_array_equal(l, ref_l)


def test_usp_emulator_divisibility_error():
    q = rnd((1, 16, 6, 4), 60)
    with pytest.raises(ValueError):
        oracle.usp_emulate(q, q, q, 0, 4, 1)  # 6 % 4 != 0
