"""GPU parity of the attention kernels against the fp64 oracle.

bf16 inputs -> tcgen05/TMEM/TMA kernel; fp32 inputs -> SIMT kernel.  Shapes span several 128-row
Q and KV tiles with ragged tails, B > 1, Sq != Skv, both supported head dims, and the degenerate
cases of the method (one key, one query, q = 0, identity attention, large magnitudes).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2411_01738_b200 import usp
from paper_2411_01738_b200.inputs import qkv, sample_rows
from tests._util import assert_bf16, assert_f32, errors, f64

pytestmark = pytest.mark.gpu


def run_attn(q, k, v, dtype=0, out_f32=0, lse=True):
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    o = torch.empty(q.shape, dtype=torch.float32 if (dtype == 1 or out_f32) else torch.bfloat16, device="cuda")
    l = torch.empty((B, H, Sq), dtype=torch.float32, device="cuda") if lse else None
    usp.attn_fwd(q, k, v, o, l, B=B, H=H, Sq=Sq, Skv=Skv, D=D, q_strides=(Sq * H * D, H * D, D),
                 kv_strides=(Skv * H * D, H * D, D), omap=usp.RowMap.plain(B, Sq, H, D), dtype=dtype,
                 out_f32=out_f32)
    torch.cuda.synchronize()
    return o, l


SHAPES = [  # B, H, Sq, Skv, D
    (1, 2, 256, 256, 64),
    (1, 2, 256, 256, 128),
    (2, 3, 300, 333, 64),
    (1, 2, 129, 1000, 128),
    (1, 1, 1, 5, 64),
    (2, 2, 513, 127, 128),
    (1, 4, 1024, 1024, 64),
    (2, 2, 300, 333, 72),
    (1, 3, 256, 1000, 72),
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("out_f32", [0, 1])
def test_attn_bf16_vs_oracle(shape, out_f32):
    B, H, Sq, Skv, D = shape
    q, _, _ = qkv(B, Sq, H, D, seed=1000 + Sq)
    _, k, v = qkv(B, Skv, H, D, seed=2000 + Skv)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda(), dtype=0, out_f32=out_f32)
    assert_bf16(errors(o, l, ref_o, ref_l))


@pytest.mark.parametrize("shape", [(1, 2, 256, 256, 64), (2, 3, 300, 333, 72), (1, 2, 129, 500, 128), (1, 1, 7, 3, 5)],
                         ids=lambda s: "x".join(map(str, s)))
def test_attn_f32_vs_oracle(shape):
    B, H, Sq, Skv, D = shape
    q, _, _ = qkv(B, Sq, H, D, seed=3000 + Sq, dtype=torch.float32)
    _, k, v = qkv(B, Skv, H, D, seed=4000 + Skv, dtype=torch.float32)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda(), dtype=1)
    assert_f32(errors(o, l, ref_o, ref_l))


def test_q_zero_gives_mean_v():
    B, H, S, D = 1, 2, 700, 128
    _, k, v = qkv(B, S, H, D, seed=11)
    q = torch.zeros_like(k)
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda())
    ref = f64(v).mean(axis=1, keepdims=True)
    assert np.abs(f64(o) - ref).max() < 4e-3
    assert np.abs(f64(l) - math.log(S)).max() < 1e-5


def test_identity_attention_canary():
    B, H, S, D, alpha = 1, 1, 1024, 64, 200.0
    k = torch.randn(B, S, H, D, generator=torch.Generator().manual_seed(5))
    k = k / k.norm(dim=-1, keepdim=True)
    q = (alpha * k).to(torch.bfloat16)
    k = k.to(torch.bfloat16)
    v = torch.randn(B, S, H, D, generator=torch.Generator().manual_seed(6)).to(torch.bfloat16)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda())
    assert_bf16(errors(o, l, ref_o, ref_l))
    assert np.abs(f64(o) - f64(v)).max() < 0.05  # O_i ~ V_i: token bookkeeping is right


def test_two_token_D64():
    # SURVEY §8(c) worked example at D=64: q0 = 8 ln3 e0 (rounded to bf16 8.8125), k0 = e0, k1 = 0
    D = 64
    q = torch.zeros(1, 2, 1, D); q[0, 0, 0, 0] = 8 * math.log(3)
    k = torch.zeros(1, 2, 1, D); k[0, 0, 0, 0] = 1.0
    v = torch.zeros(1, 2, 1, D); v[0, 0, 0, :] = 1.0; v[0, 1, 0, :] = 5.0
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda())
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    assert_bf16(errors(o, l, ref_o, ref_l))
    assert abs(float(o[0, 0, 0, 0]) - 2.0) < 2e-2 and abs(float(l[0, 0, 0]) - math.log(4)) < 3e-3
    assert abs(float(o[0, 1, 0, 0]) - 3.0) < 2e-2 and abs(float(l[0, 0, 1]) - math.log(2)) < 1e-5


def test_large_magnitude_no_overflow():
    B, H, S, D = 1, 2, 400, 128
    q, k, v = qkv(B, S, H, D, seed=77, scale=30.0)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda())
    assert torch.isfinite(o.float()).all() and torch.isfinite(l).all()
    e = errors(o, l, ref_o, ref_l)
    assert e["o_maxabs"] <= 30 * 2e-2 and e["lse_maxabs"] <= 1e-2, e


def test_determinism():
    B, H, S, D = 1, 3, 900, 64
    q, k, v = (t.cuda() for t in qkv(B, S, H, D, seed=5))
    a = run_attn(q, k, v)
    b = run_attn(q, k, v)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])


def test_unsupported_head_dim_is_rejected():
    q = torch.zeros(1, 128, 1, 96, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(usp.XditError) as ei:
        run_attn(q, q, q)
    assert ei.value.status == "UNSUPPORTED"


@pytest.mark.parametrize("D", [64, 72, 128])
@pytest.mark.parametrize("Skv", [4096, 1000])
def test_attn_tail_split_vs_oracle(D, Skv):
    """160 work items on 148 SMs: the last 12 (query-tile pair, head) items are split over key
    ranges and merged by the tail kernel.  Rows of the split items and of full items both match."""
    B, H, Sq = 1, 10, 4096
    q, _, _ = qkv(B, Sq, H, D, seed=500 + D)
    _, k, v = qkv(B, Skv, H, D, seed=600 + D)
    qc, kc, vc = q.cuda(), k.cuda(), v.cuda()
    o = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
    l = torch.empty((B, H, Sq), dtype=torch.float32, device="cuda")
    scratch = torch.empty(usp.attn_scratch_bytes(D) // 4, dtype=torch.float32, device="cuda")
    n0 = usp.launch_count()
    usp.attn_fwd(qc, kc, vc, o, l, B=B, H=H, Sq=Sq, Skv=Skv, D=D, q_strides=(Sq * H * D, H * D, D),
                 kv_strides=(Skv * H * D, H * D, D), omap=usp.RowMap.plain(B, Sq, H, D), scratch=scratch)
    torch.cuda.synchronize()
    launches = usp.launch_count() - n0
    if torch.cuda.get_device_properties(0).multi_processor_count == 148:
        assert launches == 2  # attention + tail merge
    heads = [0, 8, 9]
    rows = sample_rows(Sq, 64, extra=[1024, 1279, 1280, 4095, 3839, 3840])
    ref_o, ref_l = oracle.attention_rows(f64(q[:, :, heads]), f64(k[:, :, heads]), f64(v[:, :, heads]), rows.numpy())
    got_o = o[:, rows.cuda()][:, :, heads]
    got_l = l[:, heads][:, :, rows.cuda()]
    assert_bf16(errors(got_o, got_l, ref_o, ref_l))


@pytest.mark.parametrize("D", [64, 72, 128])
@pytest.mark.parametrize("Skv", [100, 300, 777])
@pytest.mark.parametrize("dynamic", [False, True])
def test_attn_persistent_many_units_vs_oracle(D, Skv, dynamic):
    """The persistent CTA pairs run several work units each (B=2, H=40, Sq=600: 240 units on 74
    pairs), with 1, 3 and 7 key tiles per unit (odd and even counts flip which softmax warp of a
    lane quarter starts the next unit) and a ragged last query tile; units handed out round-robin
    (no scratch) or by the scratch's atomic counter (dynamic, which also enables the tail split)."""
    B, H, Sq = 2, 40, 600
    q, _, _ = qkv(B, Sq, H, D, seed=700 + D + Skv)
    _, k, v = qkv(B, Skv, H, D, seed=800 + D + Skv)
    o = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
    l = torch.empty((B, H, Sq), dtype=torch.float32, device="cuda")
    scratch = torch.empty(usp.attn_scratch_bytes(D) // 4, dtype=torch.float32, device="cuda") if dynamic else None
    for _ in range(2):  # the second launch re-zeroes the unit counter
        usp.attn_fwd(q.cuda(), k.cuda(), v.cuda(), o, l, B=B, H=H, Sq=Sq, Skv=Skv, D=D,
                     q_strides=(Sq * H * D, H * D, D), kv_strides=(Skv * H * D, H * D, D),
                     omap=usp.RowMap.plain(B, Sq, H, D), scratch=scratch)
    torch.cuda.synchronize()
    heads = [0, 17, 39]
    ref_o, ref_l = oracle.attention(f64(q[:, :, heads]), f64(k[:, :, heads]), f64(v[:, :, heads]))
    assert_bf16(errors(o[:, :, heads], l[:, heads], ref_o, ref_l))
    # every head has been written (a unit lost by the hand-out would leave garbage rows)
    assert torch.isfinite(o.float()).all() and torch.isfinite(l).all()


def test_attn_persistent_deterministic_across_handout():
    """Dynamic hand-out changes which pair runs a unit, never its arithmetic: the output is
    bitwise identical with and without the counter when no tail split applies (items % 74 == 0)."""
    B, H, Sq, D = 1, 37, 512, 128  # 2 x 37 = 74 items: no partial round, no tail split
    q, k, v = (t.cuda() for t in qkv(B, Sq, H, D, seed=4242))
    outs = []
    for dyn in (False, True):
        o = torch.empty(q.shape, dtype=torch.bfloat16, device="cuda")
        l = torch.empty((B, H, Sq), dtype=torch.float32, device="cuda")
        scratch = torch.empty(usp.attn_scratch_bytes(D) // 4, dtype=torch.float32, device="cuda") if dyn else None
        usp.attn_fwd(q, k, v, o, l, B=B, H=H, Sq=Sq, Skv=Sq, D=D, q_strides=(Sq * H * D, H * D, D),
                     kv_strides=(Sq * H * D, H * D, D), omap=usp.RowMap.plain(B, Sq, H, D), scratch=scratch)
        torch.cuda.synchronize()
        outs.append((o, l))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("D", [64, 72, 128])
@pytest.mark.parametrize("pattern", ["jump_up", "jump_down", "climb"])
def test_attn_reference_max_paths_vs_oracle(D, pattern):
    """Reading R1' (deferred reconciliation of the running max): key tiles whose scores jump far
    above the unit's reference (x20: the exp2 row sum overflows 2^64, the tile is redone against its
    own max and the reference moves, rescaling O), far below it (later P underflow), or climb
    steadily (references reconciled by exact powers of two every tile)."""
    B, H, Sq, Skv = 1, 2, 300, 1500
    g = torch.Generator().manual_seed(31 + D)
    q = torch.randn(B, Sq, H, D, generator=g) * 3.0
    k = torch.randn(B, Skv, H, D, generator=g)
    v = torch.randn(B, Skv, H, D, generator=g)
    if pattern == "jump_up":
        k[:, 384:] *= 20.0
    elif pattern == "jump_down":
        k[:, :256] *= 20.0
    else:
        k *= torch.linspace(1.0, 12.0, Skv).view(1, Skv, 1, 1)
    q, k, v = (t.to(torch.bfloat16) for t in (q, k, v))
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    o, l = run_attn(q.cuda(), k.cuda(), v.cuda())
    assert_bf16(errors(o, l, ref_o, ref_l), scaled=True)  # peaky rows: |O*| up to max|V|
