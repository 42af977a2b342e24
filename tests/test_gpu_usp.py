"""USP parity on one GPU (SURVEY §4 "1-GPU virtual-rank harness" and §8(a) a1-a10).

* `xdit_usp_attention` at N=1 (the bench's launch configuration) against the fp64 oracle, on small
  shapes in full and at BASELINE.json's full sizes on sampled rows (rows are independent, so a
  sampled check is an exact subset check).
* Every (ulysses, ring) split with u*r in {2, 4, 8}, driven as u*r virtual ranks through the
  library's exported stage kernels (pack -> [all-to-all as tensor copies] -> unpack -> ring of
  attention + LSE merge -> final write into the reverse-all-to-all buffer -> [copies] -> unpack),
  i.e. the exact kernel sequence xdit_usp_attention enqueues around NCCL, compared per rank with the
  oracle -- "the computation yields the same results as the serial version" (§4.1.1).
"""
import math

import numpy as np
import pytest
import torch

import oracle
from paper_2411_01738_b200 import usp
from paper_2411_01738_b200.inputs import WORKLOADS, qkv, sample_rows, seed_for
from tests._util import assert_bf16, assert_f32, errors, f64

pytestmark = pytest.mark.gpu


def local_index(S_txt, S_img, N, g):
    to, tl, io, il = usp.shard(S_txt, S_img, N, g)
    return torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)])


# ------------------------------------------------------------------------------ N = 1 via the ABI
@pytest.mark.parametrize("B,H,S_txt,S_img,D", [(1, 4, 0, 1024, 64), (2, 3, 33, 400, 64), (1, 2, 17, 300, 128),
                                             (2, 4, 0, 520, 72)])
@pytest.mark.parametrize("with_lse", [True, False])
def test_usp_n1_full(B, H, S_txt, S_img, D, with_lse):
    S = S_txt + S_img
    q, k, v = qkv(B, S, H, D, seed=S + D)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    with usp.Comm(1, 1) as comm:
        out, lse = usp.attention(q.cuda(), k.cuda(), v.cuda(), S_txt=S_txt, S_img=S_img, comm=comm,
                                 return_lse=with_lse)
        torch.cuda.synchronize()
    assert_bf16(errors(out, lse, ref_o, ref_l if with_lse else None))


def test_usp_n1_f32():
    B, H, S_txt, S_img, D = 1, 3, 10, 200, 72
    q, k, v = qkv(B, S_txt + S_img, H, D, seed=9, dtype=torch.float32)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    with usp.Comm(1, 1) as comm:
        out, lse = usp.attention(q.cuda(), k.cuda(), v.cuda(), S_txt=S_txt, S_img=S_img, comm=comm)
        torch.cuda.synchronize()
    assert_f32(errors(out, lse, ref_o, ref_l))


def test_usp_n1_errors():
    q = torch.zeros(1, 64, 2, 64, dtype=torch.bfloat16, device="cuda")
    with usp.Comm(1, 1) as comm:
        with pytest.raises(usp.XditError) as e:  # (u, r) must match the handle
            usp.attention(q, q, q, S_txt=0, S_img=64, comm=comm, ulysses=2, ring=1)
        assert e.value.status == "COMM_MISMATCH"
        q96 = torch.zeros(1, 64, 2, 96, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(usp.XditError) as e:  # bf16 path: D in {64, 128}
            usp.attention(q96, q96, q96, S_txt=0, S_img=64, comm=comm)
        assert e.value.status == "UNSUPPORTED"
        qm = torch.zeros(64 * 2 * 64 + 1, dtype=torch.bfloat16, device="cuda")[1:].view(1, 64, 2, 64)
        with pytest.raises(usp.XditError) as e:  # 2-byte offset pointer
            usp.attention(qm, qm, qm, S_txt=0, S_img=64, comm=comm)
        assert e.value.status == "ALIGNMENT"
        with pytest.raises(usp.XditError) as e:  # H % ulysses is checked before enqueue
            usp.plan(1, 6, 0, 64, 64, 4, 1, 0)
        assert e.value.status == "DIVISIBILITY"


@pytest.mark.parametrize("name", ["flux", "cogvideox", "sd3", "pixart"])
def test_usp_n1_full_size_sampled(name):
    """BASELINE.json full sizes, launch configuration of bench.py (N=1), sampled rows x 2 heads."""
    w = WORKLOADS[name]
    B = w.B  # one CFG group
    torch.manual_seed(0)
    q, k, v = qkv(B, w.S, w.H, w.D, seed=seed_for(w), device="cuda")
    with usp.Comm(1, 1) as comm:
        out, lse = usp.attention(q, k, v, S_txt=w.S_txt, S_img=w.S_img, comm=comm)
        torch.cuda.synchronize()
    heads = [0, w.H - 1]
    rows = sample_rows(w.S, 96, extra=[w.S_txt - 1, w.S_txt, 127, 128, w.S - 129])
    qs, ks, vs = (f64(t[:, :, heads]) for t in (q, k, v))
    ref_o, ref_l = oracle.attention_rows(qs, ks, vs, rows.numpy())
    got_o = out[:, rows.cuda()][:, :, heads]
    got_l = lse[:, heads][:, :, rows.cuda()]
    assert_bf16(errors(got_o, got_l, ref_o, ref_l))


# ------------------------------------------------------------------------------ virtual-rank harness
def make_fmap(B, Lmax, Hh, D, seg_off, nseg, chunk_bytes, eb):
    m = usp.RowMap()
    m.nseg = nseg
    for p in range(9):
        m.seg_off[p] = seg_off[min(p, nseg)]
    m.o_seg, m.o_b, m.o_s, m.o_h = chunk_bytes // eb, Lmax * Hh * D, Hh * D, D
    m.l_seg, m.l_b, m.l_h = chunk_bytes // 4, Hh * Lmax, Lmax
    return m


def align16(x):
    return (x + 15) // 16 * 16


def run_virtual_usp(q, k, v, S_txt, S_img, u, r, f32=False, kv_out=None):
    """Every stage of xdit_usp_attention for all u*r ranks on one GPU; all-to-all and ring P2P are
    tensor copies between the virtual ranks' buffers.  Returns per-rank (out, lse).  kv_out (a
    list): also run xdit_usp_attention_kv's retention stage (xdit_kv_retain after the all-to-all and
    for every incoming ring block) and append each rank's [2, B, H/u, S, D] KV buffer."""
    B, S, H, D = q.shape
    N = u * r
    eb = 4 if f32 else 2
    dt = torch.float32 if f32 else torch.bfloat16
    plans = [usp.plan(B, H, S_txt, S_img, D, u, r, g) for g in range(N)]
    Hh, Lmax = plans[0].Hh, plans[0].Lmax
    loc = [local_index(S_txt, S_img, N, g) for g in range(N)]
    xs = [[t[:, loc[g]].contiguous().cuda() for t in (q, k, v)] for g in range(N)]
    # a2: pack
    send = []
    for g in range(N):
        sb = torch.zeros((u, 3, B, Lmax, Hh, D), dtype=dt, device="cuda")
        if u > 1:
            for t in range(3):
                usp.uly_pack(xs[g][t], sb, B=B, L=plans[g].S_loc, Lmax=Lmax, H=H, D=D, u=u, slot=t, nslots=3,
                             elem_bytes=eb)
        send.append(sb)
    # a3: all-to-all within each Ulysses row {i*u + p}: recv_g[p] = send_{i*u+p}[j]
    blocks = []
    for g in range(N):
        i, j = g // u, g % u
        if u > 1:
            recv = torch.stack([send[i * u + p][j] for p in range(u)])
            lens = [plans[i * u + p].S_loc for p in range(u)]
            Sb = plans[g].S_blk
            blk = [torch.empty((B, Sb, Hh, D), dtype=dt, device="cuda") for _ in range(3)]
            for t in range(3):  # a4: unpack
                usp.uly_unpack(recv, blk[t], B=B, Lmax=Lmax, Hh=Hh, D=D, u=u, lens=lens, slot=t, nslots=3,
                               elem_bytes=eb)
            # data movement is exact: the block is the ring block's rows, head block j (C6/C7)
            rows_i = torch.cat([loc[i * u + p] for p in range(u)])
            for t, src in enumerate((q, k, v)):
                want = src[:, rows_i][:, :, j * Hh:(j + 1) * Hh].cuda()
                assert torch.equal(blk[t], want), f"rank {g} slot {t}: pack/a2a/unpack mismatch"
        else:
            blk = xs[g]
        blocks.append(blk)
    S_sp = S_txt + S_img
    blk_off = [sum(plans[x * u].S_blk for x in range(ib)) for ib in range(r)]
    kvbuf = [torch.full((2, B, Hh, S_sp, D), float("nan"), dtype=dt, device="cuda") for _ in range(N)] \
        if kv_out is not None else None

    def retain(g, kb, vb, src):
        Sx = plans[src * u].S_blk
        st = (Sx * Hh * D, Hh * D, D)
        usp.kv_retain(kb, vb, kvbuf[g], B=B, Hh=Hh, S_blk=Sx, S_total=S_sp, seq_off=blk_off[src], D=D, strides=st)

    # a5-a8: ring loop per rank; final O/LSE written through the rowmap into the reverse-a2a buffer
    ochunk_o = align16(B * Lmax * Hh * D * eb)
    ochunk = ochunk_o + align16(B * Hh * Lmax * 4)
    osend, outs = [], []
    for g in range(N):
        P = plans[g]
        i, j = g // u, g % u
        Sb = P.S_blk
        qb = blocks[g][0]
        if u > 1:
            ob = torch.zeros(u * ochunk, dtype=torch.uint8, device="cuda")
            fmap = make_fmap(B, Lmax, Hh, D, list(P.seg_off), u, ochunk, eb)
            dst, dst_l = ob.data_ptr(), ob.data_ptr() + ochunk_o
        else:
            o_final = torch.empty((B, P.S_loc, H, D), dtype=dt, device="cuda")
            l_final = torch.empty((B, H, P.S_loc), dtype=torch.float32, device="cuda")
            fmap = usp.RowMap.plain(B, P.S_loc, H, D)
            dst, dst_l = o_final, l_final
            ob = (o_final, l_final)
        qs = (Sb * Hh * D, Hh * D, D)
        if kvbuf is not None:
            retain(g, blocks[g][1], blocks[g][2], i)
        if r == 1:
            usp.attn_fwd(qb, blocks[g][1], blocks[g][2], dst, dst_l, B=B, H=Hh, Sq=Sb, Skv=Sb, D=D, q_strides=qs,
                         kv_strides=qs, omap=fmap, dtype=1 if f32 else 0, out_f32=int(f32))
        else:
            acc_o = torch.empty((B, Sb, Hh, D), dtype=torch.float32, device="cuda")
            acc_l = torch.empty((B, Hh, Sb), dtype=torch.float32, device="cuda")
            tmp_o, tmp_l = torch.empty_like(acc_o), torch.empty_like(acc_l)
            amap = usp.RowMap.plain(B, Sb, Hh, D)
            for s in range(r):
                src = P.ring_src[s]
                assert src == (i - s) % r
                kb, vb = blocks[src * u + j][1], blocks[src * u + j][2]  # block held after s ring steps
                if kvbuf is not None and s > 0:
                    retain(g, kb, vb, src)
                Skv = P.ring_rows[s]
                ks = (Skv * Hh * D, Hh * D, D)
                o_s, l_s = (acc_o, acc_l) if s == 0 else (tmp_o, tmp_l)
                usp.attn_fwd(qb, kb, vb, o_s, l_s, B=B, H=Hh, Sq=Sb, Skv=Skv, D=D, q_strides=qs, kv_strides=ks,
                             omap=amap, dtype=1 if f32 else 0, out_f32=1)
                if s > 0:
                    last = s == r - 1
                    usp.lse_merge(acc_o, acc_l, tmp_o, tmp_l, B=B, S=Sb, Hh=Hh, D=D,
                                  final=dst if last else None, final_lse=dst_l if last else None,
                                  final_map=fmap if last else None, final_dtype=1 if f32 else 0)
        osend.append(ob)
    # a9-a10: reverse all-to-all (copies) and unpack to [B, L, H, D] / [B, H, L]
    for g in range(N):
        P = plans[g]
        i, j = g // u, g % u
        if u == 1:
            outs.append(osend[g])
            continue
        orecv = torch.stack([osend[i * u + p].view(u, ochunk)[j] for p in range(u)]).contiguous()
        out = torch.empty((B, P.S_loc, H, D), dtype=dt, device="cuda")
        lse = torch.empty((B, H, P.S_loc), dtype=torch.float32, device="cuda")
        usp.uly_unpack_out(orecv.data_ptr(), orecv.data_ptr() + ochunk_o, ochunk, ochunk, out, lse, B=B, L=P.S_loc,
                           Lmax=Lmax, Hh=Hh, D=D, u=u, elem_bytes=eb)
        # the rows of rank g inside peer p's block output, before the reverse exchange
        seg = [plans[i * u + p].seg_off for p in range(u)]
        for p in range(u):
            peer = osend[i * u + p].view(u, ochunk)[j][:ochunk_o].view(dt).view(B, Lmax, Hh, D)[:, :P.S_loc]
            assert torch.equal(out[:, :, p * Hh:(p + 1) * Hh], peer), f"rank {g} peer {p}: reverse unpack mismatch"
        outs.append((out, lse))
    torch.cuda.synchronize()
    if kv_out is not None:
        kv_out.extend(kvbuf)
    return outs, loc


SPLITS = [(2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2), (2, 4), (1, 8)]


@pytest.mark.parametrize("u,r", SPLITS, ids=lambda x: str(x))
@pytest.mark.parametrize("B,H,S_txt,S_img,D", [(2, 8, 33, 400, 64), (1, 8, 0, 1024, 128), (2, 8, 0, 700, 72)])
def test_virtual_usp_bf16(u, r, B, H, S_txt, S_img, D):
    S = S_txt + S_img
    q, k, v = qkv(B, S, H, D, seed=100 + u * 10 + r)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, u, r)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        assert_bf16(errors(o, l, ref_o[:, idx], ref_l[:, :, idx]))


@pytest.mark.parametrize("u,r", [(2, 2), (4, 1), (1, 4)], ids=lambda x: str(x))
def test_virtual_usp_f32(u, r):
    B, H, S_txt, S_img, D = 1, 4, 9, 150, 64
    q, k, v = qkv(B, S_txt + S_img, H, D, seed=7, dtype=torch.float32)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, u, r, f32=True)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        assert_f32(errors(o, l, ref_o[:, idx], ref_l[:, :, idx]))


def test_virtual_usp_toy_2x2_config0():
    """BASELINE.json configs[0]: toy B=1, H=4, D=64, 1024 tokens, Ulysses=2 x Ring=2 vs the oracle."""
    w = WORKLOADS["toy"]
    q, k, v = qkv(w.B, w.S, w.H, w.D, seed=seed_for(w))
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    outs, loc = run_virtual_usp(q, k, v, w.S_txt, w.S_img, 2, 2)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        assert_bf16(errors(o, l, ref_o[:, idx], ref_l[:, :, idx]))


def test_virtual_usp_deterministic():
    q, k, v = qkv(1, 300, 4, 64, seed=3)
    a, _ = run_virtual_usp(q, k, v, 10, 290, 2, 2)
    b, _ = run_virtual_usp(q, k, v, 10, 290, 2, 2)
    for (o1, l1), (o2, l2) in zip(a, b):
        assert torch.equal(o1, o2) and torch.equal(l1, l2)


@pytest.mark.parametrize("u,r", [(8, 1), (2, 4), (1, 8)], ids=lambda x: str(x))
def test_virtual_usp_flux_full_size_sampled(u, r):
    """Flux.1 4096px (BASELINE.json configs[3]) split over 8 virtual ranks at full size: the exact
    per-rank kernel launches of an 8-GPU USP call (pack, unpack, ring of attention + merge, final
    write into the reverse exchange buffer, unpack), checked on sampled rows of two heads per rank."""
    w = WORKLOADS["flux"]
    q, k, v = qkv(w.B, w.S, w.H, w.D, seed=seed_for(w))  # CPU, bit-reproducible
    outs, loc = run_virtual_usp(q, k, v, w.S_txt, w.S_img, u, r)
    heads = [1, w.H - 2]
    qs, ks, vs = (f64(t[:, :, heads]) for t in (q, k, v))
    for g in (0, 3, 7):
        o, l = outs[g]
        L = o.shape[1]
        pick = sample_rows(L, 24, extra=[63, 64, L - 1])
        rows = loc[g][pick].numpy()
        ref_o, ref_l = oracle.attention_rows(qs, ks, vs, rows)
        assert_bf16(errors(o[:, pick.cuda()][:, :, heads], l[:, heads][:, :, pick.cuda()], ref_o, ref_l))


def test_usp_call_is_cuda_graph_capturable():
    """The call never allocates nor synchronises the host (workspace is reserved up front), so it
    can be captured in a CUDA graph and replayed; replays give the same bits as eager calls."""
    B, H, S_txt, S_img, D = 1, 4, 31, 480, 128
    q, k, v = (t.cuda() for t in qkv(B, S_txt + S_img, H, D, seed=21))
    with usp.Comm(1, 1) as comm:
        out = torch.empty_like(q)
        lse = torch.empty((B, H, S_txt + S_img), dtype=torch.float32, device="cuda")
        usp.attention(q, k, v, S_txt=S_txt, S_img=S_img, comm=comm, out=out, lse=lse)  # reserve + warm up
        torch.cuda.synchronize()
        ref_o, ref_l = out.clone(), lse.clone()
        out.zero_(); lse.zero_()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                usp.attention(q, k, v, S_txt=S_txt, S_img=S_img, comm=comm, out=out, lse=lse)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref_o) and torch.equal(lse, ref_l)


@pytest.mark.parametrize("u,r,S_txt,S_img", [(2, 2, 3, 200), (1, 4, 2, 130), (4, 1, 0, 9), (2, 2, 5, 0)],
                         ids=["txt<N", "txt<N-ring", "tiny", "text-only"])
def test_virtual_usp_degenerate_shards(u, r, S_txt, S_img):
    """Shards where some ranks hold no text tokens, a tiny sequence (ragged rows of 2-3 tokens per
    rank) and a text-only sequence (reading C5: only an EMPTY shard is an error)."""
    B, H, D = 2, 4, 64
    q, k, v = qkv(B, S_txt + S_img, H, D, seed=77 + u + r)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, u, r)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        assert_bf16(errors(o, l, ref_o[:, idx], ref_l[:, :, idx]))


def test_virtual_usp_peaky_ring_merge():
    """Large-magnitude scores (q, k x3, so logits x9): ring partials with very different LSEs must
    merge exactly.  Rows this peaky reach |O*| ~ max|V| ~ 4.5, where one bf16 output ulp (0.031)
    alone exceeds 2e-2, so the max-abs gate is taken relative to max(1, |O*|) (reading C11)."""
    B, H, D, S_txt, S_img = 1, 4, 128, 40, 600
    q, k, _ = qkv(B, S_txt + S_img, H, D, seed=91, scale=3.0)
    _, _, v = qkv(B, S_txt + S_img, H, D, seed=92)
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, 1, 4)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        e = errors(o, l, ref_o[:, idx], ref_l[:, :, idx])
        assert e["o_maxscaled"] <= 2e-2 and e["o_rell2"] <= 1e-2 and e["lse_maxabs"] <= 1e-3, e


def test_usp_n1_single_token():
    q, k, v = (t.cuda() for t in qkv(1, 1, 2, 64, seed=5))
    with usp.Comm(1, 1) as comm:
        out, lse = usp.attention(q, k, v, S_txt=0, S_img=1, comm=comm)
        torch.cuda.synchronize()
    assert torch.equal(out, v)  # one key: O = V exactly
    s = float((q.float() * k.float()).sum()) / 8.0
    assert abs(float(lse[0, 0, 0]) - (float((q[0, 0, 0].float() * k[0, 0, 0].float()).sum()) / 8.0)) < 1e-5


# ------------------------------------------------------------------ KV retention
@pytest.mark.parametrize("u,r", [(2, 1), (1, 2), (2, 2), (4, 2), (2, 4), (1, 8)], ids=lambda x: str(x))
def test_virtual_usp_kv_retention(u, r):
    """Every virtual rank's KV buffer equals the oracle's (reading R2) bit for bit, ranks
    of one head block agree, and the attention result is unchanged."""
    B, H, S_txt, S_img, D = 2, 8, 33, 400, 64
    q, k, v = qkv(B, S_txt + S_img, H, D, seed=900 + u * 10 + r)
    kv = []
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, u, r, kv_out=kv)
    for g in range(u * r):
        want = oracle.kv_keep(f64(k), f64(v), S_txt, u, r, g)
        assert np.array_equal(f64(kv[g]), want), f"rank {g}: retained KV differs from the oracle"
        assert torch.equal(kv[g], kv[g % u])
    ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        assert_bf16(errors(o, l, ref_o[:, idx], ref_l[:, :, idx]))


@pytest.mark.parametrize("S_txt,S_img,D", [(0, 300, 64), (77, 1000, 128), (5, 700, 72)])
def test_usp_attention_kv_n1(S_txt, S_img, D):
    """xdit_usp_attention_kv at N = 1 (through the C ABI): same output as xdit_usp_attention and the
    retained buffer is the head-major K, V (oracle.kv_keep with u = r = 1)."""
    B, H = 2, 4
    q, k, v = (t.cuda() for t in qkv(B, S_txt + S_img, H, D, seed=77 + D))
    buf = torch.full((2, B, H, S_txt + S_img, D), float("nan"), dtype=torch.bfloat16, device="cuda")
    with usp.Comm(1, 1) as comm:
        o1, l1 = usp.attention(q, k, v, S_txt=S_txt, S_img=S_img, comm=comm)
        o2, l2 = usp.attention(q, k, v, S_txt=S_txt, S_img=S_img, comm=comm, kv_keep=buf)
        torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert np.array_equal(f64(buf), oracle.kv_keep(f64(k), f64(v), S_txt, 1, 1, 0))
