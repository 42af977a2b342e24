"""Rank bodies of the multi-process -m gpu tests (tests/_mp.py launches them).

Every body runs the PRODUCT call path -- paper_2411_01738_b200.usp.attention and friends, i.e. the
C ABI of libxdit_usp.so with NCCL between the ranks -- on seeded inputs that every rank regenerates
identically, and checks ITS OWN rows against the fp64 oracle ("the computation yields the same
results as the serial version").  Results are appended to `res["checks"]`.
"""
import numpy as np

from tests._mp import setup, teardown


def _local_index(usp, torch, S_txt, S_img, N, g):
    to, tl, io, il = usp.shard(S_txt, S_img, N, g)
    return torch.cat([torch.arange(to, to + tl), S_txt + torch.arange(io, io + il)])


# ------------------------------------------------------------------------------ USP, small shapes
def usp_splits(rank, world, port, res, splits, cases, backend="nccl"):
    """Every (ulysses, ring) split of the world on small ragged shapes: each rank's output and LSE
    against the full fp64 oracle, bitwise run-to-run determinism (reading C12), the retained KV
    buffer bit-exact against oracle.kv_keep (NEXT 1, R2), and the per-phase timing record."""
    import torch

    import oracle
    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv
    from tests._util import assert_bf16, assert_f32, errors, f64

    setup(rank, world, port, backend)
    for (u, r) in splits:
        comm = usp.Comm(u, r)
        if backend == "nccl":
            assert comm.source.startswith("torch"), comm.source
        for ci, (B, H, S_txt, S_img, D, dt, keep) in enumerate(cases):
            dtype = torch.float32 if dt == "f32" else torch.bfloat16
            S = S_txt + S_img
            q, k, v = qkv(B, S, H, D, seed=500 + ci, dtype=dtype)
            idx = _local_index(usp, torch, S_txt, S_img, world, rank)
            ql, kl, vl = (t[:, idx].contiguous().cuda() for t in (q, k, v))
            kv_keep = torch.zeros(2, B, H // u, S, D, dtype=dtype, device="cuda") if keep else None
            comm.profile(True)
            o1, l1 = usp.attention(ql, kl, vl, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r,
                                   kv_keep=kv_keep)
            ph = comm.phases()
            comm.profile(False)
            o2, l2 = usp.attention(ql, kl, vl, S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r)
            torch.cuda.synchronize()
            ref_o, ref_l = oracle.attention_rows(f64(q), f64(k), f64(v), idx.numpy())
            e = errors(o1, l1, ref_o, ref_l)
            (assert_f32 if dt == "f32" else assert_bf16)(e)
            assert torch.equal(o1, o2) and torch.equal(l1, l2), "second call differs"
            if keep:
                ref_kv = oracle.kv_keep(f64(k), f64(v), S_txt, u, r, rank)
                assert (f64(kv_keep) == ref_kv).all(), "kv_keep differs from oracle.kv_keep"
            assert ph is not None and len(ph["attn_ms"]) == r and ph["total_ms"] > 0, ph
            assert (ph["a2a_in_bytes"] > 0) == (u > 1) and len(ph["ring_bytes"]) == r - 1, ph
            res["checks"].append({"u": u, "r": r, "case": ci, **e})
        torch.cuda.synchronize()
        comm.destroy()
    teardown()


# ------------------------------------------------------------------ BASELINE configs, full size
def _heads_sample(H, u):
    """Heads checked against the oracle: the first and last head of every Ulysses block (<= 6)."""
    Hh = H // u
    hs = sorted({j * Hh for j in range(u)} | {j * Hh + Hh - 1 for j in range(u)})
    if len(hs) > 6:
        hs = hs[:3] + hs[-3:]
    return hs


def baseline_configs(rank, world, port, res, cases, rows_per_rank=24):
    """BASELINE.json workloads at FULL size through the product call: cases = [(workload, cfg, u, r)],
    cfg * u * r == world.  CFG groups are independent SP groups on their own batch (the
    group's global inputs seeded per group, as bench.py does); each rank checks a sample of its own
    rows -- the first and last row of its text and image shards and a strided sample -- on the first
    and last head of every Ulysses block, against the fp64 oracle evaluated on exactly those
    (row, head) pairs (rows are independent, so the sample is an exact subset check)."""
    import torch
    import torch.distributed as dist

    import oracle
    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import WORKLOADS, qkv, seed_for
    from tests._util import assert_bf16, errors

    dev = setup(rank, world, port)
    for (name, cfg, u, r) in cases:
        w = WORKLOADS[name]
        sp = u * r
        assert cfg * sp == world
        c, g = rank // sp, rank % sp
        groups = [dist.new_group(list(range(x * sp, (x + 1) * sp))) for x in range(cfg)]
        B = w.B * w.cfg // cfg
        comm = usp.Comm(u, r, group=groups[c] if sp > 1 else None)
        gq, gk, gv = qkv(B, w.S, w.H, w.D, seed=seed_for(w, c), device=torch.device("cuda", dev))
        to, tl, io, il = usp.shard(w.S_txt, w.S_img, sp, g)
        idx = torch.cat([torch.arange(to, to + tl), w.S_txt + torch.arange(io, io + il)])
        ql, kl, vl = (t.index_select(1, idx.to(gq.device)).contiguous() for t in (gq, gk, gv))
        out, lse = usp.attention(ql, kl, vl, S_txt=w.S_txt, S_img=w.S_img, comm=comm, ulysses=u, ring=r)
        torch.cuda.synchronize()
        L = len(idx)
        loc = set(np.linspace(0, L - 1, rows_per_rank).astype(int).tolist()) | {0, L - 1}
        if tl:
            loc |= {tl - 1, tl}
        loc = sorted(x for x in loc if 0 <= x < L)
        hs = _heads_sample(w.H, u)
        grow = idx[loc]
        hsel = torch.tensor(hs, device=gq.device)
        qs = gq[:, grow.to(gq.device)].index_select(2, hsel)
        ks, vs = (t.index_select(2, hsel) for t in (gk, gv))
        f = lambda t: t.to("cpu", torch.float64).numpy()  # noqa: E731
        ref_o, ref_l = oracle.attention(f(qs), f(ks), f(vs))
        got_o = out[:, loc].index_select(2, hsel.to(out.device))
        got_l = lse[:, :, loc].index_select(1, hsel.to(lse.device))
        e = errors(got_o, got_l, ref_o, ref_l)
        assert_bf16(e)
        res["checks"].append({"workload": name, "cfg": cfg, "u": u, "r": r, "rows": len(loc), "heads": hs, **e})
        del gq, gk, gv
        torch.cuda.synchronize()
        comm.destroy()
        dist.barrier()
    teardown()


# ------------------------------------------------------------------------------ CUDA graph replay
def graph_replay(rank, world, port, res, splits):
    """The multi-rank call (NCCL sends/receives on the caller's and the side stream) captured in a
    CUDA graph: every replay, and an eager call between replays, equals the eager result bitwise."""
    import torch

    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv

    setup(rank, world, port)
    for (u, r) in splits:
        comm = usp.Comm(u, r)
        S_txt, S_img, H, D = 7, 300, 8, 64
        q, k, v = qkv(1, S_txt + S_img, H, D, seed=11 + u)
        idx = _local_index(usp, torch, S_txt, S_img, world, rank)
        ql, kl, vl = (t[:, idx].contiguous().cuda() for t in (q, k, v))
        kw = dict(S_txt=S_txt, S_img=S_img, comm=comm, ulysses=u, ring=r)
        ref_o, ref_l = usp.attention(ql, kl, vl, **kw)
        torch.cuda.synchronize()
        out, lse = torch.empty_like(ref_o), torch.empty_like(ref_l)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                usp.attention(ql, kl, vl, out=out, lse=lse, **kw)
        torch.cuda.synchronize()
        for rep in range(4):
            out.zero_()
            lse.zero_()
            g.replay()
            if rep == 1:
                o2, l2 = usp.attention(ql, kl, vl, **kw)
                torch.cuda.synchronize()
                assert torch.equal(o2, ref_o) and torch.equal(l2, ref_l), "eager call after a replay differs"
            torch.cuda.synchronize()
            assert torch.equal(out, ref_o) and torch.equal(lse, ref_l), f"replay {rep} differs (u={u}, r={r})"
        res["checks"].append({"u": u, "r": r})
        del g
        comm.destroy()
    teardown()


# ------------------------------------------------------------------------------ error paths
def error_paths(rank, world, port, res):
    """Errors are return codes raised before anything is enqueued (include/xdit_usp.h): a call larger
    than the reservation -> WORKSPACE, (u, r) other than the handle's -> COMM_MISMATCH, a p2p op on
    an out-of-range peer -> INVALID_ARG, KV-buffer rows beyond S_buf -> INVALID_ARG; a valid call
    afterwards still runs (no half-enqueued collective stranded a peer)."""
    import torch

    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv

    setup(rank, world, port)
    L = usp.lib()
    comm = usp.Comm(world, 1)
    H, D = 2 * world, 64
    comm.reserve(1, H, 0, 64 * world, D, 2)
    q = torch.zeros(1, 4096, H, D, dtype=torch.bfloat16, device="cuda")
    rc = L.xdit_usp_attention(usp._ptr(q), usp._ptr(q), usp._ptr(q), usp._ptr(q), None, 1, H, 0, 4096 * world, D,
                              world, 1, usp._stream(None), comm.handle)
    assert usp.XDIT_STATUS[rc] == "WORKSPACE", (rc, usp.last_error())
    res["checks"].append("workspace")
    rc = L.xdit_usp_attention(usp._ptr(q), usp._ptr(q), usp._ptr(q), usp._ptr(q), None, 1, H, 0, 64 * world, D,
                              1, world, usp._stream(None), comm.handle)
    assert usp.XDIT_STATUS[rc] == "COMM_MISMATCH", (rc, usp.last_error())
    res["checks"].append("mismatch")
    try:
        comm.p2p([(world, "send", q)])
        raise AssertionError("p2p to an out-of-range peer was accepted")
    except usp.XditError as e:
        assert e.status == "INVALID_ARG", e
    res["checks"].append("p2p_peer")
    buf = torch.zeros(2, 1, H // world, 64, D, dtype=torch.bfloat16, device="cuda")
    rc = L.xdit_usp_attention_buf(usp._ptr(q), usp._ptr(q), usp._ptr(q), usp._ptr(q), None, usp._ptr(buf), 1, H, 0,
                                  64 * world, D, world, 1, 64, 0, 1, 0, usp._stream(None), comm.handle)
    assert usp.XDIT_STATUS[rc] == "INVALID_ARG", (rc, usp.last_error())
    res["checks"].append("buf_rows")
    S_txt, S_img = 5, 64 * world
    gq, gk, gv = qkv(1, S_txt + S_img, H, D, seed=3)
    idx = _local_index(usp, torch, S_txt, S_img, world, rank)
    o, _ = usp.attention(*(t[:, idx].contiguous().cuda() for t in (gq, gk, gv)), S_txt=S_txt, S_img=S_img, comm=comm,
                         ulysses=world, ring=1)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all()
    res["checks"].append("valid_after")
    comm.destroy()
    teardown()


# ------------------------------------------------------------------------------ NEXT 2: CFG tail
def cfg_tail(rank, world, port, res, cases):
    """CFG step tail over NCCL (NEXT 2, reading R3): rank 0 = conditional, rank 1 = unconditional;
    every rank's combined eps against oracle.cfg_combine (exact at g = 0, 1)."""
    import torch

    import oracle
    from paper_2411_01738_b200 import usp

    setup(rank, world, port)
    comm = usp.Comm(2, 1)
    for ci, (n, dt, g) in enumerate(cases):
        dtype = torch.float32 if dt == "f32" else torch.bfloat16
        gen = torch.Generator().manual_seed(70 + ci)
        both = torch.randn(2, n, generator=gen).to(dtype)
        out = usp.cfg_tail(both[rank].cuda(), g, comm=comm)
        out2 = usp.cfg_tail(both[rank].cuda(), g, comm=comm)
        torch.cuda.synchronize()
        c, u = both[0].double().numpy(), both[1].double().numpy()
        ref = oracle.cfg_combine(c, u, g)
        got = out.double().cpu().numpy()
        bound = (abs(g) * np.abs(c) + abs(1 - g) * np.abs(u)) * 2.0 ** -22 + (np.abs(ref) * 2.0 ** -8 if dt == "bf16" else 0)
        assert np.all(np.abs(got - ref) <= bound + 1e-30)
        assert torch.equal(out, out2)
        if g in (0.0, 1.0):
            assert torch.equal(out.cpu(), both[1 if g == 0.0 else 0]), "combine not exact at g in {0, 1}"
        res["checks"].append({"case": ci})
    comm.destroy()
    teardown()


# ------------------------------------------------------------------------------ NEXT 4: VAE bands
def vae_bands(rank, world, port, res, cases):
    """Patch-parallel VAE decode, one process per row band, halos over NCCL (vae.decode_band): each
    band equals the same rows of the one-device GPU decode bit for bit and of the fp64 oracle."""
    import torch

    from oracle import vae as ovae
    from paper_2411_01738_b200 import usp, vae

    setup(rank, world, port)
    comm = usp.Comm(world, 1)
    for ci, (h, c, w, widths, tc) in enumerate(cases):
        rng = np.random.default_rng(80 + ci)
        lat = rng.standard_normal((h, c, w)).astype(np.float32)
        L, cin = [], c
        for co in list(widths) + [3]:
            L.append(((rng.standard_normal((co, cin, 3, 3)) / np.sqrt(9 * cin)).astype(np.float32),
                      (rng.standard_normal(co) * 0.1).astype(np.float32)))
            cin = co
        dec = vae.Decoder(L, tc=tc)
        o, n = vae.bands(h, world)[rank]
        x0 = dec.prepare(torch.from_numpy(lat).cuda())
        mine = vae.decode_band(x0[o:o + n].contiguous(), dec, comm)
        whole = vae.decode(x0, dec)
        torch.cuda.synchronize()
        up = 2 ** len(widths)
        assert torch.equal(mine, whole[o * up:(o + n) * up]), "band differs from the one-device decode"
        want = ovae.serial_decode(lat, [(a.astype(np.float64), b.astype(np.float64)) for a, b in L])
        want = want[o * up:(o + n) * up]
        if tc:
            got = mine[:, :, :3].permute(0, 2, 1).double().cpu().numpy()
            err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
            assert err <= 2e-2, err
        else:
            err = float(np.abs(mine.cpu().double().numpy() - want).max() / np.abs(want).max())
            assert err <= 1e-5, err
        res["checks"].append({"case": ci, "err": err, "band_rows": int(mine.shape[0])})
    comm.destroy()
    teardown()


# ------------------------------------------------------------------ NEXT 3: PipeFusion (x SP) mesh
def _pf_weights(L, H, D, seed):
    rng = np.random.default_rng(seed)
    return [tuple(rng.uniform(0.2, 0.4, (H, D)).astype(np.float32) for _ in range(2)) +
            (rng.uniform(0.5, 1.5, (H, D)).astype(np.float32), rng.uniform(0.4, 0.8, (H, D)).astype(np.float32))
            for _ in range(L)]


def pipefusion_mesh(rank, world, port, res, meshes, cases):
    """PipeFusion over a pipefusion_degree x sp_degree mesh, one process per device:
    meshes = [(pp, ulysses, ring)] with pp * ulysses * ring == world; cases = [(B, S_txt, S_img, H, D,
    L, T, M, warmup, dtype)].  Stage-0 ranks check the final latent against the fp64 PipeFusion
    oracle with the same (pp, M) -- SP is exact, so the hybrid must not change the staleness pattern
     -- and, for pure PipeFusion (sp = 1), bitwise against the one-device schedule;
    after the run every rank compares its KV buffers with the other ranks of its head block (the
    paper's consistency requirement): identical bit for bit."""
    import torch
    import torch.distributed as dist

    from oracle import pipefusion as opf
    from paper_2411_01738_b200 import pipefusion as pf
    from paper_2411_01738_b200 import usp
    from paper_2411_01738_b200.inputs import qkv

    setup(rank, world, port)
    for (pp, u, r) in meshes:
        sp = u * r
        assert pp * sp == world
        d, g = rank // sp, rank % sp
        stage_groups = [dist.new_group(list(range(x * sp, (x + 1) * sp))) for x in range(pp)]
        chain_groups = [dist.new_group(list(range(y, world, sp))) for y in range(sp)]
        spc = usp.Comm(u, r, group=stage_groups[d] if sp > 1 else None)
        chain = usp.Comm(pp, 1, group=chain_groups[g] if pp > 1 else None)
        for ci, (B, S_txt, S_img, H, D, L, T, M, warmup, dt) in enumerate(cases):
            dtype = torch.float32 if dt == "f32" else torch.bfloat16
            x0 = qkv(B, S_txt + S_img, H, D, seed=40 + ci, dtype=dtype)[0]
            W = _pf_weights(L, H, D, 40 + ci)
            kw = dict(T=T, M=M, warmup=warmup, sigma=0.5, S_txt=S_txt)
            kv_out = []
            x = pf.run_mesh(x0.cuda(), W, stage=d, stages=pp, chain=chain, sp_comm=spc, kv_out=kv_out, **kw)
            torch.cuda.synchronize()
            # KV consistency: ranks (i, j) of one stage with the same head block j hold identical buffers
            if sp > 1 and r > 1:
                for li, kvb in enumerate(kv_out):
                    allb = [torch.empty_like(kvb) for _ in range(sp)]
                    dist.all_gather(allb, kvb.contiguous(), group=stage_groups[d])
                    for q in range(sp):
                        if q % u == g % u:
                            assert torch.equal(allb[q], kvb), f"KV buffer of block {li} differs from SP rank {q}"
            chk = {"pp": pp, "u": u, "r": r, "case": ci}
            if d == 0:
                if sp == 1:
                    same = pf.run(x0.cuda(), pf.SyntheticDiT(W), stages=pp, **kw)
                    torch.cuda.synchronize()
                    assert torch.equal(x, same), "stage processes differ from the one-device schedule"
                W64 = [tuple(a.astype(np.float64) for a in wl) for wl in W]
                if sp == 1:
                    want, _ = opf.pipefusion(x0.double().numpy(), W64, **kw)
                else:  # the hybrid oracle (equal to pure PipeFusion, pinned in test_pipefusion_oracle.py)
                    want, _ = opf.hybrid(x0.double().numpy(), W64, u=u, r=r, **kw)
                got = x.double().cpu().numpy()
                if dt == "f32":
                    err = float(np.abs(got - want).max() / np.abs(want).max())
                    assert err <= 1e-3, err
                else:
                    err = float(np.linalg.norm(got - want) / np.linalg.norm(want))
                    assert err <= 2e-2, err
                chk["err"] = err
            res["checks"].append(chk)
            dist.barrier()
        torch.cuda.synchronize()
        spc.destroy()
        chain.destroy()
        dist.barrier()
    teardown()
