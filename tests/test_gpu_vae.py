"""Patch-parallel VAE decode on the GPU (reading R5).

* `xdit_vae_conv3x3` against the fp64 oracle conv (fp32 FFMA: relative error ~1e-6);
* the decode on one device against `oracle.vae.serial_decode`;
* bands with halo rows (virtual devices, in one process) reproduce the one-device decode BIT FOR BIT
  -- the kernel sums every pixel in one fixed order, so patch parallelism is exact;
* one process per band, halos over NCCL: tests/test_gpu_multiproc.py.
"""
import numpy as np
import pytest
import torch

from oracle import vae as ovae
from paper_2411_01738_b200 import vae

pytestmark = pytest.mark.gpu


def make_layers(c, widths, seed, out=3):
    rng = np.random.default_rng(seed)
    L, ci = [], c
    for co in list(widths) + [out]:
        L.append(((rng.standard_normal((co, ci, 3, 3)) / np.sqrt(9 * ci)).astype(np.float32),
                  (rng.standard_normal(co) * 0.1).astype(np.float32)))
        ci = co
    return L


@pytest.mark.parametrize("H,Ci,W,Co,act", [(5, 3, 7, 4, 0), (40, 20, 70, 33, 1), (17, 64, 33, 16, 0), (3, 8, 129, 130, 1)])
def test_conv3x3_vs_oracle(H, Ci, W, Co, act):
    rng = np.random.default_rng(H * W)
    x = rng.standard_normal((H, Ci, W)).astype(np.float32)
    w = rng.standard_normal((Co, Ci, 3, 3)).astype(np.float32)
    b = rng.standard_normal(Co).astype(np.float32)
    ext = torch.zeros(H + 2, Ci, W)
    ext[1:-1] = torch.from_numpy(x)
    got = vae.conv(ext.cuda(), torch.from_numpy(w).cuda(), torch.from_numpy(b).cuda(), bool(act)).cpu().double().numpy()
    want = ovae.conv3x3(x, w, b)
    if act:
        want = ovae.upsample2(ovae.silu(want))
    scale = np.abs(w).sum(axis=(1, 2, 3)).max() * np.abs(x).max()
    assert np.abs(got - want).max() <= 1e-6 * scale


def test_decode_vs_oracle_and_bands_bitwise():
    lat = np.random.default_rng(5).standard_normal((24, 4, 20)).astype(np.float32)
    L = make_layers(4, (32, 16), 6)
    dec = vae.Decoder(L)
    img = vae.decode(torch.from_numpy(lat).cuda(), dec)
    want = ovae.serial_decode(lat, [(w.astype(np.float64), b.astype(np.float64)) for w, b in L])
    got = img.cpu().double().numpy()
    assert got.shape == want.shape == (96, 3, 80)
    assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()
    # virtual devices: every band convolved with its neighbours' boundary rows as halos
    for N in (2, 3, 4):
        x = [torch.from_numpy(lat[o:o + n]).cuda() for o, n in vae.bands(24, N)]
        for i, (w, b) in enumerate(dec.layers):
            ext = []
            for g, xb in enumerate(x):
                e = torch.zeros((xb.shape[0] + 2,) + tuple(xb.shape[1:]), device="cuda")
                e[1:-1] = xb
                if g > 0:
                    e[0] = x[g - 1][-1]
                if g + 1 < N:
                    e[-1] = x[g + 1][0]
                ext.append(e)
            x = [vae.conv(e, w, b, i < len(dec.layers) - 1) for e in ext]
        assert torch.equal(torch.cat(x), img), f"N={N}: banded decode differs from the one-device decode"


def test_conv_errors():
    from paper_2411_01738_b200 import usp
    x = torch.zeros(4, 2, 8, device="cuda")
    with pytest.raises(usp.XditError) as e:
        usp._check(usp.lib().xdit_vae_conv3x3(usp._ptr(x), 2, 0, 8, usp._ptr(x), usp._ptr(x), usp._ptr(x), 1, 0, None),
                   "xdit_vae_conv3x3")
    assert e.value.status == "INVALID_ARG"


def _bf(a):
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16)


@pytest.mark.parametrize("H,Ci,W,Co,act", [(3, 64, 128, 128, 0), (5, 40, 200, 130, 1), (4, 128, 96, 3, 0),
                                           (2, 8, 300, 64, 1), (6, 256, 130, 256, 1)])
def test_conv3x3_tc_vs_oracle(H, Ci, W, Co, act):
    """tcgen05 implicit-GEMM conv (bf16 in, fp32 accumulate, bf16 out) vs the fp64 oracle on the same
    bf16-rounded inputs: one bf16 rounding of the output (2^-8 relative) plus fp32 accumulation.
    Ragged pixel strips (W % 128), output-channel blocks (Co % 128) and channel chunks (Ci % 64)."""
    rng = np.random.default_rng(H * W + Ci)
    x = _bf(rng.standard_normal((H, Ci, W)))
    w = _bf(rng.standard_normal((Co, Ci, 3, 3)) / np.sqrt(9 * Ci))
    b = torch.from_numpy(rng.standard_normal(Co).astype(np.float32))
    dec = vae.Decoder([(w.float().numpy(), b.numpy())], tc=True)
    wt, bd = dec.layers[0]
    ext = torch.zeros(H + 2, W, Ci, dtype=torch.bfloat16)
    ext[1:-1] = x.permute(0, 2, 1)
    got = vae.conv(ext.cuda(), wt, bd, bool(act)).cpu().double().numpy()  # [H'][W'][Co(+pad)]
    want = ovae.conv3x3(x.double().numpy(), w.double().numpy(), b.double().numpy())
    if act:
        want = ovae.upsample2(ovae.silu(want))
    want = want.transpose(0, 2, 1)
    got = got[:, :, :Co]
    scale = np.abs(w.double().numpy()).sum(axis=(1, 2, 3)).max() * np.abs(x.double().numpy()).max()
    assert np.all(np.abs(got - want) <= 2.0 ** -8 * np.abs(want) + 1e-5 * scale)


def test_decode_tc_vs_oracle_and_bands_bitwise():
    lat = np.random.default_rng(7).standard_normal((24, 4, 150)).astype(np.float32)
    L = make_layers(4, (64, 32), 8)
    dec = vae.Decoder(L, tc=True)
    x0 = dec.prepare(torch.from_numpy(lat).cuda())
    img = vae.decode(x0, dec)  # [96][600][8] (3 channels + zero padding)
    want = ovae.serial_decode(lat, [(w.astype(np.float64), b.astype(np.float64)) for w, b in L]).transpose(0, 2, 1)
    got = img[:, :, :3].double().cpu().numpy()
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 2e-2, rel  # bf16 activations between layers
    for N in (2, 3, 4):
        x = [x0[o:o + n] for o, n in vae.bands(24, N)]
        for i, (w, b) in enumerate(dec.layers):
            ext = []
            for g, xb in enumerate(x):
                e = torch.zeros((xb.shape[0] + 2,) + tuple(xb.shape[1:]), dtype=xb.dtype, device="cuda")
                e[1:-1] = xb
                if g > 0:
                    e[0] = x[g - 1][-1]
                if g + 1 < N:
                    e[-1] = x[g + 1][0]
                ext.append(e)
            x = [vae.conv(e, w, b, i < len(dec.layers) - 1) for e in ext]
        assert torch.equal(torch.cat(x), img), f"N={N}: banded tc decode differs from the one-device decode"
