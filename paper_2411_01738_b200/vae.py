"""Patch-parallel VAE decode -- SURVEY §8(f) NEXT 4 (§4.3; reading R5).

Host orchestration only: every conv runs in the library -- `xdit_vae_conv3x3` (SIMT fp32,
activations [H][C][W]) or, with tc=True, `xdit_vae_conv3x3_bf16` (tcgen05 implicit GEMM, bf16
activations [H][W][C], channels padded to a multiple of 8) -- with the stage's SiLU and x2 upsample
fused into the store; halo rows move between devices with xdit_p2p (NCCL).  In both
layouts a row of the feature map is contiguous.  The decoder: per stage a 3x3 conv + SiLU + nearest
x2 upsample, then a final 3x3 conv to 3 channels.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

from . import usp


def bands(h: int, N: int) -> List[Tuple[int, int]]:
    """Balanced contiguous row bands (np.array_split convention) of h latent rows over N devices."""
    if N < 1 or h < N:
        raise ValueError("need 1 <= N <= rows")
    base, rem = divmod(h, N)
    out, off = [], 0
    for g in range(N):
        n = base + (1 if g < rem else 0)
        out.append((off, n))
        off += n
    return out


def _pad8(n: int) -> int:
    return (n + 7) // 8 * 8


class Decoder:
    """layers: [(w [Co][Ci][3][3], b [Co])]; all but the last are upsampling stages.
    tc=False: fp32 weights as given (SIMT kernel); tc=True: bf16 tap-major weights [9][Co][Ci'] with
    Ci' = Ci rounded up to a multiple of 8 (zero rows: exact), for the tcgen05 kernel."""

    def __init__(self, layers: Sequence, device="cuda", tc: bool = False):
        import torch
        self.tc = tc
        self.layers = []
        for w, b in layers:
            w = torch.as_tensor(w, dtype=torch.float32)
            b = torch.as_tensor(b, dtype=torch.float32).contiguous().to(device)
            if tc:
                Co, Ci = w.shape[:2]
                wt = torch.zeros(9, Co, _pad8(Ci))
                wt[:, :, :Ci] = w.permute(2, 3, 0, 1).reshape(9, Co, Ci)
                w = wt.to(torch.bfloat16)
            self.layers.append((w.contiguous().to(device), b))

    def prepare(self, latent):
        """The latent in this decoder's layout: fp32 [h][c][w] as given, or for tc bf16 [h][w][c'] with
        zero channels up to c' (a multiple of 8)."""
        import torch
        if not self.tc:
            return latent
        h, c, w = latent.shape
        x = torch.zeros((h, w, _pad8(c)), dtype=torch.bfloat16, device=latent.device)
        x[:, :, :c] = latent.permute(0, 2, 1)
        return x


def conv(ext, w, b, act_up: bool, stream=None):
    """One decoder conv on a halo-extended band: fp32 ext [H+2][Ci][W] with w [Co][Ci][3][3]
    (xdit_vae_conv3x3), or bf16 ext [H+2][W][Ci] with tap-major w [9][Co][Ci] (xdit_vae_conv3x3_bf16)."""
    import torch
    if ext.dtype == torch.bfloat16:
        Hp2, W, Ci = ext.shape
        H, Co = Hp2 - 2, w.shape[1]
        # channels padded to a multiple of 8 (zeros): the kernel's TMA stores and the next conv's loads
        out = torch.empty((2 * H, 2 * W, _pad8(Co)) if act_up else (H, W, _pad8(Co)), dtype=torch.bfloat16,
                          device=ext.device)
        usp._check(usp.lib().xdit_vae_conv3x3_bf16(usp._ptr(ext), H, Ci, W, usp._ptr(w), usp._ptr(b), usp._ptr(out),
                                                   Co, 1 if act_up else 0, usp._stream(stream)), "xdit_vae_conv3x3_bf16")
        return out
    Hp2, Ci, W = ext.shape
    H, Co = Hp2 - 2, w.shape[0]
    out = torch.empty((2 * H, Co, 2 * W) if act_up else (H, Co, W), dtype=torch.float32, device=ext.device)
    usp._check(usp.lib().xdit_vae_conv3x3(usp._ptr(ext), H, Ci, W, usp._ptr(w), usp._ptr(b), usp._ptr(out), Co,
                                          1 if act_up else 0, usp._stream(stream)), "xdit_vae_conv3x3")
    return out


def decode(latent, dec: Decoder):
    """Single-device decode: the whole image is one band with zero halo rows.  latent: fp32 [h][c][w]
    (SIMT decoder) or already in the tc decoder's layout (Decoder.prepare)."""
    import torch
    x = latent
    for i, (w, b) in enumerate(dec.layers):
        ext = torch.zeros((x.shape[0] + 2,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        ext[1:-1].copy_(x)
        x = conv(ext, w, b, i < len(dec.layers) - 1)
    return x


def decode_band(band, dec: Decoder, comm):
    """Patch-parallel decode, one process per band: this rank (= comm.rank of N) holds latent rows
    `band` ([h_g][c][w] fp32, or [h_g][w][c'] bf16 for a tc decoder).  Before every conv it sends
    its first row to rank g-1 and its last row to rank g+1 (their bottom / top halos) and receives
    theirs into its own halo rows -- one xdit_p2p group (NCCL) per conv, "the exchange of the
    boundary data for convolutional operators"; the image edges keep zero halos (= the
    serial zero padding).  Collective over the comm's ranks.  Returns this rank's decoded band."""
    import torch
    N, g = comm.size, comm.rank
    st = torch.cuda.current_stream()
    x = band
    for i, (w, b) in enumerate(dec.layers):
        h = x.shape[0]
        ext = torch.zeros((h + 2,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
        ext[1:-1].copy_(x)
        ops = []
        if g > 0:  # my first row -> g-1's bottom halo; g-1's last row -> my top halo
            ops += [(g - 1, "send", ext[1]), (g - 1, "recv", ext[0])]
        if g < N - 1:
            ops += [(g + 1, "send", ext[h]), (g + 1, "recv", ext[h + 1])]
        if ops:
            comm.p2p(ops, stream=st)
        x = conv(ext, w, b, i < len(dec.layers) - 1)
    return x
