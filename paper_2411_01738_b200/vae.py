"""Patch-parallel VAE decode -- SURVEY §8(f) NEXT 4 (§4.3; reading R5).

Host orchestration only: every conv runs in the library's `xdit_vae_conv3x3` (conv + bias, the
stage's SiLU and x2 upsample fused into the store); halo rows move between devices through the
peer-transport mailbox.  Activations are fp32 [H][C][W].  The decoder: per stage a 3x3 conv + SiLU +
nearest x2 upsample, then a final 3x3 conv to 3 channels.
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


class Decoder:
    """layers: [(w [Co][Ci][3][3], b [Co])]; all but the last are upsampling stages."""

    def __init__(self, layers: Sequence, device="cuda"):
        import torch
        self.layers = [(torch.as_tensor(w, dtype=torch.float32).contiguous().to(device),
                        torch.as_tensor(b, dtype=torch.float32).contiguous().to(device)) for w, b in layers]


def conv(ext, w, b, act_up: bool, stream=None):
    """xdit_vae_conv3x3 on a halo-extended band ext [H+2][Ci][W]; returns the new band."""
    import torch
    Hp2, Ci, W = ext.shape
    H, Co = Hp2 - 2, w.shape[0]
    out = torch.empty((2 * H, Co, 2 * W) if act_up else (H, Co, W), dtype=torch.float32, device=ext.device)
    usp._check(usp.lib().xdit_vae_conv3x3(usp._ptr(ext), H, Ci, W, usp._ptr(w), usp._ptr(b), usp._ptr(out), Co,
                                          1 if act_up else 0, usp._stream(stream)), "xdit_vae_conv3x3")
    return out


def decode(latent, dec: Decoder):
    """Single-device decode: the whole image is one band with zero halo rows."""
    import torch
    x = latent
    for i, (w, b) in enumerate(dec.layers):
        ext = torch.zeros((x.shape[0] + 2,) + tuple(x.shape[1:]), dtype=torch.float32, device=x.device)
        ext[1:-1].copy_(x)
        x = conv(ext, w, b, i < len(dec.layers) - 1)
    return x


def decode_band(band, dec: Decoder, comm):
    """Patch-parallel decode, one process per band: this rank (= comm.rank of N) holds latent rows
    `band` [h_g][c][w]; before every conv it sends its first row to rank g-1 and its last row to rank
    g+1 (their bottom / top halos) through the mailbox and receives theirs.  Collective.  Returns
    this rank's band of the decoded image."""
    import torch
    N, g = comm.ulysses * comm.ring, comm.rank
    st = torch.cuda.current_stream()
    # halo row bytes of the widest layer input, two spaces (layer parity) per source
    rows = []
    C, W = band.shape[1], band.shape[2]
    for i, (w, _) in enumerate(dec.layers):
        rows.append(C * W * 4)
        C = w.shape[0]
        W = W * 2 if i < len(dec.layers) - 1 else W
    rb = (max(rows) + 255) // 256 * 256
    comm.mailbox(2 * rb)
    tags = comm.__dict__.setdefault("_vae_tags", {})
    x = band
    for i, (w, b) in enumerate(dec.layers):
        h = x.shape[0]
        ext = torch.empty((h + 2,) + tuple(x.shape[1:]), dtype=torch.float32, device=x.device)
        ext[1:-1].copy_(x)
        for nb, row in ((g - 1, x[0]), (g + 1, x[h - 1])):  # my boundary rows -> the neighbours
            if 0 <= nb < N:
                t = tags[("out", nb)] = tags.get(("out", nb), 0) + 1
                if t > 2:
                    comm.wait_ack(nb, t - 2, stream=st)
                comm.put(nb, row, t, offset=(t % 2) * rb, stream=st)
        for nb, dst in ((g - 1, ext[0]), (g + 1, ext[h + 1])):  # the neighbours' rows -> my halos
            if 0 <= nb < N:
                t = tags[("in", nb)] = tags.get(("in", nb), 0) + 1
                comm.wait(nb, t, stream=st)
                dst.copy_(comm.mailbox_view(nb, tuple(dst.shape), torch.float32, offset=(t % 2) * rb))
                comm.ack(nb, t, stream=st)
            else:
                dst.zero_()
        x = conv(ext, w, b, i < len(dec.layers) - 1)
    return x
