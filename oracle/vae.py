"""fp64 oracle for the patch-parallel VAE decode -- TEST INFRASTRUCTURE.

Only ``tests/`` may import this module; the product package never does and shares no code with it.
Plain numpy fp64, explicit loops over the 3x3 taps.

What it follows (§4.3):
  * "an autodecoder module employs a VAE to decode the image (size h/8 x w/8 x c) ... from the latent
    space into images in the pixel space (h x w x 3)" and "The VAE applies multiple convolutional
    neural networks for upsampling";
  * "We divide the feature maps in the latent space into multiple patches and perform parallel VAE
    decoding across different devices. This requires the exchange of the boundary data for
    convolutional operators";
  * "Patch parallelism reduces the peak memory for intermediate activations to 1/N".

Reading (R5; SPEC S:540-575 vae_parallel): a tiny decoder -- per stage a 3x3 conv
(zero padding 1, bias) + SiLU + nearest-neighbour x2 upsample, then a final 3x3 conv to 3 channels.
Activations are [H][C][W] (row-major over height, so a row band and a halo row are contiguous).
Patch parallelism splits the latent rows into N balanced contiguous bands; before every conv a band
receives one boundary row from each neighbour (zeros at the image edge = the serial zero padding),
so the decode is exact: every output pixel is the same sum as in the serial decode.

Functions:
  conv3x3(x, w, b)                       x [H][Ci][W], w [Co][Ci][3][3], b [Co] -> [H][Co][W]
  silu(x), upsample2(x)
  serial_decode(latent, layers)          layers: [(w, b)] per conv, last one without SiLU/upsample
  bands(h, N)                            -> [(row_off, rows)] (np.array_split)
  halo(band_list, g)                     -> band g extended with its neighbours' boundary rows
  patch_parallel_decode(latent, layers, N)
"""
from __future__ import annotations

import numpy as np


def conv3x3(x, w, b):
    """Zero-padded 3x3 convolution (cross-correlation, as in conv2d) over [H][Ci][W]."""
    x = np.asarray(x, np.float64)
    H, Ci, W = x.shape
    Co = w.shape[0]
    xp = np.zeros((H + 2, Ci, W + 2))
    xp[1:H + 1, :, 1:W + 1] = x
    return _conv_valid_rows(xp, w, b)


def _conv_valid_rows(xp, w, b):
    """xp [H+2][Ci][W+2] already padded: out[y][co][x] = b[co] + sum_{ci,dy,dx} w[co,ci,dy,dx] xp[y+dy][ci][x+dx]."""
    Hp, Ci, Wp = xp.shape
    H, W = Hp - 2, Wp - 2
    out = np.empty((H, w.shape[0], W))
    out[:] = np.asarray(b, np.float64)[None, :, None]
    for dy in range(3):
        for dx in range(3):
            # [H][Ci][W] window times [Co][Ci] tap -> [H][Co][W]
            win = xp[dy:dy + H, :, dx:dx + W]
            out += np.einsum("oc,hcw->how", np.asarray(w, np.float64)[:, :, dy, dx], win)
    return out


def silu(x):
    return x / (1.0 + np.exp(-x))


def upsample2(x):
    """Nearest-neighbour x2 in both spatial dims of [H][C][W]."""
    return np.repeat(np.repeat(x, 2, axis=0), 2, axis=2)


def serial_decode(latent, layers):
    """latent [h][c][w] -> image [h 2^s][3][w 2^s]; layers = s stage convs + the final conv."""
    x = np.asarray(latent, np.float64)
    for i, (w, b) in enumerate(layers):
        x = conv3x3(x, w, b)
        if i < len(layers) - 1:
            x = upsample2(silu(x))
    return x


def bands(h: int, N: int):
    """Balanced contiguous row bands of h rows over N devices (np.array_split convention)."""
    if N < 1 or h < N:
        raise ValueError("need 1 <= N <= rows")
    base, rem = divmod(h, N)
    out, off = [], 0
    for g in range(N):
        n = base + (1 if g < rem else 0)
        out.append((off, n))
        off += n
    return out


def halo(band_list, g):
    """Band g extended by one row on each side: the neighbours' boundary rows, zeros at the edges
    ("exchange of the boundary data"; the zero rows are the serial conv's zero padding)."""
    x = band_list[g]
    top = band_list[g - 1][-1:] if g > 0 else np.zeros_like(x[:1])
    bot = band_list[g + 1][:1] if g + 1 < len(band_list) else np.zeros_like(x[:1])
    return np.concatenate([top, x, bot], axis=0)


def patch_parallel_decode(latent, layers, N: int):
    """Each of N devices holds a row band; before each conv it receives its halo rows, convolves its
    band only (the output keeps the band's rows), and upsamples locally.  Returns the concatenation of
    the final bands and the per-layer band row counts (the 1/N activation footprint)."""
    x = np.asarray(latent, np.float64)
    bl = [x[o:o + n] for (o, n) in bands(x.shape[0], N)]
    rows = []
    for i, (w, b) in enumerate(layers):
        ext = [halo(bl, g) for g in range(N)]
        new = []
        for e in ext:
            ep = np.zeros((e.shape[0], e.shape[1], e.shape[2] + 2))
            ep[:, :, 1:-1] = e
            y = _conv_valid_rows(ep, w, b)
            if i < len(layers) - 1:
                y = upsample2(silu(y))
            new.append(y)
        bl = new
        rows.append([y.shape[0] for y in bl])
    return np.concatenate(bl, axis=0), rows
