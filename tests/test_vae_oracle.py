"""Pins of the patch-parallel VAE oracle (oracle/vae.py).

conv3x3 against a brute-force 7-deep loop on tiny inputs and two closed forms (a centre-tap identity
kernel; a constant input's interior response = bias + input * sum of taps); the decoder's linearity
limit (zero latent and biases -> zero image); patch parallelism against the serial decode (exact by
construction) for several N, the band rows shrinking as 1/N, halo edge semantics.
"""
import itertools

import numpy as np
import pytest

from oracle import vae


def layers(c, widths, seed, out=3):
    rng = np.random.default_rng(seed)
    L, ci = [], c
    for co in list(widths) + [out]:
        L.append((rng.standard_normal((co, ci, 3, 3)) / np.sqrt(9 * ci), rng.standard_normal(co) * 0.1))
        ci = co
    return L


def test_conv3x3_brute_force():
    rng = np.random.default_rng(0)
    H, Ci, W, Co = 5, 3, 6, 4
    x, w, b = rng.standard_normal((H, Ci, W)), rng.standard_normal((Co, Ci, 3, 3)), rng.standard_normal(Co)
    want = np.zeros((H, Co, W))
    for y, co, xx in itertools.product(range(H), range(Co), range(W)):
        s = b[co]
        for ci, dy, dx in itertools.product(range(Ci), range(3), range(3)):
            yy, xs = y + dy - 1, xx + dx - 1
            if 0 <= yy < H and 0 <= xs < W:
                s += w[co, ci, dy, dx] * x[yy, ci, xs]
        want[y, co, xx] = s
    assert np.allclose(vae.conv3x3(x, w, b), want, rtol=0, atol=1e-13)


def test_conv3x3_closed_forms():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((6, 2, 7))
    w = np.zeros((2, 2, 3, 3))
    w[0, 0, 1, 1] = w[1, 1, 1, 1] = 1.0  # centre tap identity
    assert np.array_equal(vae.conv3x3(x, w, np.zeros(2)), x)
    w = rng.standard_normal((3, 2, 3, 3))
    b = rng.standard_normal(3)
    y = vae.conv3x3(np.full((6, 2, 7), 2.0), w, b)
    assert np.allclose(y[1:-1, :, 1:-1], (b + 2.0 * w.sum(axis=(1, 2, 3)))[None, :, None], atol=1e-13)


def test_upsample_and_linearity():
    x = np.arange(12.0).reshape(2, 2, 3)
    u = vae.upsample2(x)
    assert u.shape == (4, 2, 6) and u[3, 1, 5] == x[1, 1, 2] and u[2, 0, 1] == x[1, 0, 0]
    L = [(w, np.zeros_like(b)) for (w, b) in layers(4, (8, 8), 2)]
    assert np.array_equal(vae.serial_decode(np.zeros((6, 4, 6)), L), np.zeros((24, 3, 24)))


def test_halo_edges_are_zero_padding():
    bl = [np.full((2, 1, 3), float(g + 1)) for g in range(3)]
    e0, e1, e2 = (vae.halo(bl, g) for g in range(3))
    assert (e0[0] == 0).all() and (e0[-1] == 2).all()
    assert (e1[0] == 1).all() and (e1[-1] == 3).all()
    assert (e2[0] == 2).all() and (e2[-1] == 0).all()


@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_patch_parallel_equals_serial(N):
    rng = np.random.default_rng(3)
    lat = rng.standard_normal((8, 4, 10))
    L = layers(4, (16, 8), 4)
    want = vae.serial_decode(lat, L)
    got, rows = vae.patch_parallel_decode(lat, L, N)
    assert got.shape == want.shape == (32, 3, 40)
    assert np.allclose(got, want, rtol=0, atol=1e-12)  # SPEC S:557 "equals serial_decode within 1e-12"
    assert max(rows[-1]) == -(-8 // N) * 4  # each device holds ceil(h/N) 2^s rows: ~1/N


def test_bands():
    assert vae.bands(10, 4) == [(0, 3), (3, 3), (6, 2), (8, 2)]
    with pytest.raises(ValueError):
        vae.bands(3, 4)
