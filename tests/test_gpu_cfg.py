"""the CFG combine kernel against the fp64 oracle (reading R3, P:409-414,
S:200-208); argument checks of the step tail."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2411_01738_b200 import usp
from tests._util import f64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("g", [0.0, 1.0, 4.5, 7.5, -1.25])
@pytest.mark.parametrize("n", [8, 4096, 16 * 128 * 128 + 8])
def test_cfg_combine_vs_oracle(dtype, g, n):
    gen = torch.Generator().manual_seed(n + int(g * 10))
    c = torch.randn(n, generator=gen).to(dtype)
    u = torch.randn(n, generator=gen).to(dtype)
    out = usp.cfg_combine(c.cuda(), u.cuda(), g)
    torch.cuda.synchronize()
    ref = oracle.cfg_combine(f64(c), f64(u), g)
    got = f64(out)
    if dtype == torch.float32:  # |g c| + |(1-g) u| bounds the fp32 cancellation error
        bound = (abs(g) * np.abs(f64(c)) + abs(1 - g) * np.abs(f64(u))) * 2.0 ** -22
        assert np.all(np.abs(got - ref) <= bound + 1e-30)
    else:  # one RNE rounding of the fp32 result (half a bf16 ulp) plus the fp32 cancellation error
        bound = np.abs(ref) * 2.0 ** -8 + (abs(g) * np.abs(f64(c)) + abs(1 - g) * np.abs(f64(u))) * 2.0 ** -22
        assert np.all(np.abs(got - ref) <= bound + 1e-30)
    if g == 0.0:
        assert torch.equal(out.cpu(), u)  # g = 0 gives eps_uncond exactly
    if g == 1.0:
        assert torch.equal(out.cpu(), c)  # g = 1 gives eps_cond exactly


def test_cfg_combine_in_place_and_errors():
    c = torch.randn(64, device="cuda", dtype=torch.bfloat16)
    u = torch.randn(64, device="cuda", dtype=torch.bfloat16)
    ref = oracle.cfg_combine(f64(c), f64(u), 3.0)
    usp.cfg_combine(c, u, 3.0, out=u)  # out aliases eps_uncond
    torch.cuda.synchronize()
    assert np.all(np.abs(f64(u) - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-6)
    with pytest.raises(usp.XditError) as e:
        usp.cfg_combine(c[:7], c[:7], 1.0)  # n % 8 != 0
    assert e.value.status == "ALIGNMENT"


def test_cfg_tail_needs_a_cfg_pair():
    x = torch.zeros(64, device="cuda", dtype=torch.bfloat16)
    with usp.Comm(1, 1) as comm:
        with pytest.raises(usp.XditError) as e:
            usp.cfg_tail(x, 2.0, comm=comm)
    assert e.value.status == "COMM_MISMATCH"
