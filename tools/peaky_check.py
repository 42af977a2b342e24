"""Error anatomy of tests/test_gpu_usp.py::test_virtual_usp_peaky_ring_merge for the loaded library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2411_01738_b200.inputs import qkv  # noqa: E402
from tests._util import f64  # noqa: E402
from tests.test_gpu_usp import run_virtual_usp  # noqa: E402

B, H, D, S_txt, S_img = 1, 4, 128, 40, 600
q, k, _ = qkv(B, S_txt + S_img, H, D, seed=91, scale=3.0)
_, _, v = qkv(B, S_txt + S_img, H, D, seed=92)
ref_o, ref_l = oracle.attention(f64(q), f64(k), f64(v))
for u, r in [(1, 1), (1, 4), (4, 1)]:
    outs, loc = run_virtual_usp(q, k, v, S_txt, S_img, u, r)
    worst = (0, None)
    for g, (o, l) in enumerate(outs):
        idx = loc[g].numpy()
        d = np.abs(f64(o) - ref_o[:, idx])
        i = np.unravel_index(np.argmax(d), d.shape)
        if d[i] > worst[0]:
            worst = (float(d[i]), (g, int(idx[i[1]]), i[2], i[3], float(ref_o[:, idx][i]), float(f64(o)[i])))
    print(f"{os.environ.get('XDIT_LIB', 'base')} u={u} r={r}: max|dO| {worst[0]:.4f} at (rank, row, head, col, ref, got) {worst[1]}")
