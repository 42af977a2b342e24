"""Measure xdit_vae_conv3x3 on SD-VAE-like decoder layer shapes; one JSON line each.
FLOPs = 2*H*W*Ci*Co*9 (x4 output pixels are stores, not FLOPs); peak = FP32 FFMA
148 SMs x 128 lanes x 2 FLOP x SM clock, at the max clock from MEASURED_PEAKS.json."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01738_b200 import vae
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
    mhz = float(json.load(f).get("sm_max_mhz", 1965.0))
peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
for (H, W, Ci, Co, act) in [(128, 128, 512, 512, 1), (256, 256, 256, 256, 1), (512, 512, 128, 128, 0)]:
    ext = torch.randn(H + 2, Ci, W, device="cuda")
    w = torch.randn(Co, Ci, 3, 3, device="cuda") / 30
    b = torch.randn(Co, device="cuda")
    for _ in range(2):
        vae.conv(ext, w, b, bool(act))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        vae.conv(ext, w, b, bool(act))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    fl = 2.0 * H * W * Ci * Co * 9
    print(json.dumps({"kernel": "vae_conv3x3_kernel", "shape": {"H": H, "W": W, "Ci": Ci, "Co": Co, "act_up": act},
                      "ms": ms, "tflops": fl / ms / 1e9, "roofline": {"bound": "alu", "peak": peak, "unit": "TFLOP/s",
                      "peak_source": "FP32 FFMA: 148 SMs x 128 lanes x 2 x max SM clock", "frac": fl / ms / 1e9 / peak}}), flush=True)
