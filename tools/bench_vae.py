"""Measure the VAE decoder conv on SD-VAE-like decoder layer shapes; one JSON
line per (kernel, shape).  FLOPs = 2*H*W*Ci*Co*9 (the x4 upsampled pixels are stores, not FLOPs).
  * vae_conv3x3_kernel (SIMT fp32): peak = FP32 FFMA 148 SMs x 128 lanes x 2 FLOP x max SM clock
    (DESIGN.md §7.6);
  * vae_conv_tc_kernel (tcgen05 bf16): peak = measured bf16 dense peak (MEASURED_PEAKS.json)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_01738_b200 import vae
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
    mp = json.load(f)
mhz = float(mp.get("sm_max_mhz", 1965.0))
bf16_peak = float(mp["bf16_tflops"])
peak = 148 * 128 * 2 * mhz * 1e6 / 1e12
def timeit(fn, iters=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


for (H, W, Ci, Co, act) in [(128, 128, 512, 512, 1), (256, 256, 256, 256, 1), (512, 512, 128, 128, 0)]:
    fl = 2.0 * H * W * Ci * Co * 9
    ext = torch.randn(H + 2, Ci, W, device="cuda")
    w = torch.randn(Co, Ci, 3, 3, device="cuda") / 30
    b = torch.randn(Co, device="cuda")
    ms = timeit(lambda: vae.conv(ext, w, b, bool(act)))
    print(json.dumps({"kernel": "vae_conv3x3_kernel", "dtype": "f32", "shape": {"H": H, "W": W, "Ci": Ci, "Co": Co, "act_up": act},
                      "ms": ms, "tflops": fl / ms / 1e9, "roofline": {"bound": "alu", "peak": peak, "unit": "TFLOP/s",
                      "peak_source": "FP32 FFMA: 148 SMs x 128 lanes x 2 x max SM clock", "frac": fl / ms / 1e9 / peak}}), flush=True)
    dec = vae.Decoder([(w.cpu().numpy(), b.cpu().numpy())], tc=True)
    wt, bd = dec.layers[0]
    ext_t = torch.randn(H + 2, W, Ci, device="cuda").to(torch.bfloat16)
    ms = timeit(lambda: vae.conv(ext_t, wt, bd, bool(act)), iters=20)
    print(json.dumps({"kernel": "vae_conv_tcp_kernel", "dtype": "bf16", "shape": {"H": H, "W": W, "Ci": Ci, "Co": Co, "act_up": act},
                      "ms": ms, "tflops": fl / ms / 1e9, "roofline": {"bound": "tensor", "peak": bf16_peak, "unit": "TFLOP/s",
                      "peak_source": "measured bf16 burst (MEASURED_PEAKS.json bf16_tflops)", "frac": fl / ms / 1e9 / bf16_peak}}), flush=True)
