#!/bin/bash
# A/B of the VAE conv output-channel block (XDIT_VAE_COT=128 vs 256), then the VAE parity tests on 256.
for rep in 1 2; do for c in 128 256; do echo "COT=$c"; XDIT_VAE_COT=$c timeout 200 python tools/bench_vae.py 2>&1 | grep vae_conv_tc; done; done
XDIT_VAE_COT=256 timeout 300 python -m pytest tests/test_gpu_vae.py -q 2>&1 | tail -2
