#!/bin/bash
# ncu source-level capture of the D=64 (CogVideoX) and D=128 (Flux) pair kernel: per-SASS warp-state
# samples, to see where the MMA-issuer warp spends its tile period.
python tools/run_attn.py --B 1 --H 48 --S 17776 --D 64 --iters 5 > gpurun_out/r3_base_d64.txt 2>&1
python tools/run_attn.py --B 1 --H 24 --S 66048 --D 128 --iters 3 > gpurun_out/r3_base_d128.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_2sm -s 1 -c 1 \
  -o gpurun_out/r3_ncu_d64 python tools/run_attn.py --B 1 --H 48 --S 17776 --D 64 --iters 2 > gpurun_out/r3_ncu_d64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_2sm -s 1 -c 1 \
  -o gpurun_out/r3_ncu_d128 python tools/run_attn.py --B 1 --H 24 --S 16384 --D 128 --iters 2 > gpurun_out/r3_ncu_d128.log 2>&1
echo done
