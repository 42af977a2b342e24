#!/bin/bash
# D = 72: one N = 96 PV MMA (three 16-column SW32 V atoms per CTA, XDIT_D72_WIDE_PV) vs N = 64 + N = 32.
XDIT_LIB=paper_2411_01738_b200/libxdit_usp_wide.so timeout -s KILL 300 python -m pytest tests/test_gpu_attn.py -q -x -k "72" 2>&1 | tail -3
bash tools/ab_attn.sh "--S 4096 --D 72 --H 32 --iters 20" base wide
bash tools/ab_attn.sh "--S 16384 --D 72 --H 16 --iters 5" base wide
