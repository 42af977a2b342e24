#!/bin/bash
# One cross-CTA arrival per CTA and step (named barrier of the parity's four warps) vs four.
XDIT_LIB=paper_2411_01738_b200/libxdit_usp_few.so timeout -s KILL 300 python -m pytest tests/test_gpu_attn.py -q -x 2>&1 | tail -2
bash tools/ab_attn.sh "--S 17776 --D 64 --H 48 --iters 6" base few
bash tools/ab_attn.sh "--S 66048 --D 128 --H 24 --iters 3" base few
bash tools/ab_attn.sh "--S 4096 --D 72 --H 32 --iters 20" base few
