#!/bin/bash
# A/B of the three-warp rotation kernel (XDIT_ATTN_KERNEL=3rot) against the default CTA-pair kernel,
# interleaved, same process image; then the attention parity tests on the 3rot kernel.
for rep in 1 2; do
  for a in "--S 17776 --D 64 --H 48 --iters 6" "--S 66048 --D 128 --H 24 --iters 3" "--S 4096 --D 72 --H 32 --iters 20" "--S 4429 --D 64 --H 48 --iters 20"; do
    for k in 2sm 3rot; do printf "%-5s %-40s " $k "$a"; XDIT_ATTN_KERNEL=$k timeout -s KILL 90 python tools/run_attn.py $a 2>&1 | tail -1; done
  done
done
