#!/bin/bash
# A/B of the exp2 FMA-pipe offload (XDIT_EXP_EMU = column pairs of every 8 on the polynomial) for the
# CTA-pair kernel at D = 64 / 72, through bench.py (sustained, events), interleaved twice.
for rep in 1 2; do
  for c in cogvideox sd3 pixart; do
    for e in 0 1 2 3; do
      printf "%-10s EMU=%d " $c $e
      XDIT_EXP_EMU=$e timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print(round(d['value'],1), 'kernel', round(r['achieved'],1), 'sm_mhz', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
    done
  done
done
