#!/bin/bash
# A/B timing of kernel variants built with `python -m paper_2411_01738_b200.build --tag=T -D...`:
#   bash tools/ab_attn.sh "<run_attn args>" tag1 tag2 ...   (tag "base" = the in-tree library)
# Interleaves the variants twice so clock / power drift hits all of them alike.
args="$1"; shift
for rep in 1 2; do
  for t in "$@"; do
    if [ "$t" = base ]; then lib=""; else lib="paper_2411_01738_b200/libxdit_usp_$t.so"; fi
    printf "%-10s " "$t"; XDIT_LIB=$lib timeout -s KILL 60 python tools/run_attn.py $args 2>&1 | tail -1
  done
done
