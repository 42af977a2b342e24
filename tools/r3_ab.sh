#!/bin/bash
# Same-session A/B of tagged kernel builds on the four workload shapes, parity of each tag first.
#   bash tools/r3_ab.sh <out-prefix> tag1 tag2 ...   ("base" = the in-tree library)
out=$1; shift
for t in "$@"; do
  [ "$t" = base ] && continue
  XDIT_LIB=paper_2411_01738_b200/libxdit_usp_$t.so timeout 240 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2 | sed "s/^/$t parity: /" >> gpurun_out/${out}.txt
done
for shape in "--B 1 --H 24 --S 66048 --D 128 --iters 4" "--B 1 --H 48 --S 17776 --D 64 --iters 8" \
             "--B 2 --H 16 --S 4096 --D 72 --iters 30" "--B 2 --H 24 --S 4429 --D 64 --iters 30"; do
  echo "== $shape" >> gpurun_out/${out}.txt
  bash tools/ab_attn.sh "$shape" "$@" >> gpurun_out/${out}.txt 2>&1
done
echo done
