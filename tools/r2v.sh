XDIT_LIB=paper_2411_01738_b200/libxdit_usp_wide.so timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -1
for args in "--B 2 --H 16 --S 4096 --D 72 --iters 30" "--B 1 --H 37 --S 16384 --D 72 --iters 8"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" base wide base wide
done
