XDIT_LIB=paper_2411_01738_b200/libxdit_usp_kv1.so timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -1
for args in "--B 1 --H 24 --S 66048 --D 128 --iters 4" "--B 1 --H 48 --S 17776 --D 64 --iters 8" "--B 2 --H 16 --S 4096 --D 72 --iters 30" "--B 2 --H 24 --S 4429 --D 64 --iters 30"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" base kv1 base kv1
done
