for t in e2 p16 r200; do
  XDIT_LIB=paper_2411_01738_b200/libxdit_usp_$t.so timeout 240 python -m pytest tests/test_gpu_attn.py -x -q -k "64" 2>&1 | tail -1 | sed "s/^/$t parity: /" >> gpurun_out/r3_ab_d64tune.txt
done
for shape in "--B 1 --H 48 --S 17776 --D 64 --iters 8" "--B 2 --H 24 --S 4429 --D 64 --iters 30"; do
  echo "== $shape" >> gpurun_out/r3_ab_d64tune.txt
  bash tools/ab_attn.sh "$shape" base e2 p16 r200 >> gpurun_out/r3_ab_d64tune.txt 2>&1
done
