XDIT_LIB=paper_2411_01738_b200/libxdit_usp_arow.so timeout 300 python -m pytest tests/test_gpu_vae.py -x -q > gpurun_out/r3_arow_parity.txt 2>&1; echo rc=$? >> gpurun_out/r3_arow_parity.txt
for rep in 1 2; do
  for t in base arow; do
    lib=""; [ $t != base ] && lib=paper_2411_01738_b200/libxdit_usp_$t.so
    echo "== $t" >> gpurun_out/r3_ab_arow.txt; XDIT_LIB=$lib timeout 120 python tools/bench_vae.py 2>&1 | grep tcp_kernel >> gpurun_out/r3_ab_arow.txt
  done
done
