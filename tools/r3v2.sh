for rep in 1 2; do
  for t in base vst4 vfs; do
    lib=""; [ $t != base ] && lib=paper_2411_01738_b200/libxdit_usp_$t.so
    echo "== $t" >> gpurun_out/r3_ab_vae2.txt; XDIT_LIB=$lib timeout 120 python tools/bench_vae.py 2>&1 | grep tc_kernel >> gpurun_out/r3_ab_vae2.txt
  done
done
XDIT_LIB=paper_2411_01738_b200/libxdit_usp_vfs.so timeout 600 python -m pytest tests/test_gpu_vae.py -x -q > gpurun_out/r3_vae_fs_parity.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vae_conv_tc2 -s 2 -c 1 -o gpurun_out/r3_ncu_vae2 python tools/bench_vae.py > gpurun_out/r3_ncu_vae2.log 2>&1
