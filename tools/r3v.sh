timeout 600 python -m pytest tests/test_gpu_vae.py -x -q > gpurun_out/r3_vae_parity.txt 2>&1; echo rc=$? >> gpurun_out/r3_vae_parity.txt
for rep in 1 2; do
  echo "== pair (base)" >> gpurun_out/r3_ab_vae_pair.txt; timeout 120 python tools/bench_vae.py 2>&1 | grep tc_kernel >> gpurun_out/r3_ab_vae_pair.txt
  echo "== one-CTA" >> gpurun_out/r3_ab_vae_pair.txt; XDIT_LIB=paper_2411_01738_b200/libxdit_usp_vae1.so timeout 120 python tools/bench_vae.py 2>&1 | grep tc_kernel >> gpurun_out/r3_ab_vae_pair.txt
done
