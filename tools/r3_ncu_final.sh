# ncu evidence for the final kernel: launch list of the default bench command, and --set full of the
# attention kernel at the Flux (D = 128) and CogVideoX (D = 64, TS-MMA QK^T) shapes
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r3_launches.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:attn_fwd_2sm -s 1 -c 1 -o gpurun_out/r3f_ncu_d64 python tools/run_attn.py --B 1 --H 48 --S 17776 --D 64 --iters 2 > gpurun_out/r3f_ncu_d64.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:attn_fwd_2sm -s 1 -c 1 -o gpurun_out/r3f_ncu_d128 python tools/run_attn.py --B 1 --H 24 --S 66048 --D 128 --iters 2 > gpurun_out/r3f_ncu_d128.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:vae_conv_tcp -s 2 -c 1 -o gpurun_out/r3f_ncu_vae python tools/bench_vae.py > gpurun_out/r3f_ncu_vae.log 2>&1
