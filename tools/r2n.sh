# round-2 ncu evidence: launch list of the default bench (Flux N=1) + one full capture per workload shape
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench_flux_n1.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_launches_bench.log 2>&1
for spec in "flux:--B 1 --H 24 --S 66048 --D 128" "cogvideox:--B 1 --H 48 --S 17776 --D 64" \
            "pixart:--B 2 --H 16 --S 4096 --D 72" "sd3:--B 2 --H 24 --S 4429 --D 64"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_2sm -s 1 -c 1 \
      -o gpurun_out/r02_ncu_$name python tools/run_attn.py $args --iters 2 > gpurun_out/r02_ncu_$name.log 2>&1
done
