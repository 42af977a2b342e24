#!/bin/bash
# r01 (second session) evidence: bench lines for every config, ncu launch list of the PipeFusion
# step, ncu full capture of the VAE conv kernel and of the PipeFusion patch attention.
set -x
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_flux.json 2> gpurun_out/bench_flux.err
for c in pixart sd3 cogvideox toy; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pf_cogvideox.csv python tools/bench_pipefusion.py --config cogvideox --M 4 --L 4 --iters 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vae_conv -s 2 -c 1 -o gpurun_out/prof_vae_conv python tools/bench_vae.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:pf_prep -s 3 -c 1 -o gpurun_out/prof_pf_prep python tools/bench_pipefusion.py --config cogvideox --M 4 --L 4 --iters 2 > /dev/null 2>&1
ls -la gpurun_out
