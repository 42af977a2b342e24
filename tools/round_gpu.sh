#!/bin/bash
# One GPU session: tests, bench lines, sanitizer, ncu evidence.  Outputs under gpurun_out/.
set -x
timeout 900 python -m pytest tests/ -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_flux.json 2> gpurun_out/bench_flux.err
XDIT_EXP_EMU=2 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_flux_emu2.json 2>&1
for c in pixart sd3 cogvideox toy; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --cpu-seconds 8 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 300 compute-sanitizer --tool memcheck python tools/run_attn.py --B 1 --H 2 --S 300 --Skv 333 --D 128 --iters 1 > gpurun_out/memcheck.txt 2>&1
timeout 300 compute-sanitizer --tool racecheck python tools/run_attn.py --B 1 --H 1 --S 256 --Skv 200 --D 72 --iters 1 > gpurun_out/racecheck.txt 2>&1
timeout 300 compute-sanitizer --tool racecheck python tools/run_attn.py --B 1 --H 2 --S 300 --Skv 333 --D 128 --iters 1 > gpurun_out/racecheck_2sm.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_flux.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 1 -c 1 -o gpurun_out/prof_flux_r01_2sm python tools/run_attn.py --S 66048 --iters 2 > /dev/null 2>&1
ls -la gpurun_out
