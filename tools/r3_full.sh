#!/bin/bash
# Full GPU check of the committed kernel: smoke, every -m gpu test, the bench lines of all
# workloads, the reference arm, the ncu launch list of the default bench.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r3_smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -x -q -rf > gpurun_out/r3_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/r3_bench_flux.json 2> gpurun_out/r3_bench_flux.err; echo bench=$?
for c in cogvideox pixart sd3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r3_bench_$c.json 2> gpurun_out/r3_bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r3_bench_reference.json 2> gpurun_out/r3_bench_reference.err
echo done
