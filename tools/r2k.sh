python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2k_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/r2k_pytest.log 2>&1; echo pytest=$?
for c in flux cogvideox pixart sd3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2k_bench_$c.json 2> gpurun_out/r2k_bench_$c.err; done
