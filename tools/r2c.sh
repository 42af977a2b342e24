set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_usp.py tests/test_gpu_pipefusion.py -x -q -rf > gpurun_out/r2c_pytest.log 2>&1; echo pytest=$?
timeout 600 python tools/sweep_items.py > gpurun_out/r2c_sweep_items.txt 2>&1
for c in flux cogvideox pixart sd3; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2c_bench_$c.json 2> gpurun_out/r2c_bench_$c.err; done
