python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rf_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -rf > gpurun_out/rf_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/rf_bench_flux.json 2> gpurun_out/rf_bench_flux.err; echo bench=$?
for c in cogvideox pixart sd3 toy; do timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/rf_bench_$c.json 2> gpurun_out/rf_bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/rf_bench_reference.json 2> gpurun_out/rf_bench_reference.err
timeout 300 python tools/bench_pipefusion.py --config flux > gpurun_out/rf_pipefusion_flux.json 2>&1
timeout 300 python tools/bench_pipefusion.py --config cogvideox > gpurun_out/rf_pipefusion_cogvideox.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd_2sm -s 1 -c 1 -o gpurun_out/rf_ncu_flux python tools/run_attn.py --B 1 --H 24 --S 66048 --D 128 --iters 2 > gpurun_out/rf_ncu_flux.log 2>&1
