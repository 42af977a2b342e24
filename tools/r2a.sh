set -x
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -rf --durations=25 > gpurun_out/r2a_pytest.log 2>&1; echo pytest=$?
timeout 300 python bench.py > gpurun_out/r2a_bench_n1.json 2> gpurun_out/r2a_bench_n1.err; echo bench=$?
timeout 300 python bench.py --gpus 2 --share-gpu --no-cpu-baseline > gpurun_out/r2a_bench_share2.json 2> gpurun_out/r2a_bench_share2.err; echo share2=$?
