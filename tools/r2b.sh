set -x
./tools/probe/cluster_occ > gpurun_out/r2b_cluster_occ.txt 2>&1
timeout 600 python tools/sweep_items.py > gpurun_out/r2b_sweep_items.txt 2>&1
timeout 300 python bench.py --gpus 2 --share-gpu --no-cpu-baseline --no-t1 --steps 3 > gpurun_out/r2b_share2.json 2> gpurun_out/r2b_share2.err; echo share2=$?
