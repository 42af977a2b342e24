timeout 400 python bench.py --gpus 8 --share-gpu --config sd3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sg8_sd3.json 2> gpurun_out/sg8_sd3.err; echo sd3_8=$?
timeout 400 python bench.py --gpus 4 --share-gpu --config cogvideox --steps 3 --warmup 3 > gpurun_out/sg4_cog.json 2> gpurun_out/sg4_cog.err; echo cog_4=$?
timeout 600 python bench.py --gpus 8 --share-gpu --config cogvideox --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sg8_cog.json 2> gpurun_out/sg8_cog.err; echo cog_8=$?
