timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2 > gpurun_out/r3_stage_parity.txt
bash tools/r3_ab.sh r3_ab_stage head base
XDIT_LIB=paper_2411_01738_b200/libxdit_usp_prof.so timeout 120 python tools/trace_boundary.py --S 4429 --H 24 --D 64 > gpurun_out/r3_trace_boundary_d64d.txt 2>&1
