timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2
for e in 0 2 3 4; do echo "EMU=$e"; XDIT_EXP_EMU=$e python tools/run_attn.py --S 66048 --iters 3 | tail -1; XDIT_EXP_EMU=$e python tools/run_attn.py --S 17776 --D 64 --H 48 --iters 4 | tail -1; done
