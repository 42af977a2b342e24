for d in 0 1 2; do echo "DIAG=$d"; XDIT_DIAG=$d python tools/run_attn.py --S 66048 --iters 3 | tail -1; XDIT_DIAG=$d python tools/run_attn.py --S 17776 --D 64 --H 48 --iters 4 | tail -1; done
