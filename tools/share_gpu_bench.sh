#!/bin/bash
# Functional check of bench.py's N > 1 path on a 1-GPU box: every rank on cuda:0 (XDIT_SHARE_GPU=1,
# gloo process group), peer-memory transport.  Timings are NOT scaling numbers (ranks time-share one GPU).
run() { XDIT_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 \
          --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $1 --steps 3 --warmup 3 "${@:2}"; }
run 2 --config sd3
run 4 --config toy --ulysses 2 --ring 2
run 4 --config sd3 --ulysses 1 --ring 4
run 4 --config cogvideox
run 8 --config pixart --ulysses 2 --ring 4
