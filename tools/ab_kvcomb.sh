bash tools/ab_attn.sh "--S 17776 --D 64 --H 48 --iters 6" base comb
bash tools/ab_attn.sh "--S 66048 --D 128 --H 24 --iters 3" base comb
bash tools/ab_attn.sh "--S 4096 --D 72 --H 32 --iters 20" base comb
bash tools/ab_attn.sh "--S 4429 --D 64 --H 48 --iters 20" base comb
