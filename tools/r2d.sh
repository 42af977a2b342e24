# same-session A/B: round-1 kernel (old) vs persistent (base), bench shapes + a long D=72 shape
for args in "--B 1 --H 24 --S 66048 --D 128 --iters 4" "--B 1 --H 48 --S 17776 --D 64 --iters 8" \
            "--B 2 --H 16 --S 4096 --D 72 --iters 30" "--B 2 --H 24 --S 4429 --D 64 --iters 30" \
            "--B 1 --H 37 --S 16384 --D 72 --iters 8" "--B 1 --H 37 --S 16384 --D 128 --iters 8"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" old base old base
done
