for args in "--B 1 --H 48 --S 17776 --D 64 --iters 8" "--B 2 --H 24 --S 4429 --D 64 --iters 30" "--B 2 --H 16 --S 4096 --D 72 --iters 30"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" base r208 r200 r192 r208e12 e12
done
