for args in "--B 1 --H 48 --S 17776 --D 64 --iters 8" "--B 2 --H 16 --S 4096 --D 72 --iters 30" "--B 1 --H 37 --S 16384 --D 72 --iters 8"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" base s16 s24 s10 e6 e12 r224 r208
done
