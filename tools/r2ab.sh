for args in "--B 1 --H 24 --S 66048 --D 128 --iters 4" "--B 1 --H 37 --S 16384 --D 128 --iters 8"; do
  echo "== $args"
  bash tools/ab_attn.sh "$args" base emu16 e16r224 e16st9 e16r224st9 emu0
  bash tools/ab_attn.sh "$args" base emu16 e16r224 e16st9 e16r224st9 emu0
done
