for args in "--B 1 --H 10 --S 4096 --D 128 --iters 2 --scratch 0" "--B 1 --H 10 --S 4096 --D 128 --iters 2 --scratch 1" "--B 1 --H 10 --S 4096 --D 64 --iters 2 --scratch 1" "--B 1 --H 10 --S 4096 --Skv 1000 --D 128 --iters 2 --scratch 1"; do
  echo "== $args"; timeout 60 python tools/run_attn.py $args 2>&1 | tail -2; echo rc=$?
done
