for tool in memcheck racecheck synccheck; do
  for args in "--B 1 --H 3 --S 700 --Skv 333 --D 64" "--B 2 --H 5 --S 600 --Skv 1000 --D 72" "--B 1 --H 2 --S 300 --Skv 1300 --D 128"; do
    for sc in 0 1; do
      echo "== $tool $args scratch=$sc"
      timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/run_attn.py $args --iters 1 --scratch $sc 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|error|Error|hazard" | head -5
    done
  done
done
