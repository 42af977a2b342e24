for args in "--B 1 --H 3 --S 700 --Skv 333 --D 64" "--B 2 --H 5 --S 600 --Skv 1000 --D 72"; do
  for sc in 0 1; do
    echo "== racecheck $args scratch=$sc"
    timeout 600 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/run_attn.py $args --iters 1 --scratch $sc 2>&1 | grep -E "RACECHECK SUMMARY|Error|hazards" | head -6
  done
done
timeout 300 python -m pytest tests/test_gpu_attn.py -x -q 2>&1 | tail -2
