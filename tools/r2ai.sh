for t in base s8 r216 e8 prev; do
  if [ $t = base ]; then unset XDIT_LIB; else export XDIT_LIB=paper_2411_01738_b200/libxdit_usp_$t.so; fi
  echo "== $t"; timeout 30 python tools/run_attn.py --B 1 --H 10 --S 4096 --D 128 --iters 2 --scratch 1 2>&1 | tail -1; echo rc=$?
done
