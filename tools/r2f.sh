export XDIT_LIB=paper_2411_01738_b200/libxdit_usp_prof.so
for args in "--S 17776 --H 48 --D 64" "--S 17776 --H 48 --D 64 --diag 1" "--S 66048 --H 24 --D 128" "--S 66048 --H 24 --D 128 --diag 1" "--B 2 --S 4096 --H 16 --D 72"; do
  timeout 120 python tools/trace_attn.py $args; echo
done
