# score3 with a compile-time two-scenario slice (default) vs runtime slice width (tools/_var_nols2)
timeout 1200 python -m pytest tests -m gpu -x -q -k "large or c3 or c4 or iteration_scores or s24 or c2_benchmark or m40" 2>&1 | tail -2
for v in new old new old; do
  if [ $v = old ]; then export KRONRED_LIB=tools/_var_nols2/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c4 3e-3 0.2 --bucket 5000 2>&1 | grep "total device"
  timeout 300 python tools/iter_profile.py c3 3e-3 0.9 --bucket 9000 2>&1 | grep "total device"
done
unset KRONRED_LIB; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "total device"
