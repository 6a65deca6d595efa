# loop iterations per conditional-graph body: 8 (default) vs 16 vs 4
for v in 8 16 4 8 16; do
  if [ $v = 8 ]; then unset KRONRED_LIB; else export KRONRED_LIB=tools/_var_u$v/libkronred_b200.so; fi
  echo "== unroll $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "total device"
done
