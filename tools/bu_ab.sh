# backward suffix loop unroll (BR_SUFFIX_UNROLL 1 / 2 / 4 default / 8)
for v in 4 8 4 8; do
  if [ $v = 0 ]; then unset KRONRED_LIB; else export KRONRED_LIB=tools/_var_bu$v/libkronred_b200.so; fi
  echo "== u$v $(timeout 120 python tools/micro/base_refresh.py c2 2>&1 | tail -1) | $(timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep 'total device')"
done
