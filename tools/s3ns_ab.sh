# score3 row-split program (S = 2, 4): 3-slot ring (default) vs 2-slot ring (S3_NS_SPLIT=2)
run() { echo "== $1 $2 $(timeout 600 python tools/iter_profile.py $2 --bucket 100000 2>&1 | grep 'total device\|^sum' | tr '\n' '|')"; }
for rep in 1 2; do
for c in "c4 3e-3 0.8" "c3 3e-3 0.9" "c2"; do
  unset KRONRED_LIB; run new "$c"
  KRONRED_LIB=tools/_var_ns2/libkronred_b200.so run ns2 "$c"
done
done
