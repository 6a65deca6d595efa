# score3 register budget (S3_MIN_BLOCKS 3 default vs 4, 5) on the L = 2 large feeders and C2
for v in new mb4 mb5 new mb4; do
  case $v in new) unset KRONRED_LIB;; *) export KRONRED_LIB=tools/_var_$v/libkronred_b200.so;; esac
  for c in "c3 3e-3 0.3" "c4 3e-3 0.2" "c2"; do
    echo "== $v $c $(timeout 600 python tools/iter_profile.py $c --bucket 100000 2>&1 | grep 'total device\|^sum' | tr '\n' '|')"
  done
done
