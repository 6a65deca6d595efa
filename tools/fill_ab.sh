# S = 2 threshold (S3_FILL2_16 sixteenths of the budget): build variants
for v in 16 14 15 17 18 16 15 17; do
  if [ $v = 16 ]; then unset KRONRED_LIB; else export KRONRED_LIB=tools/_var_f2_$v/libkronred_b200.so; fi
  echo "== f2 $v $(timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep 'total device\|^ *[0-9]*- *[0-9]' | sed 's/  */ /g' | cut -c1-60 | tr '\n' '|')"
done
