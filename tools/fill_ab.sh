# S = 4 threshold (S3_FILL4_16 sixteenths of the budget): build variants
for v in 16 14 13 11 9 16 13 11; do
  if [ $v = 16 ]; then unset KRONRED_LIB; else export KRONRED_LIB=tools/_var_f4_$v/libkronred_b200.so; fi
  echo "== f4 $v $(timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep 'total device\|^ *[0-9]*- *[0-9]' | sed 's/  */ /g' | cut -c1-60 | tr '\n' '|')"
done
