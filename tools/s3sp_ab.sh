# register budget of the score3 row-split program: S3_MIN_BLOCKS_SPLIT 3 (default, 168 regs) vs 4 (128 regs)
run() { echo "== $1 $2 $(timeout 600 python tools/iter_profile.py $2 --bucket 1000 2>&1 | grep 'total device\|^ *[0-9]*- *[0-9]' | sed 's/  */ /g' | cut -c1-40 | tr '\n' '|')"; }
for c in "c4 3e-3 0.8" "c3 3e-3 0.9" "c2"; do
  unset KRONRED_LIB; run new "$c"
  KRONRED_LIB=tools/_var_sp4/libkronred_b200.so run sp4 "$c"
done
