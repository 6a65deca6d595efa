# score1 on the large feeders (KRONRED_FORCE_S1, item sizes) vs score3, C4 prefixes
for L in 24 96; do
  for v in s3 s1g16 s1g16b; do
    unset KRONRED_FORCE_S1 KRONRED_S1_GK
    if [ $v = s1g16 ]; then export KRONRED_FORCE_S1=1 KRONRED_S1_GK=16,16,8; fi
    if [ $v = s1g16b ]; then export KRONRED_FORCE_S1=1 KRONRED_S1_GK=16,8,4; fi
    echo "== L$L $v $(timeout 600 python tools/r1r2_ab.py . $L 0.01 2>&1 | tail -1)"
  done
done
