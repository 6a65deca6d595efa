# score1 candidates per item per split (KRONRED_S1_GK = S1,S2,S4)
for g in 8,8,4 4,8,4 8,8,4 4,8,4; do
  echo "== gk $g $(KRONRED_S1_GK=$g timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep 'total device\|^ *[0-9]*- *[0-9]' | sed 's/  */ /g' | cut -c1-60 | tr '\n' '|')"
done
