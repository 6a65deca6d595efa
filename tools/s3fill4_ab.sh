# S = 4 threshold on the two-scenario large feeders: 11/16 of the fill (before) vs 14/16 (default)
run() { echo "== $1 $2 $(timeout 600 python tools/iter_profile.py $2 --bucket 100000 2>&1 | grep 'total device\|^sum' | tr '\n' '|')"; }
for rep in 1 2; do
for c in "c4 3e-3 0.8" "c3 3e-3 0.9"; do
  KRONRED_S3_FILL4=11 run f11 "$c"
  run f14 "$c"
done
done
