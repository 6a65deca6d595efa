# score3 split launches on the L = 2 large feeders: round-2 final (KRONRED_S3_FULL_SMEM + one-CTA fill)
# against per-split smem and the one-wave fill (default)
run() { echo "== $1 $2 $(timeout 600 python tools/iter_profile.py $2 --bucket 100000 2>&1 | grep 'total device\|^sum' | tr '\n' '|')"; }
for c in "c4 3e-3 0.8" "c3 3e-3 0.9" "c2"; do
  KRONRED_S3_FULL_SMEM=1 KRONRED_S3_FILL=18944 run old "$c"
  run new "$c"
done
