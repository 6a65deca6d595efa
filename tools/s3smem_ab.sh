# score3 split launches: dynamic smem sized for G / S staging slots (default) vs the S = 1 size
# (KRONRED_S3_FULL_SMEM), with the automatic split, S = 2 forced, and a one-wave fill
run() { echo "== $1 $2 $(timeout 600 python tools/iter_profile.py $2 --bucket 100000 2>&1 | grep 'total device\|^sum' | tr '\n' '|')"; }
for rep in 1 2; do
for c in "c3 3e-3 0.3" "c4 3e-3 0.2" "c4 3e-3 0.8"; do
  KRONRED_S3_FULL_SMEM=1 run full "$c"
  run new "$c"
  KRONRED_S3_S=2 run newS2 "$c"
  KRONRED_S3_FILL=56832 run newfill "$c"
done
done
