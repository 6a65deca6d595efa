# score3 geometry on the large feeders at L = 24 / 96 (KRONRED_S3_G x KRONRED_S3_LS <= 128 threads), C4 prefixes
for L in 96 24; do
  for geo in "16 8" "8 16" "4 32" "12 8" "10 12"; do
    set -- $geo
    echo "== L$L G=$1 Ls=$2 $(KRONRED_S3_G=$1 KRONRED_S3_LS=$2 timeout 600 python tools/r1r2_ab.py . $L 0.01 2>&1 | tail -1)"
  done
done
