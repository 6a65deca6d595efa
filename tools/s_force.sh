for v in auto 1 auto 1; do
  if [ $v = auto ]; then unset KRONRED_S3_S; else export KRONRED_S3_S=$v; fi
  echo "== S $v"; timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep -v "^loop\|^ iters\|pick start"
done
