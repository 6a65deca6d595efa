for v in nocl; do
  unset KRONRED_NO_RCLUSTER KRONRED_NO_RWAIT
  if [ $v = nocl ]; then export KRONRED_NO_RCLUSTER=1; fi
  if [ $v = norw ]; then export KRONRED_NO_RWAIT=1; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 --out gpurun_out/tl.tsv 2>&1 | grep "after pick\|^sum\|wait" | sort -u
done
