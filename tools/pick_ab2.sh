for v in new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  timeout 300 python tools/iter_profile.py c2 --bucket 500 --out gpurun_out/tl_$v.tsv > /dev/null 2>&1
done
