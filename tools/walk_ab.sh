# A/B of the working tree's library against a baseline build (tools/_var_head), same box
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or large or golden or c5" 2>&1 | tail -2
for v in new head new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | tail -2
done
KRONRED_LIB=tools/_var_brtrace/libkronred_b200.so timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "^walk" | head -20
