# A/B: the working tree's library against the last commit's (tools/_var_head), same box
for v in new head new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py ${1:-c2} --bucket 500 2>&1 | grep "after pick\|^sum\|total device\|pick start" | sort -u
done
