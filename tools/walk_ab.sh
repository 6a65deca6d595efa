# path walk: parity subset, then A/B timeline against the last commit (tools/_var_head) and the serial walk
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or large or golden or m40 or h2k or exchange" 2>&1 | tail -2
for v in new head serial new head; do
  unset KRONRED_LIB KRONRED_SERIAL_WALK
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; fi
  if [ $v = serial ]; then export KRONRED_SERIAL_WALK=1; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|total device" | sort -u
done
