# scorers as a programmatic chain (default) vs the switch node (KRONRED_SWITCH=1): parity subset + timelines
timeout 1200 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or large or exchange or complex or live or m40 or h2k" 2>&1 | tail -2
for v in new head new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|^sum\|total device\|pick start" | sort -u
done
unset KRONRED_LIB
timeout 300 python tools/iter_profile.py c3 3e-3 0.9 --bucket 9000 2>&1 | grep "total device"
KRONRED_LIB=tools/_var_head/libkronred_b200.so timeout 300 python tools/iter_profile.py c3 3e-3 0.9 --bucket 9000 2>&1 | grep "total device"
