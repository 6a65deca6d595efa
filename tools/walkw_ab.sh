# warp-wide walk with row-split general steps: parity subset + A/B timeline against the last commit
timeout 1200 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or large or golden or m40 or h2k or pq or rad or s24 or exchange" 2>&1 | tail -2
for v in new head new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|total device" | sort -u
done
