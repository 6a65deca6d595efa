# forward general steps load-first: parity subset + A/B timeline (tools/_var_head = last commit)
timeout 900 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or large or golden or m40 or h2k or pq or rad" 2>&1 | tail -2
timeout 120 python tools/micro/base_refresh.py c2
KRONRED_LIB=tools/_var_head/libkronred_b200.so timeout 120 python tools/micro/base_refresh.py c2
for v in new head new head; do
  if [ $v = head ]; then export KRONRED_LIB=tools/_var_head/libkronred_b200.so; else unset KRONRED_LIB; fi
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 500 2>&1 | grep "after pick\|total device" | sort -u
done
