# plain tiles: one fast-sqrt vote per 8 rows (default) vs per 4-row pass (tools/_var_tv0) vs last commit
timeout 1200 python -m pytest tests -m gpu -x -q -k "c2 or c1 or incremental or full_run or m40 or h2k or split or iteration_scores" 2>&1 | tail -2
for v in new tv0 head new tv0 head; do
  case $v in new) unset KRONRED_LIB;; head) export KRONRED_LIB=tools/_var_head/libkronred_b200.so;; *) export KRONRED_LIB=tools/_var_$v/libkronred_b200.so;; esac
  echo "== $v $(timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep 'total device\|^ *[0-9]*- *[0-9]' | sed 's/  */ /g' | cut -c1-60 | tr '\n' '|')"
done
