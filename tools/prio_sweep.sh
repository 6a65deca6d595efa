for v in prio noprio; do
  if [ $v = noprio ]; then export KRONRED_NO_PRIO=1; else unset KRONRED_NO_PRIO; fi
  timeout 300 python tools/split_sweep.py c2 3e-3 --runs 3 --S 0 --bucket 100 2>/dev/null | sed "s/^/$v /" | cut -c1-400
done
