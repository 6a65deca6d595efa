# score1 ring depths per split (S1_NS1/2/4): A/B of build variants
for v in new r444 r343 r355 head new r444 r343 r355 head; do
  case $v in new) unset KRONRED_LIB;; head) export KRONRED_LIB=tools/_var_head/libkronred_b200.so;; *) export KRONRED_LIB=tools/_var_$v/libkronred_b200.so;; esac
  echo "== $v"; timeout 300 python tools/iter_profile.py c2 --bucket 200 2>&1 | grep "total device\|^ *[0-9]*- *[0-9]" | awk '{print $0}' | sed 's/  */ /g' | cut -c1-60 | tr '\n' '|'; echo
done
