# score3 Z staging L2 policy: evict_first (default) vs evict_normal (S3_Z_EVICT_FIRST=0), C4 prefixes
for rep in 1 2; do
for L in 24 96; do
  unset KRONRED_LIB; echo "== def L$L $(timeout 600 python tools/r1r2_ab.py . $L 0.01 2>&1 | tail -1)"
  KRONRED_LIB=tools/_var_ev0/libkronred_b200.so; export KRONRED_LIB; echo "== ev0 L$L $(timeout 600 python tools/r1r2_ab.py . $L 0.01 2>&1 | tail -1)"; unset KRONRED_LIB
done
unset KRONRED_LIB; echo "== def c4L2 $(timeout 600 python tools/iter_profile.py c4 3e-3 0.2 --bucket 100000 2>&1 | grep 'total device')"
KRONRED_LIB=tools/_var_ev0/libkronred_b200.so; export KRONRED_LIB; echo "== ev0 c4L2 $(timeout 600 python tools/iter_profile.py c4 3e-3 0.2 --bucket 100000 2>&1 | grep 'total device')"; unset KRONRED_LIB
done
